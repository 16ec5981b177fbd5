/*
 * gf_oracle.c -- CPU double-precision ORACLE for the Gabor Fields hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_2602_05081_b200/) never imports, links or runs it,
 * and this file shares no code, header, table or constant generator with it.
 *
 * Plain, slow, obviously-correct: brute force over ALL primitives (no BVH),
 * every quantity in double, each function citing the passage it follows.
 * Citations "P:Lnnn" are lines of PAPER.md (arXiv 2602.05081, LaTeX source);
 * readings where the paper is silent/garbled are the C-numbers of DESIGN.md §3.
 *
 *   kernel ............ Eq. 6        g = (8pi^3|S|)^-1/2 e^{-1/2 x'S^-1 x} cos(w.x)
 *   modulation ........ P:L183                        w_vec = R S^-1 (w,w,w)^T
 *   extinction ........ Eq. 1        kappa = sum alpha_i K_i, K_i bounded by ellipsoid (C7)
 *   optical depth ..... Eq. 2-3       tau_i = alpha_i int K_i dt ; T = exp(-sum tau_i)
 *   segment integral .. App. A finite form, scalars a,beta,gamma,B,delta
 *   complex erf ....... Eq. 13 Maclaurin series, run to convergence in double (C5)
 *   segments .......... Eq. 4        entry/exit events, active set per segment
 *   free flight ....... Eq. 5, bisection, first crossing (C16/C17)
 *   masks ............. P:L344-L350                  visible iff (V_r & V_l) != 0 (32-bit groups, C24)
 *   level strategies .. Table B1, readings C13/C14
 *   orient. strategies  Table B2, readings C11/C12/C15
 *   pipeline .......... P:L352-L365 (sample mask, intersect, distance sample / integrate, reweight, recurse)
 *   tomography ........ P:L363 (accumulate tau, exp after all samples)
 *   Philox4x32-10 ..... counter RNG (Salmon et al. 2011); same stream layout as the GPU
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fPIC -shared -o liboracle.so gf_oracle.c -lm -lpthread
 */
#include <complex.h>
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_PI 3.14159265358979323846
#define OR_MAXG 32

/* ------------------------------------------------------------------------- */
/* Scene                                                                      */
/* ------------------------------------------------------------------------- */
typedef struct {
    int n, P, K, G;    /* G = n_bands * G0 groups in all (C24)                           */
    int G0, n_bands;   /* groups per band 1 + (P-1) K; spatial bands (cfg5 distance bands) */
    double *mu;    /* 3n  kernel mean                                   */
    double *sinv;  /* 9n  Sigma^-1 = R S^-2 R^T (row major)             */
    double *wvec;  /* 3n  omega_vec = R S^-1 (w,w,w)^T         */
    double *norm;  /* n   (8 pi^3 |Sigma|)^-1/2  (Eq. 6)                 */
    double *alpha; /* n   kernel weight alpha_i (Eq. 1)                  */
    double *E2;    /* n   squared whitened extent (C7/C8; default 3^2)   */
    int *group;    /* n   group id g(l,b) (C10/C11/C24)                  */
    int *bin;      /* n   orientation bin (derived if not given)         */
    int *level;    /* n   pyramid level                                  */
    float *omega;  /* n   modulation scalar as given (fp32)              */
    float bin_axes[3 * 32];
    float lfmax[8];  /* max world frequency |omega_vec| per level (F3)     */
    float f0[32];    /* representative whitened frequency per group (C12)  */
} or_scene;

/* quaternion (x,y,z,w) -> rotation matrix R (row major), normalised in double */
static void quat_to_R_d(const double *q, double R[9]) {
    double x = q[0], y = q[1], z = q[2], w = q[3];
    double nn = sqrt(x * x + y * y + z * z + w * w);
    x /= nn; y /= nn; z /= nn; w /= nn;
    R[0] = 1 - 2 * (y * y + z * z); R[1] = 2 * (x * y - w * z);     R[2] = 2 * (x * z + w * y);
    R[3] = 2 * (x * y + w * z);     R[4] = 1 - 2 * (x * x + z * z); R[5] = 2 * (y * z - w * x);
    R[6] = 2 * (x * z - w * y);     R[7] = 2 * (y * z + w * x);     R[8] = 1 - 2 * (x * x + y * y);
}

/* Per-primitive derived quantities from (q, s, omega) in double:
 *   Sigma^-1 = R S^-2 R^T, omega_vec = R S^-1 (w,w,w)^T, norm = (8 pi^3 |Sigma|)^-1/2 (Eq. 6). */
static void derive_d(const double *q, const double *sx, double w, double sinv[9], double wvec[3], double *norm) {
    double R[9];
    quat_to_R_d(q, R);
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
            double acc = 0;
            for (int k = 0; k < 3; ++k) acc += R[3 * r + k] * R[3 * c + k] / (sx[k] * sx[k]);
            sinv[3 * r + c] = acc;
        }
    for (int r = 0; r < 3; ++r) {
        double acc = 0;
        for (int k = 0; k < 3; ++k) acc += R[3 * r + k] * w / sx[k];
        wvec[r] = acc;
    }
    *norm = 1.0 / sqrt(8.0 * OR_PI * OR_PI * OR_PI * sx[0] * sx[0] * sx[1] * sx[1] * sx[2] * sx[2]);
}

/* Orientation bin (C11): argmax_k |d . o_k| with d = direction of omega_vec,
 * ties -> lower k.  Integer decided by floating point, so it is taken in fp32
 * (the kernel's precision, task rule) with explicit fmaf so that no contraction
 * choice of the compiler changes it.  d is taken unnormalised (argmax is scale
 * free): d = R S^-1 (1,1,1)^T. */
static int derive_bin_f32(const float *qf, const float *sf, int K, const float *axes) {
    float x = qf[0], y = qf[1], z = qf[2], w = qf[3];
    float nn = sqrtf(fmaf(x, x, fmaf(y, y, fmaf(z, z, w * w))));
    x = x / nn; y = y / nn; z = z / nn; w = w / nn;
    float R[9];
    R[0] = 1.0f - 2.0f * fmaf(y, y, z * z); R[1] = 2.0f * fmaf(x, y, -(w * z)); R[2] = 2.0f * fmaf(x, z, w * y);
    R[3] = 2.0f * fmaf(x, y, w * z);        R[4] = 1.0f - 2.0f * fmaf(x, x, z * z); R[5] = 2.0f * fmaf(y, z, -(w * x));
    R[6] = 2.0f * fmaf(x, z, -(w * y));     R[7] = 2.0f * fmaf(y, z, w * x);     R[8] = 1.0f - 2.0f * fmaf(x, x, y * y);
    float i0 = 1.0f / sf[0], i1 = 1.0f / sf[1], i2 = 1.0f / sf[2];
    float d[3];
    for (int r = 0; r < 3; ++r) d[r] = fmaf(R[3 * r + 0], i0, fmaf(R[3 * r + 1], i1, R[3 * r + 2] * i2));
    int best = 0; float bestv = -1.0f;
    for (int k = 0; k < K; ++k) {
        const float *o = axes + 3 * k;
        float a = fabsf(fmaf(d[0], o[0], fmaf(d[1], o[1], d[2] * o[2])));
        if (a > bestv) { bestv = a; best = k; }
    }
    return best;
}

static void level_fmax_of(or_scene *s);
static void group_f0_of(or_scene *s);

/* Build the per-primitive double data.  level/bin may be NULL (bin==NULL or
 * 255 -> derived, level==NULL -> omega==0 ? 0 : 1); band NULL -> 0, n_bands >= 1
 * spatial bands (group id band * G0 + g(l,b), G0 = 1 + (P-1) K, C24).  Returns NULL
 * on bad input. */
or_scene *or_scene_create(int n, const float *mu, const float *quat, const float *scale,
                          const float *alpha, const float *omega, const float *extent,
                          const uint8_t *level, const uint8_t *bin, int P, int K,
                          const float *bin_axes, const uint8_t *band, int n_bands) {
    if (n_bands < 1) n_bands = 1;
    if (n < 0 || P < 1 || K < 1 || n_bands * (1 + (P - 1) * K) > OR_MAXG) return NULL;
    or_scene *s = (or_scene *)calloc(1, sizeof(or_scene));
    s->n = n; s->P = P; s->K = K; s->G0 = 1 + (P - 1) * K; s->n_bands = n_bands; s->G = n_bands * s->G0;
    if (bin_axes) memcpy(s->bin_axes, bin_axes, sizeof(float) * 3 * K);
    size_t nn = n > 0 ? (size_t)n : 1;
    s->mu = malloc(sizeof(double) * 3 * nn);   s->sinv = malloc(sizeof(double) * 9 * nn);
    s->wvec = malloc(sizeof(double) * 3 * nn); s->norm = malloc(sizeof(double) * nn);
    s->alpha = malloc(sizeof(double) * nn);    s->E2 = malloc(sizeof(double) * nn);
    s->group = malloc(sizeof(int) * nn);       s->bin = malloc(sizeof(int) * nn);
    s->level = malloc(sizeof(int) * nn);       s->omega = malloc(sizeof(float) * nn);
    for (int i = 0; i < n; ++i) {
        const double qd[4] = {quat[4 * i], quat[4 * i + 1], quat[4 * i + 2], quat[4 * i + 3]};
        const double sx[3] = {scale[3 * i], scale[3 * i + 1], scale[3 * i + 2]};
        derive_d(qd, sx, omega[i], s->sinv + 9 * i, s->wvec + 3 * i, s->norm + i);
        for (int k = 0; k < 3; ++k) s->mu[3 * i + k] = mu[3 * i + k];
        s->alpha[i] = alpha[i];
        s->omega[i] = omega[i];
        double E = extent ? extent[i] : 3.0;
        s->E2[i] = E * E;
        int l = level ? level[i] : (omega[i] == 0.0f ? 0 : 1);
        if (l >= P) l = P - 1;
        s->level[i] = l;
        int b = (bin && bin[i] != 255) ? bin[i] : (l == 0 ? 0 : derive_bin_f32(quat + 4 * i, scale + 3 * i, K, s->bin_axes));
        if (b >= K) b = K - 1;
        s->bin[i] = b;
        int bd = band ? band[i] : 0;
        if (bd >= n_bands) bd = n_bands - 1;
        s->group[i] = bd * s->G0 + ((l == 0) ? 0 : 1 + (l - 1) * K + b);  /* C24 group id */
    }
    level_fmax_of(s);
    group_f0_of(s);
    return s;
}

void or_scene_destroy(or_scene *s) {
    if (!s) return;
    free(s->mu); free(s->sinv); free(s->wvec); free(s->norm); free(s->alpha); free(s->E2);
    free(s->group); free(s->bin); free(s->level); free(s->omega); free(s);
}

int or_scene_groups(const or_scene *s, int *group_out, int *bin_out) {
    for (int i = 0; i < s->n; ++i) { group_out[i] = s->group[i]; if (bin_out) bin_out[i] = s->bin[i]; }
    return s->n;
}

/* ------------------------------------------------------------------------- */
/* Scene-derived policy parameters                                            */
/* ------------------------------------------------------------------------- */
/* Maximum world frequency |omega_vec| = |R S^-1 (w,w,w)^T| of each Gabor level
   (reading F3: "discard all levels that contain Gabor primitives with frequencies above the
   threshold"); level 0 (Gaussians) 0.  Double, rounded to fp32 once. */
static void level_fmax_of(or_scene *s) {
    double mx[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int i = 0; i < s->n; ++i) {
        const double *w = s->wvec + 3 * i;
        double f = sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
        if (s->level[i] > 0 && f > mx[s->level[i]]) mx[s->level[i]] = f;
    }
    for (int l = 0; l < 8; ++l) s->lfmax[l] = (float)mx[l];
}

static int cmp_float(const void *a, const void *b) {
    float x = *(const float *)a, y = *(const float *)b;
    return x < y ? -1 : (x > y ? 1 : 0);
}
/* Representative whitened frequency of each group (reading C12): the whitened
   frequency |k_W| = sqrt(3) omega (C2) of the level's median member, median = middle element
   of the sorted fp32 omegas (even count: the fp32 mean of the two middle ones), shared by all
   bins (and bands) of a level; level 0: 0. */
static void group_f0_of(or_scene *s) {
    for (int g = 0; g < 32; ++g) s->f0[g] = 0.0f;
    float *v = malloc(sizeof(float) * (s->n > 0 ? s->n : 1));
    for (int l = 1; l < s->P; ++l) {
        int m = 0;
        for (int i = 0; i < s->n; ++i) if (s->level[i] == l) v[m++] = s->omega[i];
        if (m == 0) continue;
        qsort(v, m, sizeof(float), cmp_float);
        volatile float med = (m & 1) ? v[m / 2] : (v[m / 2 - 1] + v[m / 2]) / 2.0f;
        float f0 = (float)((double)med * sqrt(3.0));
        for (int bd = 0; bd < s->n_bands; ++bd)
            for (int b = 0; b < s->K; ++b) s->f0[bd * s->G0 + 1 + (l - 1) * s->K + b] = f0;
    }
    free(v);
}

void or_scene_info(const or_scene *s, float *lfmax8, float *f0_32) {
    if (lfmax8) memcpy(lfmax8, s->lfmax, sizeof(float) * 8);
    if (f0_32) memcpy(f0_32, s->f0, sizeof(float) * 32);
}

/* Accelerated motion blur (readings M1-M3): per group the mean of its members'
   omega_vec (signs aligned with the member of largest |omega_vec|, first index on ties: +-omega_vec
   is the same cosine), k = |mean . d| (d normalised), attenuation of the box filter of length m
   along d on a cosine of angular frequency k = |sin(m k / 2) / (m k / 2)| (M2); group culled iff
   attenuation < threshold.  Level-0 groups and empty groups are kept. */
void or_motion_blur_mask(const or_scene *s, const float dir[3], float m, float threshold, uint32_t *mask_out,
                         float *att_out) {
    double d[3] = {dir[0], dir[1], dir[2]};
    double dn = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    for (int k = 0; k < 3; ++k) d[k] /= dn;
    uint32_t mask = 0;
    for (int g = 0; g < s->G; ++g) {
        double att = 1.0;
        int ref = -1;
        double refn = -1.0;
        for (int i = 0; i < s->n; ++i) {
            if (s->group[i] != g) continue;
            const double *w = s->wvec + 3 * i;
            double f = sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
            if (f > refn) { refn = f; ref = i; }
        }
        if (g % s->G0 != 0 && ref >= 0) {
            const double *r = s->wvec + 3 * ref;
            double sum[3] = {0, 0, 0};
            long cnt = 0;
            for (int i = 0; i < s->n; ++i) {
                if (s->group[i] != g) continue;
                const double *w = s->wvec + 3 * i;
                double sg = (w[0] * r[0] + w[1] * r[1] + w[2] * r[2]) < 0.0 ? -1.0 : 1.0;
                for (int k = 0; k < 3; ++k) sum[k] += sg * w[k];
                ++cnt;
            }
            double k = fabs((sum[0] * d[0] + sum[1] * d[1] + sum[2] * d[2]) / (double)cnt);
            double x = 0.5 * (double)m * k;
            att = (x == 0.0) ? 1.0 : fabs(sin(x) / x);
        }
        if (att_out) att_out[g] = (float)att;
        if (att >= threshold) mask |= 1u << g;
    }
    *mask_out = mask;
}

/* Adaptive clamping (Eq. 15; reading C8'): the whitened radius beyond which the
   untruncated line integral of a ray is below eps in the worst case ||W v|| = 1/s_max and
   Omega^2 = |k_W|^2 = 3 omega^2:  E = min(3, sqrt(max(0, -2 ln(eps 2 pi s1 s2 s3 / (alpha s_max))
   - 3 omega^2))), floored at 1e-3 (the loader requires E > 0).  Double, rounded to fp32 once. */
void or_adaptive_extent(long n, const float *scale, const float *alpha, const float *omega, float eps, float *out) {
    for (long i = 0; i < n; ++i) {
        double s0 = scale[3 * i], s1 = scale[3 * i + 1], s2 = scale[3 * i + 2];
        double smax = s0 > s1 ? (s0 > s2 ? s0 : s2) : (s1 > s2 ? s1 : s2);
        double a = alpha[i] > 1e-30f ? alpha[i] : 1e-30;
        double w = omega[i];
        double arg = -2.0 * log((double)eps * 2.0 * OR_PI * s0 * s1 * s2 / (a * smax)) - 3.0 * w * w;
        double E = sqrt(arg > 0.0 ? arg : 0.0);
        if (E > 3.0) E = 3.0;
        if (E < 1e-3) E = 1e-3;
        out[i] = (float)E;
    }
}

/* ------------------------------------------------------------------------- */
/* Kernel evaluation, Eq. 6, truncated at the ellipsoid (C7)     */
/* ------------------------------------------------------------------------- */
double or_eval_kernel(const or_scene *s, int i, const double x[3], int truncated) {
    double d[3] = {x[0] - s->mu[3 * i], x[1] - s->mu[3 * i + 1], x[2] - s->mu[3 * i + 2]};
    const double *M = s->sinv + 9 * i;
    double q = 0;
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) q += d[r] * M[3 * r + c] * d[c];
    if (truncated && q > s->E2[i]) return 0.0;
    const double *wv = s->wvec + 3 * i;
    return s->norm[i] * exp(-0.5 * q) * cos(wv[0] * d[0] + wv[1] * d[1] + wv[2] * d[2]);
}

/* ------------------------------------------------------------------------- */
/* Complex erf by its Maclaurin series, Eq. 13:                 */
/*   erf(z) = 2/sqrt(pi) sum_n (-1)^n z^(2n+1) / (n! (2n+1))                    */
/* run to convergence (term < 1e-17 |sum|, <= 200 terms) -- reading C5.       */
/* ------------------------------------------------------------------------- */
double complex or_erf(double complex z) {
    double complex zz = z * z;
    /* domain guard: the alternating series loses ~|z|^2/ln(10) digits; beyond |z|^2 = 24 the
       double result is no longer trustworthy to 1e-8, so fail loudly (NaN) instead. */
    if (cabs(zz) > 24.0) return NAN + I * NAN;
    double complex p = z;   /* (-1)^n z^(2n+1) / n! */
    double complex sum = z;
    for (int n = 1; n < 200; ++n) {
        p = p * (-zz) / (double)n;
        double complex term = p / (double)(2 * n + 1);
        sum += term;
        if (cabs(term) < 1e-17 * cabs(sum)) break;
    }
    return sum * (2.0 / sqrt(OR_PI));
}

void or_erf_parts(double re, double im, double *out) {
    double complex r = or_erf(re + I * im);
    out[0] = creal(r); out[1] = cimag(r);
}

/* ------------------------------------------------------------------------- */
/* Per (ray, primitive) scalars, App. A                          */
/* ------------------------------------------------------------------------- */
typedef struct {
    double a, beta, gamma, B, delta;
    double r2;          /* gamma - beta^2/a : squared perpendicular distance */
    int hit;            /* chord of the ellipsoid intersects [t0,t1] with positive length */
    double tin, tout;   /* chord clipped to [t0,t1] */
} or_pair;

static void pair_setup(const or_scene *s, int i, const double o[3], const double v[3],
                       double t0, double t1, or_pair *p) {
    const double *M = s->sinv + 9 * i;
    double d[3] = {o[0] - s->mu[3 * i], o[1] - s->mu[3 * i + 1], o[2] - s->mu[3 * i + 2]};
    double Mv[3], Md[3];
    for (int r = 0; r < 3; ++r) {
        Mv[r] = M[3 * r] * v[0] + M[3 * r + 1] * v[1] + M[3 * r + 2] * v[2];
        Md[r] = M[3 * r] * d[0] + M[3 * r + 1] * d[1] + M[3 * r + 2] * d[2];
    }
    p->a = v[0] * Mv[0] + v[1] * Mv[1] + v[2] * Mv[2];      /* a     = v^T S^-1 v */
    p->beta = v[0] * Md[0] + v[1] * Md[1] + v[2] * Md[2];   /* beta  = v^T S^-1 d */
    p->gamma = d[0] * Md[0] + d[1] * Md[1] + d[2] * Md[2];  /* gamma = d^T S^-1 d */
    const double *wv = s->wvec + 3 * i;
    p->B = wv[0] * v[0] + wv[1] * v[1] + wv[2] * v[2];      /* B     = w^T v */
    p->delta = wv[0] * d[0] + wv[1] * d[1] + wv[2] * d[2];  /* delta = w^T d */
    /* perpendicular distance^2, computed from the closest-approach offset
       (d + tc v) to avoid the gamma - beta^2/a cancellation for far origins */
    double tc = -p->beta / p->a;
    double dc[3] = {d[0] + tc * v[0], d[1] + tc * v[1], d[2] + tc * v[2]};
    double r2 = 0;
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) r2 += dc[r] * M[3 * r + c] * dc[c];
    p->r2 = r2;
    /* ellipsoid: a t^2 + 2 beta t + gamma <= E^2  (C7) */
    p->hit = 0;
    if (r2 < s->E2[i]) {
        double ht = sqrt((s->E2[i] - r2) / p->a);
        double ta = tc - ht, tb = tc + ht;
        if (ta < t0) ta = t0;
        if (tb > t1) tb = t1;
        if (tb > ta) { p->hit = 1; p->tin = ta; p->tout = tb; }
    }
}

/* App. A finite-domain closed form, alpha NOT applied:
 *   I = (8pi^3|S|)^-1/2 Re{ e^{i delta} e^{-gamma/2} sqrt(pi/2a) e^{(-beta+iB)^2/2a}
 *                          [erf(sqrt(a/2) t1 - zeta) - erf(sqrt(a/2) t0 - zeta)] },
 *   zeta = (-beta + iB)/sqrt(2a).
 * The exponentials are combined before evaluation,
 *   e^{-gamma/2} e^{(-beta+iB)^2/2a} = e^{-r2/2} e^{-B^2/2a} e^{-i beta B/a},
 * so that e^{beta^2/2a} (which overflows for far origins) is never formed. */
static double seg_integral(const or_scene *s, int i, const or_pair *p, double ta, double tb) {
    if (!(tb > ta)) return 0.0;
    double a = p->a, sq2a = sqrt(2.0 * a);
    double complex zeta = (-p->beta + I * p->B) / sq2a;
    double complex z1 = sqrt(a / 2.0) * tb - zeta;
    double complex z0 = sqrt(a / 2.0) * ta - zeta;
    double complex derf = or_erf(z1) - or_erf(z0);
    double mag = exp(-0.5 * p->r2 - p->B * p->B / (2.0 * a));
    double phase = p->delta - p->beta * p->B / a;
    double complex val = cexp(I * phase) * derf;
    return s->norm[i] * sqrt(OR_PI / (2.0 * a)) * mag * creal(val);
}

/* Public: integral of kernel i (alpha not applied, truncated at E) along
   o + t v over [t0,t1]. */
double or_prim_integral(const or_scene *s, int i, const float *ray_o, const float *ray_v,
                        double t0, double t1) {
    double o[3] = {ray_o[0], ray_o[1], ray_o[2]}, v[3] = {ray_v[0], ray_v[1], ray_v[2]};
    or_pair p;
    pair_setup(s, i, o, v, t0, t1, &p);
    if (!p.hit) return 0.0;
    return seg_integral(s, i, &p, p.tin, p.tout);
}

/* Untruncated full-line integral: App. A boxed infinite limit. */
double or_prim_integral_infinite(const or_scene *s, int i, const float *ray_o, const float *ray_v) {
    double o[3] = {ray_o[0], ray_o[1], ray_o[2]}, v[3] = {ray_v[0], ray_v[1], ray_v[2]};
    or_pair p;
    pair_setup(s, i, o, v, -INFINITY, INFINITY, &p);
    double a = p.a;
    return s->norm[i] * sqrt(2.0 * OR_PI / a) * exp(-0.5 * p.r2) * exp(-p.B * p.B / (2.0 * a)) *
           cos(p.delta - p.beta * p.B / a);
}

/* ------------------------------------------------------------------------- */
/* Brute-force optical depth, Eq. 2-3 with masks                */
/* ------------------------------------------------------------------------- */
typedef struct { double s, c; } neum;  /* Neumaier compensated sum */
static void neum_add(neum *n, double x) {
    double t = n->s + x;
    if (fabs(n->s) >= fabs(x)) n->c += (n->s - t) + x; else n->c += (x - t) + n->s;
    n->s = t;
}
static double neum_get(const neum *n) { return n->s + n->c; }

/* tau = sum over visible i of w_g(i) alpha_i int K_i ; also A = sum |.| and per-group tau */
/* fmax: foveation (reading F4): a primitive whose frequency along the ray |omega_vec . v|
   exceeds fmax is not integrated (INFINITY: off) */
static double trace_one_f(const or_scene *s, const double o[3], const double v[3], double t0, double t1,
                          uint32_t mask, const float *wts, double fmax, double *abs_out, double *grp_out,
                          int *nhits);
static double trace_one(const or_scene *s, const double o[3], const double v[3], double t0, double t1,
                        uint32_t mask, const float *wts, double *abs_out, double *grp_out, int *nhits) {
    return trace_one_f(s, o, v, t0, t1, mask, wts, INFINITY, abs_out, grp_out, nhits);
}
static double trace_one_f(const or_scene *s, const double o[3], const double v[3], double t0, double t1,
                          uint32_t mask, const float *wts, double fmax, double *abs_out, double *grp_out,
                          int *nhits) {
    neum tau = {0, 0}, A = {0, 0};
    neum grp[OR_MAXG];
    memset(grp, 0, sizeof(grp));
    int nh = 0;
    for (int i = 0; i < s->n; ++i) {
        int g = s->group[i];
        if (!((mask >> g) & 1u)) continue;
        or_pair p;
        pair_setup(s, i, o, v, t0, t1, &p);
        if (!p.hit) continue;
        if (fabs(p.B) > fmax) continue;  /* foveation: frequency along the ray above the threshold */
        ++nh;
        double w = wts ? (double)wts[g] : 1.0;
        double ti = w * s->alpha[i] * seg_integral(s, i, &p, p.tin, p.tout);
        neum_add(&tau, ti);
        neum_add(&A, fabs(ti));
        neum_add(&grp[g], ti);
    }
    if (abs_out) *abs_out = neum_get(&A);
    if (grp_out)
        for (int g = 0; g < s->G; ++g) grp_out[g] = neum_get(&grp[g]);
    if (nhits) *nhits = nh;
    return neum_get(&tau);
}

/* ------------------------------------------------------------------------- */
/* Thread pool helper                                                          */
/* ------------------------------------------------------------------------- */
typedef void (*or_work_fn)(void *ctx, long idx);
typedef struct { or_work_fn fn; void *ctx; long n; long next; pthread_mutex_t mu; } or_pool;
static void *pool_worker(void *arg) {
    or_pool *pl = (or_pool *)arg;
    for (;;) {
        pthread_mutex_lock(&pl->mu);
        long i = pl->next++;
        pthread_mutex_unlock(&pl->mu);
        if (i >= pl->n) break;
        pl->fn(pl->ctx, i);
    }
    return NULL;
}
static void run_parallel(or_work_fn fn, void *ctx, long n, int nthreads) {
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    or_pool pl = {fn, ctx, n, 0};
    pthread_mutex_init(&pl.mu, NULL);
    if (nthreads == 1) { pool_worker(&pl); pthread_mutex_destroy(&pl.mu); return; }
    pthread_t th[256];
    for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, pool_worker, &pl);
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    pthread_mutex_destroy(&pl.mu);
}

typedef struct {
    const or_scene *s; const float *rays; uint32_t mask; const float *wts;
    double *tau, *A, *grp; int *nhits;
} trace_ctx;
static void trace_work(void *c, long r) {
    trace_ctx *t = (trace_ctx *)c;
    const float *ry = t->rays + 8 * r;
    double o[3] = {ry[0], ry[1], ry[2]}, v[3] = {ry[4], ry[5], ry[6]};
    double A;
    double grp[OR_MAXG];
    int nh;
    t->tau[r] = trace_one(t->s, o, v, ry[3], ry[7], t->mask, t->wts, &A, grp, &nh);
    if (t->A) t->A[r] = A;
    if (t->grp) memcpy(t->grp + (size_t)r * t->s->G, grp, sizeof(double) * t->s->G);
    if (t->nhits) t->nhits[r] = nh;
}

/* rays: n x 8 floats (ox,oy,oz,tmin,dx,dy,dz,tmax). wts: G floats or NULL (=1). */
void or_trace(const or_scene *s, const float *rays, long n, uint32_t mask, const float *wts,
              double *tau, double *A, double *grp, int *nhits, int nthreads) {
    trace_ctx c = {s, rays, mask, wts, tau, A, grp, nhits};
    run_parallel(trace_work, &c, n, nthreads);
}

/* Backward of tau w.r.t. the opacities (the alpha part):
   tau_r = sum_i w_g(i) alpha_i I_i(r) is linear in alpha, so
   grad[i] = sum_r dl[r] w_g(i) I_i(r), I_i the closed-form integral of kernel i with alpha = 1 (App. A).
   Plain double loops over rays and primitives (no BVH). */
void or_grad_alpha(const or_scene *s, const float *rays, long n, uint32_t mask, const float *wts,
                   const double *dl, double *grad) {
    for (int i = 0; i < s->n; ++i) grad[i] = 0.0;
    for (long r = 0; r < n; ++r) {
        const float *ray = rays + 8 * r;
        double o[3] = {ray[0], ray[1], ray[2]}, v[3] = {ray[4], ray[5], ray[6]};
        for (int i = 0; i < s->n; ++i) {
            int g = s->group[i];
            if (!((mask >> g) & 1u)) continue;
            or_pair p;
            pair_setup(s, i, o, v, ray[3], ray[7], &p);
            if (!p.hit) continue;
            double w = wts ? (double)wts[g] : 1.0;
            grad[i] += dl[r] * w * seg_integral(s, i, &p, p.tin, p.tout);
        }
    }
}

/* Backward of tau w.r.t. every primitive parameter, by its
 * plain definition: the derivative of the single-primitive optical depth
 *   tau_ri(theta) = alpha int_{chord} g(x(t); mu, q, s, omega) dt   (Eq. 2, Eq. 6, truncated at E, C7)
 * w.r.t. theta = (mu_x, mu_y, mu_z, q_x, q_y, q_z, q_w, s_x, s_y, s_z, omega, alpha), taken as the
 * limit of the central difference quotient: Richardson-extrapolated central differences of the
 * closed-form forward (App. A) in double, (4 D(h/2) - D(h)) / 3, truncation error O(h^4).  The
 * chord endpoints move with theta (pair_setup recomputed for every perturbed primitive), so the
 * result includes the truncation-boundary terms.  Steps: mu 1e-3 min(s), q 1e-3 |q|, s_k 1e-3 s_k,
 * omega 1e-3 max(1, |omega|), alpha 1e-3 max(1, |alpha|).  Valid away from grazing chords (tau is
 * not differentiable where a chord appears: r2 = E^2) -- callers keep |r2/E^2 - 1| well above h.
 *   grad[12 i + k] += sum_r dl[r] w_g(i) d tau_ri / d theta_k ;  gabs the same sum of |.| (scale).
 * theta_in: n x 12 floats, the primitive's load inputs in that order (the scene's own float data). */
typedef struct {
    const or_scene *s; const float *theta; const float *rays; long n; uint32_t mask; const float *wts;
    const double *dl; double *grad; double *gabs;
} gradp_ctx;

static double tau_theta(const double th[12], double E2, const double o[3], const double v[3], double t0,
                        double t1) {
    double mu[3] = {th[0], th[1], th[2]}, sinv[9], wvec[3], norm, alpha = th[11], E2v = E2;
    or_scene s1;
    memset(&s1, 0, sizeof(s1));
    s1.n = 1; s1.mu = mu; s1.sinv = sinv; s1.wvec = wvec; s1.norm = &norm; s1.alpha = &alpha; s1.E2 = &E2v;
    derive_d(th + 3, th + 7, th[10], sinv, wvec, &norm);
    or_pair p;
    pair_setup(&s1, 0, o, v, t0, t1, &p);
    if (!p.hit) return 0.0;
    return alpha * seg_integral(&s1, 0, &p, p.tin, p.tout);
}

static void gradp_work(void *c_, long i) {
    const gradp_ctx *c = (const gradp_ctx *)c_;
    const or_scene *s = c->s;
    const int g = s->group[i];
    if (!((c->mask >> g) & 1u)) return;
    const double w = c->wts ? (double)c->wts[g] : 1.0;
    double th[12], hs[12];
    for (int k = 0; k < 12; ++k) th[k] = c->theta[12 * i + k];
    const double smin = fmin(th[7], fmin(th[8], th[9]));
    const double qn = sqrt(th[3] * th[3] + th[4] * th[4] + th[5] * th[5] + th[6] * th[6]);
    for (int k = 0; k < 3; ++k) hs[k] = 1e-3 * smin;
    for (int k = 3; k < 7; ++k) hs[k] = 1e-3 * qn;
    for (int k = 7; k < 10; ++k) hs[k] = 1e-3 * th[k];
    hs[10] = 1e-3 * fmax(1.0, fabs(th[10]));
    hs[11] = 1e-3 * fmax(1.0, fabs(th[11]));
    for (long r = 0; r < c->n; ++r) {
        const float *ray = c->rays + 8 * r;
        double o[3] = {ray[0], ray[1], ray[2]}, v[3] = {ray[4], ray[5], ray[6]};
        or_pair p;
        pair_setup(s, (int)i, o, v, ray[3], ray[7], &p);
        if (!p.hit || c->dl[r] == 0.0) continue;
        for (int k = 0; k < 12; ++k) {
            double D[2];
            for (int m = 0; m < 2; ++m) {
                const double h = m == 0 ? hs[k] : 0.5 * hs[k];
                double tp[12], tm[12];
                memcpy(tp, th, sizeof(th)); memcpy(tm, th, sizeof(th));
                tp[k] += h; tm[k] -= h;
                D[m] = (tau_theta(tp, s->E2[i], o, v, ray[3], ray[7]) - tau_theta(tm, s->E2[i], o, v, ray[3], ray[7])) /
                       (2.0 * h);
            }
            const double d = (4.0 * D[1] - D[0]) / 3.0;
            c->grad[12 * i + k] += c->dl[r] * w * d;
            c->gabs[12 * i + k] += fabs(c->dl[r] * w * d);
        }
    }
}

void or_grad_params(const or_scene *s, const float *theta, const float *rays, long n, uint32_t mask,
                    const float *wts, const double *dl, double *grad, double *gabs, int nthreads) {
    for (long i = 0; i < 12L * s->n; ++i) { grad[i] = 0.0; gabs[i] = 0.0; }
    gradp_ctx c = {s, theta, rays, n, mask, wts, dl, grad, gabs};
    run_parallel(gradp_work, &c, s->n, nthreads);
}

/* candidate set of one ray (prims whose clipped chord has positive length) */
int or_candidates(const or_scene *s, const float *ray, uint32_t mask, int *ids, int cap, double *r2_out) {
    double o[3] = {ray[0], ray[1], ray[2]}, v[3] = {ray[4], ray[5], ray[6]};
    int m = 0;
    for (int i = 0; i < s->n; ++i) {
        if (!((mask >> s->group[i]) & 1u)) continue;
        or_pair p;
        pair_setup(s, i, o, v, ray[3], ray[7], &p);
        if (!p.hit) continue;
        if (m < cap) { ids[m] = i; if (r2_out) r2_out[m] = p.r2 / s->E2[i]; }
        ++m;
    }
    return m;
}

/* r2/E2 of a given (ray, prim) pair, for grazing classification of set differences */
double or_pair_r2_rel(const or_scene *s, int i, const float *ray) {
    double o[3] = {ray[0], ray[1], ray[2]}, v[3] = {ray[4], ray[5], ray[6]};
    or_pair p;
    pair_setup(s, i, o, v, ray[3], ray[7], &p);
    return p.r2 / s->E2[i];
}

/* ------------------------------------------------------------------------- */
/* Philox4x32-10 (Salmon et al., SC'11), written independently of the GPU one */
/* ------------------------------------------------------------------------- */
void or_philox(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int r = 0; r < 10; ++r) {
        uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
        k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Stream layout: uniform k of stream st at path vertex d of
   (pixel, sample) = word (k&3) of Philox(ctr=(pixel, sample, d, st<<16 | k>>2),
   key=(seed_lo, seed_hi)), mapped to (x>>8)*2^-24 in [0,1) (C16). */
enum { ST_EXT = 0, ST_NEE = 1, ST_SCAT = 2, ST_CAM = 3 };
static uint32_t stream_word(uint64_t seed, uint32_t pix, uint32_t smp, uint32_t d, uint32_t st, uint32_t k) {
    uint32_t ctr[4] = {pix, smp, d, (st << 16) | (k >> 2)};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t o[4];
    or_philox(ctr, key, o);
    return o[k & 3];
}
static float u01(uint32_t x) { return (float)(x >> 8) * (1.0f / 16777216.0f); }

float or_uniform(uint64_t seed, uint32_t pix, uint32_t smp, uint32_t d, uint32_t st, uint32_t k) {
    return u01(stream_word(seed, pix, smp, d, st, k));
}

/* ------------------------------------------------------------------------- */
/* LOD policies: Table B1 (levels) x Table B2 (orientation bins)              */
/* ------------------------------------------------------------------------- */
typedef struct {
    uint32_t static_mask;
    int32_t level_strategy;  /* 0 DET 1 UNIFORM 2 POWERLAW 3 UNIFORM_CV 4 POWERLAW_CV 5 POWERLAW_CV_ACCUM */
    float beta;
    int32_t orient_strategy; /* 0 DET 1 THRESH_CULL 2 UNIFORM 3 IMPORTANCE 4 THRESH_UNIFORM */
    float delta;
} or_policy;

/* Evaluate a policy for one ray segment.  ul = level uniform; uo[l-1] = the
   orientation uniform of Gabor level l; dir = ray direction (fp32); f0[g] =
   representative whitened frequency of group g (C12).  Writes mask and G
   weights (weights of unselected groups are 0). */
void or_policy_eval(const or_scene *s, const or_policy *pol, const float dir[3], float ul, const float *uo,
                    const float *f0, uint32_t *mask_out, float *w_out) {
    int P = s->P, K = s->K, G = s->G0;  /* draws over the G0 groups of one band */
    double lw[8];       /* per-level weight; 0 = level not selected */
    for (int l = 0; l < 8; ++l) lw[l] = 0.0;
    double om = 1.0 - pol->beta;
    uint32_t m24 = (uint32_t)(ul * 16777216.0f);  /* exact: ul = m24 * 2^-24 */
    switch (pol->level_strategy) {
    case 1: { /* Uniform: level floor(u P), weight P (Table B1 row 2) */
        int j = (int)(((uint64_t)m24 * (uint64_t)P) >> 24);
        lw[j] = P;
        break;
    }
    case 2: { /* Power law: x = u^(1/(1-beta)), bucket [j/P,(j+1)/P], weight 1/(b^(1-b)-a^(1-b)) (C13) */
        int j = 0;
        for (int k = 1; k < P; ++k) if ((double)ul >= pow((double)k / P, om)) j = k;
        lw[j] = 1.0 / (pow((double)(j + 1) / P, om) - pow((double)j / P, om));
        break;
    }
    case 3: { /* Uniform + CV: level 0 (w=1) + one of 1..P-1, weight P-1 */
        lw[0] = 1.0;
        if (P > 1) { int j = 1 + (int)(((uint64_t)m24 * (uint64_t)(P - 1)) >> 24); lw[j] = P - 1; }
        break;
    }
    case 4: { /* Power law + CV: level 0 (w=1) + Gabor level from P-1 power-law buckets (C13) */
        lw[0] = 1.0;
        if (P > 1) {
            int Q = P - 1, k = 0;
            for (int q = 1; q < Q; ++q) if ((double)ul >= pow((double)q / Q, om)) k = q;
            lw[1 + k] = 1.0 / (pow((double)(k + 1) / Q, om) - pow((double)k / Q, om));
        }
        break;
    }
    case 5: { /* Power law + CV (Accum.): k by power law, render levels 0..k, w_j = 1/(1-(j/P)^(1-b)) (C14) */
        int kk = 0;
        for (int q = 1; q < P; ++q) if ((double)ul >= pow((double)q / P, om)) kk = q;
        for (int j = 0; j <= kk; ++j) lw[j] = 1.0 / (1.0 - pow((double)j / P, om));
        break;
    }
    default: /* Deterministic */
        for (int l = 0; l < P; ++l) lw[l] = 1.0;
    }
    uint32_t mask = 0;
    float w[OR_MAXG];
    for (int g = 0; g < OR_MAXG; ++g) w[g] = 0.0f;
    if (lw[0] != 0.0) { mask |= 1u; w[0] = (float)lw[0]; }  /* Gaussians never orientation-masked (C15) */
    for (int l = 1; l < P; ++l) {
        if (lw[l] == 0.0) continue;
        float bw[32];
        for (int b = 0; b < K; ++b) bw[b] = 0.0f;
        float a[32];
        for (int b = 0; b < K; ++b) {
            const float *o = s->bin_axes + 3 * b;
            a[b] = fabsf(fmaf(dir[0], o[0], fmaf(dir[1], o[1], dir[2] * o[2])));  /* a_i = |v . o_i| */
        }
        float u = uo[l - 1];
        uint32_t mu24 = (uint32_t)(u * 16777216.0f);
        switch (pol->orient_strategy) {
        case 1: /* Threshold culling: bins with a_i <= delta, weight 1 */
            for (int b = 0; b < K; ++b) if (a[b] <= pol->delta) bw[b] = 1.0f;
            break;
        case 2: { /* Uniform: one bin, weight K */
            int b = (int)(((uint64_t)mu24 * (uint64_t)K) >> 24);
            bw[b] = (float)K;
            break;
        }
        case 3: { /* Importance: p_i = w_i/W, weight W/w_i, w_i = exp(-f0^2 a_i^2 / 2) (C12) */
            float wi[32], W = 0.0f;
            for (int b = 0; b < K; ++b) {
                float f = f0 ? f0[1 + (l - 1) * K + b] : 0.0f;
                float x = f * a[b];
                wi[b] = expf(-0.5f * (x * x));
                W += wi[b];
            }
            if (!(W > 0.0f) || !isfinite(W)) { /* degenerate -> uniform fallback */
                int b = (int)(((uint64_t)mu24 * (uint64_t)K) >> 24);
                bw[b] = (float)K;
            } else {
                float t = u * W, c = 0.0f;
                int pick = K - 1;
                for (int b = 0; b < K; ++b) { c += wi[b]; if (t < c) { pick = b; break; } }
                bw[pick] = W / wi[pick];
            }
            break;
        }
        case 4: { /* Threshold + uniform: a_i <= delta weight 1; one of the rest, weight N_above */
            int nab = 0;
            for (int b = 0; b < K; ++b) { if (a[b] <= pol->delta) bw[b] = 1.0f; else ++nab; }
            if (nab > 0) {
                int pickn = (int)(((uint64_t)mu24 * (uint64_t)nab) >> 24), c = 0;
                for (int b = 0; b < K; ++b)
                    if (!(a[b] <= pol->delta)) { if (c == pickn) { bw[b] = (float)nab; break; } ++c; }
            }
            break;
        }
        default:
            for (int b = 0; b < K; ++b) bw[b] = 1.0f;
        }
        for (int b = 0; b < K; ++b) {
            if (bw[b] == 0.0f) continue;
            int g = 1 + (l - 1) * K + b;
            mask |= 1u << g;
            w[g] = (float)(lw[l] * (double)bw[b]);
        }
    }
    /* spatial bands (C24): the same draw applies to every band's copy of the groups */
    for (int bd = 1; bd < s->n_bands; ++bd) {
        mask |= (mask & ((1u << G) - 1u)) << (bd * G);
        for (int g = 0; g < G; ++g) w[bd * G + g] = w[g];
    }
    mask &= pol->static_mask;
    for (int g = 0; g < s->G; ++g) { if (!((mask >> g) & 1u)) w[g] = 0.0f; w_out[g] = w[g]; }
    *mask_out = mask;
}

/* batch form for the unbiasedness pins: n draws, uo has (P-1) uniforms per draw */
void or_policy_eval_batch(const or_scene *s, const or_policy *pol, const float *dirs, const float *ul,
                          const float *uo, const float *f0, long n, uint32_t *masks, float *w) {
    for (long i = 0; i < n; ++i)
        or_policy_eval(s, pol, dirs + 3 * i, ul[i], uo + (size_t)i * (s->P > 1 ? s->P - 1 : 1), f0, masks + i,
                       w + (size_t)i * s->G);
}

/* ------------------------------------------------------------------------- */
/* Free-flight distance sampling, Eq. 5 by segments (Eq. 4) and  */
/* bisection.  t* = first t with cumulative tau >= tau* (C17).        */
/* ------------------------------------------------------------------------- */
typedef struct { double t; int id; int kind; } or_event;  /* kind 0 enter, 1 exit */
static int ev_cmp(const void *x, const void *y) {
    const or_event *a = (const or_event *)x, *b = (const or_event *)y;
    if (a->t < b->t) return -1;
    if (a->t > b->t) return 1;
    if (a->id != b->id) return a->id < b->id ? -1 : 1;
    return a->kind - b->kind;
}

typedef struct { int idx; or_pair p; double w; } or_active;

static double active_sum(const or_scene *s, const or_active *act, const int *on, int nact, double ta, double tb) {
    neum acc = {0, 0};
    for (int k = 0; k < nact; ++k) {
        if (!on[k]) continue;
        const or_active *A = act + k;
        double lo = ta > A->p.tin ? ta : A->p.tin, hi = tb < A->p.tout ? tb : A->p.tout;
        neum_add(&acc, A->w * s->alpha[A->idx] * seg_integral(s, A->idx, &A->p, lo, hi));
    }
    return neum_get(&acc);
}

/* returns 1 and *t_out on collision, 0 on escape; *tau_total = tau over the
   whole ray if escaped (for diagnostics). */
static int free_flight_f(const or_scene *s, const double o[3], const double v[3], double t0, double t1,
                         uint32_t mask, const float *wts, double xi, double fmax, double *t_out);
int or_free_flight(const or_scene *s, const double o[3], const double v[3], double t0, double t1,
                   uint32_t mask, const float *wts, double xi, double *t_out) {
    return free_flight_f(s, o, v, t0, t1, mask, wts, xi, INFINITY, t_out);
}
static int free_flight_f(const or_scene *s, const double o[3], const double v[3], double t0, double t1,
                         uint32_t mask, const float *wts, double xi, double fmax, double *t_out) {
    double tstar = -log1p(-xi);  /* tau* = -ln(1 - xi)  (Eq. 5) */
    if (tstar <= 0.0) { *t_out = t0; return 1; }
    int cap = 64, nact = 0;
    or_active *act = malloc(sizeof(or_active) * cap);
    for (int i = 0; i < s->n; ++i) {
        int g = s->group[i];
        if (!((mask >> g) & 1u)) continue;
        or_pair p;
        pair_setup(s, i, o, v, t0, t1, &p);
        if (!p.hit) continue;
        if (fabs(p.B) > fmax) continue;  /* foveation (F4) */
        if (nact == cap) { cap *= 2; act = realloc(act, sizeof(or_active) * cap); }
        act[nact].idx = i; act[nact].p = p; act[nact].w = wts ? wts[g] : 1.0;
        ++nact;
    }
    or_event *ev = malloc(sizeof(or_event) * (2 * nact + 1));
    for (int k = 0; k < nact; ++k) {
        ev[2 * k].t = act[k].p.tin;  ev[2 * k].id = k; ev[2 * k].kind = 0;
        ev[2 * k + 1].t = act[k].p.tout; ev[2 * k + 1].id = k; ev[2 * k + 1].kind = 1;
    }
    qsort(ev, 2 * nact, sizeof(or_event), ev_cmp);
    int *on = calloc(nact > 0 ? nact : 1, sizeof(int));
    double cum = 0.0;
    int found = 0;
    for (int e = 0; e < 2 * nact; ++e) {
        /* apply the event, then the segment [ev[e].t, ev[e+1].t] has a constant active set */
        on[ev[e].id] = ev[e].kind == 0;
        if (e + 1 >= 2 * nact) break;
        double ta = ev[e].t, tb = ev[e + 1].t;
        if (!(tb > ta)) continue;
        double seg = active_sum(s, act, on, nact, ta, tb);
        if (cum + seg >= tstar) {
            /* bisection in the bracketing segment to |dt| <= 1e-12 (1+|t|) */
            double lo = ta, hi = tb;
            for (int it = 0; it < 200 && (hi - lo) > 1e-12 * (1.0 + fabs(lo)); ++it) {
                double mid = 0.5 * (lo + hi);
                double f = cum + active_sum(s, act, on, nact, ta, mid) - tstar;
                if (f >= 0.0) hi = mid; else lo = mid;
            }
            *t_out = 0.5 * (lo + hi);
            found = 1;
            break;
        }
        cum += seg;
    }
    free(on); free(ev); free(act);
    return found;
}

/* tau(ta, tb) of a set of chords, each clipped to [ta, tb] (chords outside add nothing) */
static double clipped_sum(const or_scene *s, const or_active *act, int nact, double ta, double tb) {
    neum acc = {0, 0};
    for (int k = 0; k < nact; ++k) {
        const or_active *A = act + k;
        double lo = ta > A->p.tin ? ta : A->p.tin, hi = tb < A->p.tout ? tb : A->p.tout;
        if (!(hi > lo)) continue;
        neum_add(&acc, A->w * s->alpha[A->idx] * seg_integral(s, A->idx, &A->p, lo, hi));
    }
    return neum_get(&acc);
}

/* Diagnostics of a candidate free-flight distance t_q (tests of the GPU root, C17): out[0] =
   tau(t0, t_q) by the closed form; out[1] = the largest cumulative tau at an event point (chord
   entry/exit) before t_q, i.e. how close an EARLIER segment end came to tau*; out[2] = tau*. */
void or_free_flight_diag(const or_scene *s, const float *ray, uint32_t mask, const float *wts, double xi, double t_q,
                         double *out) {
    double o[3] = {ray[0], ray[1], ray[2]}, v[3] = {ray[4], ray[5], ray[6]};
    double t0 = ray[3], t1 = ray[7];
    int cap = 64, nact = 0;
    or_active *act = malloc(sizeof(or_active) * cap);
    for (int i = 0; i < s->n; ++i) {
        int g = s->group[i];
        if (!((mask >> g) & 1u)) continue;
        or_pair p;
        pair_setup(s, i, o, v, t0, t1, &p);
        if (!p.hit) continue;
        if (nact == cap) { cap *= 2; act = realloc(act, sizeof(or_active) * cap); }
        act[nact].idx = i; act[nact].p = p; act[nact].w = wts ? wts[g] : 1.0;
        ++nact;
    }
    out[0] = clipped_sum(s, act, nact, t0, t_q);
    double best = -INFINITY;
    for (int k = 0; k < nact; ++k) {
        const double te[2] = {act[k].p.tin, act[k].p.tout};
        for (int e = 0; e < 2; ++e) {
            if (!(te[e] < t_q)) continue;
            double c = clipped_sum(s, act, nact, t0, te[e]);
            if (c > best) best = c;
        }
    }
    out[1] = best;
    out[2] = -log1p(-xi);
    free(act);
}

int or_free_flight_f(const or_scene *s, const float *ray, uint32_t mask, const float *wts, double xi, double *t_out) {
    double o[3] = {ray[0], ray[1], ray[2]}, v[3] = {ray[4], ray[5], ray[6]};
    return or_free_flight(s, o, v, ray[3], ray[7], mask, wts, xi, t_out);
}

/* ------------------------------------------------------------------------- */
/* Path estimator -- tomography, single and multiple scattering */
/* ------------------------------------------------------------------------- */
typedef struct {
    int32_t mode;          /* 0 TOMO, 1 SCATTER */
    int32_t width, height, max_depth, jitter;
    float cam_pos[3], cam_fwd[3], cam_right[3], cam_up[3];  /* right/up pre-scaled by tan(fov/2)(*aspect) */
    float albedo, hg_g, sun_dir[3], sun_E, env_L;
    uint64_t seed;
    or_policy ext, nee;
    const float *group_f0;  /* G floats (C12), NULL -> the scene's medians (group_f0_of) */
    int32_t foveation;      /* foveated rendering: mode bits, 1 levels, 2 continuous */
    float fov_gaze[2], fov_f0, fov_slope, fov_jitter;
    int32_t motion_blur;    /* motion-blur reference */
    float mb_dir[3], mb_m;
} or_render_desc;

/* Foveation threshold of a pixel ("a linear relationship between eccentricity and the
   frequency threshold", readings F1-F3, F5): e = |(px+0.5, py+0.5) - gaze| / max(W, H),
   f_max = max(0, f0 - slope e), stochastic smoothing f_max (1 + jitter (2u - 1)) with u of stream 6.
   fp32, one rounding per operation (the GPU evaluates the same expression bit for bit). */
#define ST_FOV 6u
static float fov_fmax(const or_render_desc *d, uint32_t pix, uint32_t smp) {
    float px = (float)(pix % (uint32_t)d->width), py = (float)(pix / (uint32_t)d->width);
    volatile float dx = (px + 0.5f) - d->fov_gaze[0], dy = (py + 0.5f) - d->fov_gaze[1];
    volatile float dd = dx * dx;
    volatile float ee = dy * dy;
    float e = sqrtf(dd + ee) / (float)(d->width > d->height ? d->width : d->height);
    volatile float se = d->fov_slope * e;
    float fm = d->fov_f0 - se;
    if (!(fm > 0.0f)) fm = 0.0f;
    if (d->fov_jitter > 0.0f) {
        float u = or_uniform(d->seed, pix, smp, 0, ST_FOV, 0);
        volatile float tu = 2.0f * u;
        volatile float j = d->fov_jitter * (tu - 1.0f);
        fm = fm * (1.0f + j);
    }
    return fm;
}
/* Level masking ("discard all levels that contain Gabor primitives with frequencies above
   the threshold", reading F3): level l >= 1 kept iff its maximum frequency <= f_max; level 0 kept */
static uint32_t fov_mask(const or_scene *s, const or_render_desc *d, float fm) {
    (void)d;
    uint32_t m = 1u;
    for (int l = 1; l < s->P; ++l)
        if (s->lfmax[l] <= fm)
            for (int b = 0; b < s->K; ++b) m |= 1u << (1 + (l - 1) * s->K + b);
    for (int bd = 1; bd < s->n_bands; ++bd) m |= (m & ((1u << s->G0) - 1u)) << (bd * s->G0);
    return m;
}
float or_fov_fmax(const or_render_desc *d, uint32_t pix, uint32_t smp) { return fov_fmax(d, pix, smp); }

/* camera ray in fp32 with explicit fused ops (bit-identical to the GPU) */
static void camera_ray(const or_render_desc *d, int px, int py, float jx, float jy, float o[3], float v[3]) {
    float fx = (float)px + jx, fy = (float)py + jy;
    float iw2 = 2.0f / (float)d->width, ih2 = 2.0f / (float)d->height;
    float sx = fmaf(fx, iw2, -1.0f), sy = fmaf(-fy, ih2, 1.0f);
    float r[3];
    for (int k = 0; k < 3; ++k) r[k] = fmaf(sy, d->cam_up[k], fmaf(sx, d->cam_right[k], d->cam_fwd[k]));
    float len = sqrtf(fmaf(r[0], r[0], fmaf(r[1], r[1], r[2] * r[2])));
    for (int k = 0; k < 3; ++k) { v[k] = r[k] / len; o[k] = d->cam_pos[k]; }
}

/* Henyey-Greenstein phase function (reading C19) */
static double hg_eval(double g, double cost) {
    double den = 1.0 + g * g - 2.0 * g * cost;
    return (1.0 - g * g) / (4.0 * OR_PI * den * sqrt(den));
}
static void hg_sample(double g, const double v[3], double u1, double u2, double out[3]) {
    double cost;
    if (fabs(g) < 1e-3) cost = 1.0 - 2.0 * u1;
    else { double q = (1.0 - g * g) / (1.0 - g + 2.0 * g * u1); cost = (1.0 + g * g - q * q) / (2.0 * g); }
    if (cost > 1.0) cost = 1.0;
    if (cost < -1.0) cost = -1.0;
    double sint = sqrt(fmax(0.0, 1.0 - cost * cost)), phi = 2.0 * OR_PI * u2;
    /* orthonormal basis around v (Duff et al. 2017) */
    double sgn = v[2] >= 0.0 ? 1.0 : -1.0;
    double a = -1.0 / (sgn + v[2]), b = v[0] * v[1] * a;
    double t1[3] = {1.0 + sgn * v[0] * v[0] * a, sgn * b, -sgn * v[0]};
    double t2[3] = {b, sgn + v[1] * v[1] * a, -v[1]};
    for (int k = 0; k < 3; ++k) out[k] = sint * cos(phi) * t1[k] + sint * sin(phi) * t2[k] + cost * v[k];
    double n = sqrt(out[0] * out[0] + out[1] * out[1] + out[2] * out[2]);
    for (int k = 0; k < 3; ++k) out[k] /= n;
}

static void eval_pol(const or_scene *s, const or_render_desc *d, const or_policy *pol, const float dir[3],
                     uint32_t pix, uint32_t smp, uint32_t dep, uint32_t st, uint32_t k_level,
                     uint32_t *mask, float *w) {
    float ul = or_uniform(d->seed, pix, smp, dep, st, k_level);
    float uo[8];
    for (int l = 1; l < s->P; ++l) uo[l - 1] = or_uniform(d->seed, pix, smp, dep, st, k_level + l);
    or_policy_eval(s, pol, dir, ul, uo, d->group_f0 ? d->group_f0 : s->f0, mask, w);
}

/* one (pixel, sample) path; returns the estimate, *nrays = ray queries traced */
double or_path(const or_scene *s, const or_render_desc *d, uint32_t pix, uint32_t smp, int *nrays) {
    int px = (int)(pix % (uint32_t)d->width), py = (int)(pix / (uint32_t)d->width);
    float jx = 0.5f, jy = 0.5f;
    if (d->jitter) { jx = or_uniform(d->seed, pix, smp, 0, ST_CAM, 0); jy = or_uniform(d->seed, pix, smp, 0, ST_CAM, 1); }
    float of[3], vf[3];
    camera_ray(d, px, py, jx, jy, of, vf);
    if (d->motion_blur) {
        /* P:L656 "a convolution with a 1D box filter oriented in direction d and with size m": the
           field at exposure time u is shifted by s = m (u - 1/2) d, the same as a camera at -s
           (readings M1, M2); fp32, one rounding per operation */
        float u = or_uniform(d->seed, pix, smp, 0, 7u, 0);
        volatile float sh = d->mb_m * (u - 0.5f);
        for (int k = 0; k < 3; ++k) {
            volatile float sk = sh * d->mb_dir[k];
            of[k] = of[k] - sk;
        }
    }
    int nr = 0;
    uint32_t mask;
    float w[OR_MAXG];
    /* foveation: one threshold per (pixel, sample) for every ray of the path */
    /* foveation mode bit 0: level masking (F3), bit 1: the continuous per-primitive check (F4) */
    const float fth = d->foveation ? fov_fmax(d, pix, smp) : INFINITY;
    const float fmx = (d->foveation & 2) ? fth : INFINITY;
    const uint32_t fovm = (d->foveation & 1) ? fov_mask(s, d, fth) : 0xFFFFFFFFu;
    if (d->mode == 0) {  /* tomography: tau-hat of the camera ray */
        eval_pol(s, d, &d->ext, vf, pix, smp, 0, ST_EXT, 1, &mask, w);
        mask &= fovm;
        double o[3] = {of[0], of[1], of[2]}, v[3] = {vf[0], vf[1], vf[2]};
        double tau = trace_one_f(s, o, v, 0.0, INFINITY, mask, w, fmx, NULL, NULL, NULL);
        if (nrays) *nrays = 1;
        return tau;
    }
    double o[3] = {of[0], of[1], of[2]}, v[3] = {vf[0], vf[1], vf[2]};
    double beta = 1.0, L = 0.0;
    double sun[3] = {d->sun_dir[0], d->sun_dir[1], d->sun_dir[2]};
    for (int dep = 0; dep < d->max_depth; ++dep) {
        float vfl[3] = {(float)v[0], (float)v[1], (float)v[2]};
        eval_pol(s, d, &d->ext, vfl, pix, smp, dep, ST_EXT, 1, &mask, w);
        mask &= fovm;
        double xi = or_uniform(d->seed, pix, smp, dep, ST_EXT, 0);
        double tstar;
        ++nr;
        if (!free_flight_f(s, o, v, 0.0, INFINITY, mask, w, xi, fmx, &tstar)) {
            L += beta * d->env_L;  /* escape -> environment */
            break;
        }
        double x[3] = {o[0] + tstar * v[0], o[1] + tstar * v[1], o[2] + tstar * v[2]};
        /* next-event estimation toward the directional light with its own policy */
        uint32_t mn;
        float wn[OR_MAXG];
        eval_pol(s, d, &d->nee, d->sun_dir, pix, smp, dep, ST_NEE, 0, &mn, wn);
        mn &= fovm;
        double tn = trace_one_f(s, x, sun, 0.0, INFINITY, mn, wn, fmx, NULL, NULL, NULL);
        ++nr;
        double cost = v[0] * sun[0] + v[1] * sun[1] + v[2] * sun[2];
        L += beta * d->albedo * hg_eval(d->hg_g, cost) * exp(-tn) * d->sun_E;
        if (dep + 1 >= d->max_depth) break;
        double nv[3];
        hg_sample(d->hg_g, v, or_uniform(d->seed, pix, smp, dep, ST_SCAT, 0), or_uniform(d->seed, pix, smp, dep, ST_SCAT, 1), nv);
        beta *= d->albedo;
        for (int k = 0; k < 3; ++k) { o[k] = x[k]; v[k] = nv[k]; }
    }
    if (nrays) *nrays = nr;
    return L;
}

typedef struct {
    const or_scene *s; const or_render_desc *d; const int32_t *pix; int spp_begin, spp_count;
    double *out; int *nrays;
} render_ctx;
static void render_work(void *c, long idx) {
    render_ctx *r = (render_ctx *)c;
    long p = idx / r->spp_count, k = idx % r->spp_count;
    int nr = 0;
    r->out[idx] = or_path(r->s, r->d, (uint32_t)r->pix[p], (uint32_t)(r->spp_begin + k), &nr);
    if (r->nrays) r->nrays[idx] = nr;
}

/* out[p*spp_count + k] = estimate of sample spp_begin+k at probe pixel pix[p] */
void or_render_probes(const or_scene *s, const or_render_desc *d, const int32_t *pix, long n_probe,
                      int spp_begin, int spp_count, double *out, int *nrays, int nthreads) {
    render_ctx c = {s, d, pix, spp_begin, spp_count, out, nrays};
    run_parallel(render_work, &c, n_probe * spp_count, nthreads);
}

/* camera ray exposed for tests */
void or_camera_ray(const or_render_desc *d, int px, int py, float jx, float jy, float *o, float *v) {
    camera_ray(d, px, py, jx, jy, o, v);
}
double or_hg_eval(double g, double cost) { return hg_eval(g, cost); }
void or_hg_sample(double g, const double *v, double u1, double u2, double *out) { hg_sample(g, v, u1, u2, out); }
size_t or_sizeof_render_desc(void) { return sizeof(or_render_desc); }
size_t or_sizeof_policy(void) { return sizeof(or_policy); }
