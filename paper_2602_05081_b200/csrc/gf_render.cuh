// gf_render.cuh -- device building blocks of the render path shared by its translation units:
// gf_render.cu (wavefront orchestration, camera rays, accumulation), gf_ff.cu (one-pass free flight of
// extension rays), gf_ffa_pkt.cu / gf_ffa_w.cu (free flight pass A), gf_ffb.cu (pass B, tracking
// estimators), gf_nee.cu (next-event estimation, tomography).
// Without relocatable device code every unit compiles its own copy of these inline functions.
#pragma once
#include <algorithm>

#include "gf_device.cuh"
#include "gf.h"
#include "gf_internal.h"

namespace gfk {

#ifndef GF_FF_COARSE
#define GF_FF_COARSE 16
#endif
#ifndef GF_FF_FINE
#define GF_FF_FINE 1
#endif

// qcount slots: queue counts and work cursors
enum { QC_A = 0, QC_B = 1, QC_NEXT = 2, QC_W = 3, CUR_A = 4, CUR_W = 5, CUR_N = 6, QC_O = 7, CUR_O = 8, QC_V = 9,
       CUR_V = 10 };
#ifndef GF_REC_CAP
#define GF_REC_CAP 2048
#endif
constexpr int kRecCap = GF_REC_CAP;  // records per warp buffer: pass-B windows and the tracking estimators
#ifndef GF_REFS
#define GF_REFS 0  // 1: pass A keeps each ray's hit list and solves the crossing bin from it in-kernel
                  // (measured slower: the traversal kernels lose occupancy to the resolve's registers)
#endif
constexpr int kRefCapW = 4096;  // hit-list entries per ray of the warp-per-ray pass A (more: re-traversal)
constexpr int kRefCapL = 512;   // hit-list entries per lane of the packet pass A
constexpr int kRefWarp = GF_REFS ? (kRefCapW > 32 * kRefCapL ? kRefCapW : 32 * kRefCapL) : 32;  // u32 per warp buffer
// pixel of path p in this pass (-1 if p maps outside the image / shard)
__device__ __forceinline__ int32_t path_pixel(const RenderDev& R, int64_t p) {
    const int64_t gp = R.path_base + p;
    if (R.probe) return gp < R.n_total ? R.probe[gp] : -1;
    return shard_path_pixel(gp, R.cam.W, R.cam.H, R.shard_kind, R.shard_rank, R.shard_world);
}

// warp-aggregated queue push (called by all 32 lanes of the warp)
__device__ __forceinline__ void push(uint32_t* q, uint32_t* cnt, bool pred, uint32_t val) {
    const unsigned m = __ballot_sync(0xFFFFFFFFu, pred);
    if (!m) return;
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(m) - 1;
    uint32_t base = 0;
    if (lane == leader) base = atomicAdd(cnt, (uint32_t)__popc(m));
    base = __shfl_sync(0xFFFFFFFFu, base, leader);
    if (pred) q[base + __popc(m & ((1u << lane) - 1u))] = val;
}

// dynamic fetch of 32 work items per warp (all lanes call it)
__device__ __forceinline__ bool fetch(uint32_t* work, uint32_t count, uint32_t& base) {
    uint32_t b = 0;
    if ((threadIdx.x & 31) == 0) b = atomicAdd(work, 32u);
    base = __shfl_sync(0xFFFFFFFFu, b, 0);
    return base < count;
}

__device__ __forceinline__ void count_rays(unsigned long long* c, bool active) {
    const unsigned m = __ballot_sync(0xFFFFFFFFu, active);
    if ((threadIdx.x & 31) == 0 && m) atomicAdd(c, (unsigned long long)__popc(m));
}

__device__ __forceinline__ float3 ld3(const float* x, const float* y, const float* z, uint32_t p) {
    return make_float3(x[p], y[p], z[p]);
}

// Foveated rendering (readings F1-F5 in DESIGN.md §3): per pixel a
// frequency threshold linear in the eccentricity, f_max = max(0, f_fovea - slope e), e = |pixel centre -
// gaze| / max(W, H), jittered by (1 + sigma (2u - 1)) (u: stream 6, k = 0, per pixel and sample);
// levels whose maximum frequency exceeds f_max are masked for every ray of the path, and a remaining
// primitive is skipped when its frequency along the ray |omega_vec . d| exceeds f_max (prim_setup).
// Correctly rounded fp32 ops: the oracle computes the same f_max bit for bit.
template <bool FOV>
__device__ __forceinline__ float fov_fmax(const RenderDev& R, uint32_t pix, uint32_t sample) {
    if (!FOV || !R.fov) return INFINITY;
    const float px = (float)(pix % (uint32_t)R.cam.W), py = (float)(pix / (uint32_t)R.cam.W);
    const float dx = __fsub_rn(__fadd_rn(px, 0.5f), R.fov_gaze[0]), dy = __fsub_rn(__fadd_rn(py, 0.5f), R.fov_gaze[1]);
    const float e = __fdiv_rn(__fsqrt_rn(__fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy))),
                              (float)max(R.cam.W, R.cam.H));
    float fm = fmaxf(0.0f, __fsub_rn(R.fov_f0, __fmul_rn(R.fov_slope, e)));
    if (R.fov_jitter > 0.0f) {
        const float u = stream_u(R.seed, pix, sample, 0, ST_FOV, 0);
        fm = __fmul_rn(fm, __fadd_rn(1.0f, __fmul_rn(R.fov_jitter, __fsub_rn(__fmul_rn(2.0f, u), 1.0f))));
    }
    return fm;
}
template <bool FOV>
__device__ __forceinline__ uint32_t fov_mask(const RenderDev& R, float fm) {
    if (!FOV || !(R.fov & 1)) return 0xFFFFFFFFu;  // mode bit 0: level masking (F3)
    uint32_t m = 1u;  // level 0 (Gaussians, frequency 0) always
    for (int l = 1; l < R.sc.P; ++l)
        if (R.fov_lfmax[l] <= fm)
            for (int b = 0; b < R.sc.K; ++b) m |= 1u << (1 + (l - 1) * R.sc.K + b);
    for (int bd = 1; bd < R.sc.n_bands; ++bd) m |= (m & ((1u << R.sc.G0) - 1u)) << (bd * R.sc.G0);
    return m;
}
// mode bit 1: the continuous per-primitive check (F4) uses the threshold, else none
__device__ __forceinline__ float fov_prim(const RenderDev& R, float fm) { return (R.fov & 2) ? fm : INFINITY; }


// Motion-blur reference (readings M1-M3): the field moves by s = m (u - 1/2) dir during
// the exposure (a box filter of length m along dir); a sample at time u sees the field shifted by s,
// i.e. the whole path runs in the static field from the camera origin shifted by -s.  u: stream 7,
// k = 0, depth 0, per (pixel, sample); correctly rounded fp32 as in the oracle.
__device__ __forceinline__ void mb_shift(const RenderDev& R, uint32_t pix, uint32_t sample, float3& o) {
    if (!R.mb) return;
    const float u = stream_u(R.seed, pix, sample, 0, ST_MB, 0);
    const float sh = __fmul_rn(R.mb_m, __fsub_rn(u, 0.5f));
    o.x = __fsub_rn(o.x, __fmul_rn(sh, R.mb_dir[0]));
    o.y = __fsub_rn(o.y, __fmul_rn(sh, R.mb_dir[1]));
    o.z = __fsub_rn(o.z, __fmul_rn(sh, R.mb_dir[2]));
}

// ---------------------------------------------------------------- free flight: common per-ray set-up
struct FFRay {
    float3 o, d;
    uint32_t pix, mask;
    float fth;           // foveation threshold (INFINITY: off)
    double tstar;        // tau* = -ln(1 - xi)
    float tlo, thi;      // the ray's scene interval (root box within [tmin, tmax])
    float bw, ibw;       // t-bin width and its inverse
    const float* w;      // group weights (stochastic masks: the path's row of R.pw, k_policy)
};

// Per-ray set-up, identical in both passes (recomputed, deterministic): mask and weights (a3),
// tau* (Eq. 5, C16) and [tlo, thi].  Returns 0 if the ray collides at its origin (tau* = 0), 1 if
// it misses the scene (escape), 2 if it must be traced.
template <bool STOCH, bool FOV>
__device__ __forceinline__ int ff_begin(const RenderDev& R, uint32_t p, int32_t sample, int32_t depth, FFRay& f) {
    f.pix = R.pix[p];
    f.o = ld3(R.ox, R.oy, R.oz, p);
    f.d = ld3(R.dx, R.dy, R.dz, p);
    f.fth = fov_fmax<FOV>(R, f.pix, (uint32_t)sample);
    // stochastic masks: drawn once per path and depth by k_policy (out of the traversal kernels, whose
    // instruction cache the Table B1/B2 code would share), the same for pass A and pass B
    f.w = R.pw + (size_t)p * kMaxGroups;
    f.mask = fov_mask<FOV>(R, f.fth) & (STOCH ? R.pmask[p] : R.ext.static_mask);
    const float xi = stream_u(R.seed, f.pix, (uint32_t)sample, (uint32_t)depth, ST_EXT, 0);
    f.tstar = -log1p(-(double)xi);  // tau* = -ln(1 - xi)   (Eq. 5, C16)
    const float t0 = R.trays ? R.trays[8 * (R.path_base + p) + 3] : 0.0f;  // gf_trace_free_flight: the ray's
    const float t1 = R.trays ? R.trays[8 * (R.path_base + p) + 7] : INFINITY;  // [tmin, tmax]; render: [0, inf)
    f.tlo = f.thi = t0;
    f.bw = f.ibw = 0.0f;
    if (f.tstar <= 0.0) return 0;
    const RayDev r = make_ray(f.o, f.d, 0.0f, INFINITY);
    if (R.n_nodes == 0 || !slab_range(r, R.root_lo, R.root_hi, t0, t1, f.tlo, f.thi)) return 1;
    f.bw = (f.thi - f.tlo) * (1.0f / GF_FF_COARSE);  // coarse bin width (kNC coarse bins, below)
    f.ibw = f.bw > 0.0f ? 1.0f / f.bw : 0.0f;
    return 2;
}

// GF_EST_UNIFORM (reading U1): t* uniform in the crossing bin k, no root finding
__device__ __forceinline__ float ff_uniform_t(const RenderDev& R, const FFRay& f, int32_t sample, int32_t depth, int k) {
    const float a = k <= 0 ? f.tlo : fmaf((float)k, f.bw, f.tlo);
    const float b = k >= GF_FF_COARSE - 1 ? f.thi : fmaf((float)(k + 1), f.bw, f.tlo);
    return fminf(fmaf(stream_u(R.seed, f.pix, (uint32_t)sample, (uint32_t)depth, ST_UNI, 0), b - a, a), b);
}

__device__ __forceinline__ void ff_escape(const RenderDev& R, uint32_t p) {
    R.L[p] += R.beta[p] * R.env_L;  // escape -> environment
    if (R.tout) R.tout[R.path_base + p] = INFINITY;
}
// the collision point becomes the path's new origin
__device__ __forceinline__ void ff_collide(const RenderDev& R, uint32_t p, const FFRay& f, float t, float kap = 0.0f) {
    R.fkap[p] = kap;
    R.ox[p] = fmaf(t, f.d.x, f.o.x);
    R.oy[p] = fmaf(t, f.d.y, f.o.y);
    R.oz[p] = fmaf(t, f.d.z, f.o.z);
    if (R.tout) R.tout[R.path_base + p] = t;
}

// Camera-projective box test of a depth-0 ray (camera BVH, see gf_launch_build_frame): the ray is the
// point (a, b) = (d.r, d.u) / d.f and its depth q.f = t d.f covers [t0, t1] d.f.
struct CamPt {
    float pa, pb, dfw;
};
__device__ __forceinline__ CamPt cam_point(const RenderDev& R, float3 d) {
    CamPt c;
    c.dfw = fmaf(d.x, R.cb[6], fmaf(d.y, R.cb[7], d.z * R.cb[8]));
    c.pa = fmaf(d.x, R.cb[0], fmaf(d.y, R.cb[1], d.z * R.cb[2])) / c.dfw;
    c.pb = fmaf(d.x, R.cb[3], fmaf(d.y, R.cb[4], d.z * R.cb[5])) / c.dfw;
    return c;
}
template <bool CAM>
__device__ __forceinline__ bool ff_box(const RayDev& r, const CamPt& c, float4 lo, float4 hi, float t0, float t1) {
    if (CAM)
        return lo.x <= c.pa && c.pa <= hi.x && lo.y <= c.pb && c.pb <= hi.y && hi.z >= t0 * c.dfw && lo.z <= t1 * c.dfw;
    return slab(r, lo, hi, t0, t1);
}

// ---------------------------------------------------------------- free flight: the first crossing (C17)
// Reading C17 at 1/64 of the ray's scene interval [t_lo, t_hi]: t* is the root inside the first of 64
// equal t-bins whose right edge reaches tau*.  Found hierarchically:
//  coarse: the 8 coarse bins' exact integrals (App. A closed form at the coarse edges), split into the
//    Gaussian part G_m (non-negative, kappa_i >= 0) and the Gabor part, plus each coarse bin's Gabor
//    mass M_m (sum over the Gabor chords touching it of their envelope integral 2 amp e^{Omega^2/2} >=
//    int |kappa_i|).  C_m = prefix; k1 = the first coarse edge with C_m >= tau*.  Inside coarse bin m,
//    tau(t) <= C_{m-1} + G_m + M_m =: U_m, so a coarse bin m < k1 with U_m < tau* cannot hold a fine
//    edge reaching tau*; the first one with U_m >= tau* (s0) starts the fine search.
//  fine: the 8 fine edges of each coarse bin from s0 to k1 exactly, from the chords inside it: the first
//    fine edge reaching tau* brackets the root (none: escape).
//  root: safeguarded Halley / bisection inside that fine bin over its chords.
// coarse and fine bins (resolution 1/(kNC kNF)); kNF = 1: uniform kNC bins, no fine search
constexpr int kNC = GF_FF_COARSE, kNF = GF_FF_FINE;
constexpr int kNRows = kNF > 1 ? 3 : 2;  // coarse rows per ray: Gaussian, Gabor (and Gabor mass)
static_assert(kNC >= 2 && kNC <= 32 && kNF >= 1 && kNF <= 32, "free-flight bins");
__device__ __forceinline__ float ff_edge(const FFRay& f, int m) {  // right edge of coarse bin m (-1: tlo)
    return m < 0 ? f.tlo : (m >= kNC - 1 ? f.thi : fmaf((float)(m + 1), f.bw, f.tlo));
}
__device__ __forceinline__ int ff_bin(const FFRay& f, float t) {
    return min(kNC - 1, max(0, (int)((t - f.tlo) * f.ibw)));
}
// right edge of fine bin j of coarse bin m
__device__ __forceinline__ float ff_fedge(const FFRay& f, int m, int j) {
    return j >= kNF - 1 ? ff_edge(f, m) : fmaf((float)(j + 1), f.bw * (1.0f / kNF), ff_edge(f, m - 1));
}

// The series erf of Eq. 13 (GF_ERF_CALL: out of line, one copy per translation unit -- smaller code, but
// every call spills the caller's live registers; measured slower, so inline by default).
#ifndef GF_ERF_CALL
#define GF_ERF_CALL 0
#endif
#if GF_ERF_CALL
static __device__ __noinline__
#else
__device__ __forceinline__
#endif
float2 erf_c(float u, float Om) {
    const float zr = u * kRsqrt2, zi = -Om * kRsqrt2;
    return erf_horner<kErfTerms>(zr, zi, fmaf(zr, zr, -zi * zi), 2.0f * zr * zi);
}

// Rare pieces (midpoint rule / Gauss-Legendre, seg_J): one out-of-line copy per translation unit
// instead of an inlined copy at every call site.
static __device__ __noinline__ float seg_J_rare(Setup s, float ua, float ub) {
    Work wk;
    return seg_J(s, ua, ub, wk);
}

// Coarse pass of one hit, lane-local (packet kernel): its pieces into the Gaussian (hg) or Gabor (hb)
// columns, its envelope mass into hm for every coarse bin it touches (stride between bins).
template <bool COUNT>
__device__ __forceinline__ void coarse_chord(const Setup& s, float cj, const FFRay& f, float* hg, float* hb, float* hm,
                                             int stride, Work& wk) {
    const float ta = fmaf(s.u0 - s.bp, s.ij, s.tc), tb = fmaf(s.u1 - s.bp, s.ij, s.tc);
    const int ka = ff_bin(f, ta), kb = ff_bin(f, tb);
    const bool gabor = s.Om != 0.0f;
    float* h = gabor ? hb : hg;
    if (kNF > 1 && gabor) {  // (the bound is only needed for the fine search)
        const float mass = cj * __expf(-0.5f * s.r2);  // >= int |kappa_i| over the chord (envelope)
        for (int m = ka; m <= kb; ++m) hm[m * stride] += mass;
    }
    const float wmax = 0.5f * (fmaxf(s.u0 * s.u0, s.u1 * s.u1) + s.Om * s.Om);
    if ((wmax > kWMaxSeries && gabor) || s.u1 - s.u0 < 1e-4f) {  // rare: piece by piece (GL / midpoint)
        if (COUNT) ++wk.gl;
        float ua = s.u0;
        for (int m = ka; m < kb; ++m) {
            const float ub = fminf(fmaxf(fmaf(s.j, ff_edge(f, m) - s.tc, s.bp), ua), s.u1);
            h[m * stride] += cj * seg_J_rare(s, ua, ub);
            ua = ub;
        }
        h[kb * stride] += cj * seg_J_rare(s, ua, s.u1);
        return;
    }
    float sp, cp;
    sincos_red(s.phi0, &sp, &cp);
    const float amp = cj * 0.5f * __expf(-0.5f * (s.r2 + s.Om * s.Om));
    // one erf call site: F at u0, at the coarse edges inside the chord, at u1; a symmetric full chord
    // inside one bin needs only F(h), F(-h) = -conj F(h) (the pair symmetry of P:L252)
    const bool sym = ka == kb && s.u0 == -s.h && s.u1 == s.h;
    const int ne = kb - ka + 1;
    float2 Fa = make_float2(0.0f, 0.0f);
    for (int e = sym ? 1 : 0; e <= ne; ++e) {
        const float u = e == 0 ? s.u0 : (e == ne ? s.u1 : fminf(fmaxf(fmaf(s.j, ff_edge(f, ka + e - 1) - s.tc, s.bp), s.u0), s.u1));
        const float2 F = gabor ? erf_c(u, s.Om) : make_float2(erff(u * kRsqrt2), 0.0f);
        if (sym) Fa = make_float2(-F.x, F.y);
        if (e > 0) h[(ka + e - 1) * stride] += amp * fmaf(cp, F.x - Fa.x, -sp * (F.y - Fa.y));
        Fa = F;
    }
    if (COUNT) wk.erf(s.Om, (uint32_t)(sym ? 1 : ne + 1));
}

// Decision of the coarse pass from the coarse bins (G_m, B_m Gabor signed, M_m Gabor mass) of one ray:
// k1 = first coarse edge with C_m >= tau* (kNC: none), s0 = first coarse bin m <= k1 with U_m >= tau*
// (kNC: none, then the ray escapes), *cstart = C_{s0 - 1}.  Returns k1 | s0 << 8.
__device__ __forceinline__ int coarse_decide(const double* g, const double* b, const double* mm, double tstar,
                                             double* cstart) {
    double c = 0.0;
    int k1 = kNC, s0 = kNC;
    *cstart = 0.0;
    for (int m = 0; m < kNC && k1 == kNC; ++m) {
        const double u = c + g[m] + mm[m];  // bound of tau inside coarse bin m
        if (s0 == kNC && u >= tstar) { s0 = m; *cstart = c; }
        c += g[m] + b[m];
        if (c >= tstar) k1 = m;
    }
    if (s0 > k1) s0 = k1;  // (the crossing bin itself: C_k1 >= tau* implies U_k1 >= tau*)
    if (kNF == 1) {  // uniform bins: the first edge reaching tau* is the answer at this resolution
        s0 = k1;
        c = 0.0;
        for (int m = 0; m < k1; ++m) c += g[m] + b[m];
        *cstart = c;
    }
    return k1 | (s0 << 8);
}

// tuning knobs (compile-time; bench variants are built with -D overrides)
#ifndef GF_MINB_PKT
#define GF_MINB_PKT 6  // k_ffa_pkt blocks per SM
#endif
#ifndef GF_PACKET
#define GF_PACKET 1  // depth-0 (camera) rays under a static mask: packet traversal (k_ffa_pkt)
#endif

// ---------------------------------------------------------------- pass B: root inside the window
// Per-record chord data of a hit record (a, b) = ((u0, u1, Omega, phi0), (amp, j, t_c, b')):
// full-chord integral amp (G(u1) - G(u0)), amp G(u0) (NaN for a midpoint / Gauss-Legendre record),
// amp cos phi0, -amp sin phi0.  gabor: the series for Omega != 0 (else the real erf).
template <bool COUNT>
__device__ __forceinline__ float4 chord_aux(float4 a, float4 b, bool gabor, Work& wk) {
    float full, g0 = 0.0f, ac = 0.0f, as = 0.0f;
    const float wmax = 0.5f * (fmaxf(a.x * a.x, a.y * a.y) + a.z * a.z);
    if (a.y - a.x < 1e-4f || (wmax > kWMaxSeries && a.z != 0.0f)) {
        // rare: midpoint / Gauss-Legendre (seg_J with e^{-r2/2} and 1/2 e^{-Om^2/2} in amp)
        Setup s;
        s.r2 = 0.0f; s.h = INFINITY; s.bp = b.w; s.j = b.y; s.ij = 1.0f / b.y; s.tc = b.z;
        s.Om = a.z; s.phi0 = a.w;
        full = 2.0f * b.x * __expf(0.5f * a.z * a.z) * seg_J_rare(s, a.x, a.y);
        if (COUNT) ++wk.gl;
        g0 = __int_as_float(0x7fc00000);  // NaN marks a special record
    } else {
        float sp = 0.0f, cp = 1.0f;
        if (gabor || a.w != 0.0f) sincos_red(a.w, &sp, &cp);
        ac = b.x * cp; as = -b.x * sp;
        float2 F1;
        if (!gabor) { F1 = make_float2(erff(a.y * kRsqrt2), 0.0f); if (COUNT) ++wk.erfr; }
        else { F1 = erf_shift(a.y, a.z); if (COUNT) ++wk.erfc; }
        const float G1 = fmaf(ac, F1.x, as * F1.y);
        if (a.x == -a.y) {
            g0 = -fmaf(ac, F1.x, -as * F1.y);  // F(-h) = -conj F(h)
        } else {
            float2 F0;
            if (!gabor) { F0 = make_float2(erff(a.x * kRsqrt2), 0.0f); if (COUNT) ++wk.erfr; }
            else { F0 = erf_shift(a.x, a.z); if (COUNT) ++wk.erfc; }
            g0 = fmaf(ac, F0.x, as * F0.y);
        }
        full = G1 - g0;
    }
    return make_float4(full, g0, ac, as);
}

// Records of the chords of one ray inside [t0, t1] (clipped to it) into rec (Gaussians from the
// front, Gabors from the back); ng + nb may exceed cap (then only the records that fit are written).
template <bool STOCH, bool COUNT, class BoxHit>
__device__ __forceinline__ void emit_records_b(const GNode* __restrict__ nodes, const GNode2* __restrict__ nodes2,
                                               uint32_t n_nodes, int stk_limit, const GPrim* __restrict__ prims,
                                               const RayDev& r, float t0, float t1, uint32_t mask, const float* w,
                                               WarpTrav& sm, float4* __restrict__ rec, uint32_t cap, uint32_t& ng,
                                               uint32_t& nb, Work& wk, BoxHit&& boxhit) {
    const unsigned FULL = 0xFFFFFFFFu;
    const unsigned lt = (1u << (threadIdx.x & 31)) - 1u;
    ng = nb = 0;
    warp_traverse_b<COUNT>(nodes, nodes2, n_nodes, stk_limit, mask, sm, wk, [&](bool valid, uint32_t ref) {
        bool hit = false;
        Setup s;
        float cj = 0.0f;
        if (valid) {
            const GPrim* pp = prims + (ref & kRefIdx);
            GPrim P;
            P.a = __ldg(&pp->a);
            if (COUNT) ++wk.tests;
            if (sphere_pretest(P.a, r, t0, t1)) {
                P.b = __ldg(&pp->b); P.c = __ldg(&pp->c); P.d = __ldg(&pp->d);
                hit = prim_setup(P, r, t0, t1, s);
                cj = P.d.w * s.ij;
                if (STOCH) cj *= w[ref >> 27];
            }
        }
        const bool hg = hit && s.Om == 0.0f, hb = hit && s.Om != 0.0f;
        const unsigned mg = __ballot_sync(FULL, hg), mb = __ballot_sync(FULL, hb);
        if (hit) {
            if (COUNT) ++wk.hits;
            const uint32_t slot = hg ? ng + __popc(mg & lt) : cap - 1 - (nb + __popc(mb & lt));
            if (ng + nb + __popc(mg) + __popc(mb) <= cap) {
                const float amp = 0.5f * cj * __expf(-0.5f * (s.r2 + s.Om * s.Om));
                rec[2 * slot] = make_float4(s.u0, s.u1, s.Om, s.phi0);
                rec[2 * slot + 1] = make_float4(amp, s.j, s.tc, s.bp);
            }
        }
        ng += __popc(mg);
        nb += __popc(mb);
    }, boxhit);
    __syncwarp();
}

// Equal bins [lo, hi] of one ray: right edge of bin m, bin of a t (the same arithmetic everywhere).
struct Bins {
    float lo, hi, w, iw;
    int n;
    __device__ __forceinline__ float edge(int m) const { return m < 0 ? lo : (m >= n - 1 ? hi : fmaf((float)(m + 1), w, lo)); }
    __device__ __forceinline__ int bin(float t) const { return min(n - 1, max(0, (int)((t - lo) * iw))); }
};
__device__ __forceinline__ Bins coarse_bins(const FFRay& f) { return Bins{f.tlo, f.thi, f.bw, f.ibw, kNC}; }
__device__ __forceinline__ Bins fine_bins(const FFRay& f, int m) {
    const float w = f.bw * (1.0f / kNF);
    return Bins{ff_edge(f, m - 1), ff_edge(f, m), w, w > 0.0f ? 1.0f / w : 0.0f, kNF};
}

// Chord t-range and the whitened u of a world t of record (ra, rb) = ((u0, u1, Omega, phi0), (amp, j, t_c, b')).
__device__ __forceinline__ void rec_trange(float4 ra, float4 rb, float& ta, float& tb) {
    const float ij = 1.0f / rb.y;
    ta = fmaf(ra.x - rb.w, ij, rb.z);
    tb = fmaf(ra.y - rb.w, ij, rb.z);
}
__device__ __forceinline__ float rec_u(float4 rb, float t) { return fmaf(rb.y, t - rb.z, rb.w); }
// a special record (midpoint / Gauss-Legendre, NaN amp G(u0) in its chord data): its partial integral
__device__ __forceinline__ float rec_rare(float4 ra, float4 rb, float ua, float ub) {
    Setup s;
    s.r2 = 0.0f; s.h = INFINITY; s.bp = rb.w; s.j = rb.y; s.ij = 1.0f / rb.y; s.tc = rb.z;
    s.Om = ra.z; s.phi0 = ra.w;
    return 2.0f * rb.x * __expf(0.5f * ra.z * ra.z) * seg_J_rare(s, ua, ub);
}

// sum of row r of lane-private columns (col[r * 32 + l]), rotated so that lanes read distinct banks
__device__ __forceinline__ double row_sum(const float* col0, int r) {
    const int lane = threadIdx.x & 31;
    const float* row = col0 + r * 32;
    double v = 0.0;
#pragma unroll 8
    for (int c = 0; c < 32; ++c) v += (double)row[(c + lane) & 31];
    return v;
}

// Pieces of the records' chords clipped to the bins' range into lane-private columns (bin m at
// [m * 32], this lane's column): Gaussian records into cg, Gabor records into cb, and (if cm) each Gabor
// chord's envelope mass into every bin it touches.  A clipped chord [ua, ub] in bins ka..kb adds
// -G(ua) to bin ka, +G(ub) to bin kb and, at an edge e inside it, +G(u(e)) / -G(u(e)) to the bins on
// either side (G(u) = Re{e^{i phi0} F(u)} amp, App. A: the pieces telescope to the chord's integral).
// G(u0), G(u1) come from the chord data x = (full, amp G(u0), amp cos phi0, -amp sin phi0); the other
// series values through the warp queue q (32 erf_c at a time).  All 32 lanes call it.
template <bool COUNT>
__device__ __forceinline__ void bin_records(const float4* __restrict__ rec, const float4* __restrict__ aux, uint32_t cap,
                                            uint32_t ng, uint32_t nb, const Bins& B, float* cg, float* cb, float* cm,
                                            WarpEnd& q, Work& wk) {
    const unsigned FULL = 0xFFFFFFFFu;
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    float* colg = cg + lane;
    float* colb = cb + lane;
    int nq = 0;
    auto run = [&](int take) {
        const bool v = lane < take;
        const float4 e = v ? q.e[1][nq - take + lane] : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        const uint32_t bb = v ? __float_as_uint(q.e[0][nq - take + lane].x) : 0u;
        nq -= take;
        __syncwarp();
        if (v) {
            if (COUNT) ++wk.erfc;
            const float2 F = erf_c(e.x, e.y);
            const float val = fmaf(e.z, F.x, e.w * F.y);
            colb[(bb & 0xFFu) * 32] += val;
            if ((bb >> 8) != 0xFFu) colb[(bb >> 8) * 32] -= val;
        }
    };
    const uint32_t nside[2] = {ng, nb};
#pragma unroll 1
    for (int side = 0; side < 2; ++side) {
        const uint32_t n = nside[side];
        for (uint32_t base = 0; base < n; base += 32) {
            const uint32_t i = base + lane;
            float4 ra = make_float4(0.0f, 0.0f, 0.0f, 0.0f), rb = ra, x = ra;
            int ka = 0, kb = 0, ne = 0;
            bool lo_in = true, hi_in = true;
            float ua = 0.0f, ub = 0.0f;
            if (i < n) {
                const uint32_t slot = side == 0 ? i : cap - 1 - i;
                ra = rec[2 * slot]; rb = rec[2 * slot + 1]; x = aux[slot];
                float ta, tb;
                rec_trange(ra, rb, ta, tb);
                if (tb > B.lo && ta < B.hi) {
                    lo_in = ta >= B.lo;
                    hi_in = tb <= B.hi;
                    ka = B.bin(lo_in ? ta : B.lo);
                    kb = B.bin(hi_in ? tb : B.hi);
                    ua = lo_in ? ra.x : fminf(fmaxf(rec_u(rb, B.lo), ra.x), ra.y);
                    ub = hi_in ? ra.y : fminf(fmaxf(rec_u(rb, B.hi), ra.x), ra.y);
                    if (cm && side == 1) {
                        const float mass = 2.0f * rb.x * __expf(0.5f * ra.z * ra.z);  // >= int |kappa_i|
                        for (int m = ka; m <= kb; ++m) cm[m * 32 + lane] += mass;
                    }
                    float* col = side == 0 ? colg : colb;
                    if (x.y != x.y) {  // special record: pieces lane-local
                        float u0 = ua;
                        for (int m = ka; m < kb; ++m) {
                            const float u1 = fminf(fmaxf(rec_u(rb, B.edge(m)), u0), ub);
                            col[m * 32] += rec_rare(ra, rb, u0, u1);
                            u0 = u1;
                        }
                        col[kb * 32] += rec_rare(ra, rb, u0, ub);
                    } else if (side == 0) {  // Gaussian: G(u) = amp erf(u / sqrt2), real erf inline
                        const float Ga = lo_in ? x.y : x.z * erff(ua * kRsqrt2);
                        const float Gb = hi_in ? x.y + x.x : x.z * erff(ub * kRsqrt2);
                        col[ka * 32] -= Ga;
                        col[kb * 32] += Gb;
                        for (int m = ka; m < kb; ++m) {
                            const float g = x.z * erff(fminf(fmaxf(rec_u(rb, B.edge(m)), ra.x), ra.y) * kRsqrt2);
                            col[m * 32] += g;
                            col[(m + 1) * 32] -= g;
                        }
                        if (COUNT) wk.erfr += (uint32_t)(kb - ka + !lo_in + !hi_in);
                    } else {  // Gabor: known ends here, the series values through the queue
                        if (lo_in) col[ka * 32] -= x.y;
                        if (hi_in) col[kb * 32] += x.y + x.x;
                        ne = (!lo_in) + (!hi_in) + (kb - ka);
                    }
                }
            }
            for (int e = 0; __any_sync(FULL, e < ne); ++e) {
                const bool mine = e < ne;
                const unsigned mm = __ballot_sync(FULL, mine);
                if (mine) {
                    int k = e;
                    float4 ent;
                    uint32_t bb;
                    if (!lo_in && k == 0) {
                        ent = make_float4(ua, ra.z, -x.z, -x.w);
                        bb = (uint32_t)ka | 0xFF00u;
                    } else {
                        k -= !lo_in;
                        if (!hi_in && k == 0) {
                            ent = make_float4(ub, ra.z, x.z, x.w);
                            bb = (uint32_t)kb | 0xFF00u;
                        } else {
                            const int m = ka + k - !hi_in;
                            ent = make_float4(fminf(fmaxf(rec_u(rb, B.edge(m)), ra.x), ra.y), ra.z, x.z, x.w);
                            bb = (uint32_t)m | ((uint32_t)(m + 1) << 8);
                        }
                    }
                    q.e[1][nq + __popc(mm & lt)] = ent;
                    q.e[0][nq + __popc(mm & lt)].x = __uint_as_float(bb);
                }
                nq += __popc(mm);
                GF_CHECK(nq <= kWEnd);
                __syncwarp();
                if (nq >= 32) run(32);
            }
        }
    }
    while (nq > 0) run(min(nq, 32));
    __syncwarp();
}

// Uniform bins (kNF == 1), warp version: the first coarse edge whose cumulative tau reaches tau* from the
// lane columns (rows G and Gabor): lane m holds bin m, an inclusive scan gives the edge values.
// Only the edges of bins 0 .. kmax count (their chords all in).  Returns k1 | k1 << 8 (kNC: escape),
// *cstart = tau before bin k1.
__device__ __forceinline__ int coarse_first_warp(const float* cols, double tstar, double* cstart, int kmax = kNC - 1,
                                                 double* upto = nullptr) {
    const unsigned FULL = 0xFFFFFFFFu;
    const int lane = threadIdx.x & 31;
    const double v = lane <= kmax ? row_sum(cols, lane) + row_sum(cols + kNC * 32, lane) : 0.0;
    double incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double u = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += u;
    }
    const unsigned hit = __ballot_sync(FULL, lane <= kmax && incl >= tstar);
    const int k1 = hit ? __ffs(hit) - 1 : kNC;
    *cstart = __shfl_sync(FULL, incl - v, hit ? k1 : 0);
    if (upto) *upto = __shfl_sync(FULL, incl, max(kmax, 0));  // tau at the right edge of bin kmax
    return k1 | (k1 << 8);
}

// coarse decision from the warp's lane columns (rows: G at [0], Gabor at [kNC*32], mass at [2*kNC*32])
__device__ __forceinline__ int coarse_decide_warp(const float* cols, double tstar, double* cstart) {
    const int lane = threadIdx.x & 31;
    double g = 0.0, b = 0.0, m = 0.0;
    if (lane < kNC) {
        g = row_sum(cols, lane);
        b = row_sum(cols + kNC * 32, lane);
        if (kNF > 1) m = row_sum(cols + 2 * kNC * 32, lane);
    }
    double G[kNC], B[kNC], M[kNC];
#pragma unroll
    for (int k = 0; k < kNC; ++k) {
        G[k] = __shfl_sync(0xFFFFFFFFu, g, k);
        B[k] = __shfl_sync(0xFFFFFFFFu, b, k);
        M[k] = __shfl_sync(0xFFFFFFFFu, m, k);
    }
    return coarse_decide(G, B, M, tstar, cstart);
}

// Root of f(t) = c0 + tau(a, t) - tau* in the window [a, b] over the records overlapping it (whole warp):
// first their chord data become (G(u1), base = G at max(u0, u(a)), amp cos, -amp sin) -- one erf for a
// chord straddling a -- and their slots are listed in shared memory (wl, <= kWinCap; beyond that every
// record is scanned with a range test); then safeguarded Halley (Newton if its denominator
// degenerates, bisection if a step leaves the bracket) to 1e-6 of the window (2 ulp of t at least).
// Each evaluation: a chord wholly before t adds G(u1) - base, one straddling t queues the endpoint
// u(t) (one erf, 32 at a time, type-uniform) and adds its kappa and d kappa / dt terms.
constexpr int kWinCap = 256;
template <bool COUNT>
__device__ __noinline__ float window_root(const float4* __restrict__ rec, float4* __restrict__ aux, uint32_t cap,
                                          uint32_t ng, uint32_t nb, float a, float b, double c0, double tstar,
                                          uint16_t* wl, WarpEnd& q, Work& wk) {
    const unsigned FULL = 0xFFFFFFFFu;
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    // 1. window records: chord data -> (G1, base, ac, as); list of their slots (Gaussians first)
    int nw[2] = {0, 0}, nq = 0;
    auto runb = [&](int take) {
        const bool v = lane < take;
        const float4 e = v ? q.e[1][nq - take + lane] : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        const uint32_t slot = v ? __float_as_uint(q.e[0][nq - take + lane].x) : 0u;
        nq -= take;
        __syncwarp();
        if (v) {
            if (COUNT) ++wk.erfc;
            const float2 F = erf_c(e.x, e.y);
            aux[slot].y = fmaf(e.z, F.x, e.w * F.y);
        }
    };
    const uint32_t nside[2] = {ng, nb};
    bool over = false;
#pragma unroll 1
    for (int side = 0; side < 2; ++side) {
        const uint32_t n = nside[side];
        for (uint32_t base = 0; base < n; base += 32) {
            const uint32_t i = base + lane;
            bool inw = false, push = false;
            float4 e = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
            uint32_t slot = 0;
            if (i < n) {
                slot = side == 0 ? i : cap - 1 - i;
                const float4 ra = rec[2 * slot], rb = rec[2 * slot + 1];
                float4 x = aux[slot];
                float ta, tb;
                rec_trange(ra, rb, ta, tb);
                inw = tb > a && ta < b;
                if (inw && x.y == x.y) {
                    const float g1 = x.y + x.x;
                    if (ta < a) {  // straddles the window start: base = G(u(a))
                        const float ua = fminf(fmaxf(rec_u(rb, a), ra.x), ra.y);
                        if (side == 0) {
                            x.y = x.z * erff(ua * kRsqrt2);
                            if (COUNT) ++wk.erfr;
                        } else {
                            push = true;
                            e = make_float4(ua, ra.z, x.z, x.w);
                        }
                    }
                    x.x = g1;
                    aux[slot] = x;
                }
            }
            const unsigned mw = __ballot_sync(FULL, inw);
            const int tot = nw[0] + nw[1];
            if (inw && tot + __popc(mw & lt) < kWinCap) wl[tot + __popc(mw & lt)] = (uint16_t)slot;
            nw[side] += __popc(mw);
            const unsigned m = __ballot_sync(FULL, push);
            if (m) {
                if (push) {
                    q.e[1][nq + __popc(m & lt)] = e;
                    q.e[0][nq + __popc(m & lt)].x = __uint_as_float(slot);
                }
                nq += __popc(m);
                __syncwarp();
                if (nq >= 32) runb(32);
            }
        }
    }
    while (nq > 0) runb(min(nq, 32));
    over = nw[0] + nw[1] > kWinCap;
    __syncwarp();
    // 2. Halley
    int nq0 = 0, nq1 = 0;
    double acc = 0.0;
    auto run = [&](int t, int take) {
        int& nqx = t == 0 ? nq0 : nq1;
        const bool v = lane < take;
        const float4 e = v ? q.e[t][nqx - take + lane] : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        nqx -= take;
        __syncwarp();
        if (v) {
            if (t == 0) {
                if (COUNT) ++wk.erfr;
                acc += (double)(e.z * erff(e.x * kRsqrt2));
            } else {
                if (COUNT) ++wk.erfc;
                const float2 F = erf_c(e.x, e.y);
                acc += (double)fmaf(e.z, F.x, e.w * F.y);
            }
        }
    };
    auto eval = [&](float t, double& kap_out, double& dkap_out) -> double {
        if (COUNT && lane == 0) ++wk.root;
        acc = 0.0;
        float part = 0.0f, kap = 0.0f, dkap = 0.0f;
#pragma unroll 1
        for (int side = 0; side < 2; ++side) {
            const uint32_t n = over ? nside[side] : (uint32_t)nw[side];
            for (uint32_t base = 0; base < n; base += 32) {
                const uint32_t i = base + lane;
                bool push = false;
                float4 e = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
                if (i < n) {
                    const uint32_t slot = over ? (side == 0 ? i : cap - 1 - i) : wl[(side == 0 ? 0 : nw[0]) + i];
                    const float4 ra = rec[2 * slot], rb = rec[2 * slot + 1];
                    bool inw = true;
                    if (over) {
                        float ta, tb;
                        rec_trange(ra, rb, ta, tb);
                        inw = tb > a && ta < b;
                    }
                    const float ut = rec_u(rb, t);
                    if (inw && ut > ra.x) {  // a window chord that t has reached
                        const float4 x = aux[slot];
                        if (ut >= ra.y) {
                            part += x.y == x.y ? x.x - x.y : rec_rare(ra, rb, fmaxf(ra.x, rec_u(rb, a)), ra.y);
                        } else {
                            float sp, cp;
                            sincos_red(fmaf(ra.z, ut, ra.w), &sp, &cp);
                            const float kk = rb.x * rb.y * 0.79788456080286536f * __expf(0.5f * (ra.z * ra.z - ut * ut));
                            kap += kk * cp;
                            dkap -= kk * rb.y * fmaf(ut, cp, ra.z * sp);  // d kappa / dt (Halley step)
                            if (x.y != x.y) {
                                part += rec_rare(ra, rb, fmaxf(ra.x, rec_u(rb, a)), ut);
                            } else {
                                part -= x.y;
                                push = true;
                                e = make_float4(ut, ra.z, x.z, x.w);
                            }
                        }
                    }
                }
                const unsigned m = __ballot_sync(FULL, push);
                if (m) {
                    int& nqx = side == 0 ? nq0 : nq1;
                    if (push) q.e[side][nqx + __popc(m & lt)] = e;
                    nqx += __popc(m);
                    GF_CHECK(nqx <= kWEnd);
                    __syncwarp();
                    if (nqx >= 32) run(side, 32);
                }
            }
        }
        while (nq0 > 0) run(0, min(nq0, 32));
        while (nq1 > 0) run(1, min(nq1, 32));
        double xs = acc + (double)part, k = kap, dk = dkap;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            xs += __shfl_xor_sync(FULL, xs, o);
            k += __shfl_xor_sync(FULL, k, o);
            dk += __shfl_xor_sync(FULL, dk, o);
        }
        kap_out = k;
        dkap_out = dk;
        return c0 + xs - tstar;
    };
    const float wlen = b - a;
    float lo = a, hi = b, t = a + 0.5f * wlen;
    const float tol = fmaxf(1e-6f * wlen, 2.4e-7f * fmaxf(fabsf(a), fabsf(b)));
    double kap = 0.0, dkap = 0.0;
    for (int it = 0; it < 40; ++it) {
        const double fv = eval(t, kap, dkap);
        if (fv >= 0.0) hi = t; else lo = t;
        if (!(hi - lo > tol)) break;
        if (fabs(fv) <= 1e-6 * (1.0 + tstar)) break;  // |tau(t) - tau*| at the fp32 noise floor of the sums
        const double den = 2.0 * kap * kap - fv * dkap;
        float tn = (kap > 0.0) ? (float)((double)t - (den > 0.0 ? 2.0 * fv * kap / den : fv / kap)) : 0.5f * (lo + hi);
        const bool newton = tn > lo && tn < hi;
        if (!newton) tn = 0.5f * (lo + hi);
        const bool small = newton && fabsf(tn - t) <= tol;  // converged step
        t = tn;
        if (small) break;
    }
    return t;
}

// Root of f(t) = c0 + tau(a, t) - tau* over records CLIPPED to the window [a, b] (pass B with uniform
// bins: every record is a window record, chord data x = (full, amp G(u0), amp cos, -amp sin)): each
// evaluation scans the records -- a chord wholly before t adds its full integral, one straddling t
// queues the endpoint u(t) (one erf, 32 at a time, type-uniform) and adds its kappa and d kappa / dt
// terms; safeguarded Halley (Newton / bisection) to 1e-6 of the window (2 ulp of t at least).
template <bool COUNT>
__device__ __forceinline__ float window_root_clip(const float4* __restrict__ rec, const float4* __restrict__ aux,
                                                  uint32_t cap, uint32_t ng, uint32_t nb, float a, float b, double c0,
                                                  double tstar, WarpEnd& q, Work& wk, float* kap_out = nullptr,
                                                  double wtot = 0.0) {
    const unsigned FULL = 0xFFFFFFFFu;
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const uint32_t nside[2] = {ng, nb};
    int nq0 = 0, nq1 = 0;
    double acc = 0.0;
    auto run = [&](int t, int take) {
        int& nq = t == 0 ? nq0 : nq1;
        const bool v = lane < take;
        const float4 e = v ? q.e[t][nq - take + lane] : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        nq -= take;
        __syncwarp();
        if (v) {
            if (t == 0) {
                if (COUNT) ++wk.erfr;
                acc += (double)(e.z * erff(e.x * kRsqrt2));
            } else {
                if (COUNT) ++wk.erfc;
                const float2 F = erf_c(e.x, e.y);
                acc += (double)fmaf(e.z, F.x, e.w * F.y);
            }
        }
    };
    auto eval = [&](float t, double& kap_out, double& dkap_out) -> double {
        if (COUNT && lane == 0) ++wk.root;
        acc = 0.0;
        float part = 0.0f, kap = 0.0f, dkap = 0.0f;
#pragma unroll 1
        for (int side = 0; side < 2; ++side) {
            const uint32_t n = nside[side];
            for (uint32_t base = 0; base < n; base += 32) {
                const uint32_t i = base + lane;
                bool push = false;
                float4 e = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
                if (i < n) {
                    const uint32_t slot = side == 0 ? i : cap - 1 - i;
                    const float4 ra = rec[2 * slot], rb = rec[2 * slot + 1];
                    const float ut = rec_u(rb, t);
                    if (ut > ra.x) {
                        const float4 x = aux[slot];
                        if (ut >= ra.y) {
                            part += x.x;
                        } else {
                            float sp, cp;
                            sincos_red(fmaf(ra.z, ut, ra.w), &sp, &cp);
                            const float kk = rb.x * rb.y * 0.79788456080286536f * __expf(0.5f * (ra.z * ra.z - ut * ut));
                            kap += kk * cp;
                            dkap -= kk * rb.y * fmaf(ut, cp, ra.z * sp);  // d kappa / dt (Halley step)
                            if (x.y != x.y) {  // special record: lane-local partial integral
                                part += rec_rare(ra, rb, ra.x, ut);
                            } else {
                                part -= x.y;
                                push = true;
                                e = make_float4(ut, ra.z, x.z, x.w);
                            }
                        }
                    }
                }
                const unsigned m = __ballot_sync(FULL, push);
                if (m) {
                    int& nq = side == 0 ? nq0 : nq1;
                    if (push) q.e[side][nq + __popc(m & lt)] = e;
                    nq += __popc(m);
                    GF_CHECK(nq <= kWEnd);
                    __syncwarp();
                    if (nq >= 32) run(side, 32);
                }
            }
        }
        while (nq0 > 0) run(0, min(nq0, 32));
        while (nq1 > 0) run(1, min(nq1, 32));
        double xs = acc + (double)part, k = kap, dk = dkap;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            xs += __shfl_xor_sync(FULL, xs, o);
            k += __shfl_xor_sync(FULL, k, o);
            dk += __shfl_xor_sync(FULL, dk, o);
        }
        kap_out = k;
        dkap_out = dk;
        return c0 + xs - tstar;
    };
    const float wlen = b - a;
    // start where tau, linear over the window (wtot = tau over it), reaches tau*; the midpoint without it
    const double fr = wtot > 0.0 ? fmin(0.95, fmax(0.05, (tstar - c0) / wtot)) : 0.5;
    float lo = a, hi = b, t = a + (float)fr * wlen;
    const float tol = fmaxf(1e-6f * wlen, 2.4e-7f * fmaxf(fabsf(a), fabsf(b)));
    double kap = 0.0, dkap = 0.0;
    for (int it = 0; it < 40; ++it) {
        const double fv = eval(t, kap, dkap);
        if (fv >= 0.0) hi = t; else lo = t;
        if (!(hi - lo > tol)) break;
        if (fabs(fv) <= 1e-6 * (1.0 + tstar)) break;
        const double den = 2.0 * kap * kap - fv * dkap;
        float tn = (kap > 0.0) ? (float)((double)t - (den > 0.0 ? 2.0 * fv * kap / den : fv / kap)) : 0.5f * (lo + hi);
        const bool newton = tn > lo && tn < hi;
        if (!newton) tn = 0.5f * (lo + hi);
        const bool small = newton && fabsf(tn - t) <= tol;
        t = tn;
        if (small) break;
    }
    if (kap_out) *kap_out = (float)kap;  // (at the last evaluated t)
    return t;
}

// Pass B from the ray's hit list (refs: primitive index in the traversed BVH's order | group << 27, as pass A
// met them): the warp tests each listed primitive against the window [a, b] (sphere pre-test + prim_setup:
// the traversal's predicate), writes the records of the chords inside it (clipped to it) and their chord
// data, and solves the root there (window_root_clip) -- no second traversal.  false if the window's chords
// exceed the record buffer.
template <bool STOCH, bool COUNT>
__device__ __forceinline__ bool window_from_refs(const uint32_t* __restrict__ refs, uint32_t n,
                                                 const GPrim* __restrict__ prims, const RayDev& r, const float* w,
                                                 float a, float b, double c0, double tstar, float4* __restrict__ rec,
                                                 float4* __restrict__ aux, uint32_t cap, WarpEnd& q, Work& wk, float& t) {
    const unsigned FULL = 0xFFFFFFFFu;
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    uint32_t ng = 0, nb = 0;
    for (uint32_t base = 0; base < n; base += 32) {
        const uint32_t i = base + lane;
        bool hit = false;
        Setup s;
        float cj = 0.0f;
        if (i < n) {
            const uint32_t ref = refs[i];
            const GPrim* pp = prims + (ref & kRefIdx);
            GPrim P;
            P.a = __ldg(&pp->a);
            if (sphere_pretest(P.a, r, a, b)) {
                P.b = __ldg(&pp->b); P.c = __ldg(&pp->c); P.d = __ldg(&pp->d);
                hit = prim_setup(P, r, a, b, s);
                cj = P.d.w * s.ij;
                if (STOCH) cj *= w[ref >> 27];
            }
        }
        const bool hg = hit && s.Om == 0.0f, hb = hit && s.Om != 0.0f;
        const unsigned mg = __ballot_sync(FULL, hg), mb = __ballot_sync(FULL, hb);
        if (hit) {
            const uint32_t slot = hg ? ng + __popc(mg & lt) : cap - 1 - (nb + __popc(mb & lt));
            if (ng + nb + __popc(mg) + __popc(mb) <= cap) {
                const float amp = 0.5f * cj * __expf(-0.5f * (s.r2 + s.Om * s.Om));
                rec[2 * slot] = make_float4(s.u0, s.u1, s.Om, s.phi0);
                rec[2 * slot + 1] = make_float4(amp, s.j, s.tc, s.bp);
            }
        }
        ng += __popc(mg);
        nb += __popc(mb);
    }
    __syncwarp();
    if (ng + nb > cap) return false;
    const uint32_t nside[2] = {ng, nb};
#pragma unroll 1
    for (int side = 0; side < 2; ++side)
        for (uint32_t i = lane; i < nside[side]; i += 32) {
            const uint32_t slot = side == 0 ? i : cap - 1 - i;
            aux[slot] = chord_aux<COUNT>(rec[2 * slot], rec[2 * slot + 1], side == 1, wk);
        }
    __syncwarp();
    t = window_root_clip<COUNT>(rec, aux, cap, ng, nb, a, b, c0, tstar, q, wk);
    return true;
}

// Fine search over the records (chord data x = (full, amp G(u0), ...) already computed): coarse bins s0 ..
// kend, starting from cstart = tau before coarse bin s0; each coarse bin's 8 fine edges exactly (bin_records
// into the lane columns cf), the first fine edge reaching tau* brackets the root (window_root).  Returns
// false (escape) if no fine edge reaches tau*.
template <bool COUNT>
__device__ __forceinline__ bool resolve_records(const float4* __restrict__ rec, float4* __restrict__ aux, uint32_t cap,
                                                uint32_t ng, uint32_t nb, const FFRay& f, int s0, int kend,
                                                double cstart, float* cf, uint16_t* wl, WarpEnd& q, Work& wk,
                                                float& tout, bool clipped = false, float* kap_out = nullptr,
                                                double wtot = 0.0) {
    const unsigned FULL = 0xFFFFFFFFu;
    const int lane = threadIdx.x & 31;
    if (kNF == 1) {  // uniform bins: the root inside coarse bin s0 (= the first crossing edge), tau before it cstart
        if (s0 >= kNC) return false;
        if (clipped)  // pass B: the records are exactly the window's chords, clipped to it
            tout = window_root_clip<COUNT>(rec, aux, cap, ng, nb, ff_edge(f, s0 - 1), ff_edge(f, s0), cstart, f.tstar, q, wk,
                                            kap_out, wtot);
        else
            tout = window_root<COUNT>(rec, aux, cap, ng, nb, ff_edge(f, s0 - 1), ff_edge(f, s0), cstart, f.tstar, wl, q, wk);
        return true;
    }
    double cum = cstart;
#pragma unroll 1
    for (int m = s0; m <= kend; ++m) {
        const Bins B = fine_bins(f, m);
#pragma unroll
        for (int j = 0; j < kNF; ++j) cf[j * 32 + lane] = 0.0f;
        __syncwarp();
        bin_records<COUNT>(rec, aux, cap, ng, nb, B, cf, cf, nullptr, q, wk);
        const double v = lane < kNF ? row_sum(cf, lane) : 0.0;
        double incl = v;
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
            const double u = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += u;
        }
        const unsigned hit = __ballot_sync(FULL, lane < kNF && cum + incl >= f.tstar);
        if (hit) {
            const int j = __ffs(hit) - 1;
            const double c0 = cum + __shfl_sync(FULL, incl - v, j);
            tout = window_root<COUNT>(rec, aux, cap, ng, nb, B.edge(j - 1), B.edge(j), c0, f.tstar, wl, q, wk);
            return true;
        }
        cum += __shfl_sync(FULL, incl, kNF - 1);
    }
    return false;
}

// ---------------------------------------------------------------- tracking estimators (a9 alternative)
// Null-collision delta tracking (free flight) and ratio tracking (NEE transmittance) against a
// per-ray piecewise-constant majorant, selected by gf_render_desc.estimator = GF_EST_TRACKING.
// The ray's hit records (the same 32-byte records k_ff writes) give both the majorant -- 64 bins
// over [t_lo, t_hi], bin k holding sum_i p_i over the chords overlapping it, p_i the bound of
// |kappa_i| on its chord, amp j sqrt(2/pi) e^{(Omega^2 - u_min^2)/2} -- and kappa(t) at a tentative
// point (one warp reduction over the records straddling t, no erf).  Unbiased where kappa >= 0.

// majorant bins M[0..63] over [wa, wb] (shared, per warp)
__device__ __forceinline__ void majorant_bins(const float4* __restrict__ rec, uint32_t ng, uint32_t nb, uint32_t cap,
                                              float wa, float wb, float* M) {
    const int lane = threadIdx.x & 31;
    M[lane] = 0.0f;
    M[lane + 32] = 0.0f;
    __syncwarp();
    const float span = fmaxf(wb - wa, 1e-30f), sc = 64.0f / span, pad = 1e-5f * span;
    const uint32_t nside[2] = {ng, nb};
#pragma unroll 1
    for (int side = 0; side < 2; ++side) {
        for (uint32_t i = lane; i < nside[side]; i += 32) {
            const uint32_t slot = side == 0 ? i : cap - 1 - i;
            const float4 a = rec[2 * slot], b = rec[2 * slot + 1];
            const float um = (a.x <= 0.0f && a.y >= 0.0f) ? 0.0f : fminf(fabsf(a.x), fabsf(a.y));
            const float pk = 1.0001f * fabsf(b.x) * b.y * 0.79788456080286536f * __expf(0.5f * (a.z * a.z - um * um));
            const float ij = 1.0f / b.y;
            const float ta = fmaf(a.x - b.w, ij, b.z) - pad, tb = fmaf(a.y - b.w, ij, b.z) + pad;
            const int ka = min(63, max(0, (int)floorf((ta - wa) * sc))), kb = min(63, max(0, (int)floorf((tb - wa) * sc)));
            for (int k = ka; k <= kb; ++k) atomicAdd(&M[k], pk);
        }
    }
    __syncwarp();
}

// kappa(t) along the ray from its records (all lanes get the sum)
__device__ __forceinline__ float kappa_at(const float4* __restrict__ rec, uint32_t ng, uint32_t nb, uint32_t cap,
                                          float t) {
    const int lane = threadIdx.x & 31;
    const uint32_t nside[2] = {ng, nb};
    float kap = 0.0f;
#pragma unroll 1
    for (int side = 0; side < 2; ++side) {
        for (uint32_t i = lane; i < nside[side]; i += 32) {
            const uint32_t slot = side == 0 ? i : cap - 1 - i;
            const float4 a = rec[2 * slot], b = rec[2 * slot + 1];
            const float ut = fmaf(b.y, t - b.z, b.w);
            if (ut > a.x && ut < a.y) {
                float sp, cp;
                sincos_red(fmaf(a.z, ut, a.w), &sp, &cp);
                kap += b.x * b.y * 0.79788456080286536f * __expf(0.5f * (a.z * a.z - ut * ut)) * cp;
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) kap += __shfl_xor_sync(0xFFFFFFFFu, kap, o);
    return kap;
}

// Next tentative collision: advance t through the majorant bins by an exponential step of unit
// majorant optical depth (-ln(1-u)); false if the ray leaves [wa, wb].  k = current bin.
__device__ __forceinline__ bool majorant_step(const float* M, float wa, float wb, float u, float& t, int& k) {
    const float bw = (wb - wa) * (1.0f / 64.0f);
    float tb = -log1pf(-u);
    while (k < 64) {
        const float be = (k == 63) ? wb : wa + (float)(k + 1) * bw;
        const float m = M[k], seg = be - t;
        if (m * seg <= tb) {
            tb -= m * seg;
            t = be;
            ++k;
        } else {
            t += tb / m;
            return true;
        }
    }
    return false;
}

constexpr int kPStk = 512;  // packet traversal stack (k_ffa_pkt, k_tomo_pkt)

}  // namespace gfk

// ---- host launchers of the render kernels (one translation unit each, compiled in parallel)
int gf_persist_blocks();                 // 16 blocks of 128 threads per SM
unsigned gf_rec_grid(int64_t n_paths);   // grid of the kernels owning per-warp record buffers
void gf_launch_ffa_pkt(RenderDev& R, int32_t sample, int d, bool stoch, bool count, bool cam, unsigned grid,
                       cudaStream_t st);
void gf_launch_ffa_w(RenderDev& R, int32_t sample, int d, bool stoch, bool count, bool cam, const uint32_t* q_in,
                     int cnt_slot, int cur_slot, int ray_count, unsigned grid, cudaStream_t st);
void gf_launch_ffb(RenderDev& R, int32_t sample, int d, bool stoch, bool count, bool cam, cudaStream_t st);
bool gf_ff_onepass();
void gf_launch_ff(RenderDev& R, int32_t sample, int d, bool stoch, bool count, bool cam, const uint32_t* q_in,
                  int cnt_slot, int cur_slot, cudaStream_t st);
void gf_launch_ff_trk(RenderDev& R, int32_t sample, int d, bool stoch, bool count, cudaStream_t st);
void gf_launch_nee_rt(RenderDev& R, int32_t sample, int d, bool stoch_nee, bool count, cudaStream_t st);
void gf_launch_nee_w(RenderDev& R, int32_t sample, int d, bool stoch_nee, bool count, unsigned grid, cudaStream_t st);
void gf_launch_tomo(RenderDev& R, int32_t sample, bool stoch, bool count, bool packets, unsigned grid, cudaStream_t st);
