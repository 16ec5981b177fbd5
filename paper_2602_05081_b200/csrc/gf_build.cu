// gf_build.cu -- a1 primitive ingest and a2 LBVH build.
#include <cub/device/device_radix_sort.cuh>

#include "gf_device.cuh"
#include "gf_internal.h"

namespace gfk {

// error bits reported by the load kernel
enum : uint32_t { ERR_SCALE = 1u, ERR_EXTENT = 2u, ERR_ASSIGN = 4u, ERR_QUAT = 8u, ERR_VALUE = 16u };

// Orientation bin (reading C11): argmax_k |d . o_k|, d = R S^-1 (1,1,1)^T, ties -> lower k,
// in fp32 with correctly rounded ops in the same expression order as the decision rule of
// DESIGN.md §3 C11 (an integer decided by floating point: same precision on both sides).
__device__ int derive_bin(const float* q, const float* sc, int K, const float* axes) {
    float x = q[0], y = q[1], z = q[2], w = q[3];
    float nn = __fsqrt_rn(__fmaf_rn(x, x, __fmaf_rn(y, y, __fmaf_rn(z, z, __fmul_rn(w, w)))));
    x = __fdiv_rn(x, nn); y = __fdiv_rn(y, nn); z = __fdiv_rn(z, nn); w = __fdiv_rn(w, nn);
    float R[9];
    R[0] = __fsub_rn(1.0f, __fmul_rn(2.0f, __fmaf_rn(y, y, __fmul_rn(z, z))));
    R[1] = __fmul_rn(2.0f, __fmaf_rn(x, y, -__fmul_rn(w, z)));
    R[2] = __fmul_rn(2.0f, __fmaf_rn(x, z, __fmul_rn(w, y)));
    R[3] = __fmul_rn(2.0f, __fmaf_rn(x, y, __fmul_rn(w, z)));
    R[4] = __fsub_rn(1.0f, __fmul_rn(2.0f, __fmaf_rn(x, x, __fmul_rn(z, z))));
    R[5] = __fmul_rn(2.0f, __fmaf_rn(y, z, -__fmul_rn(w, x)));
    R[6] = __fmul_rn(2.0f, __fmaf_rn(x, z, -__fmul_rn(w, y)));
    R[7] = __fmul_rn(2.0f, __fmaf_rn(y, z, __fmul_rn(w, x)));
    R[8] = __fsub_rn(1.0f, __fmul_rn(2.0f, __fmaf_rn(x, x, __fmul_rn(y, y))));
    float i0 = __fdiv_rn(1.0f, sc[0]), i1 = __fdiv_rn(1.0f, sc[1]), i2 = __fdiv_rn(1.0f, sc[2]);
    float d[3];
    for (int r = 0; r < 3; ++r) d[r] = __fmaf_rn(R[3 * r], i0, __fmaf_rn(R[3 * r + 1], i1, __fmul_rn(R[3 * r + 2], i2)));
    int best = 0;
    float bestv = -1.0f;
    for (int k = 0; k < K; ++k) {
        float a = fabsf(__fmaf_rn(d[0], axes[3 * k], __fmaf_rn(d[1], axes[3 * k + 1], __fmul_rn(d[2], axes[3 * k + 2]))));
        if (a > bestv) { bestv = a; best = k; }
    }
    return best;
}

__global__ void k_load_prims(LoadArgs A, GPrim* out, uint8_t* gout, uint32_t* err, uint32_t* lfmax_bits) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= A.n) return;
    const float* q = A.quat + 4 * i;
    const float* sc = A.scale + 3 * i;
    uint32_t e = 0;
    float qn = sqrtf(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    if (!(fabsf(qn - 1.0f) <= 1e-5f)) e |= ERR_QUAT;
    float smin = fminf(sc[0], fminf(sc[1], sc[2])), smax = fmaxf(sc[0], fmaxf(sc[1], sc[2]));
    if (!(smin > 0.0f) || !isfinite(smax) || !(smax <= 1e6f * smin)) e |= ERR_SCALE;
    float E = A.extent ? A.extent[i] : 3.0f;
    if (!(E > 0.0f) || !isfinite(E)) e |= ERR_EXTENT;
    float alpha = A.alpha[i], om = A.omega[i];
    float mx = A.mu[3 * i], my = A.mu[3 * i + 1], mz = A.mu[3 * i + 2];
    if (!(alpha >= 0.0f) || !isfinite(alpha) || !(om >= 0.0f) || !isfinite(om) || !isfinite(mx) || !isfinite(my) ||
        !isfinite(mz))
        e |= ERR_VALUE;
    int lev;
    if (A.level) {
        lev = A.level[i];
        if (lev >= A.P) e |= ERR_ASSIGN;
    } else if (om == 0.0f) {
        lev = 0;
    } else {  // reading C10: f0 = omega |S^-1 (1,1,1)| against ascending cutoffs, last level open
        float f0 = om * sqrtf(1.0f / (sc[0] * sc[0]) + 1.0f / (sc[1] * sc[1]) + 1.0f / (sc[2] * sc[2]));
        lev = 1;
        for (int c = 0; c < A.P - 2; ++c) if (f0 >= A.cutoffs[c]) lev = c + 2;
        if (lev > A.P - 1) lev = A.P - 1;
    }
    int bin;
    if (A.bin && A.bin[i] != 255) {
        bin = A.bin[i];
        if (bin >= A.K) e |= ERR_ASSIGN;
    } else {
        bin = (lev == 0) ? 0 : derive_bin(q, sc, A.K, A.axes);
    }
    const int band = A.band ? A.band[i] : 0;
    if (band >= A.n_bands) e |= ERR_ASSIGN;
    if (e) {
        atomicOr(err, e);
        atomicMin(err + 1, (uint32_t)i);
        return;
    }
    lev = min(lev, A.P - 1);
    bin = min(bin, A.K - 1);
    int group = band * (1 + (A.P - 1) * A.K) + (lev == 0 ? 0 : 1 + (lev - 1) * A.K + bin);  // C24
    if (lev > 0) {  // reading F3: the level's maximum world frequency |omega_vec| = omega |S^-1 (1,1,1)|
        const float f = om * sqrtf(1.0f / (sc[0] * sc[0]) + 1.0f / (sc[1] * sc[1]) + 1.0f / (sc[2] * sc[2]));
        atomicMax(lfmax_bits + lev, __float_as_uint(f));  // f >= 0: the bits order like the values
    }
    // R from the normalised quaternion, W = S^-1 R^T: row k of W = (column k of R) / s_k
    float x = q[0] / qn, y = q[1] / qn, z = q[2] / qn, w = q[3] / qn;
    float R[9] = {1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
                  2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
                  2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)};
    float is0 = 1.0f / sc[0], is1 = 1.0f / sc[1], is2 = 1.0f / sc[2];
    double coef = (double)alpha / (2.0 * 3.14159265358979323846 * (double)sc[0] * (double)sc[1] * (double)sc[2]);
    const float Rs = E * smax * 1.00001f + 1e-7f;  // world bounding sphere of the ellipsoid
    GPrim P;
    P.a = make_float4(mx, my, mz, Rs * Rs);
    P.b = make_float4(R[0] * is0, R[3] * is0, R[6] * is0, om);
    P.c = make_float4(R[1] * is1, R[4] * is1, R[7] * is1, E * E);
    P.d = make_float4(R[2] * is2, R[5] * is2, R[8] * is2, (float)coef);
    out[i] = P;
    gout[i] = (uint8_t)group;
}

// ---------------------------------------------------------------------------------- build
__device__ __forceinline__ uint32_t f2ord(float f) {
    uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ord2f(uint32_t u) {
    return __uint_as_float((u & 0x80000000u) ? (u & 0x7FFFFFFFu) : ~u);
}

// Frame of the BVH boxes: rows m[0..2], m[3..5], m[6..8] are the box axes (identity: world AABBs;
// the NEE light BVH uses a frame whose third axis is the light direction).
struct Frame {
    float m[9];
    int identity;  // 1: world AABBs; 0: AABBs in the rotated frame m; 2: camera-projective boxes
    float eye[3];  // camera mode: eye; m rows = r, u, f (any basis; rays use the same floats)
};

// Camera-projective box of the ellipsoid for rays from the eye: q = x - eye, the ray through
// (a, b) is {q : q.r = a q.f, q.u = b q.f, q.f >= 0}.  a-range: the two planes q.(r - a f) = 0
// through the eye tangent to the ellipsoid, roots of (cf^2 - E^2 Mff) a^2 - 2 (cr cf - E^2 Mrf) a
// + (cr^2 - E^2 Mrr) = 0 (M = (R S)(R S)^T in the basis); the same for b; depth range q.f in
// cf -+ E sqrt(Mff).  Ellipsoids reaching the eye plane get unbounded a, b.  fp64, padded outward.
__device__ inline void camera_box(const GPrim& P, float s0, float s1, float s2, float E, const Frame& F, float* b,
                                  float* center) {
    const double v[3][3] = {{(double)P.b.x * s0, (double)P.b.y * s0, (double)P.b.z * s0},
                            {(double)P.c.x * s1, (double)P.c.y * s1, (double)P.c.z * s1},
                            {(double)P.d.x * s2, (double)P.d.y * s2, (double)P.d.z * s2}};
    const double c[3] = {(double)P.a.x - F.eye[0], (double)P.a.y - F.eye[1], (double)P.a.z - F.eye[2]};
    double cm[3], A[3][3];
    for (int a = 0; a < 3; ++a) {  // a = 0 r, 1 u, 2 f
        const float* f = F.m + 3 * a;
        cm[a] = f[0] * c[0] + f[1] * c[1] + f[2] * c[2];
        for (int k = 0; k < 3; ++k) A[a][k] = f[0] * v[k][0] + f[1] * v[k][1] + f[2] * v[k][2];
    }
    auto dotk = [&](int x, int y) { return A[x][0] * A[y][0] + A[x][1] * A[y][1] + A[x][2] * A[y][2]; };
    const double E2 = (double)E * E, Mff = dotk(2, 2), cf = cm[2];
    const double hf = sqrt(E2 * Mff);
    const double padf = 1e-4 * hf + 4e-6 * (1.0 + fabs(cf));
    b[2] = (float)(cf - hf - padf);
    b[5] = (float)(cf + hf + padf);
    center[2] = (float)cf;
    const double den = cf * cf - E2 * Mff;
    for (int a = 0; a < 2; ++a) {
        if (cf - hf > 0.0 && den > 0.0) {
            const double ca = cm[a], Maa = dotk(a, a), Maf = dotk(a, 2);
            const double disc = fmax(0.0, cf * cf * Maa - 2.0 * ca * cf * Maf + ca * ca * Mff - E2 * (Mff * Maa - Maf * Maf));
            const double mid = (ca * cf - E2 * Maf) / den, half = sqrt(E2 * disc) / den;
            const double pad = 1e-5 * (fabs(mid) + half) + 1e-7;
            b[a] = (float)(mid - half - pad);
            b[3 + a] = (float)(mid + half + pad);
            center[a] = (float)mid;
        } else {
            b[a] = -1e30f;
            b[3 + a] = 1e30f;
            center[a] = 0.0f;
        }
    }
}

// conservative AABB (in frame F) of the ellipsoid {mu + R S u : |u| <= E}:
// half-width along axis a = E |a^T (R S)|
__global__ void k_bounds(const GPrim* prims, int64_t n, float* box, uint32_t* cbounds, Frame F, float* center) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    GPrim P = prims[i];
    // W = S^-1 R^T  ->  (R S)_{jk} = R_jk s_k ; W_kj = R_jk / s_k  ->  R_jk s_k = W_kj s_k^2
    // s_k^2 = 1 / |row_k(W)|^2
    float s0 = 1.0f / (P.b.x * P.b.x + P.b.y * P.b.y + P.b.z * P.b.z);
    float s1 = 1.0f / (P.c.x * P.c.x + P.c.y * P.c.y + P.c.z * P.c.z);
    float s2 = 1.0f / (P.d.x * P.d.x + P.d.y * P.d.y + P.d.z * P.d.z);
    float E = sqrtf(P.c.w);
    float cx = P.a.x, cy = P.a.y, cz = P.a.z, hwx, hwy, hwz;
    float* b = box + 6 * i;
    if (F.identity == 2) {
        float cc[3];
        camera_box(P, s0, s1, s2, E, F, b, cc);
        cx = cc[0]; cy = cc[1]; cz = cc[2];
    } else {
    if (F.identity) {
        hwx = E * sqrtf(P.b.x * P.b.x * s0 * s0 + P.c.x * P.c.x * s1 * s1 + P.d.x * P.d.x * s2 * s2);
        hwy = E * sqrtf(P.b.y * P.b.y * s0 * s0 + P.c.y * P.c.y * s1 * s1 + P.d.y * P.d.y * s2 * s2);
        hwz = E * sqrtf(P.b.z * P.b.z * s0 * s0 + P.c.z * P.c.z * s1 * s1 + P.d.z * P.d.z * s2 * s2);
    } else {
        const float v[3][3] = {{P.b.x * s0, P.b.y * s0, P.b.z * s0},   // columns of R S
                               {P.c.x * s1, P.c.y * s1, P.c.z * s1},
                               {P.d.x * s2, P.d.y * s2, P.d.z * s2}};
        float hw[3], c[3];
        for (int a = 0; a < 3; ++a) {
            const float* f = F.m + 3 * a;
            float acc = 0.0f;
            for (int k = 0; k < 3; ++k) {
                const float dk = f[0] * v[k][0] + f[1] * v[k][1] + f[2] * v[k][2];
                acc += dk * dk;
            }
            hw[a] = E * sqrtf(acc);
            c[a] = f[0] * P.a.x + f[1] * P.a.y + f[2] * P.a.z;
        }
        hwx = hw[0]; hwy = hw[1]; hwz = hw[2];
        cx = c[0]; cy = c[1]; cz = c[2];
    }
    // outward padding: relative 1e-4 of the half width + absolute term for the slab rounding
    float padx = 1e-4f * hwx + 4e-6f * (1.0f + fabsf(cx));
    float pady = 1e-4f * hwy + 4e-6f * (1.0f + fabsf(cy));
    float padz = 1e-4f * hwz + 4e-6f * (1.0f + fabsf(cz));
    b[0] = cx - hwx - padx; b[1] = cy - hwy - pady; b[2] = cz - hwz - padz;
    b[3] = cx + hwx + padx; b[4] = cy + hwy + pady; b[5] = cz + hwz + padz;
    }
    center[3 * i] = cx; center[3 * i + 1] = cy; center[3 * i + 2] = cz;
    atomicMin(cbounds + 0, f2ord(cx)); atomicMin(cbounds + 1, f2ord(cy)); atomicMin(cbounds + 2, f2ord(cz));
    atomicMax(cbounds + 3, f2ord(cx)); atomicMax(cbounds + 4, f2ord(cy)); atomicMax(cbounds + 5, f2ord(cz));
}

__device__ __forceinline__ uint64_t expand3(uint32_t x) {
    uint64_t v = x & 0x1fffffu;
    v = (v | v << 32) & 0x1f00000000ffffull;
    v = (v | v << 16) & 0x1f0000ff0000ffull;
    v = (v | v << 8) & 0x100f00f00f00f00full;
    v = (v | v << 4) & 0x10c30c30c30c30c3ull;
    v = (v | v << 2) & 0x1249249249249249ull;
    return v;
}

#ifndef GF_VIEW_KEYS_2D
#define GF_VIEW_KEYS_2D 2  // bit 0: light frame, bit 1: camera frame (camera: cfg3 +4 %, cfg2 / cfg5 within noise; light: cfg2 NEE +18 %, so off)
#endif
__global__ void k_keys(const GPrim* prims, const uint8_t* groups, int64_t n, const uint32_t* cbounds, uint64_t* keys,
                       uint32_t* vals, Frame F, const float* center, KeyMap km) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    GPrim P = prims[i];
    float lo[3] = {ord2f(cbounds[0]), ord2f(cbounds[1]), ord2f(cbounds[2])};
    float hi[3] = {ord2f(cbounds[3]), ord2f(cbounds[4]), ord2f(cbounds[5])};
    float c[3] = {P.a.x, P.a.y, P.a.z};
    if (F.identity != 1)
        for (int a = 0; a < 3; ++a) c[a] = center[3 * i + a];
    uint32_t q[3];
    for (int k = 0; k < 3; ++k) {
        float ext = hi[k] - lo[k];
        float t = ext > 0.0f ? (c[k] - lo[k]) / ext : 0.5f;
        t = fminf(fmaxf(t, 0.0f), 1.0f);
        q[k] = min((uint32_t)(t * 524288.0f), 524287u);  // 19 bits
    }
    const uint32_t group = km.k[groups[i] & (kMaxGroups - 1)];
    if ((F.identity == 0 && (GF_VIEW_KEYS_2D & 1)) || (F.identity == 2 && (GF_VIEW_KEYS_2D & 2))) {
        // view frames: 2D Morton of the two axes across the rays (19 bits each), then the axis along
        // them (19 bits) -- the top of the tree partitions columns, the bottom orders a column
        uint64_t m2 = 0;
        for (int b = 18; b >= 0; --b) m2 = (m2 << 2) | (((q[0] >> b) & 1u) << 1) | ((q[1] >> b) & 1u);
        keys[i] = ((uint64_t)group << 57) | (m2 << 19) | q[2];
    } else {
        keys[i] = ((uint64_t)group << 57) | (expand3(q[0]) << 2) | (expand3(q[1]) << 1) | expand3(q[2]);
    }
    vals[i] = (uint32_t)i;
}

__device__ __forceinline__ int delta(const uint64_t* keys, int64_t n, int64_t i, int64_t j) {
    if (j < 0 || j >= n) return -1;
    uint64_t a = keys[i], b = keys[j];
    if (a == b) return 64 + __clz((uint32_t)(i ^ j));
    return __clzll(a ^ b);
}

// Karras 2012 radix tree: internal nodes 0..n-2, leaf k stored as n-1+k
__global__ void k_karras(const uint64_t* keys, int64_t n, int32_t* left, int32_t* right, int32_t* parent,
                         int32_t* rlo, int32_t* rhi) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n - 1) return;
    int d = (delta(keys, n, i, i + 1) - delta(keys, n, i, i - 1)) >= 0 ? 1 : -1;
    int dmin = delta(keys, n, i, i - d);
    int64_t lmax = 2;
    while (delta(keys, n, i, i + lmax * d) > dmin) lmax *= 2;
    int64_t l = 0;
    for (int64_t t = lmax / 2; t >= 1; t /= 2)
        if (delta(keys, n, i, i + (l + t) * d) > dmin) l += t;
    int64_t j = i + l * d;
    int dnode = delta(keys, n, i, j);
    int64_t s = 0;
    int64_t t = l;
    do {
        t = (t + 1) / 2;
        if (delta(keys, n, i, i + (s + t) * d) > dnode) s += t;
    } while (t > 1);
    int64_t gamma = i + s * d + (d < 0 ? -1 : 0);
    int64_t lo = i < j ? i : j, hi = i < j ? j : i;
    int32_t L = (lo == gamma) ? (int32_t)(n - 1 + gamma) : (int32_t)gamma;
    int32_t Rr = (hi == gamma + 1) ? (int32_t)(n - 1 + gamma + 1) : (int32_t)(gamma + 1);
    left[i] = L; right[i] = Rr;
    parent[L] = (int32_t)i; parent[Rr] = (int32_t)i;
    rlo[i] = (int32_t)lo; rhi[i] = (int32_t)hi;
}

struct RefitArgs {
    int64_t n;
    const int32_t *left, *right, *parent, *perm;
    const float* pbox;     // per original prim, 6 floats
    const uint8_t* group;  // original order
    float* nbox;           // 2n-1 nodes x 6
    uint32_t *nmask, *ncount, *nsize;
    uint32_t* flags;
    uint32_t leafmax;
};

__device__ __forceinline__ bool collapsed(uint32_t count, uint32_t mask, uint32_t leafmax) {
    return count <= leafmax && __popc(mask) == 1;
}

__global__ void k_refit(RefitArgs A) {
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= A.n) return;
    int64_t x = A.n - 1 + k;
    int32_t pi = A.perm[k];
    const float* pb = A.pbox + 6 * (int64_t)pi;
    for (int c = 0; c < 6; ++c) A.nbox[6 * x + c] = pb[c];
    A.nmask[x] = 1u << A.group[pi];
    A.ncount[x] = 1;
    A.nsize[x] = 1;
    __threadfence();
    while (x != 0) {
        int32_t p = A.parent[x];
        if (atomicAdd(A.flags + p, 1u) == 0) return;  // first arrival: sibling not done yet
        __threadfence();
        int32_t L = A.left[p], R = A.right[p];
        const volatile float* bl = A.nbox + 6 * (int64_t)L;
        const volatile float* br = A.nbox + 6 * (int64_t)R;
        for (int c = 0; c < 3; ++c) {
            A.nbox[6 * (int64_t)p + c] = fminf(bl[c], br[c]);
            A.nbox[6 * (int64_t)p + 3 + c] = fmaxf(bl[3 + c], br[3 + c]);
        }
        uint32_t m = ((volatile uint32_t*)A.nmask)[L] | ((volatile uint32_t*)A.nmask)[R];
        uint32_t cnt = ((volatile uint32_t*)A.ncount)[L] + ((volatile uint32_t*)A.ncount)[R];
        A.nmask[p] = m;
        A.ncount[p] = cnt;
        A.nsize[p] = collapsed(cnt, m, A.leafmax) ? 1u : 1u + ((volatile uint32_t*)A.nsize)[L] + ((volatile uint32_t*)A.nsize)[R];
        __threadfence();
        x = p;
    }
}

struct LayoutArgs {
    int64_t n;
    const int32_t *left, *right, *parent, *rlo;
    const float* nbox;
    const uint32_t *nmask, *ncount, *nsize;
    GNode* out;
    uint32_t total;
    uint32_t* max_depth;
    uint32_t leafmax;
};

__global__ void k_layout(LayoutArgs A) {
    int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t nn = 2 * A.n - 1;
    if (x >= nn) return;
    int64_t root = 0;
    if (x != root) {
        int32_t p = A.parent[x];
        if (collapsed(A.ncount[p], A.nmask[p], A.leafmax)) return;  // inside a collapsed leaf
    }
    // pre-order index: walk to the root
    uint32_t idx = 0, depth = 0;
    int64_t cur = x;
    while (cur != root) {
        int32_t p = A.parent[cur];
        idx += 1;
        ++depth;
        if (A.right[p] == cur) idx += A.nsize[A.left[p]];
        cur = p;
    }
    atomicMax(A.max_depth, depth);
    uint32_t cnt = A.ncount[x], m = A.nmask[x];
    bool leaf = collapsed(cnt, m, A.leafmax);
    uint32_t skip = idx + A.nsize[x];
    uint32_t info;
    if (leaf) {
        uint32_t first = (x >= A.n - 1) ? (uint32_t)(x - (A.n - 1)) : (uint32_t)A.rlo[x];
        info = (first << 8) | (cnt << 5) | (uint32_t)(__ffs(m) - 1);
    } else {
        info = m;
    }
    const float* b = A.nbox + 6 * x;
    GNode N;
    N.lo = make_float4(b[0], b[1], b[2], __uint_as_float(skip | (leaf ? kLeafBit : 0u)));
    N.hi = make_float4(b[3], b[4], b[5], __uint_as_float(info));
    A.out[idx] = N;
}

// children pairs for the warp traversal: internal node i has children i + 1 and skip(i + 1)
__global__ void k_pair(const GNode* __restrict__ nodes, uint32_t total, GNode2* __restrict__ out) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= total) return;
    const uint32_t sk = __float_as_uint(nodes[i].lo.w);
    if (sk & kLeafBit) return;
    const uint32_t c0 = i + 1;
    const GNode a = nodes[c0];
    const uint32_t c1 = __float_as_uint(a.lo.w) & ~kLeafBit;
    const GNode b = nodes[c1];
    const uint32_t r0 = (__float_as_uint(a.lo.w) & kLeafBit) ? kLeafBit : c0;
    const uint32_t r1 = (__float_as_uint(b.lo.w) & kLeafBit) ? kLeafBit : c1;
    GNode2 o;
    o.lo0 = make_float4(a.lo.x, a.lo.y, a.lo.z, __uint_as_float(r0));
    o.hi0 = a.hi;
    o.lo1 = make_float4(b.lo.x, b.lo.y, b.lo.z, __uint_as_float(r1));
    o.hi1 = b.hi;
    out[i] = o;
}

// as k_pair, node count read on the device (asynchronous light-BVH build)
__global__ void k_pair_dev(const GNode* __restrict__ nodes, const uint32_t* __restrict__ total, int64_t bound,
                           GNode2* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= bound || i >= (int64_t)*total) return;
    const uint32_t sk = __float_as_uint(nodes[i].lo.w);
    if (sk & kLeafBit) return;
    const uint32_t c0 = (uint32_t)i + 1;
    const GNode a = nodes[c0];
    const uint32_t c1 = __float_as_uint(a.lo.w) & ~kLeafBit;
    const GNode b = nodes[c1];
    GNode2 o;
    o.lo0 = make_float4(a.lo.x, a.lo.y, a.lo.z, __uint_as_float((__float_as_uint(a.lo.w) & kLeafBit) ? kLeafBit : c0));
    o.hi0 = a.hi;
    o.lo1 = make_float4(b.lo.x, b.lo.y, b.lo.z, __uint_as_float((__float_as_uint(b.lo.w) & kLeafBit) ? kLeafBit : c1));
    o.hi1 = b.hi;
    out[i] = o;
}

__global__ void k_gather(const GPrim* in, const int32_t* perm, int64_t n, GPrim* out, int32_t* perm_out) {
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    out[k] = in[perm[k]];
    perm_out[k] = perm[k];
}

}  // namespace gfk

// ------------------------------------------------------------------------------ host side
using namespace gfk;

static inline unsigned nblk(int64_t n, int b) { return (unsigned)((n + b - 1) / b); }

cudaError_t gf_launch_load(const LoadArgs& A, void* out, uint8_t* group, uint32_t* err, uint32_t* lfmax_bits,
                           cudaStream_t st) {
    if (A.n == 0) return cudaSuccess;
    k_load_prims<<<nblk(A.n, 256), 256, 0, st>>>(A, (GPrim*)out, group, err, lfmax_bits);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- C12: group f0 = sqrt(3) median omega
// keys (level << 32 | bits(omega)) of the Gabor members (omega >= 0: the bits order like the values),
// radix-sorted; per level its member count, then the median from the sorted run of the level.
__global__ void k_f0_keys(const GPrim* prims, const uint8_t* group, int64_t n, int G0, int K, uint64_t* keys,
                          uint32_t* vals, uint32_t* counts) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int gl = group[i] % G0, lev = gl == 0 ? 0 : 1 + (gl - 1) / K;
    keys[i] = ((uint64_t)(uint32_t)lev << 32) | __float_as_uint(prims[i].b.w);  // b.w = omega as loaded
    vals[i] = 0u;
    if (lev > 0) atomicAdd(counts + lev, 1u);
}
__global__ void k_f0_count0(uint32_t* counts, int64_t n) {
    uint32_t rest = 0;
    for (int l = 1; l < kMaxLevels; ++l) rest += counts[l];
    counts[0] = (uint32_t)n - rest;
}
__global__ void k_f0_median(const uint64_t* sorted, const uint32_t* counts, int64_t n, int P, float* f0) {
    const int l = threadIdx.x;
    if (l >= kMaxLevels) return;
    f0[l] = 0.0f;
    if (l == 0 || l >= P) return;
    uint32_t off = 0;
    for (int k = 0; k < l; ++k) off += counts[k];
    const uint32_t c = counts[l];
    if (c == 0) return;
    const float a = __uint_as_float((uint32_t)sorted[off + (c - 1) / 2]), b = __uint_as_float((uint32_t)sorted[off + c / 2]);
    const float med = (c & 1u) ? b : __fdiv_rn(__fadd_rn(a, b), 2.0f);  // numpy's median (fp32 mean of the middle two)
    f0[l] = (float)((double)med * 1.7320508075688772);  // whitened |k_W| = sqrt(3) omega (C2)
}
cudaError_t gf_launch_group_f0(const GPrim* prims, const uint8_t* group, int64_t n, int P, int K, int G0,
                               const BuildScratch& S, float* f0_dev, cudaStream_t st) {
    cudaError_t e;
    uint32_t* counts = S.flags;  // kMaxLevels counters (flags are rewritten by the BVH build afterwards)
    if ((e = cudaMemsetAsync(counts, 0, sizeof(uint32_t) * kMaxLevels, st))) return e;
    if (n > 0) {
        k_f0_keys<<<nblk(n, 256), 256, 0, st>>>(prims, group, n, G0, K, S.keys_in, S.vals_in, counts);
        size_t tb = S.sort_temp_bytes;
        if ((e = cub::DeviceRadixSort::SortPairs(S.sort_temp, tb, S.keys_in, S.keys_out, S.vals_in, S.vals_out, (int)n,
                                                 0, 64, st)))
            return e;
    }
    k_f0_count0<<<1, 1, 0, st>>>(counts, n);  // level 0 precedes level 1 in the sorted order
    k_f0_median<<<1, 32, 0, st>>>(S.keys_out, counts, n, P, f0_dev);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- motion-blur group mask (M1-M3)
// omega_vec = R S^-1 (w,w,w)^T = W^T (w,w,w)^T: w times the sum of the rows of W
__device__ __forceinline__ float3 omega_vec(const GPrim& P) {
    return make_float3(P.b.w * (P.b.x + P.c.x + P.d.x), P.b.w * (P.b.y + P.c.y + P.d.y),
                       P.b.w * (P.b.z + P.c.z + P.d.z));
}
struct MbScratch {
    unsigned long long ref[kMaxGroups];  // (bits(|omega_vec|) << 32) | ~index: max -> largest, first on ties
    double sum[kMaxGroups][3];
    unsigned long long cnt[kMaxGroups];
    float att[kMaxGroups];
    uint32_t mask;
};
__global__ void k_mb_ref(const GPrim* prims, const uint8_t* group, int64_t n, MbScratch* M) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float3 w = omega_vec(prims[i]);
    const float f = sqrtf(w.x * w.x + w.y * w.y + w.z * w.z);
    atomicMax(&M->ref[group[i]], ((unsigned long long)__float_as_uint(f) << 32) | (0xFFFFFFFFu - (uint32_t)i));
}
__global__ void k_mb_sum(const GPrim* prims, const uint8_t* group, int64_t n, MbScratch* M) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int g = group[i];
    const uint32_t ri = 0xFFFFFFFFu - (uint32_t)(M->ref[g] & 0xFFFFFFFFull);
    const float3 w = omega_vec(prims[i]), r = omega_vec(prims[ri]);
    const double sg = (w.x * r.x + w.y * r.y + w.z * r.z) < 0.0f ? -1.0 : 1.0;  // +-omega_vec: the same cosine
    atomicAdd(&M->sum[g][0], sg * w.x);
    atomicAdd(&M->sum[g][1], sg * w.y);
    atomicAdd(&M->sum[g][2], sg * w.z);
    atomicAdd(&M->cnt[g], 1ull);
}
__global__ void k_mb_fin(MbScratch* M, int G, int G0, float dx, float dy, float dz, float m, float thr) {
    __shared__ uint32_t mask;
    if (threadIdx.x == 0) mask = 0;
    __syncthreads();
    const int g = threadIdx.x;
    if (g < G) {
        double att = 1.0;
        if (g % G0 != 0 && M->cnt[g] > 0) {
            const double dn = sqrt((double)dx * dx + (double)dy * dy + (double)dz * dz);
            const double k = fabs((M->sum[g][0] * dx + M->sum[g][1] * dy + M->sum[g][2] * dz) / dn) / (double)M->cnt[g];
            const double x = 0.5 * (double)m * k;
            att = x == 0.0 ? 1.0 : fabs(sin(x) / x);  // box filter on a cosine of frequency k (M2)
        }
        M->att[g] = (float)att;
        if (att >= (double)thr) atomicOr(&mask, 1u << g);
    }
    __syncthreads();
    if (threadIdx.x == 0) M->mask = mask;
}
size_t gf_mb_scratch_bytes() { return sizeof(MbScratch); }
cudaError_t gf_launch_mb_mask(const GPrim* prims, const uint8_t* group, int64_t n, int32_t G, int32_t G0, const float* dir,
                              float m, float threshold, void* dev_scratch, uint32_t* mask_host, float* att_host,
                              cudaStream_t st) {
    cudaError_t e;
    MbScratch* M = (MbScratch*)dev_scratch;
    if ((e = cudaMemsetAsync(M, 0, sizeof(MbScratch), st))) return e;
    if (n > 0) {
        k_mb_ref<<<nblk(n, 256), 256, 0, st>>>(prims, group, n, M);
        k_mb_sum<<<nblk(n, 256), 256, 0, st>>>(prims, group, n, M);
    }
    k_mb_fin<<<1, 32, 0, st>>>(M, G, G0, dir[0], dir[1], dir[2], m, threshold);
    if ((e = cudaMemcpyAsync(mask_host, &M->mask, sizeof(uint32_t), cudaMemcpyDeviceToHost, st))) return e;
    if (att_host && (e = cudaMemcpyAsync(att_host, M->att, sizeof(float) * G, cudaMemcpyDeviceToHost, st))) return e;
    if ((e = cudaStreamSynchronize(st))) return e;
    return cudaGetLastError();
}

// ---------------------------------------------------------------- C8': adaptive extents (Eq. 15)
__global__ void k_adaptive_extent(const float* scale, const float* alpha, const float* omega, int64_t n, float eps,
                                  float* out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double s0 = scale[3 * i], s1 = scale[3 * i + 1], s2 = scale[3 * i + 2];
    const double smax = fmax(s0, fmax(s1, s2));
    const double a = fmax((double)alpha[i], 1e-30), w = omega[i];
    const double arg = -2.0 * log((double)eps * 2.0 * 3.14159265358979323846 * s0 * s1 * s2 / (a * smax)) - 3.0 * w * w;
    out[i] = (float)fmin(3.0, fmax(1e-3, sqrt(fmax(arg, 0.0))));
}
cudaError_t gf_launch_adaptive_extent(const float* scale, const float* alpha, const float* omega, int64_t n, float eps,
                                      float* out, cudaStream_t st) {
    if (n > 0) k_adaptive_extent<<<nblk(n, 256), 256, 0, st>>>(scale, alpha, omega, n, eps, out);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- 64-bit hash of a workspace (replica check)
// H = sum_i mix(word_i ^ (i * golden)) mod 2^64 (splitmix64 finaliser): order-independent reduction,
// position-sensitive words; equal builds give equal hashes.
__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__global__ void k_hash(const unsigned long long* w, size_t nw, unsigned long long* out) {
    unsigned long long h = 0;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < nw; i += (size_t)gridDim.x * blockDim.x)
        h += mix64(w[i] ^ (0x9E3779B97F4A7C15ull * (unsigned long long)(i + 1)));
    for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xFFFFFFFFu, h, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, h);
}
cudaError_t gf_launch_hash(const void* data, size_t bytes, unsigned long long* out_dev, cudaStream_t st) {
    cudaError_t e;
    if ((e = cudaMemsetAsync(out_dev, 0, sizeof(unsigned long long), st))) return e;
    const size_t nw = bytes / 8;
    if (nw > 0) k_hash<<<1184, 256, 0, st>>>((const unsigned long long*)data, nw, out_dev);
    return cudaGetLastError();
}

size_t gf_sort_temp_bytes(int64_t n) {
    size_t bytes = 0;
    if (n <= 0) return 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                    (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)n, 0, 64);
    return bytes;
}

BuildScratch gf_scratch_layout(int64_t n, char* base) {
    BuildScratch s;
    size_t off = 0;
    auto take = [&](size_t bytes) { char* p = base ? base + off : nullptr; off += (bytes + 255) & ~(size_t)255; return p; };
    int64_t nn = n > 0 ? 2 * n - 1 : 1;
    s.pbox = (float*)take(sizeof(float) * 6 * (n > 0 ? n : 1));
    s.center = (float*)take(sizeof(float) * 3 * (n > 0 ? n : 1));
    s.cbounds = (uint32_t*)take(sizeof(uint32_t) * 8);
    s.keys_in = (uint64_t*)take(sizeof(uint64_t) * (n > 0 ? n : 1));
    s.keys_out = (uint64_t*)take(sizeof(uint64_t) * (n > 0 ? n : 1));
    s.vals_in = (uint32_t*)take(sizeof(uint32_t) * (n > 0 ? n : 1));
    s.vals_out = (uint32_t*)take(sizeof(uint32_t) * (n > 0 ? n : 1));
    s.left = (int32_t*)take(sizeof(int32_t) * (n > 0 ? n : 1));
    s.right = (int32_t*)take(sizeof(int32_t) * (n > 0 ? n : 1));
    s.parent = (int32_t*)take(sizeof(int32_t) * nn);
    s.rlo = (int32_t*)take(sizeof(int32_t) * (n > 0 ? n : 1));
    s.rhi = (int32_t*)take(sizeof(int32_t) * (n > 0 ? n : 1));
    s.nbox = (float*)take(sizeof(float) * 6 * nn);
    s.nmask = (uint32_t*)take(sizeof(uint32_t) * nn);
    s.ncount = (uint32_t*)take(sizeof(uint32_t) * nn);
    s.nsize = (uint32_t*)take(sizeof(uint32_t) * nn);
    s.flags = (uint32_t*)take(sizeof(uint32_t) * (n > 0 ? n : 1));
    s.sort_temp_bytes = gf_sort_temp_bytes(n);
    s.sort_temp = take(s.sort_temp_bytes + 256);
    s.total_bytes = off;
    return s;
}

// builds into nodes/sorted; returns node count via *n_nodes (host, after sync)
cudaError_t gf_launch_build(const void* prims_v, const uint8_t* group, int64_t n, const BuildScratch& S, void* nodes_v,
                            void* nodes2_v, void* sorted_v, int32_t* perm, uint32_t* n_nodes, uint32_t* max_depth,
                            float* root_box, const KeyMap& km, cudaStream_t st) {
    const GPrim* prims = (const GPrim*)prims_v;
    GNode* nodes = (GNode*)nodes_v;
    cudaError_t e;
    *n_nodes = 0;
    *max_depth = 0;
    if (n == 0) return cudaSuccess;
    uint32_t init[8] = {0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0u, 0u, 0u, 0u, 0u};
    if ((e = cudaMemcpyAsync(S.cbounds, init, sizeof(init), cudaMemcpyHostToDevice, st))) return e;
    Frame I{{1, 0, 0, 0, 1, 0, 0, 0, 1}, 1, {0, 0, 0}};
    k_bounds<<<nblk(n, 256), 256, 0, st>>>(prims, n, S.pbox, S.cbounds, I, S.center);
    k_keys<<<nblk(n, 256), 256, 0, st>>>(prims, group, n, S.cbounds, S.keys_in, S.vals_in, I, S.center, km);
    size_t tb = S.sort_temp_bytes;
    if ((e = cub::DeviceRadixSort::SortPairs(S.sort_temp, tb, S.keys_in, S.keys_out, S.vals_in, S.vals_out, (int)n,
                                             0, 64, st)))
        return e;
    if (n > 1) {
        k_karras<<<nblk(n - 1, 256), 256, 0, st>>>(S.keys_out, n, S.left, S.right, S.parent, S.rlo, S.rhi);
        if ((e = cudaMemsetAsync(S.flags, 0, sizeof(uint32_t) * n, st))) return e;
    }
    RefitArgs R{n, S.left, S.right, S.parent, (const int32_t*)S.vals_out, S.pbox, group, S.nbox, S.nmask, S.ncount,
                S.nsize, S.flags, (uint32_t)kLeafMax};
    k_refit<<<nblk(n, 256), 256, 0, st>>>(R);
    // root (node 0 = internal root, or leaf 0 when n == 1 stored at n-1+0 = 0)
    uint32_t total = 0;
    if ((e = cudaMemcpyAsync(&total, S.nsize, sizeof(uint32_t), cudaMemcpyDeviceToHost, st))) return e;
    if ((e = cudaStreamSynchronize(st))) return e;
    if ((e = cudaMemsetAsync(S.cbounds, 0, sizeof(uint32_t), st))) return e;  // reused: max depth
    LayoutArgs L{n, S.left, S.right, S.parent, S.rlo, S.nbox, S.nmask, S.ncount, S.nsize, nodes, total, S.cbounds,
                 (uint32_t)kLeafMax};
    k_layout<<<nblk(2 * n - 1, 256), 256, 0, st>>>(L);
    k_pair<<<nblk(total, 256), 256, 0, st>>>(nodes, total, (GNode2*)nodes2_v);
    k_gather<<<nblk(n, 256), 256, 0, st>>>(prims, (const int32_t*)S.vals_out, n, (GPrim*)sorted_v, perm);
    if ((e = cudaMemcpyAsync(root_box, S.nbox, sizeof(float) * 6, cudaMemcpyDeviceToHost, st))) return e;
    if ((e = cudaMemcpyAsync(max_depth, S.cbounds, sizeof(uint32_t), cudaMemcpyDeviceToHost, st))) return e;
    if ((e = cudaStreamSynchronize(st))) return e;
    *n_nodes = total;
    return cudaGetLastError();
}

#ifndef GF_LIGHT_LEAFMAX
#define GF_LIGHT_LEAFMAX 3  // primitives per leaf of the NEE light BVH (r2, level keys: 2 slower, 4 -2 %)
#endif
#ifndef GF_CAM_LEAFMAX
#define GF_CAM_LEAFMAX 3  // primitives per leaf of the camera BVH
#endif
static_assert(GF_LIGHT_LEAFMAX >= 1 && GF_LIGHT_LEAFMAX <= kLeafMax, "warp traversal buffers hold kLeafMax per leaf");
static_assert(GF_CAM_LEAFMAX >= 1 && GF_CAM_LEAFMAX <= kLeafMax, "k_ff walks the camera BVH with kLeafMax buffers");
// Asynchronous build in frame F (host rows): same kernels, no host synchronisation; the node count
// stays on the device (S.nsize[0]) and the tree depth is written to *depth (device).
cudaError_t gf_launch_build_frame(const void* prims_v, const uint8_t* group, int64_t n, const BuildScratch& S,
                                  const float* F, const float* eye, void* nodes_v, void* nodes2_v, void* sorted_v,
                                  int32_t* perm, uint32_t* depth, const KeyMap& km, cudaStream_t st) {
    const GPrim* prims = (const GPrim*)prims_v;
    GNode* nodes = (GNode*)nodes_v;
    cudaError_t e;
    if ((e = cudaMemsetAsync(depth, 0, sizeof(uint32_t), st))) return e;
    if (n == 0) return cudaSuccess;
    Frame Fr{};
    for (int k = 0; k < 9; ++k) Fr.m[k] = F[k];
    Fr.identity = eye ? 2 : 0;
    for (int k = 0; k < 3; ++k) Fr.eye[k] = eye ? eye[k] : 0.0f;
    if ((e = cudaMemsetAsync(S.cbounds, 0xFF, sizeof(uint32_t) * 3, st))) return e;
    if ((e = cudaMemsetAsync(S.cbounds + 3, 0, sizeof(uint32_t) * 3, st))) return e;
    k_bounds<<<nblk(n, 256), 256, 0, st>>>(prims, n, S.pbox, S.cbounds, Fr, S.center);
    k_keys<<<nblk(n, 256), 256, 0, st>>>(prims, group, n, S.cbounds, S.keys_in, S.vals_in, Fr, S.center, km);
    size_t tb = S.sort_temp_bytes;
    if ((e = cub::DeviceRadixSort::SortPairs(S.sort_temp, tb, S.keys_in, S.keys_out, S.vals_in, S.vals_out, (int)n,
                                             0, 64, st)))
        return e;
    if (n > 1) {
        k_karras<<<nblk(n - 1, 256), 256, 0, st>>>(S.keys_out, n, S.left, S.right, S.parent, S.rlo, S.rhi);
        if ((e = cudaMemsetAsync(S.flags, 0, sizeof(uint32_t) * n, st))) return e;
    }
    RefitArgs R{n, S.left, S.right, S.parent, (const int32_t*)S.vals_out, S.pbox, group, S.nbox, S.nmask, S.ncount,
                S.nsize, S.flags, (uint32_t)(eye ? GF_CAM_LEAFMAX : GF_LIGHT_LEAFMAX)};
    k_refit<<<nblk(n, 256), 256, 0, st>>>(R);
    LayoutArgs L{n, S.left, S.right, S.parent, S.rlo, S.nbox, S.nmask, S.ncount, S.nsize, nodes, 0, depth,
                 (uint32_t)(eye ? GF_CAM_LEAFMAX : GF_LIGHT_LEAFMAX)};
    k_layout<<<nblk(2 * n - 1, 256), 256, 0, st>>>(L);
    k_pair_dev<<<nblk(2 * n - 1, 256), 256, 0, st>>>(nodes, S.nsize, 2 * n - 1, (GNode2*)nodes2_v);
    k_gather<<<nblk(n, 256), 256, 0, st>>>(prims, (const int32_t*)S.vals_out, n, (GPrim*)sorted_v, perm);
    return cudaGetLastError();
}

// key prefix of each group: mode GF_BVH_KEYS_GROUP the group, GF_BVH_KEYS_LEVEL its (band, level) class
KeyMap gf_keymap(const SceneDev& sc, int mode) {
    KeyMap m;
    for (int g = 0; g < kMaxGroups; ++g) {
        const int g0 = sc.G0 > 0 ? g % sc.G0 : 0, band = sc.G0 > 0 ? g / sc.G0 : 0;
        const int level = g0 == 0 ? 0 : 1 + (g0 - 1) / (sc.K > 0 ? sc.K : 1);
        m.k[g] = (uint8_t)((mode == 0 ? g : band * sc.P + level) & 127);
    }
    return m;
}
