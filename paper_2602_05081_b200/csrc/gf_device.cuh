// gf_device.cuh -- device-side building blocks of the Gabor Fields hot path (sm_100a).
//
// Data layout in HBM:
//   GPrim  64 B  = 4 x float4 : (mu.xyz, Rs^2) (W row0, omega) (W row1, E^2) (W row2, c)
//          with W = S^-1 R^T (PCA whitening, reading C1), c = alpha / (2 pi s1 s2 s3),
//          k_W = (omega, omega, omega) implicit (reading C2), Rs = E s_max the world bounding
//          sphere (one 16-byte load pre-test); the group lives in the leaf (and a side array).
//   GNode  32 B  = 2 x float4 : (lo.xyz, skip | leaf<<31) (hi.xyz, info)
//          depth-first layout, hit -> i+1, miss -> skip; info = group mask (internal) or
//          first<<8 | count<<5 | group (leaf).
//   GNode2 64 B  = the two children of internal node i (same DFS index): (lo.xyz, ref) (hi.xyz, info)
//          per child, ref = the child's DFS index (internal) or kLeafBit (leaf); used by the
//          warp-per-ray traversal, which tests both children of a node in one step.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

// Bounds checks of the shared-memory frontiers and queues (debug builds, -DGF_DEBUG_CHECKS: the
// stand-in for compute-sanitizer, which this pool does not run): a failed check prints and traps.
#ifdef GF_DEBUG_CHECKS
#include <cstdio>
#define GF_CHECK(c)                                                                         \
    do {                                                                                    \
        if (!(c)) {                                                                         \
            printf("GF_CHECK failed: %s (%s:%d)\n", #c, __FILE__, __LINE__);               \
            __trap();                                                                       \
        }                                                                                   \
    } while (0)
#else
#define GF_CHECK(c) \
    do {            \
    } while (0)
#endif

namespace gfk {

constexpr int kMaxGroups = 32;
constexpr int kMaxLevels = 8;
#ifndef GF_LEAFMAX
#define GF_LEAFMAX 3
#endif
constexpr int kLeafMax = GF_LEAFMAX;  // primitives per BVH leaf (<= 7: 3-bit count)
constexpr uint32_t kLeafBit = 0x80000000u;

struct __align__(16) GPrim {
    float4 a, b, c, d;
};
struct __align__(16) GNode {
    float4 lo, hi;
};
struct __align__(16) GNode2 {
    float4 lo0, hi0, lo1, hi1;
};

// ------------------------------------------------------------------ policy (Tables B1/B2)
struct PolicyDev {
    uint32_t static_mask;
    int32_t ls, os;
    float delta;
    double th[kMaxLevels + 1];    // (j/P)^(1-beta), j = 0..P      (B1 power law buckets)
    double psi[kMaxLevels + 1];   // (k/(P-1))^(1-beta), k = 0..P-1 (B1 PL + CV buckets, C13)
    float w_pl[kMaxLevels];       // 1/(th[j+1]-th[j])
    float w_plcv[kMaxLevels];     // 1/(psi[k+1]-psi[k])
    float w_acc[kMaxLevels];      // 1/(1-th[j])                   (C14)
};

struct SceneDev {
    int32_t P, K, G;     // G = n_bands * G0 groups in all (C24)
    int32_t G0, n_bands; // groups per spatial band (1 + (P-1) K), bands (config-5 distance bands)
    float axes[3 * 16];
    float f0[kMaxGroups];
};

// ------------------------------------------------------------------ Philox4x32-10
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
        uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
        c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
        k.x += 0x9E3779B9u;
        k.y += 0xBB67AE85u;
    }
    return c;
}
enum { ST_EXT = 0, ST_NEE = 1, ST_SCAT = 2, ST_CAM = 3, ST_TRK = 4, ST_TRK_NEE = 5, ST_FOV = 6, ST_MB = 7, ST_UNI = 8 };
// 4 uniforms k0..k0+3 of a stream (k0 multiple of 4) -- one Philox call
__device__ __forceinline__ uint4 stream_block(uint64_t seed, uint32_t pix, uint32_t smp, uint32_t d, uint32_t st,
                                              uint32_t k0) {
    return philox4x32_10(make_uint4(pix, smp, d, (st << 16) | (k0 >> 2)),
                         make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
}
__device__ __forceinline__ float u01(uint32_t x) { return (float)(x >> 8) * (1.0f / 16777216.0f); }
__device__ __forceinline__ uint32_t word(const uint4& v, int i) {
    return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w));
}
// uniform k of a stream (k < 16)
__device__ __forceinline__ float stream_u(uint64_t seed, uint32_t pix, uint32_t smp, uint32_t d, uint32_t st,
                                          uint32_t k) {
    uint4 b = stream_block(seed, pix, smp, d, st, k & ~3u);
    return u01(word(b, k & 3));
}

// Evaluate a LOD policy for one ray segment (same decisions as the oracle: integer draws,
// fp64 threshold compares, fp32 orientation arithmetic with explicitly rounded ops).
// ul: level uniform; uo[l-1]: orientation uniform of Gabor level l. Writes weights for
// selected groups into w[] (others untouched) and returns the mask.
__device__ inline uint32_t policy_eval(const PolicyDev& pol, const SceneDev& sc, float3 dir, float ul,
                                       const float* uo, float* w) {
    const int P = sc.P, K = sc.K;
    float lw[kMaxLevels];
#pragma unroll
    for (int l = 0; l < kMaxLevels; ++l) lw[l] = 0.0f;
    const uint32_t m24 = (uint32_t)(ul * 16777216.0f);
    const double ud = (double)ul;
    switch (pol.ls) {
    case 1: { int j = (int)(((uint64_t)m24 * (uint64_t)P) >> 24); lw[j] = (float)P; break; }
    case 2: {
        int j = 0;
        for (int k = 1; k < P; ++k) if (ud >= pol.th[k]) j = k;
        lw[j] = pol.w_pl[j];
        break;
    }
    case 3: {
        lw[0] = 1.0f;
        if (P > 1) { int j = 1 + (int)(((uint64_t)m24 * (uint64_t)(P - 1)) >> 24); lw[j] = (float)(P - 1); }
        break;
    }
    case 4: {
        lw[0] = 1.0f;
        if (P > 1) {
            int k = 0;
            for (int q = 1; q < P - 1; ++q) if (ud >= pol.psi[q]) k = q;
            lw[1 + k] = pol.w_plcv[k];
        }
        break;
    }
    case 5: {
        int kk = 0;
        for (int q = 1; q < P; ++q) if (ud >= pol.th[q]) kk = q;
        for (int j = 0; j <= kk; ++j) lw[j] = pol.w_acc[j];
        break;
    }
    default:
        for (int l = 0; l < P; ++l) lw[l] = 1.0f;
    }
    uint32_t mask = 0;
    if (lw[0] != 0.0f) { mask |= 1u; w[0] = lw[0]; }
    for (int l = 1; l < P; ++l) {
        if (lw[l] == 0.0f) continue;
        float a[16], bw[16];
        for (int b = 0; b < K; ++b) {
            bw[b] = 0.0f;
            a[b] = fabsf(__fmaf_rn(dir.x, sc.axes[3 * b], __fmaf_rn(dir.y, sc.axes[3 * b + 1],
                                                                   __fmul_rn(dir.z, sc.axes[3 * b + 2]))));
        }
        const float u = uo[l - 1];
        const uint32_t mu24 = (uint32_t)(u * 16777216.0f);
        switch (pol.os) {
        case 1:
            for (int b = 0; b < K; ++b) if (a[b] <= pol.delta) bw[b] = 1.0f;
            break;
        case 2: { int b = (int)(((uint64_t)mu24 * (uint64_t)K) >> 24); bw[b] = (float)K; break; }
        case 3: {
            float wi[16], W = 0.0f;
            for (int b = 0; b < K; ++b) {
                float x = __fmul_rn(sc.f0[1 + (l - 1) * K + b], a[b]);
                wi[b] = expf(__fmul_rn(-0.5f, __fmul_rn(x, x)));
                W = __fadd_rn(W, wi[b]);
            }
            if (!(W > 0.0f) || !isfinite(W)) {
                int b = (int)(((uint64_t)mu24 * (uint64_t)K) >> 24);
                bw[b] = (float)K;
            } else {
                float t = __fmul_rn(u, W), c = 0.0f;
                int pick = K - 1;
                for (int b = 0; b < K; ++b) { c = __fadd_rn(c, wi[b]); if (t < c) { pick = b; break; } }
                bw[pick] = __fdiv_rn(W, wi[pick]);
            }
            break;
        }
        case 4: {
            int nab = 0;
            for (int b = 0; b < K; ++b) { if (a[b] <= pol.delta) bw[b] = 1.0f; else ++nab; }
            if (nab > 0) {
                int pickn = (int)(((uint64_t)mu24 * (uint64_t)nab) >> 24), c = 0;
                for (int b = 0; b < K; ++b)
                    if (!(a[b] <= pol.delta)) { if (c == pickn) { bw[b] = (float)nab; break; } ++c; }
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
            w[g] = lw[l] * bw[b];
        }
    }
    // spatial bands: one draw, the same groups and weights in every band (C24)
    for (int bd = 1; bd < sc.n_bands; ++bd) {
        mask |= (mask & ((1u << sc.G0) - 1u)) << (bd * sc.G0);
        for (int g = 0; g < sc.G0; ++g) w[bd * sc.G0 + g] = w[g];
    }
    return mask & pol.static_mask;
}

// policy for segment (pix, smp, d) of stream st; level uniform at k_level, orientation at k_level+l
__device__ inline uint32_t policy_for(const PolicyDev& pol, const SceneDev& sc, float3 dir, uint64_t seed,
                                      uint32_t pix, uint32_t smp, uint32_t d, uint32_t st, uint32_t k_level,
                                      float* w) {
    if (pol.ls == 0 && pol.os == 0) return pol.static_mask;  // static: weights stay 1
    float u[12];
    uint4 b0 = stream_block(seed, pix, smp, d, st, 0);
    uint4 b1 = stream_block(seed, pix, smp, d, st, 4);
    uint4 b2 = stream_block(seed, pix, smp, d, st, 8);
    u[0] = u01(b0.x); u[1] = u01(b0.y); u[2] = u01(b0.z); u[3] = u01(b0.w);
    u[4] = u01(b1.x); u[5] = u01(b1.y); u[6] = u01(b1.z); u[7] = u01(b1.w);
    u[8] = u01(b2.x); u[9] = u01(b2.y); u[10] = u01(b2.z); u[11] = u01(b2.w);
    return policy_eval(pol, sc, dir, u[k_level], u + k_level + 1, w);
}

// ------------------------------------------------------------------ camera (fp32, correctly rounded ops)
struct CamDev {
    float pos[3], fwd[3], right[3], up[3];
    int32_t W, H;
};
__device__ __forceinline__ void camera_ray(const CamDev& c, int px, int py, float jx, float jy, float3& o,
                                           float3& v) {
    float fx = __fadd_rn((float)px, jx), fy = __fadd_rn((float)py, jy);
    float iw2 = __fdiv_rn(2.0f, (float)c.W), ih2 = __fdiv_rn(2.0f, (float)c.H);
    float sx = __fmaf_rn(fx, iw2, -1.0f), sy = __fmaf_rn(-fy, ih2, 1.0f);
    float r0 = __fmaf_rn(sy, c.up[0], __fmaf_rn(sx, c.right[0], c.fwd[0]));
    float r1 = __fmaf_rn(sy, c.up[1], __fmaf_rn(sx, c.right[1], c.fwd[1]));
    float r2 = __fmaf_rn(sy, c.up[2], __fmaf_rn(sx, c.right[2], c.fwd[2]));
    float len = __fsqrt_rn(__fmaf_rn(r0, r0, __fmaf_rn(r1, r1, __fmul_rn(r2, r2))));
    v = make_float3(__fdiv_rn(r0, len), __fdiv_rn(r1, len), __fdiv_rn(r2, len));
    o = make_float3(c.pos[0], c.pos[1], c.pos[2]);
}

// ------------------------------------------------------------------ Henyey-Greenstein (C19)
__device__ __forceinline__ float hg_eval(float g, float cost) {
    float den = 1.0f + g * g - 2.0f * g * cost;
    return (1.0f - g * g) / (4.0f * 3.14159265358979f * den * sqrtf(den));
}
__device__ inline float3 hg_sample(float g, float3 v, float u1, float u2) {
    float cost;
    if (fabsf(g) < 1e-3f) cost = 1.0f - 2.0f * u1;
    else { float q = (1.0f - g * g) / (1.0f - g + 2.0f * g * u1); cost = (1.0f + g * g - q * q) / (2.0f * g); }
    cost = fminf(1.0f, fmaxf(-1.0f, cost));
    float sint = sqrtf(fmaxf(0.0f, 1.0f - cost * cost));
    float sp, cp;
    sincospif(2.0f * u2, &sp, &cp);
    float sgn = v.z >= 0.0f ? 1.0f : -1.0f;
    float a = -1.0f / (sgn + v.z), b = v.x * v.y * a;
    float3 t1 = make_float3(1.0f + sgn * v.x * v.x * a, sgn * b, -sgn * v.x);
    float3 t2 = make_float3(b, sgn + v.y * v.y * a, -v.y);
    float3 o = make_float3(sint * cp * t1.x + sint * sp * t2.x + cost * v.x,
                           sint * cp * t1.y + sint * sp * t2.y + cost * v.y,
                           sint * cp * t1.z + sint * sp * t2.z + cost * v.z);
    float n = rsqrtf(o.x * o.x + o.y * o.y + o.z * o.z);
    return make_float3(o.x * n, o.y * n, o.z * n);
}

// ------------------------------------------------------------------ work decomposition (§8(e))
// Path p of a sample pass -> pixel.  Paths enumerate 32x32 tiles (1024 paths each) in 8x4-pixel
// warps for coherence; under tile sharding (kind 1) rank r owns tiles r, r+N, r+2N, ...
// (host + device: the C ABI exports it as gf_shard_path_pixel for the multi-process tests).
__host__ __device__ inline int32_t shard_path_pixel(int64_t p, int32_t W, int32_t H, int32_t kind, int32_t rank,
                                                    int32_t world) {
    const int64_t tiles_x = (W + 31) / 32, tiles_y = (H + 31) / 32;
    int64_t tile = p >> 10;
    if (kind == 1) tile = rank + tile * world;
    if (p < 0 || tile >= tiles_x * tiles_y) return -1;
    const int local = (int)(p & 1023), blk = local >> 5, lane = local & 31;
    const int px = (int)(tile % tiles_x) * 32 + (blk & 3) * 8 + (lane & 7);
    const int py = (int)(tile / tiles_x) * 32 + (blk >> 2) * 4 + (lane >> 3);
    if (px >= W || py >= H) return -1;
    return py * W + px;
}

// ------------------------------------------------------------------ ray / box
struct RayDev {
    float3 o, d, inv, oinv;
    float tmin, tmax;
    float fmax;  // foveation: primitives with |omega_vec . d| > fmax are skipped (INFINITY: off)
};
__device__ __forceinline__ float safe_inv(float x) {
    return 1.0f / (fabsf(x) > 1e-20f ? x : copysignf(1e-20f, x));
}
__device__ __forceinline__ RayDev make_ray(float3 o, float3 d, float tmin, float tmax, float fmax = INFINITY) {
    RayDev r;
    r.o = o; r.d = d; r.tmin = tmin; r.tmax = tmax; r.fmax = fmax;
    r.inv = make_float3(safe_inv(d.x), safe_inv(d.y), safe_inv(d.z));
    r.oinv = make_float3(o.x * r.inv.x, o.y * r.inv.y, o.z * r.inv.z);
    return r;
}
// slab test against [t0,t1]; boxes are padded at build time to absorb the rounding here
__device__ __forceinline__ bool slab(const RayDev& r, float4 lo, float4 hi, float t0, float t1) {
    float ax = fmaf(lo.x, r.inv.x, -r.oinv.x), bx = fmaf(hi.x, r.inv.x, -r.oinv.x);
    float ay = fmaf(lo.y, r.inv.y, -r.oinv.y), by = fmaf(hi.y, r.inv.y, -r.oinv.y);
    float az = fmaf(lo.z, r.inv.z, -r.oinv.z), bz = fmaf(hi.z, r.inv.z, -r.oinv.z);
    float tn = fmaxf(fmaxf(fminf(ax, bx), fminf(ay, by)), fmaxf(fminf(az, bz), t0));
    float tf = fminf(fminf(fmaxf(ax, bx), fmaxf(ay, by)), fminf(fmaxf(az, bz), t1));
    return tn <= tf;
}
__device__ __forceinline__ bool slab_range(const RayDev& r, float4 lo, float4 hi, float t0, float t1, float& tn,
                                           float& tf) {
    float ax = fmaf(lo.x, r.inv.x, -r.oinv.x), bx = fmaf(hi.x, r.inv.x, -r.oinv.x);
    float ay = fmaf(lo.y, r.inv.y, -r.oinv.y), by = fmaf(hi.y, r.inv.y, -r.oinv.y);
    float az = fmaf(lo.z, r.inv.z, -r.oinv.z), bz = fmaf(hi.z, r.inv.z, -r.oinv.z);
    tn = fmaxf(fmaxf(fminf(ax, bx), fminf(ay, by)), fmaxf(fminf(az, bz), t0));
    tf = fminf(fminf(fmaxf(ax, bx), fmaxf(ay, by)), fminf(fmaxf(az, bz), t1));
    return tn <= tf;
}

// ------------------------------------------------------------------ a5: bounding-sphere pre-test
// Conservative world-space test of the ray against the primitive's bounding sphere (mu, Rs):
// one 16-byte load rejects most leaf candidates before the whitened setup.  Margins cover the
// fp32 rounding of |D|^2 - (D.d)^2 so that no primitive accepted by prim_setup is rejected.
__device__ __forceinline__ bool sphere_pretest(float4 a, const RayDev& r, float t0, float t1) {
    const float dx = r.o.x - a.x, dy = r.o.y - a.y, dz = r.o.z - a.z;
    const float b = fmaf(dx, r.d.x, fmaf(dy, r.d.y, dz * r.d.z));
    const float c = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
    const float perp2 = fmaf(-b, b, c);
    const float slack = 1e-4f * a.w + 1e-6f * c;
    if (perp2 > a.w + slack) return false;
    const float h = sqrtf(fmaxf(a.w + slack - perp2, 0.0f)) * 1.0001f + 1e-6f * fabsf(b);
    return (-b - h <= t1) && (-b + h >= t0);
}

// ------------------------------------------------------------------ a5: whitened setup + predicate
// Per (ray, primitive): world offset re-centred at the ray's closest approach to mu with an
// error-free TwoSum (o - mu = hi + lo), so that far origins (|o-mu|/s up to 3000) keep fp32
// precision in the whitened closest point p_c (SURVEY §0 finding 7).
struct Setup {
    float r2;    // |p_c|^2, squared whitened perpendicular distance (c - b^2)
    float h;     // whitened half chord sqrt(E^2 - r2)
    float bp;    // whitened arc parameter of the re-centred point: u(t) = bp + j (t - tc)
    float j;     // |W v|  (P:L223 Jacobian)
    float ij;    // 1/|W v|
    float tc;    // re-centring parameter (world t)
    float Om;    // Omega = k_W . v_W = omega (vWx+vWy+vWz)    (C2)
    float phi0;  // phase at the closest point = k_W . p_c = d - Omega b
    float u0, u1;  // whitened chord clipped to [tmin, tmax]
};

__device__ __forceinline__ bool prim_setup(const GPrim& P, const RayDev& r, float tmin, float tmax, Setup& s) {
    // TwoSum(o, -mu): hi + lo == o - mu exactly
    float hx = __fsub_rn(r.o.x, P.a.x), hy = __fsub_rn(r.o.y, P.a.y), hz = __fsub_rn(r.o.z, P.a.z);
    float bx = __fsub_rn(hx, r.o.x), by = __fsub_rn(hy, r.o.y), bz = __fsub_rn(hz, r.o.z);
    float lx = __fadd_rn(__fsub_rn(r.o.x, __fsub_rn(hx, bx)), __fsub_rn(-P.a.x, bx));
    float ly = __fadd_rn(__fsub_rn(r.o.y, __fsub_rn(hy, by)), __fsub_rn(-P.a.y, by));
    float lz = __fadd_rn(__fsub_rn(r.o.z, __fsub_rn(hz, bz)), __fsub_rn(-P.a.z, bz));
    float tc = -fmaf(hx, r.d.x, fmaf(hy, r.d.y, hz * r.d.z));
    float Dx = __fadd_rn(__fmaf_rn(tc, r.d.x, hx), lx);
    float Dy = __fadd_rn(__fmaf_rn(tc, r.d.y, hy), ly);
    float Dz = __fadd_rn(__fmaf_rn(tc, r.d.z, hz), lz);
    // whitened offset and direction (W rows in b,c,d .xyz)
    float px = fmaf(P.b.x, Dx, fmaf(P.b.y, Dy, P.b.z * Dz));
    float py = fmaf(P.c.x, Dx, fmaf(P.c.y, Dy, P.c.z * Dz));
    float pz = fmaf(P.d.x, Dx, fmaf(P.d.y, Dy, P.d.z * Dz));
    float wx = fmaf(P.b.x, r.d.x, fmaf(P.b.y, r.d.y, P.b.z * r.d.z));
    float wy = fmaf(P.c.x, r.d.x, fmaf(P.c.y, r.d.y, P.c.z * r.d.z));
    float wz = fmaf(P.d.x, r.d.x, fmaf(P.d.y, r.d.y, P.d.z * r.d.z));
    // foveation (continuous masking): frequency along the ray omega_vec . d = omega (W d).(1,1,1)
    if (fabsf(P.b.w * (wx + wy + wz)) > r.fmax) return false;
    float jj = fmaf(wx, wx, fmaf(wy, wy, wz * wz));
    float ij = rsqrtf(jj);
    float vx = wx * ij, vy = wy * ij, vz = wz * ij;
    float bp = fmaf(px, vx, fmaf(py, vy, pz * vz));
    float cx = fmaf(-bp, vx, px), cy = fmaf(-bp, vy, py), cz = fmaf(-bp, vz, pz);
    float r2 = fmaf(cx, cx, fmaf(cy, cy, cz * cz));
    const float E2 = P.c.w;
    if (!(r2 < E2)) return false;
    float h = sqrtf(E2 - r2);
    float j = jj * ij;
    float ut0 = fmaf(j, tmin - tc, bp);
    float ut1 = (tmax == INFINITY) ? INFINITY : fmaf(j, tmax - tc, bp);
    float u0 = fmaxf(-h, ut0), u1 = fminf(h, ut1);
    if (!(u1 > u0)) return false;
    const float om = P.b.w;
    s.r2 = r2; s.h = h; s.bp = bp; s.j = j; s.ij = ij; s.tc = tc;
    s.Om = om * (vx + vy + vz);
    s.phi0 = om * (cx + cy + cz);
    s.u0 = u0; s.u1 = u1;
    return true;
}

// ------------------------------------------------------------------ a6: complex erf, Eq. 13 series
// erf(z) = 2/sqrt(pi) z sum_n a_n (z^2)^n, a_n = (-1)^n / (n! (2n+1)), evaluated by Horner in
// fp32 with N = 30 terms (reading C5: the paper's 16 terms miss the 1e-4 target near the
// ellipsoid bound; 28-32 terms reach 2.3e-7 absolute over |u| <= 3, Omega <= 2.6).
__constant__ float kErfA[32] = {
    1.000000000e+00f, -3.333333333e-01f, 1.000000000e-01f, -2.380952381e-02f, 4.629629630e-03f,
    -7.575757576e-04f, 1.068376068e-04f, -1.322751323e-05f, 1.458916900e-06f, -1.450385222e-07f,
    1.312253296e-08f, -1.089222104e-09f, 8.350702795e-11f, -5.947794014e-12f, 3.955429516e-13f,
    -2.466827010e-14f, 1.448326464e-15f, -8.032735012e-17f, 4.221407289e-18f, -2.107855191e-19f,
    1.002516493e-20f, -4.551846759e-22f, 1.977064754e-23f, -8.230149299e-25f, 3.289260349e-26f,
    -1.264107899e-27f, 4.678483516e-29f, -1.669761793e-30f, 5.754191644e-32f, -1.916942862e-33f,
    6.180307588e-35f, -1.930357209e-36f};
constexpr int kErfTerms = 30;
constexpr float kRsqrt2 = 0.70710678118654752f;
constexpr float kTwoOverSqrtPi = 1.12837916709551257f;
constexpr float kInvSqrt2Pi = 0.39894228040143268f;
constexpr float kWMaxSeries = 8.0f;  // |z^2| beyond this -> Gauss-Legendre fallback (30 terms: 2.4e-7)

template <int N>
__device__ __forceinline__ float2 erf_horner(float zr, float zi, float wr, float wi) {
    float sr = kErfA[N - 1], si = 0.0f;
#pragma unroll
    for (int n = N - 2; n >= 0; --n) {
        float tr = fmaf(sr, wr, fmaf(-si, wi, kErfA[n]));
        float ti = fmaf(sr, wi, si * wr);
        sr = tr; si = ti;
    }
    return make_float2(kTwoOverSqrtPi * fmaf(zr, sr, -zi * si), kTwoOverSqrtPi * fmaf(zr, si, zi * sr));
}

// F(u) = erf((u - i Omega)/sqrt2).  Omega == 0 (every Gaussian, omega = 0, and Gabors integrated
// exactly along their modulation plane) reduces to the real erf: erff, 2 ulp.
// Otherwise the 30-term Horner series (a warp-uniform adaptive term count was measured slower:
// four unrolled copies at every call site cost more in instruction fetch than they save).
__device__ __forceinline__ float2 erf_shift(float u, float Om) {
    if (Om == 0.0f) return make_float2(erff(u * kRsqrt2), 0.0f);
    const float zr = u * kRsqrt2, zi = -Om * kRsqrt2;
    return erf_horner<kErfTerms>(zr, zi, fmaf(zr, zr, -zi * zi), 2.0f * zr * zi);
}

__constant__ float kGLx[12] = {6.40568928626056300e-02f, 1.91118867473616311e-01f, 3.15042679696163397e-01f,
                               4.33793507626045127e-01f, 5.45421471388839563e-01f, 6.48093651936975546e-01f,
                               7.40124191578554358e-01f, 8.20001985973902947e-01f, 8.86415527004401071e-01f,
                               9.38274552002732798e-01f, 9.74728555971309474e-01f, 9.95187219997021311e-01f};
__constant__ float kGLw[12] = {1.27938195346752021e-01f, 1.25837456346828247e-01f, 1.21670472927803294e-01f,
                               1.15505668053725516e-01f, 1.07444270115965565e-01f, 9.76186521041139260e-02f,
                               8.61901615319532050e-02f, 7.33464814110801611e-02f, 5.92985849154363601e-02f,
                               4.42774388174194122e-02f, 2.85313886289335593e-02f, 1.23412297999886903e-02f};

// reduce phase to [-pi, pi] then fast sincos (|x| <= 8 in practice)
__device__ __forceinline__ void sincos_red(float x, float* s, float* c) {
    float k = rintf(x * 0.15915494309189535f);
    float r = fmaf(-k, 6.28318548202514648f, x);
    r = fmaf(-k, -1.7484555e-7f, r);
    __sincosf(r, s, c);
}

// work counters (gf_stats.work, per stage), flushed with warp-aggregated atomics
constexpr int kWorkSlots = 12;
enum { W_NODES = 0, W_TESTS = 1, W_HITS = 2, W_ERFC = 3, W_ERFR = 4, W_GL = 5, W_OVERFLOW = 6, W_ROOT = 7,
       W_PATHS = 8 };
struct Work {
    uint32_t nodes = 0, tests = 0, hits = 0, erfc = 0, erfr = 0, gl = 0, overflow = 0, root = 0, paths = 0;
    __device__ __forceinline__ void erf(float Om, uint32_t k) {
        if (Om == 0.0f) erfr += k; else erfc += k;
    }
};
__device__ __forceinline__ void flush_work(unsigned long long* w, const Work& k) {
    const unsigned long long v[9] = {k.nodes, k.tests, k.hits, k.erfc, k.erfr, k.gl, k.overflow, k.root, k.paths};
#pragma unroll
    for (int i = 0; i < 9; ++i) {
        unsigned long long x = v[i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xFFFFFFFFu, x, o);
        if ((threadIdx.x & 31) == 0 && x) atomicAdd(w + i, x);
    }
}
// per-thread variant (partial warps allowed)
__device__ __forceinline__ void flush_work_thread(unsigned long long* w, const Work& k) {
    const unsigned long long v[9] = {k.nodes, k.tests, k.hits, k.erfc, k.erfr, k.gl, k.overflow, k.root, k.paths};
#pragma unroll
    for (int i = 0; i < 9; ++i)
        if (v[i]) atomicAdd(w + i, v[i]);
}

// Segment integral of primitive with setup s over whitened [ua, ub] (alpha, W-Jacobian and
// group weight NOT applied):  Jw = 1/2 e^{-(r2+Om^2)/2} Re{e^{i phi0}[F(ub) - F(ua)]}
//   = e^{-r2/2} (2 pi)^-1/2 int_ua^ub e^{-u^2/2} cos(phi0 + Om u) du      (App. A, reading C3).
// The caller multiplies by c / j (P:L223 K).  Symmetric full chords use one endpoint:
// F(h) - F(-h) = 2 Re F(h) (the "symmetries in the pair of erf terms").
__device__ inline float seg_J(const Setup& s, float ua, float ub, Work& wk) {
    const float L = ub - ua;
    float sp, cp;
    if (L < 1e-4f) {  // midpoint rule: whitened segment below 1e-4
        float um = 0.5f * (ua + ub);
        sincos_red(fmaf(s.Om, um, s.phi0), &sp, &cp);
        return kInvSqrt2Pi * __expf(-0.5f * (s.r2 + um * um)) * cp * L;
    }
    sincos_red(s.phi0, &sp, &cp);
    const float wmax = 0.5f * (fmaxf(ua * ua, ub * ub) + s.Om * s.Om);
    if (wmax > kWMaxSeries && s.Om != 0.0f) {  // outside the series domain: 24-node Gauss-Legendre
        ++wk.gl;
        float hm = 0.5f * L, c = 0.5f * (ua + ub), acc = 0.0f;
#pragma unroll 4
        for (int k = 0; k < 12; ++k) {
            float x = hm * kGLx[k];
            float s1, c1, s2, c2;
            sincos_red(fmaf(s.Om, c + x, s.phi0), &s1, &c1);
            sincos_red(fmaf(s.Om, c - x, s.phi0), &s2, &c2);
            acc = fmaf(kGLw[k], __expf(-0.5f * (c + x) * (c + x)) * c1 + __expf(-0.5f * (c - x) * (c - x)) * c2, acc);
        }
        return kInvSqrt2Pi * __expf(-0.5f * s.r2) * hm * acc;
    }
    const float amp = 0.5f * __expf(-0.5f * (s.r2 + s.Om * s.Om));
    if (ua == -s.h && ub == s.h) {
        wk.erf(s.Om, 1);
        float2 F = erf_shift(ub, s.Om);
        return 2.0f * amp * cp * F.x;
    }
    wk.erf(s.Om, 2);
    float2 Fb = erf_shift(ub, s.Om), Fa = erf_shift(ua, s.Om);
    return amp * fmaf(cp, Fb.x - Fa.x, -sp * (Fb.y - Fa.y));
}

// One erf call site for all lanes evaluating together (SIMT-uniform): the real erf if every
// participating lane has Omega == 0, otherwise the complex series for all of them (a Gaussian lane
// in a mixed group gets the same value from the series).  Inlining erf_shift at several call sites
// instead left each copy running with ~6 of 32 lanes (ncu source view, round 1).
#ifndef GF_ERF_WARP_UNIFORM
#define GF_ERF_WARP_UNIFORM 0
#endif
__device__ __forceinline__ float2 erf_warp(float u, float Om, Work& wk) {
    const float zr = u * kRsqrt2, zi = -Om * kRsqrt2;
    if (GF_ERF_WARP_UNIFORM ? __all_sync(__activemask(), Om == 0.0f) : Om == 0.0f) {
        ++wk.erfr;
        return make_float2(erff(zr), 0.0f);
    }
    ++wk.erfc;
    return erf_horner<kErfTerms>(zr, zi, fmaf(zr, zr, -zi * zi), 2.0f * zr * zi);
}

// Rare special cases of a piece [ua, ub]: midpoint rule (whitened length < 1e-4) or
// Gauss-Legendre (outside the series domain).  Returns false if the series path applies.
__device__ __forceinline__ bool seg_J_special(const Setup& s, float ua, float ub, float& res, Work& wk) {
    const float wmax = 0.5f * (fmaxf(ua * ua, ub * ub) + s.Om * s.Om);
    if (ub - ua < 1e-4f || (wmax > kWMaxSeries && s.Om != 0.0f)) {
        res = seg_J(s, ua, ub, wk);
        return true;
    }
    return false;
}

// Segment integral of a hit over its clipped chord, SIMT-uniform version of seg_J: the series
// endpoints of all lanes go through one erf call site (a symmetric full chord needs one endpoint,
// F(h) - F(-h) = 2 Re F(h); otherwise two).
__device__ __forceinline__ float seg_J_u(const Setup& s, float ua, float ub, Work& wk) {
    float res = 0.0f;
    int ne = 0;
    if (!seg_J_special(s, ua, ub, res, wk)) ne = (ua == -s.h && ub == s.h) ? 1 : 2;
    float sp, cp;
    sincos_red(s.phi0, &sp, &cp);
    const float amp = 0.5f * __expf(-0.5f * (s.r2 + s.Om * s.Om));
    float2 Fa = make_float2(0.0f, 0.0f);
#pragma unroll 1
    for (int e = 0; e < 2; ++e) {
        if (e < ne) {
            const float2 F = erf_warp(e == 0 && ne == 2 ? ua : ub, s.Om, wk);
            if (ne == 1) res = 2.0f * amp * cp * F.x;
            else if (e == 1) res = amp * fmaf(cp, F.x - Fa.x, -sp * (F.y - Fa.y));
            Fa = F;
        }
    }
    return res;
}

// contribution of a hit over its clipped chord: c/j * Jw
__device__ __forceinline__ float hit_tau(const GPrim& P, const Setup& s, Work& wk) {
    return P.d.w * s.ij * seg_J_u(s, s.u0, s.u1, wk);
}

__device__ __forceinline__ uint32_t node_mask(uint32_t skipw, uint32_t info) {
    return (skipw & kLeafBit) ? (1u << (info & 31u)) : info;
}

// ------------------------------------------------------------------ flat warp traversal engine
// One traversal step = one node test or one primitive test (a4 + a5).  State of a ray's
// stackless depth-first traversal: next node i, leaf cursor [lk, le) and the leaf's group g.
// A second (postponed) leaf slot lets a lane keep taking node steps while it still has an
// unprocessed leaf, so node steps and primitive tests each run with most lanes of the warp.
struct Trav {
    RayDev r;
    float t0, t1;
    uint32_t mask, i, lk, le, g, lk2, le2, g2;
};
__device__ __forceinline__ void trav_begin(Trav& T, const RayDev& r, float t0, float t1, uint32_t mask) {
    T.r = r; T.t0 = t0; T.t1 = t1; T.mask = mask; T.i = 0; T.lk = 0; T.le = 0; T.g = 0;
    T.lk2 = 0; T.le2 = 0; T.g2 = 0;
}
__device__ __forceinline__ bool trav_done(const Trav& T, uint32_t n_nodes) {
    return T.lk >= T.le && T.lk2 >= T.le2 && T.i >= n_nodes;
}

// Persistent warp loop over `count` work items (all 32 lanes call it).  Each lane owns one ray;
// a lane whose ray is finished fetches the next item at once (lane-level refill).  Every
// iteration the warp executes ONE uniform operation for the lanes eligible for it:
//   NODE  lanes with no unprocessed leaf: one node test (a4);
//   PRIM  lanes inside a leaf without a pending hit: one primitive test (a5);
//   HIT   lanes with a pending accepted primitive: its fused integral (a6), batched so that the
//         expensive erf work runs once BATCH lanes have one (or nothing else can advance).
// The op with the most eligible lanes wins, so node/prim/integral code never diverge against
// each other.  Callbacks (lane-local): begin(idx) -> bool (false: item needs no traversal);
// hit(setup, coef, group, sorted prim index) -> bool done (a hit may take several ops); end().  sync() is called by all lanes once per iteration.
// BATCH = 0: no pending state -- hit() runs right inside the primitive-test op (for callbacks as
// cheap as a record store).
template <bool COUNT, int BATCH, bool SPLIT, class Begin, class Hit, class End, class Sync>
__device__ __forceinline__ void flat_loop(uint32_t* work, uint32_t count, const GNode* __restrict__ nodes,
                                          uint32_t n_nodes, const GPrim* __restrict__ prims, Trav& T, Work& wk,
                                          Begin&& begin, Hit&& hit, End&& end, Sync&& sync) {
    const unsigned FULL = 0xFFFFFFFFu;
    const int lane = threadIdx.x & 31;
    bool active = false, pend = false, exhausted = false;
    Setup s;
    float coef = 0.0f;
    uint32_t pg = 0, pidx = 0;
    while (true) {
        // finish + refill
        if (active && !pend && trav_done(T, n_nodes)) {
            end();
            active = false;
        }
        if (!exhausted) {
            const unsigned need = __ballot_sync(FULL, !active);
            if (need) {
                const int leader = __ffs(need) - 1;
                uint32_t base = 0;
                if (lane == leader) base = atomicAdd(work, (uint32_t)__popc(need));
                base = __shfl_sync(FULL, base, leader);
                if (!active) {
                    const uint32_t idx = base + __popc(need & ((1u << lane) - 1u));
                    if (idx < count) active = begin(idx);
                }
                if (base + (uint32_t)__popc(need) >= count) exhausted = true;
            }
        }
        sync();
        if (!__any_sync(FULL, active)) {
            if (exhausted) break;
            continue;
        }
        // inner loop of uniform operations until some lane finishes its ray
        while (true) {
            const bool in_leaf = active && T.lk < T.le;
            const bool e_node = active && T.i < n_nodes && (!in_leaf || T.lk2 >= T.le2);
            const bool e_prim = in_leaf && !pend;
            const unsigned m_hit = __ballot_sync(FULL, pend);
            const unsigned m_node = __ballot_sync(FULL, e_node);
            const unsigned m_prim = __ballot_sync(FULL, e_prim);
            const int n_hit = __popc(m_hit), n_node = __popc(m_node), n_prim = __popc(m_prim);
            if (n_hit > 0 && (n_hit >= BATCH || n_hit >= n_node + n_prim)) {
                // run one erf type per op (real for Omega == 0, complex otherwise): no divergence
                bool run = pend;
                if (SPLIT) {
                    const unsigned m_real = __ballot_sync(FULL, pend && s.Om == 0.0f);
                    const bool real_op = 2 * __popc(m_real) >= n_hit;
                    run = pend && ((s.Om == 0.0f) == real_op);
                }
                if (run && hit(s, coef, pg, pidx)) pend = false;  // hit() may take several ops
            } else if (n_prim > 0 && n_prim >= n_node) {
                if (e_prim) {
                    const uint32_t k = T.lk, g = T.g;
                    const GPrim* q = prims + k;
                    ++T.lk;
                    if (T.lk >= T.le && T.lk2 < T.le2) {  // promote the postponed leaf
                        T.lk = T.lk2; T.le = T.le2; T.g = T.g2; T.lk2 = T.le2 = 0;
                    }
                    GPrim P;
                    P.a = __ldg(&q->a);
                    if (COUNT) ++wk.tests;
                    if (sphere_pretest(P.a, T.r, T.t0, T.t1)) {
                        P.b = __ldg(&q->b); P.c = __ldg(&q->c); P.d = __ldg(&q->d);
                        if (prim_setup(P, T.r, T.t0, T.t1, s)) {
                            if (COUNT) ++wk.hits;
                            if (BATCH == 0) {
                                hit(s, P.d.w, g, k);
                            } else {
                                coef = P.d.w;
                                pg = g;
                                pidx = k;
                                pend = true;
                            }
                        }
                    }
                }
            } else if (n_node > 0) {
                if (e_node) {
                    const uint32_t i = T.i;
                    const float4 lo = __ldg(&nodes[i].lo), hi = __ldg(&nodes[i].hi);
                    const uint32_t sk = __float_as_uint(lo.w), info = __float_as_uint(hi.w);
                    if (COUNT) ++wk.nodes;
                    const bool h = (node_mask(sk, info) & T.mask) && slab(T.r, lo, hi, T.t0, T.t1);
                    if (h && (sk & kLeafBit)) {
                        const uint32_t lk = info >> 8, le = lk + ((info >> 5) & 7u), g = info & 31u;
                        if (T.lk >= T.le) { T.lk = lk; T.le = le; T.g = g; }
                        else { T.lk2 = lk; T.le2 = le; T.g2 = g; }
                        T.i = sk & ~kLeafBit;
                    } else {
                        T.i = h ? i + 1 : (sk & ~kLeafBit);
                    }
                }
            }
            // leave the inner loop when a lane can be finished (its slot is refilled)
            if (__any_sync(FULL, active && !pend && trav_done(T, n_nodes))) break;
        }
    }
}

// ------------------------------------------------------------------ warp-per-ray traversal
// One warp owns one ray.  Its frontier lives in shared memory: a stack of internal nodes known
// to be hit and a list of pending primitive references (sorted index | group << 27).  Every step
// is one warp-uniform operation over up to 32 entries:
//   PRIM  (>= 32 pending, or no node left): one primitive test per lane (a5), on_prims callback;
//   NODE  pop up to 32 nodes, test both children of each (a4), push the hit internal children
//         and append the primitives of the hit leaves (warp prefix sums, no atomics).
// So node tests, primitive tests and (through the callbacks' queues) the integrals all run with
// full warps instead of the divergent per-lane depth-first walk.  Stack bound: a full step grows
// the stack by <= 32; above `stk_limit` one node per step is popped (depth-first, growth <= 1
// per level), and stk_limit = kWStk - 34 - max_depth keeps it in bounds (gf_build_bvh).
#ifndef GF_NODE_PREFETCH
#define GF_NODE_PREFETCH 0  // warp traversal: L1 prefetch of the pushed children's child pairs
#endif
#ifndef GF_WSTK
#define GF_WSTK 256  // warp traversal stack entries per warp (512: -2 % -- the shared memory it frees goes to L1)
#endif
constexpr int kWStk = GF_WSTK;
constexpr int kWPrm = 32 + 64 * kLeafMax;
struct WarpTrav {
    uint32_t stk[kWStk];
    uint32_t prm[kWPrm];
};
constexpr uint32_t kRefIdx = 0x07FFFFFFu;

template <bool COUNT, class OnPrims, class BoxHit>
__device__ __forceinline__ void warp_traverse_b(const GNode* __restrict__ nodes, const GNode2* __restrict__ n2,
                                                uint32_t n_nodes, int stk_limit, uint32_t mask, WarpTrav& sm, Work& wk,
                                                OnPrims&& on_prims, BoxHit&& boxhit) {
    const unsigned FULL = 0xFFFFFFFFu;
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    int ns = 0, np = 0;
    if (n_nodes == 0) return;
    {  // root
        const float4 lo = __ldg(&nodes[0].lo), hi = __ldg(&nodes[0].hi);
        const uint32_t sk = __float_as_uint(lo.w), info = __float_as_uint(hi.w);
        if (COUNT && lane == 0) ++wk.nodes;
        if (!((node_mask(sk, info) & mask) && boxhit(lo, hi))) return;
        if (sk & kLeafBit) {
            const int cnt = (int)((info >> 5) & 7u);
            if (lane < cnt) sm.prm[lane] = ((info >> 8) + lane) | ((info & 31u) << 27);
            np = cnt;
        } else {
            if (lane == 0) sm.stk[0] = 0;
            ns = 1;
        }
        __syncwarp();
    }
    while (true) {
        if (np >= 32 || (ns == 0 && np > 0)) {
            const int take = min(np, 32);
            const bool valid = lane < take;
            const uint32_t ref = valid ? sm.prm[np - take + lane] : 0u;
            np -= take;
            __syncwarp();
            on_prims(valid, ref);
        } else if (ns > 0) {
            const int take = ns > stk_limit ? 1 : min(ns, 32);
            const bool valid = lane < take;
            const uint32_t i = valid ? sm.stk[ns - take + lane] : 0u;
            ns -= take;
            __syncwarp();
            bool h0 = false, h1 = false;
            uint32_t ref0 = 0, ref1 = 0, inf0 = 0, inf1 = 0;
            if (valid) {
                const GNode2* q = n2 + i;
                const float4 lo0 = __ldg(&q->lo0), hi0 = __ldg(&q->hi0), lo1 = __ldg(&q->lo1), hi1 = __ldg(&q->hi1);
                ref0 = __float_as_uint(lo0.w); inf0 = __float_as_uint(hi0.w);
                ref1 = __float_as_uint(lo1.w); inf1 = __float_as_uint(hi1.w);
                h0 = (node_mask(ref0, inf0) & mask) && boxhit(lo0, hi0);
                h1 = (node_mask(ref1, inf1) & mask) && boxhit(lo1, hi1);
                if (COUNT) wk.nodes += 2;
            }
            const bool i0 = h0 && !(ref0 & kLeafBit), i1 = h1 && !(ref1 & kLeafBit);
#if GF_NODE_PREFETCH
            // the children pushed now are the next steps' pops: start their child-pair loads into L1
            if (i0) asm volatile("prefetch.global.L1 [%0];" ::"l"(n2 + ref0));
            if (i1) asm volatile("prefetch.global.L1 [%0];" ::"l"(n2 + ref1));
#endif
            const unsigned b0 = __ballot_sync(FULL, i0), b1 = __ballot_sync(FULL, i1);
            if (i0) sm.stk[ns + __popc(b0 & lt)] = ref0;
            if (i1) sm.stk[ns + __popc(b0) + __popc(b1 & lt)] = ref1;
            ns += __popc(b0) + __popc(b1);
            GF_CHECK(ns <= kWStk);
            const uint32_t c0 = (h0 && (ref0 & kLeafBit)) ? ((inf0 >> 5) & 7u) : 0u;
            const uint32_t c1 = (h1 && (ref1 & kLeafBit)) ? ((inf1 >> 5) & 7u) : 0u;
            if (__any_sync(FULL, c0 + c1 > 0)) {
                uint32_t incl = c0 + c1;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t v = __shfl_up_sync(FULL, incl, o);
                    if (lane >= o) incl += v;
                }
                const uint32_t pos = (uint32_t)np + incl - (c0 + c1);
                const uint32_t v0 = (inf0 >> 8) | ((inf0 & 31u) << 27), v1 = (inf1 >> 8) | ((inf1 & 31u) << 27);
#pragma unroll
                for (uint32_t k = 0; k < (uint32_t)kLeafMax; ++k)  // predicated, no divergent loop
                    if (k < c0) sm.prm[pos + k] = v0 + k;
#pragma unroll
                for (uint32_t k = 0; k < (uint32_t)kLeafMax; ++k)
                    if (k < c1) sm.prm[pos + c0 + k] = v1 + k;
                np += (int)__shfl_sync(FULL, incl, 31);
                GF_CHECK(np <= kWPrm);
            }
            __syncwarp();
        } else {
            break;
        }
    }
}

// world-frame boxes: slab test of ray r over [t0, t1]
template <bool COUNT, class OnPrims>
__device__ __forceinline__ void warp_traverse(const GNode* __restrict__ nodes, const GNode2* __restrict__ n2,
                                              uint32_t n_nodes, int stk_limit, const RayDev& r, float t0, float t1,
                                              uint32_t mask, WarpTrav& sm, Work& wk, OnPrims&& on_prims) {
    warp_traverse_b<COUNT>(nodes, n2, n_nodes, stk_limit, mask, sm, wk, on_prims,
                           [&](float4 lo, float4 hi) { return slab(r, lo, hi, t0, t1); });
}

// Endpoint queues of the warp integrator: a hit's integral is Re{e^{i phi0} [F(u1) - F(u0)]} amp
// (seg_J), i.e. one or two erf endpoints, each queued as (u, Omega, A, B) with the contribution
// A Re F(u) + B Im F(u): symmetric full chord (F(h) - F(-h) = 2 Re F(h)): (h, Om, 2 amp cos phi0, 0);
// otherwise (u1, Om, amp cos, -amp sin) and (u0, Om, -amp cos, amp sin).  Queue 0 holds the
// Omega == 0 endpoints (real erf), queue 1 the series endpoints; a queue is evaluated 32 at a
// time with one erf type per step.
constexpr int kWEnd = 96;
struct WarpEnd {
    float4 e[2][kWEnd];
};

// tau of one ray (all 32 lanes call; the result is returned on every lane).  Weights w[g] apply
// when STOCH (stochastic LOD masks).
template <bool STOCH, bool COUNT, class BoxHit>
__device__ __forceinline__ double warp_tau_b(const GNode* __restrict__ nodes, const GNode2* __restrict__ n2,
                                             uint32_t n_nodes, int stk_limit, const GPrim* __restrict__ prims,
                                             const RayDev& r, float t0, float t1, uint32_t mask, const float* w,
                                             WarpTrav& sm, WarpEnd& q, Work& wk, BoxHit&& boxhit) {
    const unsigned FULL = 0xFFFFFFFFu;
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    double acc = 0.0;
    int nq0 = 0, nq1 = 0;
    auto run = [&](int t, int take) {
        int& nq = t == 0 ? nq0 : nq1;
        const bool valid = lane < take;
        const float4 e = valid ? q.e[t][nq - take + lane] : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        nq -= take;
        __syncwarp();
        if (valid) {
            const float zr = e.x * kRsqrt2;
            if (t == 0) {
                if (COUNT) ++wk.erfr;
                acc += (double)(e.z * erff(zr));
            } else {
                if (COUNT) ++wk.erfc;
                const float zi = -e.y * kRsqrt2;
                const float2 F = erf_horner<kErfTerms>(zr, zi, fmaf(zr, zr, -zi * zi), 2.0f * zr * zi);
                acc += (double)fmaf(e.z, F.x, e.w * F.y);
            }
        }
    };
    warp_traverse_b<COUNT>(nodes, n2, n_nodes, stk_limit, mask, sm, wk, [&](bool valid, uint32_t ref) {
        int ne = 0;
        bool real = false;
        float4 e0 = make_float4(0.0f, 0.0f, 0.0f, 0.0f), e1 = e0;
        if (valid) {
            const uint32_t k = ref & kRefIdx;
            const GPrim* pp = prims + k;
            GPrim P;
            P.a = __ldg(&pp->a);
            if (COUNT) ++wk.tests;
            Setup s;
            if (sphere_pretest(P.a, r, t0, t1)) {
                P.b = __ldg(&pp->b); P.c = __ldg(&pp->c); P.d = __ldg(&pp->d);
                if (prim_setup(P, r, t0, t1, s)) {
                    if (COUNT) ++wk.hits;
                    float cj = P.d.w * s.ij;
                    if (STOCH) cj *= w[ref >> 27];
                    float res;
                    if (seg_J_special(s, s.u0, s.u1, res, wk)) {
                        acc += (double)(cj * res);  // rare: midpoint / Gauss-Legendre, lane-local
                    } else {
                        const float amp = 0.5f * cj * __expf(-0.5f * (s.r2 + s.Om * s.Om));
                        float sp, cp;
                        sincos_red(s.phi0, &sp, &cp);
                        real = s.Om == 0.0f;
                        if (s.u0 == -s.h && s.u1 == s.h) {
                            ne = 1;
                            e0 = make_float4(s.u1, s.Om, 2.0f * amp * cp, 0.0f);
                        } else {
                            ne = 2;
                            e0 = make_float4(s.u1, s.Om, amp * cp, -amp * sp);
                            e1 = make_float4(s.u0, s.Om, -amp * cp, amp * sp);
                        }
                    }
                }
            }
        }
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            const bool mine = ne > 0 && (real == (t == 0));
            const unsigned m1 = __ballot_sync(FULL, mine), m2 = __ballot_sync(FULL, mine && ne == 2);
            if (m1) {
                int& nq = t == 0 ? nq0 : nq1;
                if (mine) {
                    q.e[t][nq + __popc(m1 & lt)] = e0;
                    if (ne == 2) q.e[t][nq + __popc(m1) + __popc(m2 & lt)] = e1;
                }
                nq += __popc(m1) + __popc(m2);
                GF_CHECK(nq <= kWEnd);
                __syncwarp();
                while (nq >= 32) run(t, 32);
            }
        }
    }, boxhit);
    while (nq0 > 0) run(0, min(nq0, 32));
    while (nq1 > 0) run(1, min(nq1, 32));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(FULL, acc, o);
    return acc;
}

template <bool STOCH, bool COUNT>
__device__ __forceinline__ double warp_tau(const GNode* __restrict__ nodes, const GNode2* __restrict__ n2,
                                           uint32_t n_nodes, int stk_limit, const GPrim* __restrict__ prims,
                                           const RayDev& r, float t0, float t1, uint32_t mask, const float* w,
                                           WarpTrav& sm, WarpEnd& q, Work& wk) {
    return warp_tau_b<STOCH, COUNT>(nodes, n2, n_nodes, stk_limit, prims, r, t0, t1, mask, w, sm, q, wk,
                                    [&](float4 lo, float4 hi) { return slab(r, lo, hi, t0, t1); });
}

}  // namespace gfk
