// gf_trace.cu -- a4 masked all-hits traversal + a5 ellipsoid clip + a6 fused line integral
// + a7 transmittance (Eq. 2-3; masks P:L344-L350).
#include <algorithm>

#include "gf_device.cuh"
#include "gf_internal.h"

namespace gfk {

// Stackless depth-first traversal with escape links over all nodes whose box meets [t0,t1]
// and whose group mask meets the ray mask; calls f(prim, group) for every primitive of every
// visited leaf.  No early exit: tau needs every overlap.
template <bool COUNT, class F>
__device__ __forceinline__ void traverse(const GNode* __restrict__ nodes, uint32_t n_nodes,
                                         const GPrim* __restrict__ prims, const RayDev& r, float t0, float t1,
                                         uint32_t mask, uint32_t& nvis, F&& f) {
    uint32_t i = 0;
    while (i < n_nodes) {
        const float4 lo = __ldg(&nodes[i].lo);
        const float4 hi = __ldg(&nodes[i].hi);
        const uint32_t sk = __float_as_uint(lo.w), info = __float_as_uint(hi.w);
        if (COUNT) ++nvis;
        const bool hit = (node_mask(sk, info) & mask) && slab(r, lo, hi, t0, t1);
        if (hit && (sk & kLeafBit)) {
            const uint32_t first = info >> 8, cnt = (info >> 5) & 7u, g = info & 31u;
            for (uint32_t k = 0; k < cnt; ++k) {
                const GPrim* p = prims + first + k;
                GPrim P;
                P.a = __ldg(&p->a);
                if (!sphere_pretest(P.a, r, t0, t1)) continue;
                P.b = __ldg(&p->b); P.c = __ldg(&p->c); P.d = __ldg(&p->d);
                f(P, g, first + k);
            }
            i = sk & ~kLeafBit;
        } else if (hit) {
            i = i + 1;
        } else {
            i = sk & ~kLeafBit;
        }
    }
}

// brute force over all primitives in input order (test path); same pre-test + predicate
template <class F>
__device__ __forceinline__ void brute(const GPrim* __restrict__ prims, const uint8_t* __restrict__ group, int64_t n,
                                     const RayDev& r, float t0, float t1, uint32_t mask, F&& f) {
    for (int64_t k = 0; k < n; ++k) {
        const uint32_t g = __ldg(group + k);
        if (!((mask >> g) & 1u)) continue;
        const GPrim* p = prims + k;
        GPrim P;
        P.a = __ldg(&p->a);
        if (!sphere_pretest(P.a, r, t0, t1)) continue;
        P.b = __ldg(&p->b); P.c = __ldg(&p->c); P.d = __ldg(&p->d);
        f(P, g, (uint32_t)k);
    }
}

template <bool BRUTE, bool COUNT, bool STOCH>
__global__ void __launch_bounds__(128) k_trace(TraceArgs A) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= A.n) return;
    const float4 r0 = __ldg((const float4*)A.rays + 2 * i);
    const float4 r1 = __ldg((const float4*)A.rays + 2 * i + 1);
    const float3 o = make_float3(r0.x, r0.y, r0.z), d = make_float3(r1.x, r1.y, r1.z);
    const RayDev r = make_ray(o, d, r0.w, r1.w);
    float w[kMaxGroups];
    uint32_t mask;
    if (STOCH) mask = policy_for(A.pol, A.sc, d, A.seed, (uint32_t)i, 0, 0, ST_EXT, 1, w);
    else mask = A.pol.static_mask;
    double tau = 0.0;
    uint32_t nvis = 0, ntest = 0, nhit = 0;
    Work wk;
    auto on_prim = [&](const GPrim& P, uint32_t g, uint32_t) {
        if (COUNT) ++ntest;
        Setup s;
        if (!prim_setup(P, r, r.tmin, r.tmax, s)) return;
        if (COUNT) ++nhit;
        float c = hit_tau(P, s, wk);
        if (STOCH) c *= w[g];
        tau += (double)c;
    };
    if (BRUTE) brute(A.prims, A.group, A.n_prims, r, r.tmin, r.tmax, mask, on_prim);
    else traverse<COUNT>(A.nodes, A.n_nodes, A.prims, r, r.tmin, r.tmax, mask, nvis, on_prim);
    A.tau[i] = (float)tau;
    if (A.T) A.T[i] = (float)exp(-tau);
    if (COUNT && A.counters) {
        A.counters[3 * i] = nvis;
        A.counters[3 * i + 1] = ntest;
        A.counters[3 * i + 2] = nhit;
    }
    if (COUNT && A.work) {
        wk.nodes = nvis; wk.tests = ntest; wk.hits = nhit; wk.paths = 1;
        flush_work_thread(A.work + kWorkSlots * STAGE_TRACE, wk);
    }
}

// BVH path: one warp per ray (warp_traverse + endpoint queues, gf_device.cuh)
template <bool COUNT, bool STOCH>
__global__ void __launch_bounds__(128) k_trace_w(TraceArgs A) {
    __shared__ WarpTrav s_t[4];
    __shared__ WarpEnd s_e[4];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    Work tot;
    for (int64_t i = (int64_t)blockIdx.x * 4 + wid; i < A.n; i += (int64_t)gridDim.x * 4) {
        const float4 r0 = __ldg((const float4*)A.rays + 2 * i);
        const float4 r1 = __ldg((const float4*)A.rays + 2 * i + 1);
        const float3 o = make_float3(r0.x, r0.y, r0.z), d = make_float3(r1.x, r1.y, r1.z);
        const RayDev r = make_ray(o, d, r0.w, r1.w);
        float w[kMaxGroups];
        uint32_t mask;
        if (STOCH) mask = policy_for(A.pol, A.sc, d, A.seed, (uint32_t)i, 0, 0, ST_EXT, 1, w);
        else mask = A.pol.static_mask;
        Work wk;
        const double tau = warp_tau<STOCH, COUNT>(A.nodes, A.nodes2, A.n_nodes, A.stk_limit, A.prims, r, r.tmin,
                                                  r.tmax, mask, w, s_t[wid], s_e[wid], wk);
        if (lane == 0) {
            A.tau[i] = (float)tau;
            if (A.T) A.T[i] = (float)exp(-tau);
        }
        if (COUNT) {
            uint32_t v[3] = {wk.nodes, wk.tests, wk.hits};
#pragma unroll
            for (int k = 0; k < 3; ++k)
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xFFFFFFFFu, v[k], o);
            if (lane == 0 && A.counters) {
                A.counters[3 * i] = v[0];
                A.counters[3 * i + 1] = v[1];
                A.counters[3 * i + 2] = v[2];
            }
            tot.nodes += wk.nodes; tot.tests += wk.tests; tot.hits += wk.hits;
            tot.erfc += wk.erfc; tot.erfr += wk.erfr; tot.gl += wk.gl;
            if (lane == 0) ++tot.paths;
        }
    }
    if (COUNT && A.work) flush_work(A.work + kWorkSlots * STAGE_TRACE, tot);
}

// Backward of tau w.r.t. the opacities (alpha part): tau is linear in alpha,
// d tau_r / d alpha_i = w_g c_i/alpha_i (1/j) J_i with c_i / alpha_i = 1 / (2 pi s1 s2 s3) =
// |W0| |W1| |W2| / (2 pi).  One warp per ray over the BVH; each hit's integral lane-local (seg_J),
// scattered into grad[perm[k]] (input order) with atomics.
template <bool STOCH>
__global__ void __launch_bounds__(128) k_grad_alpha(TraceArgs A, const float* __restrict__ dl,
                                                    float* __restrict__ grad) {
    __shared__ WarpTrav s_t[4];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    Work wk;
    for (int64_t i = (int64_t)blockIdx.x * 4 + wid; i < A.n; i += (int64_t)gridDim.x * 4) {
        const float4 r0 = __ldg((const float4*)A.rays + 2 * i);
        const float4 r1 = __ldg((const float4*)A.rays + 2 * i + 1);
        const float3 o = make_float3(r0.x, r0.y, r0.z), d = make_float3(r1.x, r1.y, r1.z);
        const RayDev r = make_ray(o, d, r0.w, r1.w);
        float w[kMaxGroups];
        uint32_t mask;
        if (STOCH) mask = policy_for(A.pol, A.sc, d, A.seed, (uint32_t)i, 0, 0, ST_EXT, 1, w);
        else mask = A.pol.static_mask;
        const float g = __ldg(dl + i);
        if (g == 0.0f) continue;
        warp_traverse<false>(A.nodes, A.nodes2, A.n_nodes, A.stk_limit, r, r.tmin, r.tmax, mask, s_t[wid], wk,
                             [&](bool valid, uint32_t ref) {
            if (!valid) return;
            const uint32_t k = ref & kRefIdx;
            const GPrim* pp = A.prims + k;
            GPrim P;
            P.a = __ldg(&pp->a);
            if (!sphere_pretest(P.a, r, r.tmin, r.tmax)) return;
            P.b = __ldg(&pp->b); P.c = __ldg(&pp->c); P.d = __ldg(&pp->d);
            Setup s;
            if (!prim_setup(P, r, r.tmin, r.tmax, s)) return;
            const float nb = sqrtf(P.b.x * P.b.x + P.b.y * P.b.y + P.b.z * P.b.z);
            const float nc = sqrtf(P.c.x * P.c.x + P.c.y * P.c.y + P.c.z * P.c.z);
            const float nd = sqrtf(P.d.x * P.d.x + P.d.y * P.d.y + P.d.z * P.d.z);
            float v = nb * nc * nd * 0.15915494309189535f * s.ij * seg_J(s, s.u0, s.u1, wk);
            if (STOCH) v *= w[ref >> 27];
            atomicAdd(grad + A.perm[k], g * v);
        });
    }
}

// ---------------------------------------------------------------- parameter gradient (§8(f) rank 4)
// Complex segment moment  J0 = e^{-r2/2} (2 pi)^-1/2 int_ua^ub e^{-u^2/2} e^{i (phi0 + Om u)} du
// (Re J0 = seg_J).  Series: 1/2 e^{-(r2+Om^2)/2} e^{i phi0} [F(ub) - F(ua)]; same midpoint and
// Gauss-Legendre special cases as seg_J.
__device__ inline float2 seg_J0c(const Setup& s, float ua, float ub, Work& wk) {
    const float L = ub - ua;
    if (L < 1e-4f) {
        const float um = 0.5f * (ua + ub);
        float sp, cp;
        sincos_red(fmaf(s.Om, um, s.phi0), &sp, &cp);
        const float e = kInvSqrt2Pi * __expf(-0.5f * (s.r2 + um * um)) * L;
        return make_float2(e * cp, e * sp);
    }
    const float wmax = 0.5f * (fmaxf(ua * ua, ub * ub) + s.Om * s.Om);
    if (wmax > kWMaxSeries && s.Om != 0.0f) {
        ++wk.gl;
        const float hm = 0.5f * L, c = 0.5f * (ua + ub);
        float ar = 0.0f, ai = 0.0f;
        for (int k = 0; k < 12; ++k) {
            const float x = hm * kGLx[k];
            float s1, c1, s2, c2;
            sincos_red(fmaf(s.Om, c + x, s.phi0), &s1, &c1);
            sincos_red(fmaf(s.Om, c - x, s.phi0), &s2, &c2);
            const float e1 = __expf(-0.5f * (c + x) * (c + x)), e2 = __expf(-0.5f * (c - x) * (c - x));
            ar = fmaf(kGLw[k], e1 * c1 + e2 * c2, ar);
            ai = fmaf(kGLw[k], e1 * s1 + e2 * s2, ai);
        }
        const float f = kInvSqrt2Pi * __expf(-0.5f * s.r2) * hm;
        return make_float2(f * ar, f * ai);
    }
    float sp, cp;
    sincos_red(s.phi0, &sp, &cp);
    const float amp = 0.5f * __expf(-0.5f * (s.r2 + s.Om * s.Om));
    wk.erf(s.Om, 2);
    const float2 Fb = erf_shift(ub, s.Om), Fa = erf_shift(ua, s.Om);
    const float dr = Fb.x - Fa.x, di = Fb.y - Fa.y;
    return make_float2(amp * fmaf(cp, dr, -sp * di), amp * fmaf(cp, di, sp * dr));
}

// Per-hit derivatives of tau_ri = c int_chord K(y(t)) dt, K(y) = (2 pi)^-1/2 e^{-|y|^2/2} cos(k.y),
// y = W (x - mu), k = omega (1,1,1), c = alpha (2 pi)^-1 |det W|.  With the whitened
// arc parameter u (y = cvec + u v) and the moments Jn = e^{-r2/2} (2 pi)^-1/2 int u^n e^{-u^2/2 + i phi(u)}:
//   J1 = i Om J0 - [E],  J2 = i Om J1 - [u E] + J0   (integration by parts), E(u) the integrand;
//   d tau/d mu    = c [ ij W^T A + sum_e K(y_e) ij/h W^T y_e ]
//   d tau/d W     = c [ -ij (A D^T + ij B d^T) - sum_e K(y_e) ij/h y_e X_e^T ]   (|det W| part: finish)
//   d tau/d omega = -c ij [ (1.cvec) Im J0 + (1.v) Im J1 ]
//   A = cvec Re J0 + v Re J1 + k Im J0,  B = cvec Re(J1 - bp J0) + v Re(J2 - bp J1) + k Im(J1 - bp J0)
// where D = o + tc d - mu, X_e = D + (u_e - bp) ij d, and e runs over chord ends on the ellipsoid
// (u = +-h: the end moves with mu and W; a clipped end at tmin/tmax does not).
// acc (16 floats per primitive, input order): mu[3], W[9] row-major, omega, alpha, sum l tau, -.
// The 15 partial sums of one hit (layout of acc, entries 0..14), loss weight l applied.
__device__ __forceinline__ void hit_grad(const GPrim& P, const Setup& s, float3 o, float3 d, float l, float* G,
                                         Work& wk) {
    // world offset at the re-centring point (TwoSum as prim_setup) and whitened vectors
    const float hx = __fsub_rn(o.x, P.a.x), hy = __fsub_rn(o.y, P.a.y), hz = __fsub_rn(o.z, P.a.z);
    const float bx = __fsub_rn(hx, o.x), by = __fsub_rn(hy, o.y), bz = __fsub_rn(hz, o.z);
    const float lx = __fadd_rn(__fsub_rn(o.x, __fsub_rn(hx, bx)), __fsub_rn(-P.a.x, bx));
    const float ly = __fadd_rn(__fsub_rn(o.y, __fsub_rn(hy, by)), __fsub_rn(-P.a.y, by));
    const float lz = __fadd_rn(__fsub_rn(o.z, __fsub_rn(hz, bz)), __fsub_rn(-P.a.z, bz));
    const float D[3] = {__fadd_rn(__fmaf_rn(s.tc, d.x, hx), lx), __fadd_rn(__fmaf_rn(s.tc, d.y, hy), ly),
                        __fadd_rn(__fmaf_rn(s.tc, d.z, hz), lz)};
    const float dv[3] = {d.x, d.y, d.z};
    const float Wm[3][3] = {{P.b.x, P.b.y, P.b.z}, {P.c.x, P.c.y, P.c.z}, {P.d.x, P.d.y, P.d.z}};
    float pv[3], vv[3], cv[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        pv[a] = fmaf(Wm[a][0], D[0], fmaf(Wm[a][1], D[1], Wm[a][2] * D[2]));
        vv[a] = fmaf(Wm[a][0], dv[0], fmaf(Wm[a][1], dv[1], Wm[a][2] * dv[2])) * s.ij;
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) cv[a] = fmaf(-s.bp, vv[a], pv[a]);
    const float om = P.b.w, cst = P.d.w;
    const float2 J0 = seg_J0c(s, s.u0, s.u1, wk);
    float E0r, E0i, E1r, E1i;
    {
        float sp, cp;
        sincos_red(fmaf(s.Om, s.u0, s.phi0), &sp, &cp);
        const float e0 = kInvSqrt2Pi * __expf(-0.5f * (s.r2 + s.u0 * s.u0));
        E0r = e0 * cp; E0i = e0 * sp;
        sincos_red(fmaf(s.Om, s.u1, s.phi0), &sp, &cp);
        const float e1 = kInvSqrt2Pi * __expf(-0.5f * (s.r2 + s.u1 * s.u1));
        E1r = e1 * cp; E1i = e1 * sp;
    }
    const float J1r = -s.Om * J0.y - (E1r - E0r), J1i = s.Om * J0.x - (E1i - E0i);
    const float J2r = -s.Om * J1i - (s.u1 * E1r - s.u0 * E0r) + J0.x;
    const float Kr = J1r - s.bp * J0.x, Ki = J1i - s.bp * J0.y, Lr = J2r - s.bp * J1r;
    float Av[3], Bv[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        Av[a] = fmaf(cv[a], J0.x, fmaf(vv[a], J1r, om * J0.y));
        Bv[a] = fmaf(cv[a], Kr, fmaf(vv[a], Lr, om * Ki));
    }
    const float ij = s.ij;
    float gmu[3], gW[3][3];
#pragma unroll
    for (int b = 0; b < 3; ++b) {
        gmu[b] = ij * fmaf(Wm[0][b], Av[0], fmaf(Wm[1][b], Av[1], Wm[2][b] * Av[2]));
#pragma unroll
        for (int a = 0; a < 3; ++a) gW[a][b] = -ij * fmaf(Av[a], D[b], ij * Bv[a] * dv[b]);
    }
    // moving chord ends on the ellipsoid
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        const float ue = e ? s.u1 : s.u0;
        if (ue != (e ? s.h : -s.h)) continue;
        const float Ke = (e ? E1r : E0r) * ij / s.h;
        float ye[3], Xe[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            ye[a] = fmaf(ue, vv[a], cv[a]);
            Xe[a] = fmaf((ue - s.bp) * ij, dv[a], D[a]);
        }
#pragma unroll
        for (int b = 0; b < 3; ++b) {
            gmu[b] = fmaf(Ke, fmaf(Wm[0][b], ye[0], fmaf(Wm[1][b], ye[1], Wm[2][b] * ye[2])), gmu[b]);
#pragma unroll
            for (int a = 0; a < 3; ++a) gW[a][b] = fmaf(-Ke * ye[a], Xe[b], gW[a][b]);
        }
    }
    const float gom = -ij * fmaf(cv[0] + cv[1] + cv[2], J0.y, (vv[0] + vv[1] + vv[2]) * J1i);
    const float nb = sqrtf(P.b.x * P.b.x + P.b.y * P.b.y + P.b.z * P.b.z);
    const float nc = sqrtf(P.c.x * P.c.x + P.c.y * P.c.y + P.c.z * P.c.z);
    const float nd = sqrtf(P.d.x * P.d.x + P.d.y * P.d.y + P.d.z * P.d.z);
    const float lc = l * cst;
#pragma unroll
    for (int b = 0; b < 3; ++b) G[b] = lc * gmu[b];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) G[3 + 3 * a + b] = lc * gW[a][b];
    G[12] = lc * gom;
    G[13] = l * nb * nc * nd * 0.15915494309189535f * ij * J0.x;
    G[14] = lc * ij * J0.x;
}

__device__ __forceinline__ void red_grad(float* acc, const float* G) {
    // four 16-byte vector atomics (sm_90+ float4 atomicAdd on global memory)
    float4* out = (float4*)acc;
    atomicAdd(out + 0, make_float4(G[0], G[1], G[2], G[3]));
    atomicAdd(out + 1, make_float4(G[4], G[5], G[6], G[7]));
    atomicAdd(out + 2, make_float4(G[8], G[9], G[10], G[11]));
    atomicAdd(out + 3, make_float4(G[12], G[13], G[14], 0.0f));
}

template <bool STOCH>
__global__ void __launch_bounds__(128) k_grad_params(TraceArgs A, const float* __restrict__ dl,
                                                     float* __restrict__ acc) {
    __shared__ WarpTrav s_t[4];
    const int wid = threadIdx.x >> 5;
    Work wk;
    for (int64_t i = (int64_t)blockIdx.x * 4 + wid; i < A.n; i += (int64_t)gridDim.x * 4) {
        const float4 r0 = __ldg((const float4*)A.rays + 2 * i);
        const float4 r1 = __ldg((const float4*)A.rays + 2 * i + 1);
        const float3 o = make_float3(r0.x, r0.y, r0.z), d = make_float3(r1.x, r1.y, r1.z);
        const RayDev r = make_ray(o, d, r0.w, r1.w);
        float w[kMaxGroups];
        uint32_t mask;
        if (STOCH) mask = policy_for(A.pol, A.sc, d, A.seed, (uint32_t)i, 0, 0, ST_EXT, 1, w);
        else mask = A.pol.static_mask;
        const float g = __ldg(dl + i);
        if (g == 0.0f) continue;
        warp_traverse<false>(A.nodes, A.nodes2, A.n_nodes, A.stk_limit, r, r.tmin, r.tmax, mask, s_t[wid], wk,
                             [&](bool valid, uint32_t ref) {
            if (!valid) return;
            const uint32_t k = ref & kRefIdx;
            const GPrim* pp = A.prims + k;
            GPrim P;
            P.a = __ldg(&pp->a);
            if (!sphere_pretest(P.a, r, r.tmin, r.tmax)) return;
            P.b = __ldg(&pp->b); P.c = __ldg(&pp->c); P.d = __ldg(&pp->d);
            Setup s;
            if (!prim_setup(P, r, r.tmin, r.tmax, s)) return;
            const float l = STOCH ? g * w[ref >> 27] : g;
            float G[15];
            hit_grad(P, s, o, d, l, G, wk);
            red_grad(acc + (size_t)A.perm[k] * 16, G);
        });
    }
}

// Coherent rays (GF_TRACE_PACKETS: consecutive rays of a pixel block): one depth-first walk of
// the scene BVH per 32 rays (a child pair is descended if any lane's slab test hits it), a hit
// leaf's primitives loaded once and tested per lane; a primitive's 15 partial sums are summed over
// the lanes (butterfly shuffles) and added with one set of vector atomics -- 32x fewer atomics on
// the primitives every ray of a block crosses.
constexpr int kGStk = 256;
#ifndef GF_GRADP_MINB
#define GF_GRADP_MINB 5  // 96 registers (a few spills), 5 blocks per SM: -13 % vs 128 registers (tools_grad_sweep.sh)
#endif
template <bool STOCH>
__global__ void __launch_bounds__(128, GF_GRADP_MINB) k_grad_pkt(TraceArgs A, const float* __restrict__ dl,
                                                  float* __restrict__ acc) {
    __shared__ uint32_t s_stk[4][kGStk];
    const unsigned FULL = 0xFFFFFFFFu;
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t* stk = s_stk[wid];
    Work wk;
    for (int64_t base = ((int64_t)blockIdx.x * 4 + wid) * 32; base < A.n; base += (int64_t)gridDim.x * 128) {
        const int64_t i = base + lane;
        const bool valid = i < A.n;
        float4 r0 = make_float4(0.0f, 0.0f, 0.0f, 0.0f), r1 = make_float4(0.0f, 0.0f, 1.0f, 0.0f);
        float g = 0.0f;
        uint32_t mask = 0;
        float w[kMaxGroups];
        if (valid) {
            r0 = __ldg((const float4*)A.rays + 2 * i);
            r1 = __ldg((const float4*)A.rays + 2 * i + 1);
            g = __ldg(dl + i);
            const float3 dd = make_float3(r1.x, r1.y, r1.z);
            if (STOCH) mask = policy_for(A.pol, A.sc, dd, A.seed, (uint32_t)i, 0, 0, ST_EXT, 1, w);
            else mask = A.pol.static_mask;
        }
        const float3 o = make_float3(r0.x, r0.y, r0.z), d = make_float3(r1.x, r1.y, r1.z);
        const RayDev r = make_ray(o, d, r0.w, r1.w);
        const bool act = valid && g != 0.0f;
        if (!__any_sync(FULL, act)) continue;
        auto boxhit = [&](uint32_t sk, uint32_t info, float4 lo, float4 hi) {
            return act && (node_mask(sk, info) & mask) && slab(r, lo, hi, r.tmin, r.tmax);
        };
        auto leaf = [&](uint32_t info, bool mine) {
            const uint32_t first = info >> 8, cnt = (info >> 5) & 7u, grp = info & 31u;
            for (uint32_t k = 0; k < cnt; ++k) {
                const GPrim* pp = A.prims + first + k;
                GPrim P;
                P.a = __ldg(&pp->a);
                const bool pass = mine && sphere_pretest(P.a, r, r.tmin, r.tmax);
                if (!__any_sync(FULL, pass)) continue;
                P.b = __ldg(&pp->b); P.c = __ldg(&pp->c); P.d = __ldg(&pp->d);
                Setup s;
                float G[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) G[j] = 0.0f;
                const bool hit = pass && prim_setup(P, r, r.tmin, r.tmax, s);
                if (!__any_sync(FULL, hit)) continue;
                if (hit) hit_grad(P, s, o, d, STOCH ? g * w[grp] : g, G, wk);
                // transposing butterfly: after the halving steps (8+4+2+1 shuffles) lane L holds the
                // partial sum of entry L>>1 over its half-warp pair; one more xor-1 completes it
#pragma unroll
                for (int half = 8; half >= 1; half >>= 1) {
                    const bool up = (lane & (2 * half)) != 0;
#pragma unroll
                    for (int j = 0; j < half; ++j) {
                        const float send = up ? G[j] : G[j + half];
                        const float keep = up ? G[j + half] : G[j];
                        G[j] = keep + __shfl_xor_sync(FULL, send, 2 * half);
                    }
                }
                G[0] += __shfl_xor_sync(FULL, G[0], 1);
                const int e = lane >> 1;
                if (!(lane & 1) && e < 15) atomicAdd(acc + (size_t)A.perm[first + k] * 16 + e, G[0]);
            }
        };
        int ns = 0;
        {
            const float4 lo = __ldg(&A.nodes[0].lo), hi = __ldg(&A.nodes[0].hi);
            const uint32_t sk = __float_as_uint(lo.w), info = __float_as_uint(hi.w);
            const bool h = boxhit(sk, info, lo, hi);
            if (__any_sync(FULL, h)) {
                if (sk & kLeafBit) leaf(info, h);
                else { stk[0] = 0; ns = 1; }
            }
        }
        while (ns > 0) {
            const uint32_t i2 = stk[--ns];
            const GNode2* q = A.nodes2 + i2;
            const float4 lo0 = __ldg(&q->lo0), hi0 = __ldg(&q->hi0), lo1 = __ldg(&q->lo1), hi1 = __ldg(&q->hi1);
            const uint32_t ref0 = __float_as_uint(lo0.w), inf0 = __float_as_uint(hi0.w);
            const uint32_t ref1 = __float_as_uint(lo1.w), inf1 = __float_as_uint(hi1.w);
            const bool h0 = boxhit(ref0, inf0, lo0, hi0), h1 = boxhit(ref1, inf1, lo1, hi1);
            const bool a0 = __any_sync(FULL, h0), a1 = __any_sync(FULL, h1);
            __syncwarp();
            if (a1) {
                if (ref1 & kLeafBit) leaf(inf1, h1);
                else { GF_CHECK(ns < kGStk); stk[ns++] = ref1; }
            }
            if (a0) {
                if (ref0 & kLeafBit) leaf(inf0, h0);
                else { GF_CHECK(ns < kGStk); stk[ns++] = ref0; }
            }
            __syncwarp();
        }
    }
}

// Chain rule to the load parameters (input order): W = S^-1 R^T (rows R_.k / s_k), |det W| = 1/(s1 s2 s3):
//   d/ds_k = -(1/s_k) [ sum l tau + sum_b dW_kb W_kb ],  d/dR_bk = dW_kb / s_k,
//   d/dq = (I - qh qh^T)/|q| J_R(qh)^T d/dR   (R(qh) of the unit quaternion (x, y, z, w)).
__global__ void k_grad_finish(const GPrim* __restrict__ prims, int64_t n, const float* __restrict__ acc,
                              const float* __restrict__ quat, float* __restrict__ grad) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const GPrim P = prims[i];
    const float* a = acc + i * 16;
    const float Wm[3][3] = {{P.b.x, P.b.y, P.b.z}, {P.c.x, P.c.y, P.c.z}, {P.d.x, P.d.y, P.d.z}};
    float gR[3][3], gs[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const float sk = rsqrtf(Wm[k][0] * Wm[k][0] + Wm[k][1] * Wm[k][1] + Wm[k][2] * Wm[k][2]);
        float dot = 0.0f;
#pragma unroll
        for (int b = 0; b < 3; ++b) {
            dot = fmaf(a[3 + 3 * k + b], Wm[k][b], dot);
            gR[b][k] = a[3 + 3 * k + b] / sk;
        }
        gs[k] = -(a[14] + dot) / sk;
    }
    const float4 q = __ldg((const float4*)quat + i);
    const float qn = sqrtf(q.x * q.x + q.y * q.y + q.z * q.z + q.w * q.w);
    const float x = q.x / qn, y = q.y / qn, z = q.z / qn, w = q.w / qn;
    // d tau / d (x, y, z, w) of the unit quaternion through R (row-major entries R_rc)
    const float gx = 2.0f * (y * (gR[0][1] + gR[1][0]) + z * (gR[0][2] + gR[2][0]) + w * (gR[2][1] - gR[1][2])) -
                     4.0f * x * (gR[1][1] + gR[2][2]);
    const float gy = 2.0f * (x * (gR[0][1] + gR[1][0]) + w * (gR[0][2] - gR[2][0]) + z * (gR[1][2] + gR[2][1])) -
                     4.0f * y * (gR[0][0] + gR[2][2]);
    const float gz = 2.0f * (w * (gR[1][0] - gR[0][1]) + x * (gR[0][2] + gR[2][0]) + y * (gR[1][2] + gR[2][1])) -
                     4.0f * z * (gR[0][0] + gR[1][1]);
    const float gw = 2.0f * (z * (gR[1][0] - gR[0][1]) + y * (gR[0][2] - gR[2][0]) + x * (gR[2][1] - gR[1][2]));
    const float pr = x * gx + y * gy + z * gz + w * gw;
    float* o = grad + i * 12;
    o[0] = a[0]; o[1] = a[1]; o[2] = a[2];
    o[3] = (gx - x * pr) / qn; o[4] = (gy - y * pr) / qn; o[5] = (gz - z * pr) / qn; o[6] = (gw - w * pr) / qn;
    o[7] = gs[0]; o[8] = gs[1]; o[9] = gs[2];
    o[10] = a[12]; o[11] = a[13];
}

template <bool BRUTE>
__global__ void __launch_bounds__(128) k_candidates(TraceArgs A) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= A.n) return;
    const float4 r0 = __ldg((const float4*)A.rays + 2 * i);
    const float4 r1 = __ldg((const float4*)A.rays + 2 * i + 1);
    const RayDev r = make_ray(make_float3(r0.x, r0.y, r0.z), make_float3(r1.x, r1.y, r1.z), r0.w, r1.w);
    const uint32_t mask = A.pol.static_mask;
    int32_t cnt = 0;
    uint32_t nvis = 0;
    int32_t* out = A.cand_ids + i * (int64_t)A.cand_cap;
    auto on_prim = [&](const GPrim& P, uint32_t, uint32_t k) {
        Setup s;
        if (!prim_setup(P, r, r.tmin, r.tmax, s)) return;
        if (cnt < A.cand_cap) out[cnt] = BRUTE ? (int32_t)k : A.perm[k];
        ++cnt;
    };
    if (BRUTE) brute(A.prims, A.group, A.n_prims, r, r.tmin, r.tmax, mask, on_prim);
    else traverse<false>(A.nodes, A.n_nodes, A.prims, r, r.tmin, r.tmax, mask, nvis, on_prim);
    A.cand_count[i] = cnt;
}

}  // namespace gfk

using namespace gfk;

cudaError_t gf_launch_trace(const TraceArgs& A, bool brute_force, bool count, cudaStream_t st) {
    if (A.n == 0) return cudaSuccess;
    count = count || A.work != nullptr;
    const unsigned grid = (unsigned)((A.n + 127) / 128);
    const bool stoch = !(A.pol.ls == 0 && A.pol.os == 0);
#define GF_T(B, C, S) k_trace<B, C, S><<<grid, 128, 0, st>>>(A)
    if (brute_force) {
        if (count) { if (stoch) GF_T(true, true, true); else GF_T(true, true, false); }
        else { if (stoch) GF_T(true, false, true); else GF_T(true, false, false); }
    } else {
        static int sms = 0;
        if (!sms) {
            int dev = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        }
        const unsigned wgrid = (unsigned)std::min<int64_t>((A.n + 3) / 4, (int64_t)sms * 16);
        if (count) {
            if (stoch) k_trace_w<true, true><<<wgrid, 128, 0, st>>>(A);
            else k_trace_w<true, false><<<wgrid, 128, 0, st>>>(A);
        } else {
            if (stoch) k_trace_w<false, true><<<wgrid, 128, 0, st>>>(A);
            else k_trace_w<false, false><<<wgrid, 128, 0, st>>>(A);
        }
    }
#undef GF_T
    return cudaGetLastError();
}

cudaError_t gf_launch_grad_alpha(const TraceArgs& A, const float* dl, float* grad, cudaStream_t st) {
    if (A.n == 0 || A.n_nodes == 0) return cudaSuccess;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const unsigned wgrid = (unsigned)std::min<int64_t>((A.n + 3) / 4, (int64_t)sms * 16);
    if (!(A.pol.ls == 0 && A.pol.os == 0)) k_grad_alpha<true><<<wgrid, 128, 0, st>>>(A, dl, grad);
    else k_grad_alpha<false><<<wgrid, 128, 0, st>>>(A, dl, grad);
    return cudaGetLastError();
}

cudaError_t gf_launch_grad_params(const TraceArgs& A, const float* dl, float* acc, bool packets, cudaStream_t st) {
    if (A.n == 0 || A.n_nodes == 0) return cudaSuccess;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const bool stoch = !(A.pol.ls == 0 && A.pol.os == 0);
    if (packets) {
        const unsigned pgrid = (unsigned)std::min<int64_t>((A.n + 127) / 128, (int64_t)sms * 16);
        if (stoch) k_grad_pkt<true><<<pgrid, 128, 0, st>>>(A, dl, acc);
        else k_grad_pkt<false><<<pgrid, 128, 0, st>>>(A, dl, acc);
        return cudaGetLastError();
    }
    const unsigned wgrid = (unsigned)std::min<int64_t>((A.n + 3) / 4, (int64_t)sms * 16);
    if (stoch) k_grad_params<true><<<wgrid, 128, 0, st>>>(A, dl, acc);
    else k_grad_params<false><<<wgrid, 128, 0, st>>>(A, dl, acc);
    return cudaGetLastError();
}

cudaError_t gf_launch_grad_finish(const GPrim* prims, int64_t n, const float* acc, const float* quat, float* grad,
                                  cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    k_grad_finish<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(prims, n, acc, quat, grad);
    return cudaGetLastError();
}

cudaError_t gf_launch_candidates(const TraceArgs& A, bool brute_force, cudaStream_t st) {
    if (A.n == 0) return cudaSuccess;
    const unsigned grid = (unsigned)((A.n + 127) / 128);
    if (brute_force) k_candidates<true><<<grid, 128, 0, st>>>(A);
    else k_candidates<false><<<grid, 128, 0, st>>>(A);
    return cudaGetLastError();
}
