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

cudaError_t gf_launch_candidates(const TraceArgs& A, bool brute_force, cudaStream_t st) {
    if (A.n == 0) return cudaSuccess;
    const unsigned grid = (unsigned)((A.n + 127) / 128);
    if (brute_force) k_candidates<true><<<grid, 128, 0, st>>>(A);
    else k_candidates<false><<<grid, 128, 0, st>>>(A);
    return cudaGetLastError();
}
