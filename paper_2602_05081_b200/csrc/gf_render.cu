// gf_render.cu -- a8 free-flight distance sampling, a9 scatter loop, a10 accumulation
// (Eq. 4-5, bisection/root finding P:L254, pipeline P:L352-L365).
//
// Wavefront over the paths of one sample pass: gen -> [ffA -> ffB -> nee] x max_depth -> finish.
//  ffA: one traversal of the ray's scene interval accumulating tau into kBins t-bins
//       (tau_total gives the escape test, the bins bracket the root);
//  ffB: one traversal restricted to the bracketing bin gathers its active primitives, then a
//       safeguarded Newton/bisection on tau(t) = tau* (derivative = kappa(t), analytic);
//  nee: shadow ray towards the directional light (analytic T), HG phase, next direction.
// Queues are warp-aggregated; work is fetched dynamically 32 paths at a time.
#include <algorithm>

#include "gf_device.cuh"
#include "gf_internal.h"

namespace gfk {

#ifndef GF_BINS
#define GF_BINS 1
#endif
constexpr int kBins = GF_BINS;
constexpr int kHitCap = 1024;  // hits recorded per path by ffA for ffB (overflow -> traversal gather)
constexpr int kWorkA = 4, kWorkB = 5, kWorkN = 6, kWorkT = 7;  // qcount slots: work cursors
constexpr int kCntT = 8, kCntO = 9, kWorkAT = 10, kWorkAI = 11, kWorkAO = 12;  // record pass A queues
constexpr int kCntB2 = 13, kWorkBW = 14;  // single-pass (record overflow) paths for ffB; warp ffB cursor
#ifndef GF_REC_CAP
#define GF_REC_CAP 1024
#endif
constexpr int kRecCap = GF_REC_CAP;  // 32-byte hit records per path (overflow -> single-pass ffA)

template <bool COUNT, class F>
__device__ __forceinline__ void traverse_r(const GNode* __restrict__ nodes, uint32_t n_nodes,
                                           const GPrim* __restrict__ prims, const RayDev& r, float t0, float t1,
                                           uint32_t mask, Work& wk, F&& f) {
    uint32_t i = 0;
    while (i < n_nodes) {
        const float4 lo = __ldg(&nodes[i].lo);
        const float4 hi = __ldg(&nodes[i].hi);
        const uint32_t sk = __float_as_uint(lo.w), info = __float_as_uint(hi.w);
        if (COUNT) ++wk.nodes;
        const bool hit = (node_mask(sk, info) & mask) && slab(r, lo, hi, t0, t1);
        if (hit && (sk & kLeafBit)) {
            const uint32_t first = info >> 8, cnt = (info >> 5) & 7u, g = info & 31u;
            for (uint32_t k = 0; k < cnt; ++k) {
                const GPrim* p = prims + first + k;
                GPrim P;
                P.a = __ldg(&p->a);
                if (COUNT) ++wk.tests;
                if (!sphere_pretest(P.a, r, t0, t1)) continue;
                P.b = __ldg(&p->b); P.c = __ldg(&p->c); P.d = __ldg(&p->d);
                f(P, g);
            }
            i = sk & ~kLeafBit;
        } else if (hit) {
            i = i + 1;
        } else {
            i = sk & ~kLeafBit;
        }
    }
}

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

// tau of a ray through the masked, weighted field (NEE, tomography, ffB overflow)
template <bool STOCH, bool COUNT>
__device__ __forceinline__ double trace_tau(const RenderDev& R, const RayDev& r, float t0, float t1, uint32_t mask,
                                            const float* w, Work& wk) {
    double tau = 0.0;
    traverse_r<COUNT>(R.nodes, R.n_nodes, R.prims, r, t0, t1, mask, wk, [&](const GPrim& P, uint32_t g) {
        Setup s;
        if (!prim_setup(P, r, t0, t1, s)) return;
        if (COUNT) ++wk.hits;
        float c = hit_tau(P, s, wk);
        if (STOCH) c *= w[g];
        tau += (double)c;
    });
    return tau;
}

__global__ void __launch_bounds__(128) k_gen(RenderDev R, int32_t sample) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // grid covers whole warps
    const int32_t pix = p < R.n_paths ? path_pixel(R, p) : -1;
    const bool ok = pix >= 0;
    if (ok) {
        float jx = 0.5f, jy = 0.5f;
        if (R.jitter) {
            uint4 b = stream_block(R.seed, (uint32_t)pix, (uint32_t)sample, 0, ST_CAM, 0);
            jx = u01(b.x); jy = u01(b.y);
        }
        float3 o, d;
        camera_ray(R.cam, pix % R.cam.W, pix / R.cam.W, jx, jy, o, d);
        R.ox[p] = o.x; R.oy[p] = o.y; R.oz[p] = o.z;
        R.dx[p] = d.x; R.dy[p] = d.y; R.dz[p] = d.z;
        R.beta[p] = 1.0f;
        R.L[p] = 0.0f;
        R.pix[p] = (uint32_t)pix;
    }
    push(R.qA, R.qcount + 0, ok, (uint32_t)p);
}

// ---------------------------------------------------------------- binned tau over [t0, t1]
// Adds one hit's partial integrals into NB equal t-bins (one erf evaluation per bin boundary
// inside the chord, the chord ends shared) and counts the primitives overlapping each bin.
// Returns the bin span ka | kb << 8 of the chord.  bins/cnts are per-thread columns of shared
// arrays (element k at [k * stride]).
template <int NB, bool COUNT>
__device__ __forceinline__ uint32_t bin_add(const Setup& s, float cj, float t0, float bw, float ibw, float* bins,
                                            uint16_t* cnts, int stride, Work& wk) {
    const float ta = fmaf(s.u0 - s.bp, s.ij, s.tc), tb = fmaf(s.u1 - s.bp, s.ij, s.tc);
    const int ka = min(NB - 1, max(0, (int)((ta - t0) * ibw)));
    const int kb = min(NB - 1, max(0, (int)((tb - t0) * ibw)));
    const uint32_t span = (uint32_t)ka | ((uint32_t)kb << 8);
    for (int m = ka; m <= kb; ++m) cnts[m * stride] = (uint16_t)min(65535, cnts[m * stride] + 1);
    if (ka == kb) {
        bins[ka * stride] += cj * seg_J(s, s.u0, s.u1, wk);
        return span;
    }
    const float wmax = 0.5f * (fmaxf(s.u0 * s.u0, s.u1 * s.u1) + s.Om * s.Om);
    float ua = s.u0;
    if ((wmax > kWMaxSeries && s.Om != 0.0f) || s.u1 - s.u0 < 1e-4f) {  // per-piece generic path
        for (int m = ka + 1; m <= kb; ++m) {
            float ub = fminf(fmaxf(fmaf(s.j, (t0 + m * bw) - s.tc, s.bp), ua), s.u1);
            bins[(m - 1) * stride] += cj * seg_J(s, ua, ub, wk);
            ua = ub;
        }
        bins[kb * stride] += cj * seg_J(s, ua, s.u1, wk);
        return span;
    }
    // shared endpoints: one erf evaluation per bin boundary inside the chord
    float sp, cp;
    sincos_red(s.phi0, &sp, &cp);
    const float amp = cj * 0.5f * __expf(-0.5f * (s.r2 + s.Om * s.Om));
    float2 Fa = erf_shift(ua, s.Om);
    for (int m = ka + 1; m <= kb; ++m) {
        float ub = fminf(fmaxf(fmaf(s.j, (t0 + m * bw) - s.tc, s.bp), ua), s.u1);
        float2 Fb = erf_shift(ub, s.Om);
        bins[(m - 1) * stride] += amp * fmaf(cp, Fb.x - Fa.x, -sp * (Fb.y - Fa.y));
        Fa = Fb;
        ua = ub;
    }
    float2 Fb = erf_shift(s.u1, s.Om);
    bins[kb * stride] += amp * fmaf(cp, Fb.x - Fa.x, -sp * (Fb.y - Fa.y));
    if (COUNT) wk.erf(s.Om, (uint32_t)(kb - ka + 2));
    return span;
}

// tuning knobs (compile-time; bench variants are built with -D overrides)
#ifndef GF_BATCH
#define GF_BATCH 0
#endif
#ifndef GF_MINB_FFA
#define GF_MINB_FFA 6
#endif
#ifndef GF_MINB_NEE
#define GF_MINB_NEE 6
#endif
#ifndef GF_SPLIT_FFA
#define GF_SPLIT_FFA 0
#endif
#ifndef GF_SPLIT_NEE
#define GF_SPLIT_NEE 0
#endif
#ifndef GF_BATCH_T
#define GF_BATCH_T 0  // record-emitting traversal: the hit callback (one 32-byte store) runs inline
#endif
#ifndef GF_MINB_T
#define GF_MINB_T 8
#endif
constexpr int kBatch = GF_BATCH;  // integrate pending hits once this many lanes (or most blocked lanes) have one

template <bool STOCH, bool COUNT>
__global__ void __launch_bounds__(128) k_tomo(RenderDev R, int32_t sample) {
    Work wk;
    Trav T;
    uint32_t p = 0;
    double tau = 0.0;
    float w[kMaxGroups];
    bool began = false;
    flat_loop<COUNT, kBatch, GF_SPLIT_NEE>(
        R.qcount + kWorkT, (uint32_t)R.n_paths, R.nodes, R.n_nodes, R.prims, T, wk,
        [&](uint32_t idx) -> bool {
            p = idx;
            const int32_t pix = path_pixel(R, p);
            if (pix < 0) return false;
            float jx = 0.5f, jy = 0.5f;
            if (R.jitter) {
                uint4 b = stream_block(R.seed, (uint32_t)pix, (uint32_t)sample, 0, ST_CAM, 0);
                jx = u01(b.x); jy = u01(b.y);
            }
            float3 o, d;
            camera_ray(R.cam, pix % R.cam.W, pix / R.cam.W, jx, jy, o, d);
            const uint32_t mask = STOCH ? policy_for(R.ext, R.sc, d, R.seed, (uint32_t)pix, (uint32_t)sample, 0,
                                                     ST_EXT, 1, w)
                                        : R.ext.static_mask;
            trav_begin(T, make_ray(o, d, 0.0f, INFINITY), 0.0f, INFINITY, mask);
            tau = 0.0;
            began = true;
            if (COUNT) ++wk.paths;
            return true;
        },
        [&](const Setup& s, float coef, uint32_t g, uint32_t k) -> bool {
            float c = coef * s.ij * seg_J(s, s.u0, s.u1, wk);
            if (STOCH) c *= w[g];
            tau += (double)c;
            return true;
        },
        [&]() { R.L[p] = (float)tau; },
        [&]() { count_rays(R.rays + 0, began); began = false; });
    if (COUNT) flush_work(R.work + kWorkSlots * STAGE_TOMO, wk);
}

// ---------------------------------------------------------------- ffA: binned tau over the ray
// Single-pass version (traversal with the bin integrals inline).  Used for the paths whose hit
// records overflow the record buffer of k_ffA_T (input queue q, counter slots cnt/work).
template <bool STOCH, bool COUNT>
__global__ void __launch_bounds__(128, GF_MINB_FFA) k_ffA(RenderDev R, int32_t sample, int32_t depth,
                                                           const uint32_t* __restrict__ q, int cnt_slot, int work_slot,
                                                           int ray_count) {
    Work wk;
    Trav T;
    uint32_t p = 0;
    double tstar = 0.0;
    float tlo = 0.0f, bw = 0.0f, ibw = 0.0f;
    // per-thread bins in shared memory, [bin][thread] (conflict-free), fp32 (a bin sums tens of terms)
    __shared__ float s_bins[kBins * 128];
    __shared__ uint16_t s_cnts[kBins * 128];
    float* bins = s_bins + threadIdx.x;
    uint16_t* cnts = s_cnts + threadIdx.x;
    float w[kMaxGroups];
    bool began = false, fin = false, collide = false;
    uint32_t fin_p = 0, nh = 0;
    auto finish = [&](int32_t bin, double cum_before, double bin_tau, int32_t nact) {
        if (bin == -2) {
            R.L[p] += R.beta[p] * R.env_L;  // escape -> environment
            collide = false;
        } else {
            R.bin[p] = bin < 0 ? bin : (bin | (nact << 16));
            R.cum[p] = cum_before;               // tau before the bracketing bin
            R.cum[p + R.n_paths] = tstar;        // tau*
            R.cum[p + 2 * R.n_paths] = bin_tau;  // tau inside the bin
            R.nhit[p] = nh;
            collide = true;
        }
        fin = true;
        fin_p = p;
    };
    flat_loop<COUNT, kBatch, GF_SPLIT_FFA>(
        R.qcount + work_slot, R.qcount[cnt_slot], R.nodes, R.n_nodes, R.prims, T, wk,
        [&](uint32_t idx) -> bool {
            p = q[idx];
            began = ray_count != 0;
            if (COUNT) ++wk.paths;
            const uint32_t pix = R.pix[p];
            const float3 o = ld3(R.ox, R.oy, R.oz, p), d = ld3(R.dx, R.dy, R.dz, p);
            const uint32_t mask = STOCH ? policy_for(R.ext, R.sc, d, R.seed, pix, (uint32_t)sample, (uint32_t)depth,
                                                     ST_EXT, 1, w)
                                        : R.ext.static_mask;
            const float xi = stream_u(R.seed, pix, (uint32_t)sample, (uint32_t)depth, ST_EXT, 0);
            tstar = -log1p(-(double)xi);  // tau* = -ln(1 - xi)   (Eq. 5, C16)
            if (tstar <= 0.0) { finish(-1, 0.0, 0.0, 0); return false; }
            const RayDev r = make_ray(o, d, 0.0f, INFINITY);
            float thi;
            if (R.n_nodes == 0 || !slab_range(r, R.root_lo, R.root_hi, 0.0f, INFINITY, tlo, thi)) {
                finish(-2, 0.0, 0.0, 0);
                return false;
            }
            bw = (thi - tlo) * (1.0f / kBins);
            ibw = bw > 0.0f ? 1.0f / bw : 0.0f;
            nh = 0;
#pragma unroll
            for (int k = 0; k < kBins; ++k) { bins[k * 128] = 0.0f; cnts[k * 128] = 0; }
            trav_begin(T, r, tlo, thi, mask);
            return true;
        },
        [&](const Setup& s, float coef, uint32_t g, uint32_t k) -> bool {
            float cj = coef * s.ij;
            if (STOCH) cj *= w[g];
            const uint32_t span = bin_add<kBins, COUNT>(s, cj, tlo, bw, ibw, bins, cnts, 128, wk);
            // hit list for ffB: (sorted primitive index | group << 24, bin span), layout [path][k]
            if (nh < (uint32_t)R.hit_cap) R.hits[(size_t)p * R.hit_cap + nh] = make_uint2(k | (g << 24), span);
            ++nh;
            return true;
        },
        [&]() {
            double cum = 0.0;
            for (int k = 0; k < kBins; ++k) {
                const double c2 = cum + (double)bins[k * 128];
                if (c2 >= tstar) { finish(k, cum, (double)bins[k * 128], cnts[k * 128]); return; }
                cum = c2;
            }
            finish(-2, 0.0, 0.0, 0);
        },
        [&]() {
            push(R.qB2, R.qcount + kCntB2, fin && collide, fin_p);
            count_rays(R.rays + 0, began);
            fin = false;
            began = false;
        });
    if (COUNT) flush_work(R.work + kWorkSlots * STAGE_FFA, wk);
}


// ---------------------------------------------------------------- ffA as two kernels
// k_ffA_T: lean traversal that emits one 32-byte record per accepted primitive,
//   a = (u0, u1, Omega, phi0), b = (amp = c/j w e^{-(r2+Omega^2)/2} / 2, j, t_c, b'),
// Gaussians (Omega == 0) from the front of the path's region, Gabors from the back;
// k_ffA_I: one warp per path expands its records into erf endpoints (chord start, every bin
//   boundary inside the chord, chord end; a symmetric single-bin chord needs one) and evaluates
//   one endpoint per lane, type-uniform (real erf for the Gaussian part, the series for the Gabor
//   part), accumulating the pieces into shared per-path bins; then brackets tau*.
// Both read/write the records, which ffB also uses, so no primitive is reloaded after traversal.
template <bool STOCH, bool COUNT>
__global__ void __launch_bounds__(128, GF_MINB_T) k_ffA_T(RenderDev R, int32_t sample, int32_t depth) {
    Work wk;
    Trav T;
    uint32_t p = 0, ng = 0, nb = 0;
    double tstar = 0.0;
    float w[kMaxGroups];
    bool began = false, fin_b = false, fin_t = false, fin_o = false;
    uint32_t fin_p = 0;
    const uint32_t cap = (uint32_t)R.rec_cap;
    auto finish_early = [&](int32_t bin) {
        if (bin == -2) {
            R.L[p] += R.beta[p] * R.env_L;  // escape -> environment
        } else {
            R.bin[p] = bin;
            R.cum[p + R.n_paths] = tstar;
            fin_b = true;
            fin_p = p;
        }
    };
    flat_loop<COUNT, GF_BATCH_T, false>(
        R.qcount + kWorkAT, R.qcount[0], R.nodes, R.n_nodes, R.prims, T, wk,
        [&](uint32_t idx) -> bool {
            p = R.qA[idx];
            began = true;
            if (COUNT) ++wk.paths;
            const uint32_t pix = R.pix[p];
            const float3 o = ld3(R.ox, R.oy, R.oz, p), d = ld3(R.dx, R.dy, R.dz, p);
            const uint32_t mask = STOCH ? policy_for(R.ext, R.sc, d, R.seed, pix, (uint32_t)sample, (uint32_t)depth,
                                                     ST_EXT, 1, w)
                                        : R.ext.static_mask;
            const float xi = stream_u(R.seed, pix, (uint32_t)sample, (uint32_t)depth, ST_EXT, 0);
            tstar = -log1p(-(double)xi);  // tau* = -ln(1 - xi)   (Eq. 5, C16)
            if (tstar <= 0.0) { finish_early(-1); return false; }
            const RayDev r = make_ray(o, d, 0.0f, INFINITY);
            float tlo, thi;
            if (R.n_nodes == 0 || !slab_range(r, R.root_lo, R.root_hi, 0.0f, INFINITY, tlo, thi)) {
                finish_early(-2);
                return false;
            }
            R.tlo[p] = tlo;
            R.tbw[p] = (thi - tlo) * (1.0f / kBins);
            R.cum[p + R.n_paths] = tstar;
            ng = nb = 0;
            trav_begin(T, r, tlo, thi, mask);
            return true;
        },
        [&](const Setup& s, float coef, uint32_t g, uint32_t k) -> bool {
            float cj = coef * s.ij;
            if (STOCH) cj *= w[g];
            if (ng + nb < cap) {
                const float amp = 0.5f * cj * __expf(-0.5f * (s.r2 + s.Om * s.Om));
                const size_t slot = (size_t)p * cap + (s.Om == 0.0f ? ng : cap - 1 - nb);
                float4* rp = R.rec + 2 * slot;
                rp[0] = make_float4(s.u0, s.u1, s.Om, s.phi0);
                rp[1] = make_float4(amp, s.j, s.tc, s.bp);
            }
            if (s.Om == 0.0f) ++ng; else ++nb;
            return true;
        },
        [&]() {
            fin_p = p;
            if (ng + nb <= cap) {
                R.nrg[p] = ng;
                R.nrb[p] = nb;
                fin_t = true;
            } else {
                R.nrg[p] = 0xFFFFFFFFu;  // overflow: the single-pass kernel redoes this path
                fin_o = true;
            }
        },
        [&]() {
            push(R.qB, R.qcount + 1, fin_b, fin_p);
            push(R.qT, R.qcount + kCntT, fin_t, fin_p);
            push(R.qO, R.qcount + kCntO, fin_o, fin_p);
            count_rays(R.rays + 0, began);
            fin_b = fin_t = fin_o = began = false;
        });
    if (COUNT) flush_work(R.work + kWorkSlots * STAGE_FFA, wk);
}

// chord bin span of a record in the path's bins [tlo, tlo + kBins bw)
__device__ __forceinline__ void rec_span(float4 a, float4 b, float tlo, float ibw, int& ka, int& kb) {
    const float ij = 1.0f / b.y;
    const float ta = fmaf(a.x - b.w, ij, b.z), tb = fmaf(a.y - b.w, ij, b.z);
    ka = min(kBins - 1, max(0, (int)((ta - tlo) * ibw)));
    kb = min(kBins - 1, max(0, (int)((tb - tlo) * ibw)));
}

template <bool COUNT>
__global__ void __launch_bounds__(128) k_ffA_I(RenderDev R) {
    __shared__ float s_bins[4][kBins];
    __shared__ uint32_t s_cnts[4][kBins];
    __shared__ int s_off[4][33];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned FULL = 0xFFFFFFFFu;
    float* bins = s_bins[wid];
    uint32_t* cnts = s_cnts[wid];
    int* off = s_off[wid];
    const uint32_t count = R.qcount[kCntT], cap = (uint32_t)R.rec_cap;
    Work wk;
    while (true) {
        uint32_t idx = 0;
        if (lane == 0) idx = atomicAdd(R.qcount + kWorkAI, 1u);
        idx = __shfl_sync(FULL, idx, 0);
        if (idx >= count) break;
        const uint32_t p = R.qT[idx];
        const float tlo = R.tlo[p], bw = R.tbw[p], ibw = bw > 0.0f ? 1.0f / bw : 0.0f;
        for (int k = lane; k < kBins; k += 32) { bins[k] = 0.0f; cnts[k] = 0; }
        __syncwarp();
        const uint32_t nside[2] = {R.nrg[p], R.nrb[p]};
#pragma unroll 1
        for (int side = 0; side < 2; ++side) {  // 0: Gaussian records (real erf), 1: Gabor records (series)
            const uint32_t n = nside[side];
            for (uint32_t base = 0; base < n; base += 32) {
                const uint32_t i = base + lane;
                const bool valid = i < n;
                float4 a = make_float4(0, 0, 0, 0), b = make_float4(0, 1, 0, 0);
                int ka = 0, kb = 0, ne = 0;
                if (valid) {
                    const size_t slot = (size_t)p * cap + (side == 0 ? i : cap - 1 - i);
                    a = R.rec[2 * slot];
                    b = R.rec[2 * slot + 1];
                    rec_span(a, b, tlo, ibw, ka, kb);
                    for (int m = ka; m <= kb; ++m) atomicAdd(&cnts[m], 1u);
                    const float wmax = 0.5f * (fmaxf(a.x * a.x, a.y * a.y) + a.z * a.z);
                    if (a.y - a.x < 1e-4f || (wmax > kWMaxSeries && a.z != 0.0f)) {
                        // rare: midpoint / Gauss-Legendre pieces, lane-local (seg_J without e^{-r2/2}
                        // and the 1/2 e^{-Om^2/2} folded into amp)
                        Setup s;
                        s.r2 = 0.0f; s.h = INFINITY; s.bp = b.w; s.j = b.y; s.ij = 1.0f / b.y; s.tc = b.z;
                        s.Om = a.z; s.phi0 = a.w;
                        const float scale = 2.0f * b.x * __expf(0.5f * a.z * a.z);  // cj e^{-r2/2}
                        float ua = a.x;
                        for (int m = ka + 1; m <= kb + 1; ++m) {
                            const float ub = (m > kb) ? a.y
                                                      : fminf(fmaxf(fmaf(b.y, (tlo + m * bw) - b.z, b.w), ua), a.y);
                            atomicAdd(&bins[m - 1], scale * seg_J(s, ua, ub, wk));
                            ua = ub;
                        }
                    } else {
                        ne = (ka == kb && a.x == -a.y) ? 1 : (kb - ka + 2);
                    }
                }
                // exclusive prefix of endpoint counts over the chunk
                int incl = ne;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int v = __shfl_up_sync(FULL, incl, o);
                    if (lane >= o) incl += v;
                }
                off[lane + 1] = incl;
                if (lane == 0) off[0] = 0;
                __syncwarp();
                const int total = __shfl_sync(FULL, incl, 31);
                for (int e0 = 0; e0 < total; e0 += 32) {
                    const int e = e0 + lane;
                    // owner record of endpoint e: largest r with off[r] <= e (binary search)
                    int lo = 0, hi = 31;
                    while (lo < hi) {
                        const int mid = (lo + hi + 1) >> 1;
                        if (off[mid] <= e) lo = mid; else hi = mid - 1;
                    }
                    const int r = lo;
                    const float u0 = __shfl_sync(FULL, a.x, r), u1 = __shfl_sync(FULL, a.y, r);
                    const float Om = __shfl_sync(FULL, a.z, r), phi = __shfl_sync(FULL, a.w, r);
                    const float amp = __shfl_sync(FULL, b.x, r), jj = __shfl_sync(FULL, b.y, r);
                    const float tc = __shfl_sync(FULL, b.z, r), bp = __shfl_sync(FULL, b.w, r);
                    const int rka = __shfl_sync(FULL, ka, r), rne = __shfl_sync(FULL, ne, r);
                    if (e < total) {
                        const int je = e - off[r];
                        float u;
                        if (rne == 1 || je == rne - 1) u = u1;
                        else if (je == 0) u = u0;
                        else u = fminf(fmaxf(fmaf(jj, (tlo + (rka + je) * bw) - tc, bp), u0), u1);
                        float sp = 0.0f, cp = 1.0f;
                        float2 F;
                        if (side == 0) {
                            F = make_float2(erff(u * kRsqrt2), 0.0f);
                            if (phi != 0.0f) sincos_red(phi, &sp, &cp);  // Gabor along its modulation plane
                            if (COUNT) ++wk.erfr;
                        } else {
                            const float zr = u * kRsqrt2, zi = -Om * kRsqrt2;
                            F = erf_horner<kErfTerms>(zr, zi, fmaf(zr, zr, -zi * zi), 2.0f * zr * zi);
                            sincos_red(phi, &sp, &cp);
                            if (COUNT) ++wk.erfc;
                        }
                        if (rne == 1) {
                            atomicAdd(&bins[rka], 2.0f * amp * cp * F.x);
                        } else {
                            const float v = amp * fmaf(cp, F.x, -sp * F.y);
                            if (je >= 1) atomicAdd(&bins[rka + je - 1], v);
                            if (je <= rne - 2) atomicAdd(&bins[rka + je], -v);
                        }
                    }
                }
                __syncwarp();
            }
        }
        __syncwarp();
        if (lane == 0) {
            const double tstar = R.cum[p + R.n_paths];
            int32_t bin = -2;
            double cum = 0.0, cum_before = 0.0, bin_tau = 0.0;
            uint32_t nact = 0;
            for (int k = 0; k < kBins; ++k) {
                const double c2 = cum + (double)bins[k];
                if (c2 >= tstar) { bin = k; cum_before = cum; bin_tau = bins[k]; nact = cnts[k]; break; }
                cum = c2;
            }
            if (bin == -2) {
                R.L[p] += R.beta[p] * R.env_L;  // escape -> environment
            } else {
                R.bin[p] = bin | (int32_t)(min(nact, 32767u) << 16);
                R.cum[p] = cum_before;
                R.cum[p + 2 * R.n_paths] = bin_tau;
                R.qB[atomicAdd(R.qcount + 1, 1u)] = p;
            }
        }
        __syncwarp();
    }
    if (COUNT) flush_work(R.work + kWorkSlots * STAGE_FFAI, wk);
}

// ---------------------------------------------------------------- ffB: root in the bracketing bin
// Active primitives of the bracket, split into Gaussians (Omega == 0: real erf, 8 floats) and
// Gabors (complex erf, 13 floats); kept in local memory.  Inside the bunny-like scenes the
// overlap depth of the level-0 Gaussians is ~150, hence the large Gaussian list.
constexpr int kCapG = 448, kCapB = 96;
struct ActG {
    float amp, kap0, j, tc, bp, u0, u1, F0;
};
struct ActB {
    float amp, kap0, Om, phi0, cp, sp, j, tc, bp, u0, u1, F0r, F0i;
};

__device__ __forceinline__ double actg_tau(const ActG& a, float t, double& kap, Work& wk) {
    float u = fmaf(a.j, t - a.tc, a.bp);
    if (!(u > a.u0)) return 0.0;
    if (u < a.u1) kap += (double)(a.kap0 * __expf(-0.5f * u * u));
    else u = a.u1;
    ++wk.erfr;
    return (double)(a.amp * (erff(u * kRsqrt2) - a.F0));
}

__device__ __forceinline__ double actb_tau(const ActB& a, float t, double& kap, Work& wk) {
    float u = fmaf(a.j, t - a.tc, a.bp);
    if (!(u > a.u0)) return 0.0;
    if (u < a.u1) {
        float sp, cp;
        sincos_red(fmaf(a.Om, u, a.phi0), &sp, &cp);
        kap += (double)(a.kap0 * __expf(-0.5f * u * u) * cp);
    } else {
        u = a.u1;
    }
    const float wmax = 0.5f * (fmaxf(a.u0 * a.u0, u * u) + a.Om * a.Om);
    if (wmax > kWMaxSeries || u - a.u0 < 1e-4f) {  // generic path (GL / midpoint): cj*J from scratch
        Setup s;
        s.r2 = 0.0f; s.h = INFINITY; s.bp = a.bp; s.j = a.j; s.ij = 1.0f / a.j; s.tc = a.tc; s.Om = a.Om;
        s.phi0 = a.phi0; s.u0 = a.u0; s.u1 = u;
        // amp = cj e^{-r2/2} e^{-Om^2/2} / 2 ; seg_J with r2 = 0 carries e^{-Om^2/2}/2 only for the series,
        // so rescale from kap0 = cj j e^{-r2/2} / sqrt(2 pi)
        return (double)(a.kap0 * s.ij * 2.5066282746310002f * seg_J(s, a.u0, u, wk));
    }
    wk.erf(a.Om, 1);
    const float2 F = erf_shift(u, a.Om);
    return (double)(a.amp * fmaf(a.cp, F.x - a.F0r, -a.sp * (F.y - a.F0i)));
}

// Per-thread version (local-memory active lists), used for the record-overflow paths (queue qB2);
// each processed path is appended to qB for the NEE stage.
template <bool STOCH, bool COUNT>
__global__ void __launch_bounds__(128) k_ffB(RenderDev R, int32_t sample, int32_t depth) {
    const uint32_t count = R.qcount[kCntB2];
    uint32_t base;
    Work wk;
    while (fetch(R.qcount + kWorkB, count, base)) {
        const uint32_t idx = base + (threadIdx.x & 31);
        if (idx >= count) continue;
        const uint32_t p = R.qB2[idx];
        R.qB[atomicAdd(R.qcount + 1, 1u)] = p;
        const int32_t binw = R.bin[p];
        const float3 o = ld3(R.ox, R.oy, R.oz, p), d = ld3(R.dx, R.dy, R.dz, p);
        float tres = 0.0f;
        if (binw >= 0) {
            const int32_t bin = binw & 0xFFFF;
            const uint32_t pix = R.pix[p];
            float w[kMaxGroups];
            const uint32_t mask = STOCH ? policy_for(R.ext, R.sc, d, R.seed, pix, (uint32_t)sample, (uint32_t)depth,
                                                     ST_EXT, 1, w)
                                        : R.ext.static_mask;
            const RayDev r = make_ray(o, d, 0.0f, INFINITY);
            float tlo, thi;
            slab_range(r, R.root_lo, R.root_hi, 0.0f, INFINITY, tlo, thi);
            const float bw = (thi - tlo) * (1.0f / kBins);
            const float ta = tlo + bin * bw;
            const float tb = (bin == kBins - 1) ? thi : tlo + (bin + 1) * bw;
            const double tstar = R.cum[p + R.n_paths];
            const double cum0 = R.cum[p], span = R.cum[p + 2 * R.n_paths];
            ActG ag[kCapG];
            ActB ab[kCapB];
            int ng = 0, nb = 0;
            auto gather = [&](const GPrim& P, uint32_t g) {
                Setup s;
                if (!prim_setup(P, r, ta, tb, s)) return;
                if (COUNT) ++wk.hits;
                float cj = P.d.w * s.ij;
                if (STOCH) cj *= w[g];
                const float kap0 = cj * s.j * kInvSqrt2Pi * __expf(-0.5f * s.r2);
                if (s.Om == 0.0f) {
                    if (ng < kCapG) {
                        ActG& a = ag[ng];
                        a.amp = 0.5f * cj * __expf(-0.5f * s.r2); a.kap0 = kap0; a.j = s.j; a.tc = s.tc; a.bp = s.bp;
                        a.u0 = s.u0; a.u1 = s.u1; a.F0 = erff(s.u0 * kRsqrt2);
                        if (COUNT) ++wk.erfr;
                    }
                    ++ng;
                } else {
                    if (nb < kCapB) {
                        ActB& a = ab[nb];
                        a.amp = 0.5f * cj * __expf(-0.5f * (s.r2 + s.Om * s.Om)); a.kap0 = kap0;
                        a.Om = s.Om; a.phi0 = s.phi0; a.j = s.j; a.tc = s.tc; a.bp = s.bp; a.u0 = s.u0; a.u1 = s.u1;
                        sincos_red(s.phi0, &a.sp, &a.cp);
                        const float2 F0 = erf_shift(s.u0, s.Om);
                        if (COUNT) wk.erf(s.Om, 1);
                        a.F0r = F0.x; a.F0i = F0.y;
                    }
                    ++nb;
                }
            };
            const bool recpath = R.nrg[p] != 0xFFFFFFFFu;
            const uint32_t nh = recpath ? 0xFFFFFFFFu : R.nhit[p];
            if (recpath) {  // the path's hit records from k_ffA_T: clip to the bracket, no primitive reload
                const float ibw = bw > 0.0f ? 1.0f / bw : 0.0f;
                const uint32_t cap = (uint32_t)R.rec_cap;
                const uint32_t nside[2] = {R.nrg[p], R.nrb[p]};
                for (int side = 0; side < 2; ++side) {
                    for (uint32_t i = 0; i < nside[side]; ++i) {
                        const size_t slot = (size_t)p * cap + (side == 0 ? i : cap - 1 - i);
                        const float4 a = R.rec[2 * slot], b = R.rec[2 * slot + 1];
                        int ka, kb;
                        rec_span(a, b, tlo, ibw, ka, kb);
                        if (COUNT) ++wk.tests;
                        if (ka > bin || kb < bin) continue;
                        const float ua = fmaxf(a.x, fmaf(b.y, ta - b.z, b.w));
                        const float ub = fminf(a.y, fmaf(b.y, tb - b.z, b.w));
                        if (!(ub > ua)) continue;
                        if (COUNT) ++wk.hits;
                        const float kap0 = b.x * b.y * 0.79788456080286536f * __expf(0.5f * a.z * a.z);
                        if (a.z == 0.0f && a.w == 0.0f) {
                            if (ng < kCapG) {
                                ActG& g = ag[ng];
                                g.amp = b.x; g.kap0 = kap0; g.j = b.y; g.tc = b.z; g.bp = b.w; g.u0 = ua; g.u1 = ub;
                                g.F0 = erff(ua * kRsqrt2);
                                if (COUNT) ++wk.erfr;
                            }
                            ++ng;
                        } else {
                            if (nb < kCapB) {
                                ActB& q = ab[nb];
                                q.amp = b.x; q.kap0 = kap0; q.Om = a.z; q.phi0 = a.w; q.j = b.y; q.tc = b.z; q.bp = b.w;
                                q.u0 = ua; q.u1 = ub;
                                sincos_red(a.w, &q.sp, &q.cp);
                                const float2 F0 = erf_shift(ua, a.z);
                                if (COUNT) wk.erf(a.z, 1);
                                q.F0r = F0.x; q.F0i = F0.y;
                            }
                            ++nb;
                        }
                    }
                }
            } else if (nh <= (uint32_t)R.hit_cap) {  // scan the path's hit list from single-pass ffA
                for (uint32_t k = 0; k < nh; ++k) {
                    const uint2 e = R.hits[(size_t)p * R.hit_cap + k];
                    if ((int)(e.y & 0xFFu) > bin || (int)(e.y >> 8) < bin) continue;
                    const GPrim* q = R.prims + (e.x & 0xFFFFFFu);
                    GPrim P;
                    P.a = __ldg(&q->a); P.b = __ldg(&q->b); P.c = __ldg(&q->c); P.d = __ldg(&q->d);
                    if (COUNT) ++wk.tests;
                    gather(P, e.x >> 24);  // (hits already passed the predicate on the full ray)
                }
            } else {
                traverse_r<COUNT>(R.nodes, R.n_nodes, R.prims, r, ta, tb, mask, wk, gather);
            }
            const bool overflow = ng > kCapG || nb > kCapB;
            if (COUNT && overflow) ++wk.overflow;
            auto eval = [&](float t, double& kap) -> double {
                kap = 0.0;
                double acc = cum0 - tstar;
                if (COUNT) ++wk.root;
                if (!overflow) {
                    for (int k = 0; k < ng; ++k) acc += actg_tau(ag[k], t, kap, wk);
                    for (int k = 0; k < nb; ++k) acc += actb_tau(ab[k], t, kap, wk);
                } else {  // list overflow: stream the bracket's primitives again (hit list or traversal)
                    auto one = [&](const GPrim& P, uint32_t g) {
                        Setup s;
                        if (!prim_setup(P, r, ta, tb, s)) return;
                        float cj = P.d.w * s.ij;
                        if (STOCH) cj *= w[g];
                        const float ut = fmaf(s.j, t - s.tc, s.bp);
                        if (!(ut > s.u0)) return;
                        if (ut < s.u1) {
                            float sp, cp;
                            sincos_red(fmaf(s.Om, ut, s.phi0), &sp, &cp);
                            kap += (double)(cj * s.j * kInvSqrt2Pi * __expf(-0.5f * (s.r2 + ut * ut)) * cp);
                        }
                        acc += (double)(cj * seg_J(s, s.u0, fminf(ut, s.u1), wk));
                    };
                    if (nh <= (uint32_t)R.hit_cap) {
                        for (uint32_t k = 0; k < nh; ++k) {
                            const uint2 e = R.hits[(size_t)p * R.hit_cap + k];
                            if ((int)(e.y & 0xFFu) > bin || (int)(e.y >> 8) < bin) continue;
                            const GPrim* q = R.prims + (e.x & 0xFFFFFFu);
                            GPrim P;
                            P.a = __ldg(&q->a); P.b = __ldg(&q->b); P.c = __ldg(&q->c); P.d = __ldg(&q->d);
                            one(P, e.x >> 24);
                        }
                    } else {
                        traverse_r<COUNT>(R.nodes, R.n_nodes, R.prims, r, ta, tb, mask, wk, one);
                    }
                }
                return acc;
            };
            float lo = ta, hi = tb;
            // initial guess: linear in the bin's own tau (from ffA)
            const double need = tstar - cum0;
            float t = ta + 0.5f * (tb - ta);
            if (span > 0.0 && need >= 0.0) t = ta + (float)(need / span) * (tb - ta);
            t = fminf(fmaxf(t, lo), hi);
            for (int it = 0; it < 48; ++it) {
                double kap;
                const double f = eval(t, kap);
                if (f >= 0.0) hi = t; else lo = t;
                if (!(hi - lo > 1e-6f * bw)) break;
                if (fabs(f) <= 1e-6 * (1.0 + tstar)) break;  // |tau(t) - tau*| at the fp32 noise floor
                float tn = (kap > 0.0) ? (float)((double)t - f / kap) : 0.5f * (lo + hi);
                const bool newton = tn > lo && tn < hi;
                if (!newton) tn = 0.5f * (lo + hi);
                const bool small = newton && fabsf(tn - t) <= 1e-5f * bw;  // converged Newton step
                t = tn;
                if (small) break;
            }
            tres = t;
        }
        // collision point becomes the new origin
        R.ox[p] = fmaf(tres, d.x, o.x);
        R.oy[p] = fmaf(tres, d.y, o.y);
        R.oz[p] = fmaf(tres, d.z, o.z);
    }
    if (COUNT) flush_work(R.work + kWorkSlots * STAGE_FFB, wk);
}


// ---------------------------------------------------------------- ffB, one warp per path
// The bracket's active primitives are the path's hit records overlapping bin k.  Lanes scan the
// records in parallel (coalesced); every Newton evaluation is a warp reduction of
//   f(t) = cum0 - tau* + sum_i amp_i [G_i(clamp(u_i(t))) - G_i(lower_i)],  G = Re(e^{i phi} F),
//   kappa(t) = sum_i kap0_i e^{-u^2/2} cos(phi_i + Omega_i u)      (derivative of tau, analytic),
// so all lanes take the same (safeguarded Newton / bisection) steps.  No per-lane lists.
template <bool COUNT>
__global__ void __launch_bounds__(128) k_ffB_W(RenderDev R) {
    const int lane = threadIdx.x & 31;
    const unsigned FULL = 0xFFFFFFFFu;
    const uint32_t count = R.qcount[1], cap = (uint32_t)R.rec_cap;
    Work wk;
    while (true) {
        uint32_t idx = 0;
        if (lane == 0) idx = atomicAdd(R.qcount + kWorkBW, 1u);
        idx = __shfl_sync(FULL, idx, 0);
        if (idx >= count) break;
        const uint32_t p = R.qB[idx];
        const int32_t binw = R.bin[p];
        const float3 o = ld3(R.ox, R.oy, R.oz, p), d = ld3(R.dx, R.dy, R.dz, p);
        float tres = 0.0f;
        if (binw >= 0) {
            const int bin = binw & 0xFFFF;
            const float tlo = R.tlo[p], bw = R.tbw[p], ibw = bw > 0.0f ? 1.0f / bw : 0.0f;
            const float ta = tlo + bin * bw;
            const float tb = tlo + (bin + 1) * bw;
            const float tbc = (bin == kBins - 1) ? INFINITY : tb;  // clip window (records end at thi)
            const double tstar = R.cum[p + R.n_paths], cum0 = R.cum[p], span = R.cum[p + 2 * R.n_paths];
            const uint32_t nside[2] = {R.nrg[p], R.nrb[p]};
            // one scan over the records: mode 0 -> S0 = sum amp G(lower); mode 1 -> sum amp G(clamp(u_t)), kappa
            auto scan = [&](int mode, float t, double& kap_out) -> double {
                float acc = 0.0f, kap = 0.0f;
#pragma unroll 1
                for (int side = 0; side < 2; ++side) {
                    for (uint32_t i = lane; i < nside[side]; i += 32) {
                        const size_t slot = (size_t)p * cap + (side == 0 ? i : cap - 1 - i);
                        const float4 a = R.rec[2 * slot], b = R.rec[2 * slot + 1];
                        int ka, kb;
                        rec_span(a, b, tlo, ibw, ka, kb);
                        if (ka > bin || kb < bin) continue;
                        const float lower = fmaxf(a.x, fmaf(b.y, ta - b.z, b.w));
                        const float upper = fminf(a.y, fmaf(b.y, tbc - b.z, b.w));
                        if (!(upper > lower)) continue;
                        if (COUNT && mode == 0) ++wk.hits;
                        const float wmax = 0.5f * (fmaxf(lower * lower, upper * upper) + a.z * a.z);
                        const bool special = upper - lower < 1e-4f || (wmax > kWMaxSeries && a.z != 0.0f);
                        float u = lower;
                        if (mode == 1) {
                            const float ut = fmaf(b.y, t - b.z, b.w);
                            if (ut > lower && ut < upper) {
                                float sp, cp;
                                sincos_red(fmaf(a.z, ut, a.w), &sp, &cp);
                                kap += b.x * b.y * 0.79788456080286536f * __expf(0.5f * (a.z * a.z - ut * ut)) * cp;
                            }
                            u = fminf(fmaxf(ut, lower), upper);
                        }
                        if (special) {  // rare: midpoint / Gauss-Legendre from lower (no S0 term)
                            if (mode == 1 && u > lower) {
                                Setup s;
                                s.r2 = 0.0f; s.h = INFINITY; s.bp = b.w; s.j = b.y; s.ij = 1.0f / b.y; s.tc = b.z;
                                s.Om = a.z; s.phi0 = a.w;
                                acc += 2.0f * b.x * __expf(0.5f * a.z * a.z) * seg_J(s, lower, u, wk);
                            }
                            continue;
                        }
                        float2 F;
                        float sp = 0.0f, cp = 1.0f;
                        if (side == 0) {
                            F = make_float2(erff(u * kRsqrt2), 0.0f);
                            if (a.w != 0.0f) sincos_red(a.w, &sp, &cp);
                            if (COUNT) ++wk.erfr;
                        } else {
                            const float zr = u * kRsqrt2, zi = -a.z * kRsqrt2;
                            F = erf_horner<kErfTerms>(zr, zi, fmaf(zr, zr, -zi * zi), 2.0f * zr * zi);
                            sincos_red(a.w, &sp, &cp);
                            if (COUNT) ++wk.erfc;
                        }
                        acc += b.x * fmaf(cp, F.x, -sp * F.y);
                    }
                }
                double x = acc, k = kap;
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) {
                    x += __shfl_xor_sync(FULL, x, off);
                    k += __shfl_xor_sync(FULL, k, off);
                }
                kap_out = k;
                return x;
            };
            double kap;
            const double S0 = scan(0, 0.0f, kap);
            auto eval = [&](float t, double& kp) -> double {
                if (COUNT) ++wk.root;
                return cum0 - tstar - S0 + scan(1, t, kp);
            };
            float lo = ta, hi = tb;
            const double need = tstar - cum0;
            float t = ta + 0.5f * (tb - ta);
            if (span > 0.0 && need >= 0.0) t = ta + (float)(need / span) * (tb - ta);
            t = fminf(fmaxf(t, lo), hi);
            for (int it = 0; it < 48; ++it) {
                const double f = eval(t, kap);
                if (f >= 0.0) hi = t; else lo = t;
                if (!(hi - lo > 1e-6f * bw)) break;
                if (fabs(f) <= 1e-6 * (1.0 + tstar)) break;  // |tau(t) - tau*| at the fp32 noise floor
                float tn = (kap > 0.0) ? (float)((double)t - f / kap) : 0.5f * (lo + hi);
                const bool newton = tn > lo && tn < hi;
                if (!newton) tn = 0.5f * (lo + hi);
                const bool small = newton && fabsf(tn - t) <= 1e-5f * bw;  // converged Newton step
                t = tn;
                if (small) break;
            }
            tres = t;
        }
        if (lane == 0) {  // collision point becomes the new origin
            R.ox[p] = fmaf(tres, d.x, o.x);
            R.oy[p] = fmaf(tres, d.y, o.y);
            R.oz[p] = fmaf(tres, d.z, o.z);
        }
        __syncwarp();
    }
    if (COUNT) flush_work(R.work + kWorkSlots * STAGE_FFB, wk);
}

// ---------------------------------------------------------------- NEE + phase sampling
template <bool STOCH, bool COUNT>
__global__ void __launch_bounds__(128, GF_MINB_NEE) k_nee(RenderDev R, int32_t sample, int32_t depth) {
    Work wk;
    Trav T;
    uint32_t p = 0, pix = 0;
    double tau = 0.0;
    float w[kMaxGroups];
    bool began = false, cont = false;
    uint32_t fin_p = 0;
    flat_loop<COUNT, kBatch, GF_SPLIT_NEE>(
        R.qcount + kWorkN, R.qcount[1], R.nodes, R.n_nodes, R.prims, T, wk,
        [&](uint32_t idx) -> bool {
            p = R.qB[idx];
            pix = R.pix[p];
            began = true;
            if (COUNT) ++wk.paths;
            const float3 x = ld3(R.ox, R.oy, R.oz, p);
            const uint32_t mask = STOCH ? policy_for(R.nee, R.sc, R.sun, R.seed, pix, (uint32_t)sample,
                                                     (uint32_t)depth, ST_NEE, 0, w)
                                        : R.nee.static_mask;
            trav_begin(T, make_ray(x, R.sun, 0.0f, INFINITY), 0.0f, INFINITY, mask);
            tau = 0.0;
            return true;
        },
        [&](const Setup& s, float coef, uint32_t g, uint32_t k) -> bool {
            float c = coef * s.ij * seg_J(s, s.u0, s.u1, wk);
            if (STOCH) c *= w[g];
            tau += (double)c;
            return true;
        },
        [&]() {
            const float3 d = ld3(R.dx, R.dy, R.dz, p);
            const float beta = R.beta[p];
            const float cost = d.x * R.sun.x + d.y * R.sun.y + d.z * R.sun.z;
            R.L[p] += beta * R.albedo * hg_eval(R.hg_g, cost) * (float)exp(-tau) * R.sun_E;
            if (depth + 1 < R.max_depth) {
                uint4 b = stream_block(R.seed, pix, (uint32_t)sample, (uint32_t)depth, ST_SCAT, 0);
                float3 nd = hg_sample(R.hg_g, d, u01(b.x), u01(b.y));
                R.dx[p] = nd.x; R.dy[p] = nd.y; R.dz[p] = nd.z;
                R.beta[p] = beta * R.albedo;
                cont = true;
                fin_p = p;
            }
        },
        [&]() {
            push(R.qNext, R.qcount + 2, cont, fin_p);
            count_rays(R.rays + 1, began);
            cont = false;
            began = false;
        });
    if (COUNT) flush_work(R.work + kWorkSlots * STAGE_NEE, wk);
}

// NEE, one warp per path (warp_tau): shadow-ray transmittance, HG phase sampling of the next
// direction.  Replaces the per-lane k_nee on the production path.
template <bool STOCH, bool COUNT>
__global__ void __launch_bounds__(128) k_nee_w(RenderDev R, int32_t sample, int32_t depth) {
    __shared__ WarpTrav s_t[4];
    __shared__ WarpEnd s_e[4];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t count = R.qcount[1];
    Work wk;
    uint32_t nray = 0;
    while (true) {
        uint32_t idx = 0;
        if (lane == 0) idx = atomicAdd(R.qcount + kWorkN, 1u);
        idx = __shfl_sync(0xFFFFFFFFu, idx, 0);
        if (idx >= count) break;
        const uint32_t p = R.qB[idx];
        const uint32_t pix = R.pix[p];
        if (COUNT && lane == 0) ++wk.paths;
        ++nray;
        const float3 x = ld3(R.ox, R.oy, R.oz, p);
        float w[kMaxGroups];
        const uint32_t mask = STOCH ? policy_for(R.nee, R.sc, R.sun, R.seed, pix, (uint32_t)sample, (uint32_t)depth,
                                                 ST_NEE, 0, w)
                                    : R.nee.static_mask;
        const double tau = warp_tau<STOCH, COUNT>(R.nodes, R.nodes2, R.n_nodes, R.stk_limit, R.prims,
                                                  make_ray(x, R.sun, 0.0f, INFINITY), 0.0f, INFINITY, mask, w,
                                                  s_t[wid], s_e[wid], wk);
        if (lane == 0) {
            const float3 d = ld3(R.dx, R.dy, R.dz, p);
            const float beta = R.beta[p];
            const float cost = d.x * R.sun.x + d.y * R.sun.y + d.z * R.sun.z;
            R.L[p] += beta * R.albedo * hg_eval(R.hg_g, cost) * (float)exp(-tau) * R.sun_E;
            if (depth + 1 < R.max_depth) {
                uint4 b = stream_block(R.seed, pix, (uint32_t)sample, (uint32_t)depth, ST_SCAT, 0);
                float3 nd = hg_sample(R.hg_g, d, u01(b.x), u01(b.y));
                R.dx[p] = nd.x; R.dy[p] = nd.y; R.dz[p] = nd.z;
                R.beta[p] = beta * R.albedo;
                R.qNext[atomicAdd(R.qcount + 2, 1u)] = p;
            }
        }
    }
    if (lane == 0 && nray) atomicAdd(R.rays + 1, (unsigned long long)nray);
    if (COUNT) flush_work(R.work + kWorkSlots * STAGE_NEE, wk);
}

// tomography (mode 0), one warp per pixel: L = tau of the camera ray
template <bool STOCH, bool COUNT>
__global__ void __launch_bounds__(128) k_tomo_w(RenderDev R, int32_t sample) {
    __shared__ WarpTrav s_t[4];
    __shared__ WarpEnd s_e[4];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    Work wk;
    uint32_t nray = 0;
    for (int64_t p = (int64_t)blockIdx.x * 4 + wid; p < R.n_paths; p += (int64_t)gridDim.x * 4) {
        const int32_t pix = path_pixel(R, p);
        if (pix < 0) continue;
        float jx = 0.5f, jy = 0.5f;
        if (R.jitter) {
            uint4 b = stream_block(R.seed, (uint32_t)pix, (uint32_t)sample, 0, ST_CAM, 0);
            jx = u01(b.x); jy = u01(b.y);
        }
        float3 o, d;
        camera_ray(R.cam, pix % R.cam.W, pix / R.cam.W, jx, jy, o, d);
        float w[kMaxGroups];
        const uint32_t mask = STOCH ? policy_for(R.ext, R.sc, d, R.seed, (uint32_t)pix, (uint32_t)sample, 0, ST_EXT, 1, w)
                                    : R.ext.static_mask;
        if (COUNT && lane == 0) ++wk.paths;
        ++nray;
        const double tau = warp_tau<STOCH, COUNT>(R.nodes, R.nodes2, R.n_nodes, R.stk_limit, R.prims,
                                                  make_ray(o, d, 0.0f, INFINITY), 0.0f, INFINITY, mask, w, s_t[wid],
                                                  s_e[wid], wk);
        if (lane == 0) R.L[p] = (float)tau;
    }
    if (lane == 0 && nray) atomicAdd(R.rays + 0, (unsigned long long)nray);
    if (COUNT) flush_work(R.work + kWorkSlots * STAGE_TOMO, wk);
}

__global__ void k_rotate(uint32_t* qc) {
    qc[0] = qc[2];
    qc[1] = 0; qc[2] = 0;
    qc[kWorkA] = 0; qc[kWorkB] = 0; qc[kWorkN] = 0;
    qc[kCntT] = 0; qc[kCntO] = 0; qc[kWorkAT] = 0; qc[kWorkAI] = 0; qc[kWorkAO] = 0;
    qc[kCntB2] = 0; qc[kWorkBW] = 0;
}

__global__ void __launch_bounds__(256) k_finish(RenderDev R, int32_t slot) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= R.n_paths) return;
    const int32_t pix = path_pixel(R, p);
    if (pix < 0) return;
    const float v = R.L[p];
    if (R.probe) {
        R.accum[(R.path_base + p) * R.spp_count + slot] = v;
    } else {
        R.accum[2 * (int64_t)pix] += v;
        R.accum[2 * (int64_t)pix + 1] += v * v;
    }
}

}  // namespace gfk

using namespace gfk;

size_t gf_render_state_bytes(int64_t n, char* base, RenderDev* R) {
    size_t off = 0;
    auto take = [&](size_t bytes) { char* p = base ? base + off : nullptr; off += (bytes + 255) & ~(size_t)255; return p; };
    const size_t nf = sizeof(float) * (size_t)n, nu = sizeof(uint32_t) * (size_t)n;
    float* ox = (float*)take(nf); float* oy = (float*)take(nf); float* oz = (float*)take(nf);
    float* dx = (float*)take(nf); float* dy = (float*)take(nf); float* dz = (float*)take(nf);
    float* beta = (float*)take(nf); float* L = (float*)take(nf);
    double* cum = (double*)take(sizeof(double) * 3 * (size_t)n);
    int32_t* bin = (int32_t*)take(nu); uint32_t* pix = (uint32_t*)take(nu); uint32_t* nhit = (uint32_t*)take(nu);
    uint2* hits = (uint2*)take(sizeof(uint2) * (size_t)kHitCap * (size_t)n);
    float4* rec = (float4*)take(sizeof(float4) * 2 * (size_t)kRecCap * (size_t)n);
    uint32_t* nrg = (uint32_t*)take(nu); uint32_t* nrb = (uint32_t*)take(nu);
    float* tlo = (float*)take(nf); float* tbw = (float*)take(nf);
    uint32_t* qA = (uint32_t*)take(nu); uint32_t* qB = (uint32_t*)take(nu); uint32_t* qN = (uint32_t*)take(nu);
    uint32_t* qT = (uint32_t*)take(nu); uint32_t* qO = (uint32_t*)take(nu); uint32_t* qB2 = (uint32_t*)take(nu);
    uint32_t* qc = (uint32_t*)take(sizeof(uint32_t) * 16);
    if (R) {
        R->ox = ox; R->oy = oy; R->oz = oz; R->dx = dx; R->dy = dy; R->dz = dz; R->beta = beta; R->L = L;
        R->cum = cum; R->bin = bin; R->pix = pix; R->nhit = nhit; R->hits = hits; R->hit_cap = kHitCap;
        R->rec = rec; R->rec_cap = kRecCap; R->nrg = nrg; R->nrb = nrb; R->tlo = tlo; R->tbw = tbw;
        R->qA = qA; R->qB = qB; R->qNext = qN; R->qT = qT; R->qO = qO; R->qB2 = qB2; R->qcount = qc;
    }
    return off;
}

static int g_persist_blocks = 0;

template <bool S, bool C>
static void launch_depth(RenderDev& R, int32_t sample, int d, unsigned pgrid, unsigned wgrid, cudaStream_t st,
                         StageTimer& T,
                         bool stoch_nee) {
    cudaEvent_t e;
    T.pre(STAGE_FFA, st, e);
    k_ffA_T<S, C><<<pgrid, 128, 0, st>>>(R, sample, d);
    T.post(STAGE_FFA, st, e);
    T.pre(STAGE_FFAI, st, e);
    k_ffA_I<C><<<pgrid, 128, 0, st>>>(R);
    T.post(STAGE_FFAI, st, e);
    T.pre(STAGE_FFA, st, e);  // record-overflow paths: single-pass kernel
    k_ffA<S, C><<<pgrid, 128, 0, st>>>(R, sample, d, R.qO, kCntO, kWorkAO, 0);
    T.post(STAGE_FFA, st, e);
    T.pre(STAGE_FFB, st, e);
    k_ffB_W<C><<<pgrid, 128, 0, st>>>(R);
    T.post(STAGE_FFB, st, e);
    T.pre(STAGE_FFB, st, e);  // record-overflow paths (appended to qB for NEE)
    k_ffB<S, C><<<pgrid, 128, 0, st>>>(R, sample, d);
    T.post(STAGE_FFB, st, e);
    T.pre(STAGE_NEE, st, e);
    if (stoch_nee) k_nee_w<true, C><<<wgrid, 128, 0, st>>>(R, sample, d);
    else k_nee_w<false, C><<<wgrid, 128, 0, st>>>(R, sample, d);
    T.post(STAGE_NEE, st, e);
}

cudaError_t gf_launch_render_pass(RenderDev& R, int32_t sample, int32_t slot, cudaStream_t st, StageTimer& T) {
    cudaError_t e;
    if (R.n_paths == 0) return cudaSuccess;
    if (!g_persist_blocks) {
        int dev = 0, sms = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        g_persist_blocks = sms * 16;
    }
    const bool cnt = R.work != nullptr;
    const bool stoch_ext = !(R.ext.ls == 0 && R.ext.os == 0);
    const bool stoch_nee = !(R.nee.ls == 0 && R.nee.os == 0);
    const unsigned grid = (unsigned)((R.n_paths + 127) / 128);
    const unsigned pgrid = (unsigned)std::min<int64_t>((int64_t)g_persist_blocks, (R.n_paths + 127) / 128);
    const unsigned wgrid = (unsigned)std::min<int64_t>((int64_t)g_persist_blocks, (R.n_paths + 3) / 4);  // warp/path
    if ((e = cudaMemsetAsync(R.qcount, 0, sizeof(uint32_t) * 16, st))) return e;
    cudaEvent_t ev;
    if (R.mode == 0) {
        T.pre(STAGE_TOMO, st, ev);
        if (stoch_ext) {
            if (cnt) k_tomo_w<true, true><<<wgrid, 128, 0, st>>>(R, sample);
            else k_tomo_w<true, false><<<wgrid, 128, 0, st>>>(R, sample);
        } else {
            if (cnt) k_tomo_w<false, true><<<wgrid, 128, 0, st>>>(R, sample);
            else k_tomo_w<false, false><<<wgrid, 128, 0, st>>>(R, sample);
        }
        T.post(STAGE_TOMO, st, ev);
    } else {
        T.pre(STAGE_GEN, st, ev);
        k_gen<<<grid, 128, 0, st>>>(R, sample);
        T.post(STAGE_GEN, st, ev);
        for (int d = 0; d < R.max_depth; ++d) {
            if (stoch_ext) {
                if (cnt) launch_depth<true, true>(R, sample, d, pgrid, wgrid, st, T, stoch_nee);
                else launch_depth<true, false>(R, sample, d, pgrid, wgrid, st, T, stoch_nee);
            } else {
                if (cnt) launch_depth<false, true>(R, sample, d, pgrid, wgrid, st, T, stoch_nee);
                else launch_depth<false, false>(R, sample, d, pgrid, wgrid, st, T, stoch_nee);
            }
            T.pre(STAGE_FINISH, st, ev);
            k_rotate<<<1, 1, 0, st>>>(R.qcount);
            T.post(STAGE_FINISH, st, ev);
            std::swap(R.qA, R.qNext);
        }
    }
    T.pre(STAGE_FINISH, st, ev);
    k_finish<<<(unsigned)((R.n_paths + 255) / 256), 256, 0, st>>>(R, slot);
    T.post(STAGE_FINISH, st, ev);
    return cudaGetLastError();
}
