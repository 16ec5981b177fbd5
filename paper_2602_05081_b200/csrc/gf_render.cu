// gf_render.cu -- a8 free-flight distance sampling, a9 scatter loop, a10 accumulation
// (Eq. 4-5, bisection/root finding P:L254, pipeline P:L352-L365).
//
// Wavefront over the paths of one sample pass: gen -> [ff -> (fallback) -> nee] x max_depth -> finish.
//  k_ff   (one warp per path): warp traversal emitting hit records, exact tau_total (escape test),
//         safeguarded Newton on tau(t) = tau* (derivative = kappa(t), analytic);
//  k_ffA + k_ffB (per thread): single-pass fallback for paths with more records than the buffer;
//  k_nee_w (one warp per path): shadow ray towards the directional light (T = e^-tau), HG phase,
//         next direction.
// Queues are warp-aggregated; warps fetch paths dynamically from the queues.
#include <algorithm>

#include "gf_device.cuh"
#include "gf_internal.h"

namespace gfk {

#ifndef GF_BINS
#define GF_BINS 1
#endif
constexpr int kBins = GF_BINS;
constexpr int kHitCap = 1024;  // hits recorded per path by ffA for ffB (overflow -> traversal gather)
// qcount slots: 0 qA count, 1 qB count, 2 qNext count, then work cursors and fallback queues
constexpr int kWorkA = 4, kWorkB = 5, kWorkN = 6;  // cursors: (unused), k_ffB, k_nee_w
constexpr int kWorkRO = 7, kCntO2 = 8;  // k_ff redo of packet-overflow paths: cursor, its overflow count
constexpr int kCntO = 9, kWorkAT = 10, kWorkAO = 12;  // record-overflow queue count; k_ff / k_ffA cursors
constexpr int kCntB2 = 13;  // single-pass ffA -> per-thread ffB queue
#ifndef GF_REC_CAP
#define GF_REC_CAP 32768
#endif
constexpr int kRecCap = GF_REC_CAP;  // hit records per k_ff warp buffer (overflow -> single-pass ffA)

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
    if (!FOV || !R.fov) return 0xFFFFFFFFu;
    uint32_t m = 1u;  // level 0 (Gaussians, frequency 0) always
    for (int l = 1; l < R.sc.P; ++l)
        if (R.fov_lfmax[l] <= fm)
            for (int b = 0; b < R.sc.K; ++b) m |= 1u << (1 + (l - 1) * R.sc.K + b);
    return m;
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
        mb_shift(R, (uint32_t)pix, (uint32_t)sample, o);
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
#ifndef GF_CAM_BVH
#define GF_CAM_BVH 1  // k_ff_pkt traverses the camera BVH (projective boxes, built per gf_render call)
#endif
#ifndef GF_PRE_PF
#define GF_PRE_PF 1  // packet resolve: load the next chunk's chord data one chunk ahead
#endif
#ifndef GF_MINB_PKT
#define GF_MINB_PKT 7  // k_ff_pkt blocks per SM (72 registers)
#endif
#ifndef GF_PACKET
#define GF_PACKET 1  // depth-0 (camera) free flight with packet traversal (k_ff_pkt)
#endif
#ifndef GF_MINB_FFA
#define GF_MINB_FFA 6
#endif
#ifndef GF_SPLIT_FFA
#define GF_SPLIT_FFA 0
#endif
constexpr int kBatch = GF_BATCH;  // integrate pending hits once this many lanes (or most blocked lanes) have one

// ---------------------------------------------------------------- ffA: binned tau over the ray
// Single-pass version (traversal with the bin integrals inline).  Used for the paths whose hit
// records overflow the record buffer of k_ff (input queue q, counter slots cnt/work).
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
            const float fmx = fov_fmax<true>(R, (uint32_t)pix, (uint32_t)sample);
            const uint32_t mask = fov_mask<true>(R, fmx) & (STOCH ? policy_for(R.ext, R.sc, d, R.seed, pix, (uint32_t)sample, (uint32_t)depth,
                                                     ST_EXT, 1, w)
                                        : R.ext.static_mask);
            const float xi = stream_u(R.seed, pix, (uint32_t)sample, (uint32_t)depth, ST_EXT, 0);
            tstar = -log1p(-(double)xi);  // tau* = -ln(1 - xi)   (Eq. 5, C16)
            if (tstar <= 0.0) { finish(-1, 0.0, 0.0, 0); return false; }
            const RayDev r = make_ray(o, d, 0.0f, INFINITY, fmx);
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
    if (COUNT) flush_work(R.work + kWorkSlots * STAGE_FFB, wk);
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
            const float fmx = fov_fmax<true>(R, (uint32_t)pix, (uint32_t)sample);
            const uint32_t mask = fov_mask<true>(R, fmx) & (STOCH ? policy_for(R.ext, R.sc, d, R.seed, pix, (uint32_t)sample, (uint32_t)depth,
                                                     ST_EXT, 1, w)
                                        : R.ext.static_mask);
            const RayDev r = make_ray(o, d, 0.0f, INFINITY, fmx);
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
            const uint32_t nh = R.nhit[p];
            if (nh <= (uint32_t)R.hit_cap) {  // scan the path's hit list from single-pass ffA
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


// Phases 2-3 of the free flight of path p (whole warp): per-record chord integrals -> tau_total ->
// escape or the root of tau(t) = tau* (Halley / Newton / bisection over the records), then the
// path's new origin or its environment contribution.  rec/aux: the ray's ng Gaussian (front) and
// nb Gabor (back) records in a region of cap records.
// Per-record chord data of a hit record (a, b): full-chord integral amp (G(u1) - G(u0)),
// amp G(u0) (NaN for a midpoint / Gauss-Legendre record), amp cos phi0, -amp sin phi0.
// gabor: the series for Omega != 0 (else the real erf).
template <bool COUNT>
__device__ __forceinline__ float4 chord_aux(float4 a, float4 b, bool gabor, Work& wk) {
    float full, g0 = 0.0f, ac = 0.0f, as = 0.0f;
    const float wmax = 0.5f * (fmaxf(a.x * a.x, a.y * a.y) + a.z * a.z);
    if (a.y - a.x < 1e-4f || (wmax > kWMaxSeries && a.z != 0.0f)) {
        // rare: midpoint / Gauss-Legendre (seg_J with e^{-r2/2} and 1/2 e^{-Om^2/2} in amp)
        Setup s;
        s.r2 = 0.0f; s.h = INFINITY; s.bp = b.w; s.j = b.y; s.ij = 1.0f / b.y; s.tc = b.z;
        s.Om = a.z; s.phi0 = a.w;
        full = 2.0f * b.x * __expf(0.5f * a.z * a.z) * seg_J(s, a.x, a.y, wk);
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

template <bool COUNT, bool PRE>
__device__ __forceinline__ void ff_resolve(const RenderDev& R, uint32_t p, float3 o, float3 d, float tlo, float thi,
                                           double tstar, const float4* __restrict__ rec, float4* __restrict__ aux,
                                           uint32_t cap, uint32_t ng, uint32_t nb, float* hist, WarpEnd& q, Work& wk) {
    const unsigned FULL = 0xFFFFFFFFu;
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    // 2. per-record full integrals -> tau_total, histogram over 64 t-bins by chord centre
    float tot = 0.0f;
    const float hscale = 64.0f / fmaxf(thi - tlo, 1e-30f);
    hist[lane] = 0.0f;
    hist[lane + 32] = 0.0f;
    __syncwarp();
    const uint32_t nside[2] = {ng, nb};
#pragma unroll 1
    for (int side = 0; side < 2; ++side) {
        for (uint32_t i = lane; i < nside[side]; i += 32) {
            const uint32_t slot = side == 0 ? i : cap - 1 - i;
            float full, tm;
            if (PRE) {  // aux = (t_a, t_b, full, amp G(u0)): the records themselves are not read
                const float4 x = aux[slot];
                full = x.z;
                tm = 0.5f * (x.x + x.y);
            } else {
                const float4 a = rec[2 * slot], b = rec[2 * slot + 1];
                const float4 x = chord_aux<COUNT>(a, b, side == 1, wk);
                aux[slot] = x;
                full = x.x;
                tm = b.z + (0.5f * (a.x + a.y) - b.w) / b.y;
            }
            tot += full;
            atomicAdd(&hist[min(63, max(0, (int)((tm - tlo) * hscale)))], full);
        }
    }
    double tau_tot = tot;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tau_tot += __shfl_xor_sync(FULL, tau_tot, o);
    if (!PRE && tau_tot < tstar) {  // escape -> environment
        if (lane == 0) R.L[p] += R.beta[p] * R.env_L;
        return;
    }
    __syncwarp();
    // 3. Newton / bisection on f(t) = tau(t) - tau*
    int nq0 = 0, nq1 = 0;
    double acc = 0.0;
    auto run = [&](int t, int take) {
        int& nq = t == 0 ? nq0 : nq1;
        const bool v = lane < take;
        const float4 e = v ? q.e[t][nq - take + lane] : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        nq -= take;
        __syncwarp();
        if (v) {
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
    auto eval = [&](float t, double& kap_out, double& dkap_out) -> double {
        if (COUNT && lane == 0) ++wk.root;
        acc = 0.0;
        float part = 0.0f, kap = 0.0f, dkap = 0.0f;
#pragma unroll 1
        for (int side = 0; side < 2; ++side) {
            const uint32_t n = nside[side];
#if GF_PRE_PF
            float4 xnext = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
            if (PRE && lane < n) xnext = aux[side == 0 ? lane : cap - 1 - lane];
#if GF_PRE_PF == 2
            float4 xnext2 = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
            if (PRE && lane + 32 < n) xnext2 = aux[side == 0 ? lane + 32 : cap - 1 - (lane + 32)];
#endif
#endif
            for (uint32_t base = 0; base < n; base += 32) {
                const uint32_t i = base + lane;
                bool push = false;
                float4 e = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
#if GF_PRE_PF == 2
                const float4 xcur = xnext;  // chord data of this chunk, loaded two chunks ahead
                xnext = xnext2;
                if (PRE && i + 64 < n) xnext2 = aux[side == 0 ? i + 64 : cap - 1 - (i + 64)];
#elif GF_PRE_PF
                const float4 xcur = xnext;  // chord data of this chunk, loaded one chunk ahead
                if (PRE && i + 32 < n) xnext = aux[side == 0 ? i + 32 : cap - 1 - (i + 32)];
#endif
                if (PRE && i < n) {  // aux = (t_a, t_b, full, amp G(u0)); records read only for straddlers
                    const uint32_t slot = side == 0 ? i : cap - 1 - i;
#if GF_PRE_PF
                    const float4 x = xcur;
#else
                    const float4 x = aux[slot];
#endif
                    if (t >= x.y) {
                        part += x.z;
                    } else if (t > x.x) {
                        const float4 a = rec[2 * slot], b = rec[2 * slot + 1];
                        const float ut = fminf(fmaxf(fmaf(b.y, t - b.z, b.w), a.x), a.y);
                        float sp, cp;
                        sincos_red(fmaf(a.z, ut, a.w), &sp, &cp);
                        const float kk = b.x * b.y * 0.79788456080286536f * __expf(0.5f * (a.z * a.z - ut * ut));
                        kap += kk * cp;
                        dkap -= kk * b.y * fmaf(ut, cp, a.z * sp);
                        if (x.w != x.w) {  // special record: lane-local partial integral
                            Setup s;
                            s.r2 = 0.0f; s.h = INFINITY; s.bp = b.w; s.j = b.y; s.ij = 1.0f / b.y; s.tc = b.z;
                            s.Om = a.z; s.phi0 = a.w;
                            part += 2.0f * b.x * __expf(0.5f * a.z * a.z) * seg_J(s, a.x, ut, wk);
                        } else {
                            float s0 = 0.0f, c0 = 1.0f;
                            if (side == 1 || a.w != 0.0f) sincos_red(a.w, &s0, &c0);
                            part -= x.w;
                            push = true;
                            e = make_float4(ut, a.z, b.x * c0, -b.x * s0);
                        }
                    }
                } else if (!PRE && i < n) {
                    const uint32_t slot = side == 0 ? i : cap - 1 - i;
                    const float4 a = rec[2 * slot], b = rec[2 * slot + 1], x = aux[slot];
                    const float ut = fmaf(b.y, t - b.z, b.w);
                    if (ut >= a.y) {
                        part += x.x;
                    } else if (ut > a.x) {
                        float sp, cp;
                        sincos_red(fmaf(a.z, ut, a.w), &sp, &cp);
                        const float kk = b.x * b.y * 0.79788456080286536f * __expf(0.5f * (a.z * a.z - ut * ut));
                        kap += kk * cp;
                        dkap -= kk * b.y * fmaf(ut, cp, a.z * sp);  // d kappa / dt (Halley step)
                        if (x.y != x.y) {  // special record: lane-local partial integral
                            Setup s;
                            s.r2 = 0.0f; s.h = INFINITY; s.bp = b.w; s.j = b.y; s.ij = 1.0f / b.y; s.tc = b.z;
                            s.Om = a.z; s.phi0 = a.w;
                            part += 2.0f * b.x * __expf(0.5f * a.z * a.z) * seg_J(s, a.x, ut, wk);
                        } else {
                            part -= x.y;
                            push = true;
                            e = make_float4(ut, a.z, x.z, x.w);
                        }
                    }
                }
                const unsigned m = __ballot_sync(FULL, push);
                if (m) {
                    int& nq = side == 0 ? nq0 : nq1;
                    if (push) q.e[side][nq + __popc(m & lt)] = e;
                    nq += __popc(m);
                    __syncwarp();
                    if (nq >= 32) run(side, 32);
                }
            }
        }
        while (nq0 > 0) run(0, min(nq0, 32));
        while (nq1 > 0) run(1, min(nq1, 32));
        double x = acc + (double)part, k = kap, dk = dkap;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            x += __shfl_xor_sync(FULL, x, o);
            k += __shfl_xor_sync(FULL, k, o);
            dk += __shfl_xor_sync(FULL, dk, o);
        }
        kap_out = k;
        dkap_out = dk;
        return x - tstar;
    };
    const float bw = thi - tlo;
    float lo = tlo, hi = thi;
    float t;
    {  // start: first crossing of tau* in the histogram's running sum (linear inside the bin)
        const float h0 = hist[2 * lane], h1 = hist[2 * lane + 1];
        float incl = h0 + h1;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const float v = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += v;
        }
        const unsigned m = __ballot_sync(FULL, (double)incl >= tstar);
        const int L = m ? __ffs(m) - 1 : 31;
        const float ts = (float)tstar, prev = incl - (h0 + h1);
        float pos;
        if (prev + h0 >= ts) pos = 2 * lane + fminf(fmaxf((ts - prev) / fmaxf(h0, 1e-30f), 0.0f), 1.0f);
        else pos = 2 * lane + 1 + fminf(fmaxf((ts - prev - h0) / fmaxf(h1, 1e-30f), 0.0f), 1.0f);
        pos = __shfl_sync(FULL, pos, L);
        t = fminf(fmaxf(tlo + pos * (bw * (1.0f / 64.0f)), lo), hi);
    }
    double kap = 0.0, dkap = 0.0;
    for (int it = 0; it < 48; ++it) {
        const double f = eval(t, kap, dkap);
        if (f >= 0.0) hi = t; else lo = t;
        if (!(hi - lo > 1e-6f * bw)) break;
        if (fabs(f) <= 1e-6 * (1.0 + tstar)) break;  // |tau(t) - tau*| at the fp32 noise floor
        // Halley step (f' = kappa, f'' = d kappa/dt: cubic convergence), Newton if its
        // denominator degenerates, bisection if the step leaves the bracket
        const double den = 2.0 * kap * kap - f * dkap;
        float tn = (kap > 0.0) ? (float)((double)t - (den > 0.0 ? 2.0 * f * kap / den : f / kap)) : 0.5f * (lo + hi);
        const bool newton = tn > lo && tn < hi;
        if (!newton) tn = 0.5f * (lo + hi);
        const bool small = newton && fabsf(tn - t) <= 1e-5f * bw;  // converged Newton step
        t = tn;
        if (small) break;
    }
    if (lane == 0) {  // collision point becomes the new origin
        R.ox[p] = fmaf(t, d.x, o.x);
        R.oy[p] = fmaf(t, d.y, o.y);
        R.oz[p] = fmaf(t, d.z, o.z);
        R.qB[atomicAdd(R.qcount + 1, 1u)] = p;
    }
}

// ---------------------------------------------------------------- free flight, one warp per path
// k_ff fuses the whole free-flight step of a path (a8):
//  1. warp_traverse over [t_lo, t_hi] (the root box span) emitting one 32-byte record per
//     accepted primitive into the warp's own record buffer (coalesced, warp prefix offsets):
//     a = (u0, u1, Omega, phi0), b = (amp = c/j w e^{-(r2+Omega^2)/2} / 2, j, t_c, b');
//     Gaussians (Omega == 0) from the front, Gabors from the back, so erf work is type-uniform;
//  2. per record its full-chord integral amp (G(u1) - G(u0)), G(u) = Re{e^{i phi0} F(u)}, and
//     amp G(u0), amp cos phi0, -amp sin phi0 (aux); tau_total = sum -> escape test (Eq. 5);
//  3. safeguarded Newton / bisection on tau(t) = tau* over the whole ray: each evaluation scans
//     the records -- a chord wholly before t adds its full integral, one straddling t queues the
//     endpoint u(t) (one erf, evaluated 32 at a time, type-uniform) and adds its kappa term --
//     so no erf is spent on chords that t has passed or not reached.
// The buffer (rec_cap records per warp) stays L2-resident between the three phases; a path with
// more records than rec_cap goes to the single-pass fallback (k_ffA + k_ffB).
// CAM: depth-0 rays from the eye traverse the camera BVH (projective boxes, see k_ff_pkt)
template <bool STOCH, bool COUNT, bool CAM, bool FOV>
__global__ void __launch_bounds__(128) k_ff(RenderDev R, int32_t sample, int32_t depth,
                                            const uint32_t* __restrict__ q_in, int cnt_slot, int cur_slot,
                                            uint32_t* __restrict__ q_over, int over_slot) {
    __shared__ WarpTrav s_t[4];
    __shared__ WarpEnd s_e[4];
    __shared__ float s_h[4][64];  // coarse tau(t) histogram of the chord integrals -> Newton start
    const unsigned FULL = 0xFFFFFFFFu;
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const uint32_t count = R.qcount[cnt_slot], cap = (uint32_t)R.rec_cap;
    float* hist = s_h[wid];
    const size_t gw = (size_t)blockIdx.x * 4 + wid;
    float4* __restrict__ rec = R.wrec + gw * cap * 2;
    float4* __restrict__ aux = R.waux + gw * cap;
    WarpEnd& q = s_e[wid];
    Work wk;
    uint32_t nray = 0;
    while (true) {
        uint32_t idx = 0;
        if (lane == 0) idx = atomicAdd(R.qcount + cur_slot, 1u);
        idx = __shfl_sync(FULL, idx, 0);
        if (idx >= count) break;
        const uint32_t p = q_in[idx];
        ++nray;
        if (COUNT && lane == 0) ++wk.paths;
        const uint32_t pix = R.pix[p];
        const float3 o = ld3(R.ox, R.oy, R.oz, p), d = ld3(R.dx, R.dy, R.dz, p);
        float w[kMaxGroups];
        const float fmx = fov_fmax<FOV>(R, (uint32_t)pix, (uint32_t)sample);
        const uint32_t mask = fov_mask<FOV>(R, fmx) & (STOCH ? policy_for(R.ext, R.sc, d, R.seed, pix, (uint32_t)sample, (uint32_t)depth,
                                                 ST_EXT, 1, w)
                                    : R.ext.static_mask);
        const float xi = stream_u(R.seed, pix, (uint32_t)sample, (uint32_t)depth, ST_EXT, 0);
        const double tstar = -log1p(-(double)xi);  // tau* = -ln(1 - xi)   (Eq. 5, C16)
        if (tstar <= 0.0) {  // collision at the origin
            if (lane == 0) R.qB[atomicAdd(R.qcount + 1, 1u)] = p;
            continue;
        }
        const RayDev r = make_ray(o, d, 0.0f, INFINITY, fmx);
        float tlo, thi;
        if (R.n_nodes == 0 || !slab_range(r, R.root_lo, R.root_hi, 0.0f, INFINITY, tlo, thi)) {
            if (lane == 0) R.L[p] += R.beta[p] * R.env_L;  // escape -> environment
            continue;
        }
        // 1. records
        uint32_t ng = 0, nb = 0;
        const float dfw = fmaf(d.x, R.cb[6], fmaf(d.y, R.cb[7], d.z * R.cb[8]));
        const float pa = fmaf(d.x, R.cb[0], fmaf(d.y, R.cb[1], d.z * R.cb[2])) / dfw;
        const float pb = fmaf(d.x, R.cb[3], fmaf(d.y, R.cb[4], d.z * R.cb[5])) / dfw;
        const float qlo = tlo * dfw, qhi = thi * dfw;
        const GPrim* __restrict__ prims = CAM ? R.cprims : R.prims;
        warp_traverse_b<COUNT>(CAM ? R.cnodes : R.nodes, CAM ? R.cnodes2 : R.nodes2, R.n_nodes,
                               CAM ? max(1, kWStk - 34 - (int)*R.cdepth) : R.stk_limit, mask, s_t[wid], wk,
                             [&](bool valid, uint32_t ref) {
            bool hit = false;
            Setup s;
            float cj = 0.0f;
            if (valid) {
                const GPrim* pp = prims + (ref & kRefIdx);
                GPrim P;
                P.a = __ldg(&pp->a);
                if (COUNT) ++wk.tests;
                if (sphere_pretest(P.a, r, tlo, thi)) {
                    P.b = __ldg(&pp->b); P.c = __ldg(&pp->c); P.d = __ldg(&pp->d);
                    hit = prim_setup(P, r, tlo, thi, s);
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
        }, [&](float4 lo, float4 hi) {
            if (CAM) return lo.x <= pa && pa <= hi.x && lo.y <= pb && pb <= hi.y && hi.z >= qlo && lo.z <= qhi;
            return slab(r, lo, hi, tlo, thi);
        });
        if (ng + nb > cap) {  // record overflow: single-pass fallback
            if (lane == 0) q_over[atomicAdd(R.qcount + over_slot, 1u)] = p;
            continue;
        }
        __syncwarp();
        ff_resolve<COUNT, false>(R, p, o, d, tlo, thi, tstar, rec, aux, cap, ng, nb, hist, q, wk);
        __syncwarp();
    }
    if (lane == 0 && nray) atomicAdd(R.rays + 0, (unsigned long long)nray);
    if (COUNT) flush_work(R.work + kWorkSlots * STAGE_FFA, wk);
}

// ---------------------------------------------------------------- free flight of coherent rays
// k_ff_pkt: depth-0 camera rays, 32 consecutive paths per warp (one 8x4 pixel block of the tiled
// path order, so the rays are nearly parallel and overlap the same primitives).  Packet traversal:
// the warp walks ONE depth-first stack; each popped node's child pair is loaded once (broadcast)
// and every lane tests it against its own ray; a child is descended if any lane's ray meets it,
// and a hit leaf's primitives are loaded once and tested by each lane against its ray.  Each lane
// writes its ray's hit records into its own region of the warp's buffer; then the warp resolves
// the rays one after another with ff_resolve (chord integrals, escape test, root).
constexpr int kPStk = 512;
template <bool STOCH, bool COUNT, bool FOV>
__global__ void __launch_bounds__(128, GF_MINB_PKT) k_ff_pkt(RenderDev R, int32_t sample, int32_t depth) {
    __shared__ uint32_t s_stk[4][kPStk];
    __shared__ WarpEnd s_e[4];
    __shared__ float s_h[4][64];
    const unsigned FULL = 0xFFFFFFFFu;
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t count = R.qcount[0], cap = (uint32_t)R.rec_cap, lcap = cap / 32;
    const size_t gw = (size_t)blockIdx.x * 4 + wid;
    float4* __restrict__ wrec = R.wrec + gw * cap * 2;
    float4* __restrict__ waux = R.waux + gw * cap;
    float4* __restrict__ myrec = wrec + (size_t)lane * lcap * 2;
    float4* __restrict__ myaux = waux + (size_t)lane * lcap;
    uint32_t* stk = s_stk[wid];
    Work wk;
    uint32_t nray = 0;
    while (true) {
        uint32_t base = 0;
        if (lane == 0) base = atomicAdd(R.qcount + kWorkAT, 32u);
        base = __shfl_sync(FULL, base, 0);
        if (base >= count) break;
        const uint32_t idx = base + lane;
        const bool valid = idx < count;
        const uint32_t p = valid ? R.qA[idx] : 0u;
        bool act = valid;
        uint32_t pix = 0, mask = 0;
        float fmx = INFINITY;
        float3 o = make_float3(0.0f, 0.0f, 0.0f), d = make_float3(0.0f, 0.0f, 1.0f);
        double tstar = 0.0;
        float w[kMaxGroups];
        if (valid) {
            ++nray;
            if (COUNT) ++wk.paths;
            pix = R.pix[p];
            o = ld3(R.ox, R.oy, R.oz, p);
            d = ld3(R.dx, R.dy, R.dz, p);
            fmx = fov_fmax<FOV>(R, pix, (uint32_t)sample);
            mask = fov_mask<FOV>(R, fmx) & (STOCH ? policy_for(R.ext, R.sc, d, R.seed, pix, (uint32_t)sample, (uint32_t)depth,
                                                          ST_EXT, 1, w)
                                             : R.ext.static_mask);
            const float xi = stream_u(R.seed, pix, (uint32_t)sample, (uint32_t)depth, ST_EXT, 0);
            tstar = -log1p(-(double)xi);  // tau* = -ln(1 - xi)   (Eq. 5, C16)
            if (tstar <= 0.0) {  // collision at the origin
                R.qB[atomicAdd(R.qcount + 1, 1u)] = p;
                act = false;
            }
        }
        const RayDev r = make_ray(o, d, 0.0f, INFINITY, fmx);
        float tlo = 0.0f, thi = 0.0f;
        if (act && (R.n_nodes == 0 || !slab_range(r, R.root_lo, R.root_hi, 0.0f, INFINITY, tlo, thi))) {
            R.L[p] += R.beta[p] * R.env_L;  // escape -> environment
            act = false;
        }
        // box test: camera BVH (projective boxes: the ray is the point (a, b) = (d.r, d.u) / d.f with depth
        // q.f = t d.f in [tlo, thi] d.f) or world slabs
        const float dfw = fmaf(d.x, R.cb[6], fmaf(d.y, R.cb[7], d.z * R.cb[8]));
        const float pa = fmaf(d.x, R.cb[0], fmaf(d.y, R.cb[1], d.z * R.cb[2])) / dfw;
        const float pb = fmaf(d.x, R.cb[3], fmaf(d.y, R.cb[4], d.z * R.cb[5])) / dfw;
        const float qlo = tlo * dfw, qhi = thi * dfw;
        auto boxhit = [&](float4 lo, float4 hi) {
            if (GF_CAM_BVH)
                return lo.x <= pa && pa <= hi.x && lo.y <= pb && pb <= hi.y && hi.z >= qlo && lo.z <= qhi;
            return slab(r, lo, hi, tlo, thi);
        };
        // packet traversal: one uniform depth-first walk for the 32 rays; each lane integrates its
        // own chords as they are found (tau_total), so only colliding rays need the records again
        uint32_t ng = 0, nb = 0;
        double tau_tot = 0.0;
        auto leaf = [&](uint32_t info, bool mine) {
            const uint32_t first = info >> 8, cnt = (info >> 5) & 7u, g = info & 31u;
            for (uint32_t k = 0; k < cnt; ++k) {
                const GPrim* pp = (GF_CAM_BVH ? R.cprims : R.prims) + first + k;
                GPrim P;
                P.a = __ldg(&pp->a);
                bool pass = false;
                if (mine) {
                    if (COUNT) ++wk.tests;
                    pass = sphere_pretest(P.a, r, tlo, thi);
                }
                if (!__any_sync(FULL, pass)) continue;
                P.b = __ldg(&pp->b); P.c = __ldg(&pp->c); P.d = __ldg(&pp->d);
                Setup s;
                if (pass && prim_setup(P, r, tlo, thi, s)) {
                    if (COUNT) ++wk.hits;
                    float cj = P.d.w * s.ij;
                    if (STOCH) cj *= w[g];
                    const bool gs = s.Om == 0.0f;
                    const float amp = 0.5f * cj * __expf(-0.5f * (s.r2 + s.Om * s.Om));
                    const float4 ra = make_float4(s.u0, s.u1, s.Om, s.phi0), rb = make_float4(amp, s.j, s.tc, s.bp);
                    const float4 xc = chord_aux<COUNT>(ra, rb, !gs, wk);  // all lanes: same primitive type
                    tau_tot += (double)xc.x;
                    // resolve layout: chord t-interval, full integral, amp G(u0)
                    const float4 x = make_float4(fmaf(s.u0 - s.bp, s.ij, s.tc), fmaf(s.u1 - s.bp, s.ij, s.tc), xc.x, xc.y);
                    if (ng + nb < lcap) {
                        const uint32_t slot = gs ? ng : lcap - 1 - nb;
                        myrec[2 * slot] = ra;
                        myrec[2 * slot + 1] = rb;
                        myaux[slot] = x;
                    }
                    if (gs) ++ng; else ++nb;
                }
            }
        };
        if (__any_sync(FULL, act)) {
            int ns = 0;
            const GNode* nd0 = GF_CAM_BVH ? R.cnodes : R.nodes;
            const float4 lo = __ldg(&nd0[0].lo), hi = __ldg(&nd0[0].hi);
            const uint32_t sk = __float_as_uint(lo.w), info = __float_as_uint(hi.w);
            if (COUNT && act) ++wk.nodes;
            const bool hr = act && (node_mask(sk, info) & mask) && boxhit(lo, hi);
            if (__any_sync(FULL, hr)) {
                if (sk & kLeafBit) leaf(info, hr);
                else { stk[0] = 0; ns = 1; }
            }
            while (ns > 0) {
                const uint32_t i = stk[--ns];
                const GNode2* q = (GF_CAM_BVH ? R.cnodes2 : R.nodes2) + i;
                const float4 lo0 = __ldg(&q->lo0), hi0 = __ldg(&q->hi0), lo1 = __ldg(&q->lo1), hi1 = __ldg(&q->hi1);
                const uint32_t ref0 = __float_as_uint(lo0.w), inf0 = __float_as_uint(hi0.w);
                const uint32_t ref1 = __float_as_uint(lo1.w), inf1 = __float_as_uint(hi1.w);
                if (COUNT && act) wk.nodes += 2;
                const bool h0 = act && (node_mask(ref0, inf0) & mask) && boxhit(lo0, hi0);
                const bool h1 = act && (node_mask(ref1, inf1) & mask) && boxhit(lo1, hi1);
                const bool a0 = __any_sync(FULL, h0), a1 = __any_sync(FULL, h1);
                if (a1) {
                    if (ref1 & kLeafBit) leaf(inf1, h1);
                    else stk[ns++] = ref1;
                }
                if (a0) {
                    if (ref0 & kLeafBit) leaf(inf0, h0);
                    else stk[ns++] = ref0;
                }
                __syncwarp();
            }
        }
        if (act && ng + nb > lcap) {  // record overflow: warp-per-ray redo
            R.qO[atomicAdd(R.qcount + kCntO, 1u)] = p;
            act = false;
        }
        if (act && tau_tot < tstar) {  // escape -> environment
            R.L[p] += R.beta[p] * R.env_L;
            act = false;
        }
        __syncwarp();
        // resolve the rays one after another with the whole warp
        unsigned todo = __ballot_sync(FULL, act);
        while (todo) {
            const int l = __ffs(todo) - 1;
            todo &= todo - 1;
            const uint32_t pl = __shfl_sync(FULL, p, l);
            const float3 ol = make_float3(__shfl_sync(FULL, o.x, l), __shfl_sync(FULL, o.y, l), __shfl_sync(FULL, o.z, l));
            const float3 dl = make_float3(__shfl_sync(FULL, d.x, l), __shfl_sync(FULL, d.y, l), __shfl_sync(FULL, d.z, l));
            const float tlol = __shfl_sync(FULL, tlo, l), thil = __shfl_sync(FULL, thi, l);
            const double tsl = __shfl_sync(FULL, tstar, l);
            const uint32_t ngl = __shfl_sync(FULL, ng, l), nbl = __shfl_sync(FULL, nb, l);
            ff_resolve<COUNT, true>(R, pl, ol, dl, tlol, thil, tsl, wrec + (size_t)l * lcap * 2, waux + (size_t)l * lcap,
                                    lcap, ngl, nbl, s_h[wid], s_e[wid], wk);
            __syncwarp();
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) nray += __shfl_xor_sync(FULL, nray, off);
    if (lane == 0 && nray) atomicAdd(R.rays + 0, (unsigned long long)nray);
    if (COUNT) flush_work(R.work + kWorkSlots * STAGE_FFA, wk);
}

// ---------------------------------------------------------------- tracking estimators (a9 alternative)
// Null-collision delta tracking (free flight) and ratio tracking (NEE transmittance) against a
// per-ray piecewise-constant majorant, selected by gf_render_desc.estimator = GF_EST_TRACKING.
// The ray's hit records (the same 32-byte records k_ff writes) give both the majorant -- 64 bins
// over [t_lo, t_hi], bin k holding sum_i p_i over the chords overlapping it, p_i the bound of
// |kappa_i| on its chord, amp j sqrt(2/pi) e^{(Omega^2 - u_min^2)/2} -- and kappa(t) at a tentative
// point (one warp reduction over the records straddling t, no erf).  Unbiased where kappa >= 0.

// hit records of one ray into rec (Gaussians from the front, Gabors from the back); false if the
// ray has more than cap records
template <bool STOCH, bool COUNT>
__device__ __forceinline__ bool emit_records(const RenderDev& R, const RayDev& r, float t0, float t1, uint32_t mask,
                                             const float* w, WarpTrav& sm, float4* __restrict__ rec, uint32_t cap,
                                             uint32_t& ng, uint32_t& nb, Work& wk) {
    const unsigned FULL = 0xFFFFFFFFu;
    const unsigned lt = (1u << (threadIdx.x & 31)) - 1u;
    ng = nb = 0;
    warp_traverse<COUNT>(R.nodes, R.nodes2, R.n_nodes, R.stk_limit, r, t0, t1, mask, sm, wk,
                         [&](bool valid, uint32_t ref) {
        bool hit = false;
        Setup s;
        float cj = 0.0f;
        if (valid) {
            const GPrim* pp = R.prims + (ref & kRefIdx);
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
    });
    __syncwarp();
    return ng + nb <= cap;
}

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

// free flight by delta tracking (one warp per path; records in the k_ff buffers)
template <bool STOCH, bool COUNT>
__global__ void __launch_bounds__(128) k_ff_trk(RenderDev R, int32_t sample, int32_t depth) {
    __shared__ WarpTrav s_t[4];
    __shared__ float s_m[4][64];
    const unsigned FULL = 0xFFFFFFFFu;
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t count = R.qcount[0], cap = (uint32_t)R.rec_cap;
    float4* __restrict__ rec = R.wrec + ((size_t)blockIdx.x * 4 + wid) * cap * 2;
    float* M = s_m[wid];
    Work wk;
    uint32_t nray = 0;
    while (true) {
        uint32_t idx = 0;
        if (lane == 0) idx = atomicAdd(R.qcount + kWorkAT, 1u);
        idx = __shfl_sync(FULL, idx, 0);
        if (idx >= count) break;
        const uint32_t p = R.qA[idx];
        ++nray;
        if (COUNT && lane == 0) ++wk.paths;
        const uint32_t pix = R.pix[p];
        const float3 o = ld3(R.ox, R.oy, R.oz, p), d = ld3(R.dx, R.dy, R.dz, p);
        float w[kMaxGroups];
        const float fmx = fov_fmax<true>(R, (uint32_t)pix, (uint32_t)sample);
        const uint32_t mask = fov_mask<true>(R, fmx) & (STOCH ? policy_for(R.ext, R.sc, d, R.seed, pix, (uint32_t)sample, (uint32_t)depth,
                                                 ST_EXT, 1, w)
                                    : R.ext.static_mask);
        const RayDev r = make_ray(o, d, 0.0f, INFINITY, fmx);
        float tlo, thi;
        if (R.n_nodes == 0 || !slab_range(r, R.root_lo, R.root_hi, 0.0f, INFINITY, tlo, thi)) {
            if (lane == 0) R.L[p] += R.beta[p] * R.env_L;
            continue;
        }
        uint32_t ng, nb;
        if (!emit_records<STOCH, COUNT>(R, r, tlo, thi, mask, w, s_t[wid], rec, cap, ng, nb, wk)) {
            if (lane == 0) R.qO[atomicAdd(R.qcount + kCntO, 1u)] = p;  // analytic single-pass fallback
            continue;
        }
        majorant_bins(rec, ng, nb, cap, tlo, thi, M);
        float t = tlo;
        int k = 0;
        bool collide = false;
        for (uint32_t j = 0; j < (1u << 20); ++j) {
            const uint4 bl = stream_block(R.seed, pix, (uint32_t)sample, (uint32_t)depth, ST_TRK, 4 * j);
            if (!majorant_step(M, tlo, thi, u01(bl.x), t, k)) break;
            if (COUNT && lane == 0) ++wk.root;
            const float kap = kappa_at(rec, ng, nb, cap, t);
            if (u01(bl.y) * M[k] < kap) { collide = true; break; }  // real collision
        }
        if (lane == 0) {
            if (collide) {
                R.ox[p] = fmaf(t, d.x, o.x);
                R.oy[p] = fmaf(t, d.y, o.y);
                R.oz[p] = fmaf(t, d.z, o.z);
                R.qB[atomicAdd(R.qcount + 1, 1u)] = p;
            } else {
                R.L[p] += R.beta[p] * R.env_L;  // escape -> environment
            }
        }
        __syncwarp();
    }
    if (lane == 0 && nray) atomicAdd(R.rays + 0, (unsigned long long)nray);
    if (COUNT) flush_work(R.work + kWorkSlots * STAGE_FFA, wk);
}

// NEE with ratio tracking: T = prod_j (1 - kappa(t_j) / M(t_j)) over the tentative points
template <bool STOCH, bool COUNT>
__global__ void __launch_bounds__(128) k_nee_rt(RenderDev R, int32_t sample, int32_t depth) {
    __shared__ WarpTrav s_t[4];
    __shared__ WarpEnd s_e[4];
    __shared__ float s_m[4][64];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t count = R.qcount[1], cap = (uint32_t)R.rec_cap;
    float4* __restrict__ rec = R.wrec + ((size_t)blockIdx.x * 4 + wid) * cap * 2;
    float* M = s_m[wid];
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
        const float fmx = fov_fmax<true>(R, (uint32_t)pix, (uint32_t)sample);
        const uint32_t mask = fov_mask<true>(R, fmx) & (STOCH ? policy_for(R.nee, R.sc, R.sun, R.seed, pix, (uint32_t)sample, (uint32_t)depth,
                                                 ST_NEE, 0, w)
                                    : R.nee.static_mask);
        const RayDev r = make_ray(x, R.sun, 0.0f, INFINITY, fmx);
        float T = 1.0f, tlo, thi;
        if (R.n_nodes > 0 && slab_range(r, R.root_lo, R.root_hi, 0.0f, INFINITY, tlo, thi)) {
            uint32_t ng, nb;
            if (emit_records<STOCH, COUNT>(R, r, tlo, thi, mask, w, s_t[wid], rec, cap, ng, nb, wk)) {
                majorant_bins(rec, ng, nb, cap, tlo, thi, M);
                float t = tlo;
                int k = 0;
                for (uint32_t j = 0; j < (1u << 20); ++j) {
                    const uint4 bl = stream_block(R.seed, pix, (uint32_t)sample, (uint32_t)depth, ST_TRK_NEE, 4 * j);
                    if (!majorant_step(M, tlo, thi, u01(bl.x), t, k)) break;
                    if (COUNT && lane == 0) ++wk.root;
                    T *= 1.0f - kappa_at(rec, ng, nb, cap, t) / M[k];
                }
            } else {  // more records than the buffer: closed-form transmittance
                T = (float)exp(-warp_tau<STOCH, COUNT>(R.nodes, R.nodes2, R.n_nodes, R.stk_limit, R.prims, r, 0.0f,
                                                       INFINITY, mask, w, s_t[wid], s_e[wid], wk));
            }
        }
        if (lane == 0) {
            const float3 d = ld3(R.dx, R.dy, R.dz, p);
            const float beta = R.beta[p];
            const float cost = d.x * R.sun.x + d.y * R.sun.y + d.z * R.sun.z;
            R.L[p] += beta * R.albedo * hg_eval(R.hg_g, cost) * T * R.sun_E;
            if (depth + 1 < R.max_depth) {
                uint4 b = stream_block(R.seed, pix, (uint32_t)sample, (uint32_t)depth, ST_SCAT, 0);
                float3 nd = hg_sample(R.hg_g, d, u01(b.x), u01(b.y));
                R.dx[p] = nd.x; R.dy[p] = nd.y; R.dz[p] = nd.z;
                R.beta[p] = beta * R.albedo;
                R.qNext[atomicAdd(R.qcount + 2, 1u)] = p;
            }
        }
        __syncwarp();
    }
    if (lane == 0 && nray) atomicAdd(R.rays + 1, (unsigned long long)nray);
    if (COUNT) flush_work(R.work + kWorkSlots * STAGE_NEE, wk);
}

// NEE, one warp per path (warp_tau): shadow-ray transmittance, HG phase sampling of the next
// direction.  Replaces the per-lane k_nee on the production path.
// LIGHT: traverse the light BVH (boxes in a frame whose third axis is the light direction, built
// per gf_render call by gf_launch_build_frame): the shadow ray is axis-parallel there, so a box test
// is two interval tests and one compare, and the boxes are tight across the rays' direction.
template <bool STOCH, bool COUNT, bool LIGHT, bool FOV>
__global__ void __launch_bounds__(128) k_nee_w(RenderDev R, int32_t sample, int32_t depth) {
    __shared__ WarpTrav s_t[4];
    __shared__ WarpEnd s_e[4];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t count = R.qcount[1];
    const int lstk = LIGHT ? max(1, kWStk - 34 - (int)*R.ldepth) : 0;
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
        const float fmx = fov_fmax<FOV>(R, (uint32_t)pix, (uint32_t)sample);
        const uint32_t mask = fov_mask<FOV>(R, fmx) & (STOCH ? policy_for(R.nee, R.sc, R.sun, R.seed, pix, (uint32_t)sample, (uint32_t)depth,
                                                 ST_NEE, 0, w)
                                    : R.nee.static_mask);
        double tau;
        if (LIGHT) {
            const float3 xp = make_float3(fmaf(R.lf[0], x.x, fmaf(R.lf[1], x.y, R.lf[2] * x.z)),
                                          fmaf(R.lf[3], x.x, fmaf(R.lf[4], x.y, R.lf[5] * x.z)),
                                          fmaf(R.lf[6], x.x, fmaf(R.lf[7], x.y, R.lf[8] * x.z)));
            tau = warp_tau_b<STOCH, COUNT>(R.lnodes, R.lnodes2, R.n_nodes, lstk, R.lprims,
                                           make_ray(x, R.sun, 0.0f, INFINITY, fmx), 0.0f, INFINITY, mask, w, s_t[wid],
                                           s_e[wid], wk, [&](float4 lo, float4 hi) {
                                               return lo.x <= xp.x && xp.x <= hi.x && lo.y <= xp.y && xp.y <= hi.y &&
                                                      hi.z >= xp.z;
                                           });
        } else {
            tau = warp_tau<STOCH, COUNT>(R.nodes, R.nodes2, R.n_nodes, R.stk_limit, R.prims,
                                         make_ray(x, R.sun, 0.0f, INFINITY, fmx), 0.0f, INFINITY, mask, w, s_t[wid],
                                         s_e[wid], wk);
        }
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
template <bool STOCH, bool COUNT, bool FOV>
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
        mb_shift(R, (uint32_t)pix, (uint32_t)sample, o);
        float w[kMaxGroups];
        const float fmx = fov_fmax<FOV>(R, (uint32_t)pix, (uint32_t)sample);
        const uint32_t mask = fov_mask<FOV>(R, fmx) & (STOCH ? policy_for(R.ext, R.sc, d, R.seed, (uint32_t)pix, (uint32_t)sample, 0, ST_EXT, 1, w)
                                    : R.ext.static_mask);
        if (COUNT && lane == 0) ++wk.paths;
        ++nray;
        const double tau = warp_tau<STOCH, COUNT>(R.nodes, R.nodes2, R.n_nodes, R.stk_limit, R.prims,
                                                  make_ray(o, d, 0.0f, INFINITY, fmx), 0.0f, INFINITY, mask, w, s_t[wid],
                                                  s_e[wid], wk);
        if (lane == 0) R.L[p] = (float)tau;
    }
    if (lane == 0 && nray) atomicAdd(R.rays + 0, (unsigned long long)nray);
    if (COUNT) flush_work(R.work + kWorkSlots * STAGE_TOMO, wk);
}

// Tomography of coherent camera rays (static mask, no foveation / motion blur): the packet walk of
// k_ff_pkt over the camera BVH for 32 consecutive pixels (one 8x4 block), each lane integrating its
// own hits lane-locally (seg_J; all lanes test the same primitive, so the erf type is uniform).
#ifndef GF_TOMO_MINB
#define GF_TOMO_MINB 8  // 64 registers, 8 blocks per SM: +12-15 % over 80 registers (cfg2 / cfg5 --tomography)
#endif
template <bool COUNT>
__global__ void __launch_bounds__(128, GF_TOMO_MINB) k_tomo_pkt(RenderDev R, int32_t sample) {
    __shared__ uint32_t s_stk[4][kPStk];
    const unsigned FULL = 0xFFFFFFFFu;
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t* stk = s_stk[wid];
    const uint32_t mask = R.ext.static_mask;
    Work wk;
    uint32_t nray = 0;
    for (int64_t base = ((int64_t)blockIdx.x * 4 + wid) * 32; base < R.n_paths; base += (int64_t)gridDim.x * 128) {
        const int64_t p = base + lane;
        const int32_t pix = p < R.n_paths ? path_pixel(R, p) : -1;
        const bool act0 = pix >= 0;
        float3 o = make_float3(0.0f, 0.0f, 0.0f), d = make_float3(0.0f, 0.0f, 1.0f);
        if (act0) {
            float jx = 0.5f, jy = 0.5f;
            if (R.jitter) {
                uint4 b = stream_block(R.seed, (uint32_t)pix, (uint32_t)sample, 0, ST_CAM, 0);
                jx = u01(b.x); jy = u01(b.y);
            }
            camera_ray(R.cam, pix % R.cam.W, pix / R.cam.W, jx, jy, o, d);
            ++nray;
            if (COUNT) ++wk.paths;
        }
        const RayDev r = make_ray(o, d, 0.0f, INFINITY);
        float tlo = 0.0f, thi = 0.0f;
        const bool act = act0 && R.n_nodes > 0 && slab_range(r, R.root_lo, R.root_hi, 0.0f, INFINITY, tlo, thi);
        const float dfw = fmaf(d.x, R.cb[6], fmaf(d.y, R.cb[7], d.z * R.cb[8]));
        const float pa = fmaf(d.x, R.cb[0], fmaf(d.y, R.cb[1], d.z * R.cb[2])) / dfw;
        const float pb = fmaf(d.x, R.cb[3], fmaf(d.y, R.cb[4], d.z * R.cb[5])) / dfw;
        const float qlo = tlo * dfw, qhi = thi * dfw;
        auto boxhit = [&](float4 lo, float4 hi) {
            return lo.x <= pa && pa <= hi.x && lo.y <= pb && pb <= hi.y && hi.z >= qlo && lo.z <= qhi;
        };
        double tau = 0.0;
        auto leaf = [&](uint32_t info, bool mine) {
            const uint32_t first = info >> 8, cnt = (info >> 5) & 7u;
            for (uint32_t k = 0; k < cnt; ++k) {
                const GPrim* pp = R.cprims + first + k;
                GPrim P;
                P.a = __ldg(&pp->a);
                bool pass = false;
                if (mine) {
                    if (COUNT) ++wk.tests;
                    pass = sphere_pretest(P.a, r, tlo, thi);
                }
                if (!__any_sync(FULL, pass)) continue;
                P.b = __ldg(&pp->b); P.c = __ldg(&pp->c); P.d = __ldg(&pp->d);
                Setup s;
                if (pass && prim_setup(P, r, tlo, thi, s)) {
                    if (COUNT) ++wk.hits;
                    tau += (double)(P.d.w * s.ij * seg_J(s, s.u0, s.u1, wk));
                }
            }
        };
        if (__any_sync(FULL, act)) {
            int ns = 0;
            const float4 lo = __ldg(&R.cnodes[0].lo), hi = __ldg(&R.cnodes[0].hi);
            const uint32_t sk = __float_as_uint(lo.w), info = __float_as_uint(hi.w);
            if (COUNT && act) ++wk.nodes;
            const bool hr = act && (node_mask(sk, info) & mask) && boxhit(lo, hi);
            if (__any_sync(FULL, hr)) {
                if (sk & kLeafBit) leaf(info, hr);
                else { stk[0] = 0; ns = 1; }
            }
            while (ns > 0) {
                const uint32_t i = stk[--ns];
                const GNode2* q = R.cnodes2 + i;
                const float4 lo0 = __ldg(&q->lo0), hi0 = __ldg(&q->hi0), lo1 = __ldg(&q->lo1), hi1 = __ldg(&q->hi1);
                const uint32_t ref0 = __float_as_uint(lo0.w), inf0 = __float_as_uint(hi0.w);
                const uint32_t ref1 = __float_as_uint(lo1.w), inf1 = __float_as_uint(hi1.w);
                if (COUNT && act) wk.nodes += 2;
                const bool h0 = act && (node_mask(ref0, inf0) & mask) && boxhit(lo0, hi0);
                const bool h1 = act && (node_mask(ref1, inf1) & mask) && boxhit(lo1, hi1);
                const bool a0 = __any_sync(FULL, h0), a1 = __any_sync(FULL, h1);
                if (a1) {
                    if (ref1 & kLeafBit) leaf(inf1, h1);
                    else stk[ns++] = ref1;
                }
                if (a0) {
                    if (ref0 & kLeafBit) leaf(inf0, h0);
                    else stk[ns++] = ref0;
                }
                __syncwarp();
            }
        }
        if (act0) R.L[p] = (float)tau;
        __syncwarp();
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) nray += __shfl_xor_sync(FULL, nray, off);
    if (lane == 0 && nray) atomicAdd(R.rays + 0, (unsigned long long)nray);
    if (COUNT) flush_work(R.work + kWorkSlots * STAGE_TOMO, wk);
}

__global__ void k_rotate(uint32_t* qc) {
    qc[0] = qc[2];
    qc[1] = 0; qc[2] = 0;
    qc[kWorkA] = 0; qc[kWorkB] = 0; qc[kWorkN] = 0;
    qc[kCntO] = 0; qc[kWorkAT] = 0; qc[kWorkAO] = 0; qc[kCntB2] = 0; qc[kWorkRO] = 0; qc[kCntO2] = 0;
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

// persistent grid: 16 blocks of 128 threads per SM (the kernels' occupancy is <= 8 resident)
static int persist_blocks() {
    static int b = 0;
    if (!b) {
        int dev = 0, sms = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        b = (sms > 0 ? sms : 148) * 16;
    }
    return b;
}

// k_ff runs one resident wave (its 26 KB of shared memory per block allow <= 8 blocks per SM), so
// record buffers exist for sms x 8 blocks x 4 warps at most
static int ff_max_blocks() { return persist_blocks() / 2; }
template <bool S, bool C>
static unsigned ff_grid(int64_t n_paths) {
    static int occ = 0;
    if (!occ) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_ff<S, C, false, false>, 128, 0);
        occ = std::max(1, std::min(occ, 8));
    }
    const int64_t blocks = (int64_t)(persist_blocks() / 16) * occ;
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(blocks, (n_paths + 3) / 4));
}

size_t gf_render_state_bytes(int64_t n, int64_t n_prims, char* base, RenderDev* R, BuildScratch* LS) {
    size_t off = 0;
    auto take = [&](size_t bytes) { char* p = base ? base + off : nullptr; off += (bytes + 255) & ~(size_t)255; return p; };
    const size_t nf = sizeof(float) * (size_t)n, nu = sizeof(uint32_t) * (size_t)n;
    float* ox = (float*)take(nf); float* oy = (float*)take(nf); float* oz = (float*)take(nf);
    float* dx = (float*)take(nf); float* dy = (float*)take(nf); float* dz = (float*)take(nf);
    float* beta = (float*)take(nf); float* L = (float*)take(nf);
    double* cum = (double*)take(sizeof(double) * 3 * (size_t)n);
    int32_t* bin = (int32_t*)take(nu); uint32_t* pix = (uint32_t*)take(nu); uint32_t* nhit = (uint32_t*)take(nu);
    uint2* hits = (uint2*)take(sizeof(uint2) * (size_t)kHitCap * (size_t)n);
    const size_t nw = (size_t)4 * (size_t)std::max<int64_t>(1, std::min<int64_t>((int64_t)ff_max_blocks(), (n + 3) / 4));
    float4* wrec = (float4*)take(sizeof(float4) * 2 * (size_t)kRecCap * nw);
    float4* waux = (float4*)take(sizeof(float4) * (size_t)kRecCap * nw);
    uint32_t* qA = (uint32_t*)take(nu); uint32_t* qB = (uint32_t*)take(nu); uint32_t* qN = (uint32_t*)take(nu);
    uint32_t* qO = (uint32_t*)take(nu); uint32_t* qB2 = (uint32_t*)take(nu); uint32_t* qO2 = (uint32_t*)take(nu);
    uint32_t* qc = (uint32_t*)take(sizeof(uint32_t) * 16);
    // light BVH (NEE): nodes, child pairs, primitives in its leaf order, permutation, depth, build scratch
    const size_t np1 = (size_t)std::max<int64_t>(n_prims, 1);
    GNode* lnodes = (GNode*)take(sizeof(GNode) * 2 * np1);
    GNode2* lnodes2 = (GNode2*)take(sizeof(GNode2) * 2 * np1);
    GPrim* lprims = (GPrim*)take(sizeof(GPrim) * np1);
    int32_t* lperm = (int32_t*)take(sizeof(int32_t) * np1);
    uint32_t* ldepth = (uint32_t*)take(sizeof(uint32_t) * 4);
    GNode* cnodes = (GNode*)take(sizeof(GNode) * 2 * np1);  // camera BVH (depth-0 packets)
    GNode2* cnodes2 = (GNode2*)take(sizeof(GNode2) * 2 * np1);
    GPrim* cprims = (GPrim*)take(sizeof(GPrim) * np1);
    int32_t* cperm = (int32_t*)take(sizeof(int32_t) * np1);
    uint32_t* cdepth = (uint32_t*)take(sizeof(uint32_t) * 4);
    const size_t lsb = gf_scratch_layout(n_prims, nullptr).total_bytes;
    char* lscratch = (char*)take(lsb);
    if (LS) *LS = gf_scratch_layout(n_prims, lscratch);
    if (R) {
        R->ox = ox; R->oy = oy; R->oz = oz; R->dx = dx; R->dy = dy; R->dz = dz; R->beta = beta; R->L = L;
        R->cum = cum; R->bin = bin; R->pix = pix; R->nhit = nhit; R->hits = hits; R->hit_cap = kHitCap;
        R->wrec = wrec; R->waux = waux; R->rec_cap = kRecCap;
        R->qA = qA; R->qB = qB; R->qNext = qN; R->qO = qO; R->qB2 = qB2; R->qO2 = qO2; R->qcount = qc;
        R->lnodes = lnodes; R->lnodes2 = lnodes2; R->lprims = lprims; R->lperm = lperm; R->ldepth = ldepth;
        R->cnodes = cnodes; R->cnodes2 = cnodes2; R->cprims = cprims; R->cperm = cperm; R->cdepth = cdepth;
    }
    return off;
}


template <bool S, bool C>
static void launch_ff(RenderDev& R, int32_t sample, int d, bool cam, const uint32_t* q_in, int cnt_slot, int cur_slot,
                      uint32_t* q_over, int over_slot, cudaStream_t st) {
    const unsigned g = ff_grid<S, C>(R.n_paths);
    if (R.fov) {
        if (cam) k_ff<S, C, true, true><<<g, 128, 0, st>>>(R, sample, d, q_in, cnt_slot, cur_slot, q_over, over_slot);
        else k_ff<S, C, false, true><<<g, 128, 0, st>>>(R, sample, d, q_in, cnt_slot, cur_slot, q_over, over_slot);
    } else {
        if (cam) k_ff<S, C, true, false><<<g, 128, 0, st>>>(R, sample, d, q_in, cnt_slot, cur_slot, q_over, over_slot);
        else k_ff<S, C, false, false><<<g, 128, 0, st>>>(R, sample, d, q_in, cnt_slot, cur_slot, q_over, over_slot);
    }
}

template <bool S, bool C>
static void launch_depth(RenderDev& R, int32_t sample, int d, unsigned pgrid, unsigned wgrid, cudaStream_t st,
                         StageTimer& T,
                         bool stoch_nee) {
    cudaEvent_t e;
    // coherent camera rays under one static mask: packet traversal
    const bool packet = GF_PACKET && d == 0 && !S && R.estimator == 0 && R.camb;  // (k_ff_pkt needs the camera BVH)
    T.pre(STAGE_FFA, st, e);
    if (R.estimator == 1) k_ff_trk<S, C><<<ff_grid<S, C>(R.n_paths), 128, 0, st>>>(R, sample, d);
    else if (packet) {
        if (R.fov) k_ff_pkt<S, C, true><<<ff_grid<S, C>(R.n_paths), 128, 0, st>>>(R, sample, d);
        else k_ff_pkt<S, C, false><<<ff_grid<S, C>(R.n_paths), 128, 0, st>>>(R, sample, d);
    } else {
        launch_ff<S, C>(R, sample, d, d == 0 && R.camb, R.qA, 0, kWorkAT, R.qO, kCntO, st);
    }
    T.post(STAGE_FFA, st, e);
    if (packet) {  // rays with more records than a packet lane holds: warp-per-ray k_ff (larger buffer),
        T.pre(STAGE_FFB, st, e);  // timed with the fallbacks (stage "ff_fallback")
        launch_ff<S, C>(R, sample, d, R.camb, R.qO, kCntO, kWorkRO, R.qO2, kCntO2, st);
        T.post(STAGE_FFB, st, e);
    }
    T.pre(STAGE_FFB, st, e);  // record-overflow paths: single-pass kernels (stage "ffB")
    if (packet) k_ffA<S, C><<<pgrid, 128, 0, st>>>(R, sample, d, R.qO2, kCntO2, kWorkAO, 0);
    else k_ffA<S, C><<<pgrid, 128, 0, st>>>(R, sample, d, R.qO, kCntO, kWorkAO, 0);
    T.post(STAGE_FFB, st, e);
    T.pre(STAGE_FFB, st, e);  // record-overflow paths (appended to qB for NEE)
    k_ffB<S, C><<<pgrid, 128, 0, st>>>(R, sample, d);
    T.post(STAGE_FFB, st, e);
    T.pre(STAGE_NEE, st, e);
    if (R.estimator == 1) {  // ratio tracking uses the k_ff record buffers (same grid)
        if (stoch_nee) k_nee_rt<true, C><<<ff_grid<S, C>(R.n_paths), 128, 0, st>>>(R, sample, d);
        else k_nee_rt<false, C><<<ff_grid<S, C>(R.n_paths), 128, 0, st>>>(R, sample, d);
    } else {
#define GF_NEE(SN, L, F) k_nee_w<SN, C, L, F><<<wgrid, 128, 0, st>>>(R, sample, d)
        if (R.fov) {
            if (R.light) { if (stoch_nee) GF_NEE(true, true, true); else GF_NEE(false, true, true); }
            else { if (stoch_nee) GF_NEE(true, false, true); else GF_NEE(false, false, true); }
        } else {
            if (R.light) { if (stoch_nee) GF_NEE(true, true, false); else GF_NEE(false, true, false); }
            else { if (stoch_nee) GF_NEE(true, false, false); else GF_NEE(false, false, false); }
        }
#undef GF_NEE
    }
    T.post(STAGE_NEE, st, e);
}

cudaError_t gf_launch_render_pass(RenderDev& R, int32_t sample, int32_t slot, cudaStream_t st, StageTimer& T) {
    cudaError_t e;
    if (R.n_paths == 0) return cudaSuccess;
    const bool cnt = R.work != nullptr;
    const bool stoch_ext = !(R.ext.ls == 0 && R.ext.os == 0);
    const bool stoch_nee = !(R.nee.ls == 0 && R.nee.os == 0);
    const unsigned grid = (unsigned)((R.n_paths + 127) / 128);
    const unsigned pgrid = (unsigned)std::min<int64_t>((int64_t)persist_blocks(), (R.n_paths + 127) / 128);
    const unsigned wgrid = (unsigned)std::min<int64_t>((int64_t)persist_blocks(), (R.n_paths + 3) / 4);  // warp/path
    if ((e = cudaMemsetAsync(R.qcount, 0, sizeof(uint32_t) * 16, st))) return e;
    cudaEvent_t ev;
    if (R.mode == 0) {
        T.pre(STAGE_TOMO, st, ev);
#define GF_TOMO(S_, C_, F_) k_tomo_w<S_, C_, F_><<<wgrid, 128, 0, st>>>(R, sample)
        if (R.camb && !stoch_ext && !R.fov && GF_PACKET && R.n_paths >= R.tomo_pkt_min) {  // coherent camera rays: packets
            const unsigned tg = (unsigned)std::min<int64_t>((int64_t)persist_blocks(), (R.n_paths + 127) / 128);
            if (cnt) k_tomo_pkt<true><<<tg, 128, 0, st>>>(R, sample);
            else k_tomo_pkt<false><<<tg, 128, 0, st>>>(R, sample);
        } else if (R.fov) {
            if (stoch_ext) { if (cnt) GF_TOMO(true, true, true); else GF_TOMO(true, false, true); }
            else { if (cnt) GF_TOMO(false, true, true); else GF_TOMO(false, false, true); }
        } else {
            if (stoch_ext) { if (cnt) GF_TOMO(true, true, false); else GF_TOMO(true, false, false); }
            else { if (cnt) GF_TOMO(false, true, false); else GF_TOMO(false, false, false); }
        }
#undef GF_TOMO
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
