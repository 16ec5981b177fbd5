// gf_ffb.cu -- a8 free flight, pass B (the root of tau(t) = tau* inside the first-crossing bin)
// and the selectable delta / ratio tracking estimators.
#include <algorithm>

#include "gf_render.cuh"

namespace gfk {

// Records of the chords of a window [a, b] (clipped to it) into the warp's buffer and their chord data
// (chord_aux); returns false if they exceed the buffer; *tot = tau over the window (whole warp).
template <bool STOCH, bool COUNT, bool CAM>
__device__ __forceinline__ bool window_records(const RenderDev& R, const FFRay& f, const RayDev& r, const CamPt& cp,
                                               float a, float b, WarpTrav& sm, float4* __restrict__ rec,
                                               float4* __restrict__ aux, uint32_t cap, uint32_t& ng, uint32_t& nb,
                                               double* tot, Work& wk) {
    const GNode* __restrict__ nodes = CAM ? R.cnodes : R.nodes;
    const GNode2* __restrict__ nodes2 = CAM ? R.cnodes2 : R.nodes2;
    const GPrim* __restrict__ prims = CAM ? R.cprims : R.prims;
    const int stk_limit = CAM ? max(1, kWStk - 34 - (int)*R.cdepth) : R.stk_limit;
    const int lane = threadIdx.x & 31;
    emit_records_b<STOCH, COUNT>(nodes, nodes2, R.n_nodes, stk_limit, prims, r, a, b, f.mask, f.w, sm, rec, cap, ng, nb,
                                 wk, [&](float4 lo, float4 hi) { return ff_box<CAM>(r, cp, lo, hi, a, b); });
    if (ng + nb > cap) return false;
    const uint32_t nside[2] = {ng, nb};
    float acc = 0.0f;
#pragma unroll 1
    for (int side = 0; side < 2; ++side)
        for (uint32_t i = lane; i < nside[side]; i += 32) {
            const uint32_t slot = side == 0 ? i : cap - 1 - i;
            const float4 x = chord_aux<COUNT>(rec[2 * slot], rec[2 * slot + 1], side == 1, wk);
            aux[slot] = x;
            acc += x.x;
        }
    double t = acc;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xFFFFFFFFu, t, o);
    *tot = t;
    __syncwarp();
    return true;
}

// k_ffb_w: one warp per path of queue qW (pass A found a coarse bin that may hold the first crossing):
// the coarse bins s0 .. k1 are re-traversed -- the world BVH, or the camera BVH for depth-0 rays (CAM) --
// emitting the records of the chords inside them, clipped to them, into the warp's buffer; then the
// fine search and the root (resolve_records).  Windows with more chords than the buffer holds are
// taken coarse bin by coarse bin, then fine bin by fine bin (exact tau of each by warp_tau), and the
// crossing fine bin is halved by the exact tau of its left half until its records fit.
// Overflow path of k_ffb_w (rare, out of line so that the common path keeps its registers): the coarse
// bins s0 .. kend one by one; a coarse bin still too full fine bin by fine bin (exact tau of each by
// warp_tau), the crossing fine bin halved by the exact tau of its left half until its records fit.
template <bool STOCH, bool COUNT, bool CAM>
__device__ __forceinline__ bool ffb_overflow(const RenderDev& R, const FFRay& f, const RayDev& r, const CamPt& cp, int s0,
                                          int kend, double cstart, WarpTrav& sm, WarpEnd& q, float* cf, uint16_t* wl,
                                          float4* __restrict__ rec, float4* __restrict__ aux, uint32_t cap, Work& wk,
                                          float& t) {
    const GNode* __restrict__ nodes = CAM ? R.cnodes : R.nodes;
    const GNode2* __restrict__ nodes2 = CAM ? R.cnodes2 : R.nodes2;
    const GPrim* __restrict__ prims = CAM ? R.cprims : R.prims;
    const int stk_limit = CAM ? max(1, kWStk - 34 - (int)*R.cdepth) : R.stk_limit;
    auto tau_over = [&](float a, float b) {
        return warp_tau_b<STOCH, COUNT>(nodes, nodes2, R.n_nodes, stk_limit, prims, r, a, b, f.mask, f.w, sm, q, wk,
                                        [&](float4 lo, float4 hi) { return ff_box<CAM>(r, cp, lo, hi, a, b); });
    };
    uint32_t ng = 0, nb = 0;
    double tot = 0.0, cum = cstart;
    for (int m = s0; m <= kend; ++m) {
        if (window_records<STOCH, COUNT, CAM>(R, f, r, cp, ff_edge(f, m - 1), ff_edge(f, m), sm, rec, aux, cap, ng, nb,
                                              &tot, wk)) {
            if (resolve_records<COUNT>(rec, aux, cap, ng, nb, f, m, m, cum, cf, wl, q, wk, t, true)) return true;
            cum += tot;
            continue;
        }
        const Bins FB = fine_bins(f, m);
        for (int j = 0; j < kNF; ++j) {
            float a = FB.edge(j - 1), b = FB.edge(j);
            const double tj = tau_over(a, b);
            if (cum + tj < f.tstar) {
                cum += tj;
                continue;
            }
            double c0 = cum;  // the first crossing fine bin: halve until its records fit
            for (int split = 0; split < 24; ++split) {
                if (window_records<STOCH, COUNT, CAM>(R, f, r, cp, a, b, sm, rec, aux, cap, ng, nb, &tot, wk)) break;
                const float mid = 0.5f * (a + b);
                const double tl = tau_over(a, mid);
                if (c0 + tl >= f.tstar) b = mid;
                else { c0 += tl; a = mid; }
            }
            if (ng + nb > cap) ng = nb = 0;  // (24 halvings: below 1e-7 of the bin) the window's midpoint
            t = window_root<COUNT>(rec, aux, cap, ng, nb, a, b, c0, f.tstar, wl, q, wk);
            return true;
        }
    }
    return false;
}

template <bool STOCH, bool COUNT, bool FOV, bool CAM>
#ifndef GF_MINB_FFB
#define GF_MINB_FFB 8  // 64 registers, 8 blocks per SM: ffB -2..-4 % against 72 registers / 7 blocks (cfg4, cfg5)
#endif
__global__ void __launch_bounds__(128, GF_MINB_FFB) k_ffb_w(RenderDev R, int32_t sample, int32_t depth, const uint32_t* __restrict__ q_in,
                                               int cnt_slot, int cur_slot) {
    __shared__ WarpTrav s_t[4];
    __shared__ WarpEnd s_e[4];
    __shared__ float s_f[4][kNF * 32];
    __shared__ uint16_t s_w[4][kWinCap];
    const unsigned FULL = 0xFFFFFFFFu;
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t count = R.qcount[cnt_slot], cap = (uint32_t)R.rec_cap;
    const size_t gw = (size_t)blockIdx.x * 4 + wid;
    float4* __restrict__ rec = R.wrec + gw * cap * 2;
    float4* __restrict__ aux = R.waux + gw * cap;
    Work wk;
    while (true) {
        uint32_t idx = 0;
        if (lane == 0) idx = atomicAdd(R.qcount + cur_slot, 1u);
        idx = __shfl_sync(FULL, idx, 0);
        if (idx >= count) break;
        const uint32_t p = q_in[idx];
        FFRay f;
        ff_begin<STOCH, FOV>(R, p, sample, depth, f);  // the same set-up as pass A
        f.mask &= R.ffg[p];  // only the groups with chords in the window (pass A): other subtrees pruned at the top
        const int ks = R.ffk[p], k1 = ks & 0xFF, s0 = ks >> 8, kend = k1 < kNC ? k1 : kNC - 1;
        const double cstart = R.ffc[p];
        const RayDev r = make_ray(f.o, f.d, 0.0f, INFINITY, fov_prim(R, f.fth));
        const CamPt cp = cam_point(R, f.d);
        uint32_t ng = 0, nb = 0;
        double tot = 0.0;
        float t = 0.0f, kap = 0.0f;
        bool col = false;
        if (window_records<STOCH, COUNT, CAM>(R, f, r, cp, ff_edge(f, s0 - 1), ff_edge(f, kend), s_t[wid], rec, aux, cap,
                                              ng, nb, &tot, wk)) {
            col = resolve_records<COUNT>(rec, aux, cap, ng, nb, f, s0, kend, cstart, s_f[wid], s_w[wid], s_e[wid], wk, t,
                                         true, &kap, tot);
        } else {  // more chords than the buffer holds: k_ffb_over (queue qV)
            if (lane == 0) {
                if (COUNT) ++wk.overflow;
                R.qV[atomicAdd(R.qcount + QC_V, 1u)] = p;
            }
            continue;
        }
        if (lane == 0) {
            if (col) {
                ff_collide(R, p, f, t, kap);
                R.qB[atomicAdd(R.qcount + QC_B, 1u)] = p;
            } else {
                ff_escape(R, p);  // no fine edge reached tau* (a coarse bin's bound only)
            }
        }
        __syncwarp();
    }
    if (COUNT) flush_work(R.work + kWorkSlots * STAGE_FFB, wk);
}
template <bool STOCH, bool COUNT, bool FOV, bool CAM>
__global__ void __launch_bounds__(128) k_ffb_over(RenderDev R, int32_t sample, int32_t depth) {
    __shared__ WarpTrav s_t[4];
    __shared__ WarpEnd s_e[4];
    __shared__ float s_f[4][kNF * 32];
    __shared__ uint16_t s_w[4][kWinCap];
    const unsigned FULL = 0xFFFFFFFFu;
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t count = R.qcount[QC_V], cap = (uint32_t)R.rec_cap;
    const size_t gw = (size_t)blockIdx.x * 4 + wid;
    float4* __restrict__ rec = R.wrec + gw * cap * 2;
    float4* __restrict__ aux = R.waux + gw * cap;
    Work wk;
    while (true) {
        uint32_t idx = 0;
        if (lane == 0) idx = atomicAdd(R.qcount + CUR_V, 1u);
        idx = __shfl_sync(FULL, idx, 0);
        if (idx >= count) break;
        const uint32_t p = R.qV[idx];
        FFRay f;
        ff_begin<STOCH, FOV>(R, p, sample, depth, f);
        f.mask &= R.ffg[p];
        const int ks = R.ffk[p], k1 = ks & 0xFF, s0 = ks >> 8, kend = k1 < kNC ? k1 : kNC - 1;
        const RayDev r = make_ray(f.o, f.d, 0.0f, INFINITY, fov_prim(R, f.fth));
        const CamPt cp = cam_point(R, f.d);
        float t = 0.0f;
        const bool col = ffb_overflow<STOCH, COUNT, CAM>(R, f, r, cp, s0, kend, R.ffc[p], s_t[wid], s_e[wid], s_f[wid],
                                                         s_w[wid], rec, aux, cap, wk, t);
        if (lane == 0) {
            if (col) {
                ff_collide(R, p, f, t);
                R.qB[atomicAdd(R.qcount + QC_B, 1u)] = p;
            } else {
                ff_escape(R, p);
            }
        }
        __syncwarp();
    }
    if (COUNT) flush_work(R.work + kWorkSlots * STAGE_FFB, wk);
}

// free flight by delta tracking (one warp per path; records in the k_ff buffers)
template <bool STOCH, bool COUNT>
__global__ void __launch_bounds__(128) k_ff_trk(RenderDev R, int32_t sample, int32_t depth) {
    __shared__ WarpTrav s_t[4];
    __shared__ float s_m[4][64];
    const unsigned FULL = 0xFFFFFFFFu;
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t count = R.qcount[QC_A], cap = (uint32_t)R.rec_cap;
    float4* __restrict__ rec = R.wrec + ((size_t)blockIdx.x * 4 + wid) * cap * 2;
    float* M = s_m[wid];
    Work wk;
    uint32_t nray = 0;
    while (true) {
        uint32_t idx = 0;
        if (lane == 0) idx = atomicAdd(R.qcount + CUR_A, 1u);
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
        const RayDev r = make_ray(o, d, 0.0f, INFINITY, fov_prim(R, fmx));
        float tlo, thi;
        if (R.n_nodes == 0 || !slab_range(r, R.root_lo, R.root_hi, 0.0f, INFINITY, tlo, thi)) {
            if (lane == 0) R.L[p] += R.beta[p] * R.env_L;
            continue;
        }
        uint32_t ng, nb;
        emit_records_b<STOCH, COUNT>(R.nodes, R.nodes2, R.n_nodes, R.stk_limit, R.prims, r, tlo, thi, mask, w, s_t[wid],
                                     rec, cap, ng, nb, wk, [&](float4 lo, float4 hi) { return slab(r, lo, hi, tlo, thi); });
        if (ng + nb > cap) {  // more chords than the buffer: the analytic free flight (passes A + B)
            if (lane == 0) R.qO[atomicAdd(R.qcount + QC_O, 1u)] = p;
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
                R.qB[atomicAdd(R.qcount + QC_B, 1u)] = p;
            } else {
                R.L[p] += R.beta[p] * R.env_L;  // escape -> environment
            }
        }
        __syncwarp();
    }
    if (lane == 0 && nray) atomicAdd(R.rays + (depth == 0 ? 0 : 1), (unsigned long long)nray);
    if (COUNT) flush_work(R.work + kWorkSlots * STAGE_FFA, wk);
}

// NEE with ratio tracking: T = prod_j (1 - kappa(t_j) / M(t_j)) over the tentative points
template <bool STOCH, bool COUNT>
__global__ void __launch_bounds__(128) k_nee_rt(RenderDev R, int32_t sample, int32_t depth) {
    __shared__ WarpTrav s_t[4];
    __shared__ WarpEnd s_e[4];
    __shared__ float s_m[4][64];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t count = R.qcount[QC_B], cap = (uint32_t)R.rec_cap;
    float4* __restrict__ rec = R.wrec + ((size_t)blockIdx.x * 4 + wid) * cap * 2;
    float* M = s_m[wid];
    Work wk;
    uint32_t nray = 0;
    while (true) {
        uint32_t idx = 0;
        if (lane == 0) idx = atomicAdd(R.qcount + CUR_N, 1u);
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
        const RayDev r = make_ray(x, R.sun, 0.0f, INFINITY, fov_prim(R, fmx));
        float T = 1.0f, tlo, thi;
        if (R.n_nodes > 0 && slab_range(r, R.root_lo, R.root_hi, 0.0f, INFINITY, tlo, thi)) {
            uint32_t ng, nb;
            emit_records_b<STOCH, COUNT>(R.nodes, R.nodes2, R.n_nodes, R.stk_limit, R.prims, r, tlo, thi, mask, w,
                                         s_t[wid], rec, cap, ng, nb, wk,
                                         [&](float4 lo, float4 hi) { return slab(r, lo, hi, tlo, thi); });
            if (ng + nb <= cap) {
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
                R.qNext[atomicAdd(R.qcount + QC_NEXT, 1u)] = p;
            }
        }
        __syncwarp();
    }
    if (lane == 0 && nray) atomicAdd(R.rays + 2, (unsigned long long)nray);
    if (COUNT) flush_work(R.work + kWorkSlots * STAGE_NEE, wk);
}

}  // namespace gfk

using namespace gfk;

// Kernels that own a per-warp record buffer (k_ffb_w, tracking) run one resident wave of at most
// 8 blocks of 4 warps per SM, so buffers exist for sms x 8 x 4 warps at most (gf_render_state_bytes).
unsigned gf_rec_grid(int64_t n_paths) {
    static int occ = 0;
    if (!occ) {
        int o1 = 0, o2 = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o1, k_ffb_w<false, false, false, false>, 128, 0);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, k_ff_trk<false, false>, 128, 0);
        occ = std::max(1, std::min(std::max(o1, o2), 8));
    }
    const int64_t blocks = (int64_t)(gf_persist_blocks() / 16) * occ;
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(blocks, (n_paths + 3) / 4));
}

void gf_launch_ffb(RenderDev& R, int32_t sample, int d, bool stoch, bool count, bool cam, cudaStream_t st) {
    const unsigned g = gf_rec_grid(R.n_paths);
    uint32_t* const q = R.qW;
    const int cs = QC_W, cu = CUR_W;
#define GF_FFB(S_, C_, F_, M_)                                              \
    do {                                                                    \
        k_ffb_w<S_, C_, F_, M_><<<g, 128, 0, st>>>(R, sample, d, q, cs, cu); \
        k_ffb_over<S_, C_, F_, M_><<<gf_persist_blocks() / 16, 128, 0, st>>>(R, sample, d); \
    } while (0)
#define GF_FFB2(S_, C_)                                                         \
    if (R.fov) { if (cam) GF_FFB(S_, C_, true, true); else GF_FFB(S_, C_, true, false); } \
    else { if (cam) GF_FFB(S_, C_, false, true); else GF_FFB(S_, C_, false, false); }
    if (stoch) { if (count) { GF_FFB2(true, true) } else { GF_FFB2(true, false) } }
    else { if (count) { GF_FFB2(false, true) } else { GF_FFB2(false, false) } }
#undef GF_FFB2
#undef GF_FFB
}

void gf_launch_ff_trk(RenderDev& R, int32_t sample, int d, bool stoch, bool count, cudaStream_t st) {
    const unsigned g = gf_rec_grid(R.n_paths);
    if (stoch) { if (count) k_ff_trk<true, true><<<g, 128, 0, st>>>(R, sample, d); else k_ff_trk<true, false><<<g, 128, 0, st>>>(R, sample, d); }
    else { if (count) k_ff_trk<false, true><<<g, 128, 0, st>>>(R, sample, d); else k_ff_trk<false, false><<<g, 128, 0, st>>>(R, sample, d); }
}

void gf_launch_nee_rt(RenderDev& R, int32_t sample, int d, bool stoch_nee, bool count, cudaStream_t st) {
    const unsigned g = gf_rec_grid(R.n_paths);
    if (stoch_nee) { if (count) k_nee_rt<true, true><<<g, 128, 0, st>>>(R, sample, d); else k_nee_rt<true, false><<<g, 128, 0, st>>>(R, sample, d); }
    else { if (count) k_nee_rt<false, true><<<g, 128, 0, st>>>(R, sample, d); else k_nee_rt<false, false><<<g, 128, 0, st>>>(R, sample, d); }
}
