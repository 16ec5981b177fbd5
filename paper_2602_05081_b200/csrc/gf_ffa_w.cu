// gf_ffa_w.cu -- a8 free flight, pass A, one warp per ray (Eq. 5; reading C17): the ray's
// optical depth integrated exactly into the 8 coarse t-bins, the escape test and the coarse bins of the
// first crossing (coarse_decide).
#include "gf_render.cuh"

namespace gfk {

// ---------------------------------------------------------------- pass A: one warp per ray
// Endpoint queue of the coarse binning (Gabor chords, the series erf): each entry (u, Omega, A, B)
// contributes v = A Re F(u) + B Im F(u) to coarse bin `plus` and -v to bin `minus` (0xFF: none),
// evaluated 32 at a time into the evaluating lane's column.  Gaussian chords (real erf) and the Gabor
// envelope masses are binned lane-locally.
constexpr int kQB = 96;  // < 32 pending + 64 pushed by one chord-end step
struct WarpBinQ {
    float4 e[kQB];
    uint32_t b[kQB];
};

template <bool STOCH, bool COUNT, bool FOV, bool CAM>
#ifdef GF_MINB_FFAW  // tuning variants: the blocks per SM the registers must allow
#define GF_LB_FFAW __launch_bounds__(128, GF_MINB_FFAW)
#else
#define GF_LB_FFAW __launch_bounds__(128)
#endif
__global__ void GF_LB_FFAW k_ffa_w(RenderDev R, int32_t sample, int32_t depth,
                                               const uint32_t* __restrict__ q_in, int cnt_slot, int cur_slot,
                                               int ray_count) {
    __shared__ WarpTrav s_t[4];
    __shared__ WarpBinQ s_q[4];
    __shared__ float s_h[4][kNRows * kNC * 32];  // per warp: G, Gabor (, mass) rows; bin m of lane l at [m * 32 + l]
#if GF_REFS
    __shared__ WarpEnd s_e[4];  // pass B from the hit list (window_from_refs)
#else
    WarpEnd* s_e = nullptr;  // (no in-kernel pass B)
#endif
    __shared__ uint32_t s_gm[4][kNC];  // per coarse bin: the groups with chords in it
    const unsigned FULL = 0xFFFFFFFFu;
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const uint32_t count = R.qcount[cnt_slot];
    float* cols = s_h[wid];
    float* cg = cols + lane;                 // this lane's private columns: conflict-free, no atomics
    float* cb = cols + kNC * 32 + lane;
    float* cm = cols + (kNRows - 1) * kNC * 32 + lane;  // (only written when kNF > 1)
    WarpBinQ& q = s_q[wid];
    const size_t gw = (size_t)blockIdx.x * 4 + wid;
    uint32_t* __restrict__ refs = R.wref + gw * kRefWarp;  // this ray's hit list
    float4* __restrict__ rec = R.wrec + gw * (size_t)R.rec_cap * 2;
    float4* __restrict__ aux = R.waux + gw * (size_t)R.rec_cap;
    const GNode* __restrict__ nodes = CAM ? R.cnodes : R.nodes;
    const GNode2* __restrict__ nodes2 = CAM ? R.cnodes2 : R.nodes2;
    const GPrim* __restrict__ prims = CAM ? R.cprims : R.prims;
    const int stk_limit = CAM ? max(1, kWStk - 34 - (int)*R.cdepth) : R.stk_limit;
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
        FFRay f;
        const int st = ff_begin<STOCH, FOV>(R, p, sample, depth, f);
        if (st == 0) {
            if (lane == 0) {
                ff_collide(R, p, f, f.tlo);
                R.qB[atomicAdd(R.qcount + QC_B, 1u)] = p;
            }
            continue;
        }
        if (st == 1) {
            if (lane == 0) ff_escape(R, p);
            continue;
        }
        const RayDev r = make_ray(f.o, f.d, 0.0f, INFINITY, fov_prim(R, f.fth));
        const CamPt cp = cam_point(R, f.d);
#pragma unroll
        for (int m = 0; m < kNC; ++m) cg[m * 32] = cb[m * 32] = cm[m * 32] = 0.0f;
        if (lane < kNC) s_gm[wid][lane] = 0u;
        __syncwarp();
        int nq1 = 0;
        uint32_t nref = 0;
        // Windows of bins [wa, wb], front to back: each window's chords, clipped to it, go into its bins and
        // the exact prefix at its edges decides -- a ray whose first crossing lies in an early window never
        // visits the rest of the scene (the edge values are the same sums as in one sweep: C17 unchanged).
        // R.ff_win 1: one split, after the bin where tau*/kappa (kappa at the path's last collision, scaled
        // by win_scale) predicts the crossing; 3: two splits (there and at 3x; measured no better); 2: windows
        // of 1, 2, 4, .. bins; 0: one sweep.
        int split = kNC;  // first bin of the second window (kNC: one window)
        if (kNF == 1 && (R.ff_win == 1 || R.ff_win == 3) && depth > 0) {
            const float k0 = R.fkap[p];
            if (k0 > 0.0f)
                split = (int)fmin((double)kNC, fmax(1.0, R.win_scale * (f.tstar / k0 - (double)f.tlo) * f.ibw + 1.0));
        }
        int ks = kNC;
        double cstart = 0.0;
        for (int wa = 0; wa < kNC;) {
        const int wb = kNF > 1 ? kNC - 1 : R.ff_win == 2 ? min(kNC - 1, 2 * wa)
                     : wa < split ? split - 1 : (R.ff_win == 3 && wa < 3 * split) ? min(kNC - 1, 3 * split - 1) : kNC - 1;
        const float wlo = ff_edge(f, wa - 1), whi = ff_edge(f, wb);
        auto run = [&](int, int take) {
            const bool v = lane < take;
            const float4 e = v ? q.e[nq1 - take + lane] : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
            const uint32_t bb = v ? q.b[nq1 - take + lane] : 0u;
            nq1 -= take;
            __syncwarp();
            if (v) {
                if (COUNT) ++wk.erfc;
                const float2 F = erf_c(e.x, e.y);
                const float val = fmaf(e.z, F.x, e.w * F.y);
                cb[(bb & 0xFFu) * 32] += val;  // (any column: the columns are summed at the end)
                if ((bb >> 8) < (uint32_t)kNC) cb[(bb >> 8) * 32] -= val;
            }
        };
        warp_traverse_b<COUNT>(nodes, nodes2, R.n_nodes, stk_limit, f.mask, s_t[wid], wk, [&](bool valid, uint32_t ref) {
            bool hit = false;
            Setup s;
            float cj = 0.0f;
            if (valid) {
                const GPrim* pp = prims + (ref & kRefIdx);
                GPrim P;
                P.a = __ldg(&pp->a);
                if (COUNT) ++wk.tests;
                if (sphere_pretest(P.a, r, wlo, whi)) {
                    P.b = __ldg(&pp->b); P.c = __ldg(&pp->c); P.d = __ldg(&pp->d);
                    hit = prim_setup(P, r, wlo, whi, s);
                    cj = P.d.w * s.ij;
                    if (STOCH) cj *= f.w[ref >> 27];
                }
            }
            if (GF_REFS) {  // the hit list for pass B
                const unsigned mh = __ballot_sync(FULL, hit);
                if (hit && nref + __popc(mh & lt) < (uint32_t)kRefCapW) refs[nref + __popc(mh & lt)] = ref;
                nref += __popc(mh);
            }
            int ne = 0, ka = 0, kb = 0;
            float amp = 0.0f, sp = 0.0f, cp_ = 1.0f;
            if (hit) {
                if (COUNT) ++wk.hits;
                ka = min(wb, max(wa, ff_bin(f, fmaf(s.u0 - s.bp, s.ij, s.tc))));  // (the chord is clipped to
                kb = min(wb, max(wa, ff_bin(f, fmaf(s.u1 - s.bp, s.ij, s.tc))));  //  the window)
                for (int m = ka; m <= kb; ++m) atomicOr(&s_gm[wid][m], 1u << (ref >> 27));
                const float wmax = 0.5f * (fmaxf(s.u0 * s.u0, s.u1 * s.u1) + s.Om * s.Om);
                if (kNF > 1 && s.Om != 0.0f) {  // Gabor envelope mass >= int |kappa_i| into every coarse bin it touches
                    const float mass = cj * __expf(-0.5f * s.r2);
                    for (int m = ka; m <= kb; ++m) cm[m * 32] += mass;
                }
                float* col = s.Om == 0.0f ? cg : cb;
                if ((wmax > kWMaxSeries && s.Om != 0.0f) || s.u1 - s.u0 < 1e-4f) {  // rare: lane-local pieces
                    float ua = s.u0;
                    for (int m = ka; m < kb; ++m) {
                        const float ub = fminf(fmaxf(fmaf(s.j, ff_edge(f, m) - s.tc, s.bp), ua), s.u1);
                        col[m * 32] += cj * seg_J_rare(s, ua, ub);
                        ua = ub;
                    }
                    col[kb * 32] += cj * seg_J_rare(s, ua, s.u1);
                    if (COUNT) ++wk.gl;
                } else if (s.Om == 0.0f) {  // Gaussian (and Omega = 0): real erf pieces, lane-local
                    const float g = 0.5f * cj * __expf(-0.5f * s.r2) * (s.phi0 == 0.0f ? 1.0f : __cosf(s.phi0));
                    float Fa = erff(s.u0 * kRsqrt2);
                    for (int m = ka; m < kb; ++m) {
                        const float ub = fminf(fmaxf(fmaf(s.j, ff_edge(f, m) - s.tc, s.bp), s.u0), s.u1);
                        const float Fb = erff(ub * kRsqrt2);
                        cg[m * 32] += g * (Fb - Fa);
                        Fa = Fb;
                    }
                    cg[kb * 32] += g * (erff(s.u1 * kRsqrt2) - Fa);
                    if (COUNT) wk.erfr += (uint32_t)(kb - ka + 2);
                } else {  // Gabor: series endpoints queued with their bins (type-uniform batches of 32)
                    amp = 0.5f * cj * __expf(-0.5f * (s.r2 + s.Om * s.Om));
                    sincos_red(s.phi0, &sp, &cp_);
                    ne = (ka == kb && s.u0 == -s.h && s.u1 == s.h) ? 1 : 2 + (kb - ka);
                }
            }
            {  // chord ends: one push step for all lanes (1 or 2 entries per lane)
                const bool has = ne > 0, two = ne > 1;
                const unsigned m1 = __ballot_sync(FULL, has), m2 = __ballot_sync(FULL, two);
                if (m1) {
                    if (has) {
                        const int o1 = nq1 + __popc(m1 & lt);
                        if (ne == 1) {  // symmetric full chord inside one bin: 2 amp cos(phi0) Re F(h)
                            q.e[o1] = make_float4(s.u1, s.Om, 2.0f * amp * cp_, 0.0f);
                            q.b[o1] = (uint32_t)ka | 0xFF00u;
                        } else {  // +G(u1) into the last bin, -G(u0) into the first
                            q.e[o1] = make_float4(s.u1, s.Om, amp * cp_, -amp * sp);
                            q.b[o1] = (uint32_t)kb | 0xFF00u;
                            const int o2 = nq1 + __popc(m1) + __popc(m2 & lt);
                            q.e[o2] = make_float4(s.u0, s.Om, -amp * cp_, amp * sp);
                            q.b[o2] = (uint32_t)ka | 0xFF00u;
                        }
                    }
                    nq1 += __popc(m1) + __popc(m2);
                    GF_CHECK(nq1 <= kQB);
                    __syncwarp();
                    while (nq1 >= 32) run(1, 32);
                }
            }
            for (int e = 2; __any_sync(FULL, e < ne); ++e) {  // coarse edges inside the chord
                const bool mine = e < ne;
                const unsigned mm = __ballot_sync(FULL, mine);
                if (mine) {
                    const int m = ka + e - 2;
                    const float u = fminf(fmaxf(fmaf(s.j, ff_edge(f, m) - s.tc, s.bp), s.u0), s.u1);
                    q.e[nq1 + __popc(mm & lt)] = make_float4(u, s.Om, amp * cp_, -amp * sp);
                    q.b[nq1 + __popc(mm & lt)] = (uint32_t)m | ((uint32_t)(m + 1) << 8);
                }
                nq1 += __popc(mm);
                __syncwarp();
                if (nq1 >= 32) run(1, 32);
            }
        }, [&](float4 lo, float4 hi) { return ff_box<CAM>(r, cp, lo, hi, wlo, whi); });
        while (nq1 > 0) run(1, min(nq1, 32));
        __syncwarp();
        ks = kNF == 1 ? coarse_first_warp(cols, f.tstar, &cstart, wb) : coarse_decide_warp(cols, f.tstar, &cstart);
        if ((ks >> 8) < kNC) break;
        wa = wb + 1;
        }
        if ((ks >> 8) == kNC) {  // no coarse bin can reach tau*: escape
            if (lane == 0) ff_escape(R, p);
            continue;
        }
        // pass B right here from the hit list (uniform bins): the root inside the crossing bin
        float t = 0.0f;
        if (GF_REFS && kNF == 1 && nref <= (uint32_t)kRefCapW &&
            window_from_refs<STOCH, COUNT>(refs, nref, prims, r, STOCH ? f.w : nullptr, ff_edge(f, (ks & 0xFF) - 1), ff_edge(f, ks & 0xFF),
                                           cstart, f.tstar, rec, aux, (uint32_t)R.rec_cap, s_e[wid], wk, t)) {
            if (lane == 0) {
                ff_collide(R, p, f, t);
                R.qB[atomicAdd(R.qcount + QC_B, 1u)] = p;
            }
        } else if (R.estimator == GF_EST_UNIFORM && kNF == 1) {  // biased: uniform in the crossing bin (U1)
            if (lane == 0) {
                ff_collide(R, p, f, ff_uniform_t(R, f, sample, depth, ks & 0xFF));
                R.qB[atomicAdd(R.qcount + QC_B, 1u)] = p;
            }
        } else if (lane == 0) {  // the crossing bin is re-traversed by pass B (k_ffb_w)
            R.ffk[p] = ks;
            R.ffc[p] = cstart;
            uint32_t g = 0;
            for (int m = ks >> 8; m <= min(ks & 0xFF, kNC - 1); ++m) g |= s_gm[wid][m];
            R.ffg[p] = g;
            R.qW[atomicAdd(R.qcount + QC_W, 1u)] = p;
        }
        __syncwarp();
    }
    if (ray_count && lane == 0 && nray) atomicAdd(R.rays + (depth == 0 ? 0 : 1), (unsigned long long)nray);
    // (the overflow re-run of a one-pass kernel's rays counts as fallback work, stage ffB)
    if (COUNT) flush_work(R.work + kWorkSlots * (ray_count ? STAGE_FFA : STAGE_FFB), wk);
}

}  // namespace gfk

using namespace gfk;

void gf_launch_ffa_w(RenderDev& R, int32_t sample, int d, bool stoch, bool count, bool cam, const uint32_t* q_in,
                     int cnt_slot, int cur_slot, int ray_count, unsigned grid, cudaStream_t st) {
#define GF_FFA(S_, C_, F_, M_) \
    k_ffa_w<S_, C_, F_, M_><<<grid, 128, 0, st>>>(R, sample, d, q_in, cnt_slot, cur_slot, ray_count)
#define GF_FFA2(S_, C_)                                                         \
    if (R.fov) { if (cam) GF_FFA(S_, C_, true, true); else GF_FFA(S_, C_, true, false); } \
    else { if (cam) GF_FFA(S_, C_, false, true); else GF_FFA(S_, C_, false, false); }
    if (stoch) { if (count) { GF_FFA2(true, true) } else { GF_FFA2(true, false) } }
    else { if (count) { GF_FFA2(false, true) } else { GF_FFA2(false, false) } }
#undef GF_FFA2
#undef GF_FFA
}
