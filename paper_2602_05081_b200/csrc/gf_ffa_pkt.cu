// gf_ffa_pkt.cu -- a8 free flight, pass A for coherent (camera) rays (Eq. 5; reading C17):
// the ray's optical depth integrated exactly into the 8 coarse t-bins (Gaussian and Gabor parts, Gabor
// envelope masses), the escape test and the coarse bins of the first crossing (coarse_decide).
#include "gf_render.cuh"

namespace gfk {

// ---------------------------------------------------------------- pass A: coherent camera rays
// k_ffa_pkt: 32 consecutive paths per warp (one 8x4 pixel block of the tiled path order: nearly
// parallel rays meeting the same nodes and primitives).  The warp walks ONE depth-first stack: each
// popped node's child pair is loaded once (broadcast) and tested by every lane against its own ray;
// a child is descended if any lane's ray meets it; a hit leaf's primitives are loaded once and
// tested per lane, and each lane bins its own chords (coarse_chord) into its columns of shared memory.
// CAM: boxes of the camera BVH (projective, depth-0 rays from the eye); else world slabs.
template <bool STOCH, bool COUNT, bool FOV, bool CAM>
__global__ void __launch_bounds__(128, GF_MINB_PKT) k_ffa_pkt(RenderDev R, int32_t sample, int32_t depth,
                                                              const uint32_t* __restrict__ q_in, int cnt_slot,
                                                              int cur_slot) {
    __shared__ uint32_t s_stk[4][kPStk];
    __shared__ float s_h[kNRows][kNC * 128];  // Gaussian pieces, Gabor pieces (, Gabor masses)
#if GF_REFS
    __shared__ WarpEnd s_e[4];  // pass B of the colliding lanes from their hit lists
#else
    WarpEnd* s_e = nullptr;  // (no in-kernel pass B)
#endif
    __shared__ uint32_t s_gm[kNC * 128];  // per lane and coarse bin: the groups with chords in the bin
    const unsigned FULL = 0xFFFFFFFFu;
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t count = R.qcount[cnt_slot];
    uint32_t* stk = s_stk[wid];
    float* hg = s_h[0] + threadIdx.x;  // coarse bin m of this lane's ray at [m * 128] (conflict-free columns)
    float* hb = s_h[1] + threadIdx.x;
    float* hm = s_h[kNRows - 1] + threadIdx.x;  // (only written when kNF > 1)
    uint32_t* gm = s_gm + threadIdx.x;
    const GNode* __restrict__ nodes = CAM ? R.cnodes : R.nodes;
    const GNode2* __restrict__ nodes2 = CAM ? R.cnodes2 : R.nodes2;
    const GPrim* __restrict__ prims = CAM ? R.cprims : R.prims;
    const size_t gw = (size_t)blockIdx.x * 4 + wid;
    uint32_t* __restrict__ wrefs = R.wref + gw * kRefWarp;  // lane l's hit list at [l * kRefCapL]
    uint32_t* __restrict__ myrefs = wrefs + lane * kRefCapL;
    float4* __restrict__ rec = R.wrec + gw * (size_t)R.rec_cap * 2;
    float4* __restrict__ aux = R.waux + gw * (size_t)R.rec_cap;
    Work wk;
    uint32_t nray = 0;
    while (true) {
        uint32_t base = 0;
        if (lane == 0) base = atomicAdd(R.qcount + cur_slot, 32u);
        base = __shfl_sync(FULL, base, 0);
        if (base >= count) break;
        const uint32_t idx = base + lane;
        const bool valid = idx < count;
        const uint32_t p = valid ? q_in[idx] : 0u;
        FFRay f;
        const int st = valid ? ff_begin<STOCH, FOV>(R, p, sample, depth, f) : -1;
        if (valid) {
            ++nray;
            if (COUNT) ++wk.paths;
        }
        if (st == 0) ff_collide(R, p, f, f.tlo);
        if (st == 1) ff_escape(R, p);
        push(R.qB, R.qcount + QC_B, st == 0, p);
        bool act = st == 2;
        const RayDev r = make_ray(valid ? f.o : make_float3(0.0f, 0.0f, 0.0f), valid ? f.d : make_float3(0.0f, 0.0f, 1.0f),
                                  0.0f, INFINITY, valid ? fov_prim(R, f.fth) : INFINITY);
        const CamPt cp = cam_point(R, r.d);
        const float t0 = act ? f.tlo : 0.0f, t1 = act ? f.thi : 0.0f;
        const uint32_t mask = act ? f.mask : 0u;
#pragma unroll
        for (int m = 0; m < kNC; ++m) {
            hg[m * 128] = hb[m * 128] = hm[m * 128] = 0.0f;  // (hm may alias hb: zero)
            gm[m * 128] = 0u;
        }
        uint32_t nref = 0;
        auto leaf = [&](uint32_t info, bool mine) {
            const uint32_t first = info >> 8, cnt = (info >> 5) & 7u, g = info & 31u;
            for (uint32_t k = 0; k < cnt; ++k) {
                const GPrim* pp = prims + first + k;
                GPrim P;
                P.a = __ldg(&pp->a);
                bool pass = false;
                if (mine) {
                    if (COUNT) ++wk.tests;
                    pass = sphere_pretest(P.a, r, t0, t1);
                }
                if (!__any_sync(FULL, pass)) continue;
                P.b = __ldg(&pp->b); P.c = __ldg(&pp->c); P.d = __ldg(&pp->d);
                Setup s;
                if (pass && prim_setup(P, r, t0, t1, s)) {
                    if (COUNT) ++wk.hits;
                    if (GF_REFS) {  // this lane's hit list for pass B
                        if (nref < (uint32_t)kRefCapL) myrefs[nref] = (first + k) | (g << 27);
                        ++nref;
                    }
                    float cj = P.d.w * s.ij;
                    if (STOCH) cj *= f.w[g];
                    coarse_chord<COUNT>(s, cj, f, hg, hb, hm, 128, wk);  // all lanes: the same primitive type
                    const int ka = ff_bin(f, fmaf(s.u0 - s.bp, s.ij, s.tc)), kb = ff_bin(f, fmaf(s.u1 - s.bp, s.ij, s.tc));
                    for (int m = ka; m <= kb; ++m) gm[m * 128] |= 1u << g;
                }
            }
        };
        if (__any_sync(FULL, act)) {
            int ns = 0;
            const float4 lo = __ldg(&nodes[0].lo), hi = __ldg(&nodes[0].hi);
            const uint32_t sk = __float_as_uint(lo.w), info = __float_as_uint(hi.w);
            if (COUNT && act) ++wk.nodes;
            const bool hr = act && (node_mask(sk, info) & mask) && ff_box<CAM>(r, cp, lo, hi, t0, t1);
            if (__any_sync(FULL, hr)) {
                if (sk & kLeafBit) leaf(info, hr);
                else { stk[0] = 0; ns = 1; }
            }
            while (ns > 0) {
                const uint32_t i = stk[--ns];
                const GNode2* q = nodes2 + i;
                const float4 lo0 = __ldg(&q->lo0), hi0 = __ldg(&q->hi0), lo1 = __ldg(&q->lo1), hi1 = __ldg(&q->hi1);
                const uint32_t ref0 = __float_as_uint(lo0.w), inf0 = __float_as_uint(hi0.w);
                const uint32_t ref1 = __float_as_uint(lo1.w), inf1 = __float_as_uint(hi1.w);
                if (COUNT && act) wk.nodes += 2;
                const bool h0 = act && (node_mask(ref0, inf0) & mask) && ff_box<CAM>(r, cp, lo0, hi0, t0, t1);
                const bool h1 = act && (node_mask(ref1, inf1) & mask) && ff_box<CAM>(r, cp, lo1, hi1, t0, t1);
                const bool a0 = __any_sync(FULL, h0), a1 = __any_sync(FULL, h1);
                if (a1) {
                    if (ref1 & kLeafBit) leaf(inf1, h1);
                    else { GF_CHECK(ns < kPStk); stk[ns++] = ref1; }
                }
                if (a0) {
                    if (ref0 & kLeafBit) leaf(inf0, h0);
                    else { GF_CHECK(ns < kPStk); stk[ns++] = ref0; }
                }
                __syncwarp();
            }
        }
        int ks = 0;
        double cstart = 0.0;
        bool uni = false;
        if (act) {
            if (kNF == 1) {  // uniform bins: the first edge reaching tau*, lane-local over this lane's columns
                double c = 0.0;
                int k1 = kNC;
                for (int m = 0; m < kNC; ++m) {
                    const double c2 = c + (double)hg[m * 128] + (double)hb[m * 128];
                    if (c2 >= f.tstar) { k1 = m; break; }
                    c = c2;
                }
                ks = k1 | (k1 << 8);
                cstart = c;
            } else {
                double g[kNC], b[kNC], mm[kNC];
#pragma unroll
                for (int m = 0; m < kNC; ++m) { g[m] = hg[m * 128]; b[m] = hb[m * 128]; mm[m] = hm[m * 128]; }
                ks = coarse_decide(g, b, mm, f.tstar, &cstart);
            }
            if ((ks >> 8) == kNC) {  // no coarse bin can reach tau*: escape
                ff_escape(R, p);
                act = false;
            } else if (R.estimator == GF_EST_UNIFORM && kNF == 1) {  // biased: uniform in the crossing bin (U1)
                ff_collide(R, p, f, ff_uniform_t(R, f, sample, depth, ks & 0xFF));
                act = false;
                uni = true;
            } else {
                R.ffk[p] = ks;
                R.ffc[p] = cstart;
                uint32_t g = 0;
                for (int m = ks >> 8; m <= min(ks & 0xFF, kNC - 1); ++m) g |= gm[m * 128];
                R.ffg[p] = g;
            }
        }
        // pass B here for the colliding lanes whose hit list fits, one lane after another with the whole
        // warp (uniform bins); the others re-traverse their crossing bin in k_ffb_w
        const bool here = GF_REFS && kNF == 1 && act && nref <= (uint32_t)kRefCapL;
        unsigned todo = __ballot_sync(FULL, here);
        bool done = false;
        while (todo) {
            const int l = __ffs(todo) - 1;
            todo &= todo - 1;
            const float3 ol = make_float3(__shfl_sync(FULL, r.o.x, l), __shfl_sync(FULL, r.o.y, l), __shfl_sync(FULL, r.o.z, l));
            const float3 dl = make_float3(__shfl_sync(FULL, r.d.x, l), __shfl_sync(FULL, r.d.y, l), __shfl_sync(FULL, r.d.z, l));
            const RayDev rl = make_ray(ol, dl, 0.0f, INFINITY, __shfl_sync(FULL, r.fmax, l));
            const int kl = __shfl_sync(FULL, ks, l) & 0xFF;
            const float lo_l = __shfl_sync(FULL, t0, l), hi_l = __shfl_sync(FULL, t1, l), bw_l = __shfl_sync(FULL, f.bw, l);
            const float wa = kl == 0 ? lo_l : fmaf((float)kl, bw_l, lo_l);  // ff_edge of the lane's bins
            const float wb = kl >= kNC - 1 ? hi_l : fmaf((float)(kl + 1), bw_l, lo_l);
            float tl = 0.0f;
            const bool ok = window_from_refs<false, COUNT>(wrefs + l * kRefCapL, __shfl_sync(FULL, nref, l), prims, rl, nullptr,
                                                           wa, wb, __shfl_sync(FULL, cstart, l),
                                                           __shfl_sync(FULL, f.tstar, l), rec, aux, (uint32_t)R.rec_cap,
                                                           s_e[wid], wk, tl);
            const float tl_l = __shfl_sync(FULL, tl, 0);
            if (lane == l && ok) {
                ff_collide(R, p, f, tl_l);
                done = true;
            }
            __syncwarp();
        }
        push(R.qB, R.qcount + QC_B, done || uni, p);
        push(R.qW, R.qcount + QC_W, act && !done, p);
        __syncwarp();
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) nray += __shfl_xor_sync(FULL, nray, off);
    if (lane == 0 && nray) atomicAdd(R.rays + (depth == 0 ? 0 : 1), (unsigned long long)nray);
    if (COUNT) flush_work(R.work + kWorkSlots * STAGE_FFA, wk);
}

}  // namespace gfk

using namespace gfk;

void gf_launch_ffa_pkt(RenderDev& R, int32_t sample, int d, bool stoch, bool count, bool cam, unsigned grid,
                       cudaStream_t st) {
#define GF_PKT(S_, C_, F_, M_) k_ffa_pkt<S_, C_, F_, M_><<<grid, 128, 0, st>>>(R, sample, d, R.qA, QC_A, CUR_A)
#define GF_PKT2(S_, C_)                                                         \
    if (R.fov) { if (cam) GF_PKT(S_, C_, true, true); else GF_PKT(S_, C_, true, false); } \
    else { if (cam) GF_PKT(S_, C_, false, true); else GF_PKT(S_, C_, false, false); }
    if (stoch) { if (count) { GF_PKT2(true, true) } else { GF_PKT2(true, false) } }
    else { if (count) { GF_PKT2(false, true) } else { GF_PKT2(false, false) } }
#undef GF_PKT2
#undef GF_PKT
}

