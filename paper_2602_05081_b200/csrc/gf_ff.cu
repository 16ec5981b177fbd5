// gf_ff.cu -- a8 free flight of extension rays in ONE pass (Eq. 5; reading C17),
// one warp per ray:
//  1. warp traversal of [t_lo, t_hi] emitting one 32-byte record per chord into the warp's buffer
//     (reused ray after ray, so its touched part stays in L2), Gaussians from the front, Gabors from
//     the back (type-uniform erf work);
//  2. per record its chord integral -> tau_total -> escape test;
//  3. unless even the Gabor envelope masses cannot lift tau to tau*: the records' chords integrated
//     exactly into the 8 coarse t-bins (one erf per coarse edge inside a chord, lane-private columns,
//     no atomics) -> the coarse bins that may hold the first crossing (coarse_decide);
//  4. their 8 fine edges each, exactly, from the records -> the first fine bin whose right edge reaches
//     tau*, and the root of tau(t) = tau* inside it: safeguarded Halley over its records
//     (resolve_records, window_root).
// Rays with more chords than the buffer holds take the two-pass kernels (gf_ffa_w.cu + gf_ffb.cu),
// which need no per-ray storage.
#include "gf_render.cuh"

namespace gfk {

#ifndef GF_FF_ONEPASS
#define GF_FF_ONEPASS 0  // 1: extension rays take the one-pass kernel (measured slower: instruction-cache bound)
#endif

template <bool STOCH, bool COUNT, bool FOV, bool CAM>
__global__ void __launch_bounds__(128) k_ff(RenderDev R, int32_t sample, int32_t depth, const uint32_t* __restrict__ q_in,
                                            int cnt_slot, int cur_slot) {
    __shared__ WarpTrav s_t[4];
    __shared__ WarpEnd s_e[4];
    __shared__ float s_h[4][kNRows * kNC * 32];  // coarse rows (G, Gabor, mass), then fine rows; [m * 32 + lane]
    __shared__ uint16_t s_w[4][kWinCap];
    const unsigned FULL = 0xFFFFFFFFu;
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const uint32_t count = R.qcount[cnt_slot], cap = (uint32_t)R.rec_cap;
    const size_t gw = (size_t)blockIdx.x * 4 + wid;
    float4* __restrict__ rec = R.wrec + gw * cap * 2;
    float4* __restrict__ aux = R.waux + gw * cap;
    float* cols = s_h[wid];
    WarpEnd& q = s_e[wid];
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
        // 1. records
        uint32_t ng = 0, nb = 0;
        emit_records_b<STOCH, COUNT>(nodes, nodes2, R.n_nodes, stk_limit, prims, r, f.tlo, f.thi, f.mask, f.w, s_t[wid],
                                     rec, cap, ng, nb, wk,
                                     [&](float4 lo, float4 hi) { return ff_box<CAM>(r, cp, lo, hi, f.tlo, f.thi); });
        if (ng + nb > cap) {  // more chords than the buffer: the two-pass kernels
            if (lane == 0) R.qO[atomicAdd(R.qcount + QC_O, 1u)] = p;
            continue;
        }
        const uint32_t nside[2] = {ng, nb};
        // 2. chord integrals -> tau_total (aux = full, amp G(u0), amp cos phi0, -amp sin phi0); Gabor masses
        float tot = 0.0f, mass = 0.0f;
#pragma unroll 1
        for (int side = 0; side < 2; ++side)
            for (uint32_t i = lane; i < nside[side]; i += 32) {
                const uint32_t slot = side == 0 ? i : cap - 1 - i;
                const float4 ra = rec[2 * slot], rb = rec[2 * slot + 1];
                const float4 x = chord_aux<COUNT>(ra, rb, side == 1, wk);
                aux[slot] = x;
                tot += x.x;
                if (side == 1) mass += 2.0f * rb.x * __expf(0.5f * ra.z * ra.z);
            }
        double ttot = tot, tmass = mass;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            ttot += __shfl_xor_sync(FULL, ttot, o);
            tmass += __shfl_xor_sync(FULL, tmass, o);
        }
        if (ttot + tmass < f.tstar) {  // tau(t) <= tau_Gauss + Gabor mass < tau* everywhere: escape
            if (lane == 0) ff_escape(R, p);
            continue;
        }
        // 3. coarse bins (Gaussian, Gabor, Gabor mass) from the records -> the coarse bins of the crossing
#pragma unroll
        for (int m = 0; m < kNRows * kNC; ++m) cols[m * 32 + lane] = 0.0f;
        __syncwarp();
        bin_records<COUNT>(rec, aux, cap, ng, nb, coarse_bins(f), cols, cols + kNC * 32,
                           kNF > 1 ? cols + 2 * kNC * 32 : nullptr, q, wk);
        double cstart;
        const int ks = kNF == 1 ? coarse_first_warp(cols, f.tstar, &cstart) : coarse_decide_warp(cols, f.tstar, &cstart);
        const int k1 = ks & 0xFF, s0 = ks >> 8;
        bool col = false;
        float t = 0.0f;
        __syncwarp();
        // 4. fine bins of coarse bins s0 .. k1 and the root in the first fine bin reaching tau*
        if (s0 < kNC)
            col = resolve_records<COUNT>(rec, aux, cap, ng, nb, f, s0, k1 < kNC ? k1 : kNC - 1, cstart, cols, s_w[wid], q,
                                         wk, t);
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
    if (lane == 0 && nray) atomicAdd(R.rays + (depth == 0 ? 0 : 1), (unsigned long long)nray);
    if (COUNT) flush_work(R.work + kWorkSlots * STAGE_FFA, wk);
}

}  // namespace gfk

using namespace gfk;

bool gf_ff_onepass() { return GF_FF_ONEPASS != 0; }

void gf_launch_ff(RenderDev& R, int32_t sample, int d, bool stoch, bool count, bool cam, const uint32_t* q_in,
                  int cnt_slot, int cur_slot, cudaStream_t st) {
    const unsigned g = gf_rec_grid(R.n_paths);
#define GF_FF(S_, C_, F_, M_) k_ff<S_, C_, F_, M_><<<g, 128, 0, st>>>(R, sample, d, q_in, cnt_slot, cur_slot)
#define GF_FF2(S_, C_)                                                         \
    if (R.fov) { if (cam) GF_FF(S_, C_, true, true); else GF_FF(S_, C_, true, false); } \
    else { if (cam) GF_FF(S_, C_, false, true); else GF_FF(S_, C_, false, false); }
    if (stoch) { if (count) { GF_FF2(true, true) } else { GF_FF2(true, false) } }
    else { if (count) { GF_FF2(false, true) } else { GF_FF2(false, false) } }
#undef GF_FF2
#undef GF_FF
}
