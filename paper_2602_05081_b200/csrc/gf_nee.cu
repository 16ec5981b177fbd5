// gf_nee.cu -- a9 next-event estimation (shadow rays to the directional light, T = e^-tau, Eq. 3) and
// a7 tomography (tau-hat of the camera rays).
#include <algorithm>

#include "gf_render.cuh"

namespace gfk {


// NEE, one warp per path (warp_tau): shadow-ray transmittance, HG phase sampling of the next
// direction.  Replaces the per-lane k_nee on the production path.
// LIGHT: traverse the light BVH (boxes in a frame whose third axis is the light direction, built
// per gf_render call by gf_launch_build_frame): the shadow ray is axis-parallel there, so a box test
// is two interval tests and one compare, and the boxes are tight across the rays' direction.
template <bool STOCH, bool COUNT, bool LIGHT, bool FOV>
#ifdef GF_MINB_NEE  // tuning variants: the blocks per SM the registers must allow
#define GF_LB_NEE __launch_bounds__(128, GF_MINB_NEE)
#else
#define GF_LB_NEE __launch_bounds__(128)
#endif
__global__ void GF_LB_NEE k_nee_w(RenderDev R, int32_t sample, int32_t depth) {
    __shared__ WarpTrav s_t[4];
    __shared__ WarpEnd s_e[4];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t count = R.qcount[QC_B];
    const int lstk = LIGHT ? max(1, kWStk - 34 - (int)*R.ldepth) : 0;
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
                                           make_ray(x, R.sun, 0.0f, INFINITY, fov_prim(R, fmx)), 0.0f, INFINITY, mask, w, s_t[wid],
                                           s_e[wid], wk, [&](float4 lo, float4 hi) {
                                               return lo.x <= xp.x && xp.x <= hi.x && lo.y <= xp.y && xp.y <= hi.y &&
                                                      hi.z >= xp.z;
                                           });
        } else {
            tau = warp_tau<STOCH, COUNT>(R.nodes, R.nodes2, R.n_nodes, R.stk_limit, R.prims,
                                         make_ray(x, R.sun, 0.0f, INFINITY, fov_prim(R, fmx)), 0.0f, INFINITY, mask, w, s_t[wid],
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
                R.qNext[atomicAdd(R.qcount + QC_NEXT, 1u)] = p;
            }
        }
    }
    if (lane == 0 && nray) atomicAdd(R.rays + 2, (unsigned long long)nray);
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
                                                  make_ray(o, d, 0.0f, INFINITY, fov_prim(R, fmx)), 0.0f, INFINITY, mask, w, s_t[wid],
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
                    else { GF_CHECK(ns < kPStk); stk[ns++] = ref1; }
                }
                if (a0) {
                    if (ref0 & kLeafBit) leaf(inf0, h0);
                    else { GF_CHECK(ns < kPStk); stk[ns++] = ref0; }
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

}  // namespace gfk

using namespace gfk;

void gf_launch_nee_w(RenderDev& R, int32_t sample, int d, bool stoch_nee, bool C_, unsigned wgrid, cudaStream_t st) {
#define GF_NEE(SN, C, L, F) k_nee_w<SN, C, L, F><<<wgrid, 128, 0, st>>>(R, sample, d)
#define GF_NEE2(C)                                                                        \
    if (R.fov) {                                                                          \
        if (R.light) { if (stoch_nee) GF_NEE(true, C, true, true); else GF_NEE(false, C, true, true); }     \
        else { if (stoch_nee) GF_NEE(true, C, false, true); else GF_NEE(false, C, false, true); }           \
    } else {                                                                              \
        if (R.light) { if (stoch_nee) GF_NEE(true, C, true, false); else GF_NEE(false, C, true, false); }   \
        else { if (stoch_nee) GF_NEE(true, C, false, false); else GF_NEE(false, C, false, false); }         \
    }
    if (C_) { GF_NEE2(true) } else { GF_NEE2(false) }
#undef GF_NEE2
#undef GF_NEE
}

void gf_launch_tomo(RenderDev& R, int32_t sample, bool stoch_ext, bool cnt, bool packets, unsigned wgrid, cudaStream_t st) {
#define GF_TOMO(S_, C_, F_) k_tomo_w<S_, C_, F_><<<wgrid, 128, 0, st>>>(R, sample)
    if (packets) {  // coherent camera rays under a static mask: packets
        const unsigned tg = (unsigned)std::min<int64_t>((int64_t)gf_persist_blocks(), (R.n_paths + 127) / 128);
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
}
