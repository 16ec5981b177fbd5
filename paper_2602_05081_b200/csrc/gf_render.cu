// gf_render.cu -- a9 scatter-loop orchestration (wavefront), camera rays, a10 accumulation; the
// free-flight (a8) kernels live in gf_ffa.cu / gf_ffb.cu, NEE and tomography in gf_nee.cu
// (Eq. 4-5, bisection/root finding P:L254, pipeline P:L352-L365).
//
// Wavefront over the paths of one sample pass: gen -> [ffA -> ffB -> nee] x max_depth -> finish.
//  ffA (pass A): one traversal of the ray's scene interval [t_lo, t_hi] integrating every hit's chord
//      EXACTLY into kNB equal t-bins (App. A closed form at the bin edges): tau_total for the escape
//      test (Eq. 5) and the first bin whose right-edge cumulative tau reaches tau* (reading C17).
//      k_ffa_pkt: 32 coherent camera rays per warp, one packet walk, lane-local integration;
//      k_ffa_w:   one warp per ray (extension rays), erf endpoints queued with their target bins.
//  ffB (pass B, k_ffb_w): one warp per colliding ray re-traverses only that bin's window, records the
//      few chords inside it and solves tau(t) = tau* there by safeguarded Halley / bisection.
//  NEE (k_nee_w): shadow ray towards the directional light (T = e^-tau), HG phase, next direction.
// No record of a whole ray is ever stored: pass A keeps kNB floats per ray on chip, pass B one
// window's records in a small (L2-resident) per-warp buffer.  Queues are warp-aggregated; warps
// fetch paths dynamically from the queues.
#include <algorithm>

#include <cub/device/device_radix_sort.cuh>

#include "gf_render.cuh"

namespace gfk {

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
    push(R.qA, R.qcount + QC_A, ok, (uint32_t)p);
}


// gf_trace_free_flight: paths = the caller's rays (pixel index = ray index for the RNG streams)
__global__ void __launch_bounds__(128) k_gen_rays(RenderDev R) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // grid covers whole warps
    const bool ok = p < R.n_paths;
    if (ok) {
        const int64_t g = R.path_base + p;
        const float4 r0 = __ldg((const float4*)R.trays + 2 * g), r1 = __ldg((const float4*)R.trays + 2 * g + 1);
        R.ox[p] = r0.x; R.oy[p] = r0.y; R.oz[p] = r0.z;
        R.dx[p] = r1.x; R.dy[p] = r1.y; R.dz[p] = r1.z;
        R.beta[p] = 1.0f;
        R.L[p] = 0.0f;
        R.pix[p] = (uint32_t)g;
    }
    push(R.qA, R.qcount + QC_A, ok, (uint32_t)p);
}

// a3 for the free flight of depth `depth`: the extension policy's mask and group weights of every path of
// queue qA (Tables B1/B2, stream 0 of the path vertex), read by pass A and pass B through ff_begin
__global__ void __launch_bounds__(128) k_policy(RenderDev R, int32_t sample, int32_t depth) {
    const uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= R.qcount[QC_A]) return;
    const uint32_t p = R.qA[idx];
    float w[kMaxGroups];
    const uint32_t m = policy_for(R.ext, R.sc, ld3(R.dx, R.dy, R.dz, p), R.seed, R.pix[p], (uint32_t)sample,
                                  (uint32_t)depth, ST_EXT, 1, w);
    R.pmask[p] = m;
    float* o = R.pw + (size_t)p * kMaxGroups;
    for (int g = 0; g < R.sc.G; ++g) o[g] = w[g];
}

// Extension-ray reordering (R.reorder, A/B): 24-bit keys = direction octant << 21 | Morton of the origin
// (7 bits per axis over the root box), sentinel 0xFFFFFF past the queue's count; CUB sorts queue qA by
// them before pass A, so that neighbouring warps trace nearby, similar rays.
__device__ __forceinline__ uint32_t spread7(uint32_t v) {
    uint32_t r = 0;
    for (int b = 0; b < 7; ++b) r |= ((v >> b) & 1u) << (3 * b);
    return r;
}
__global__ void __launch_bounds__(256) k_ext_keys(RenderDev R) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= R.n_paths) return;
    uint32_t key = 0xFFFFFFu, val = 0u;
    if (i < (int64_t)R.qcount[QC_A]) {
        val = R.qA[i];
        const float3 o = ld3(R.ox, R.oy, R.oz, val), d = ld3(R.dx, R.dy, R.dz, val);
        const float lo[3] = {R.root_lo.x, R.root_lo.y, R.root_lo.z}, hi[3] = {R.root_hi.x, R.root_hi.y, R.root_hi.z};
        const float x[3] = {o.x, o.y, o.z};
        uint32_t m = 0;
        for (int a = 0; a < 3; ++a) {
            const float u = fminf(fmaxf((x[a] - lo[a]) / fmaxf(hi[a] - lo[a], 1e-30f), 0.0f), 1.0f);
            m |= spread7((uint32_t)(u * 127.0f)) << (2 - a);
        }
        key = ((uint32_t)(d.x < 0.0f) | ((uint32_t)(d.y < 0.0f) << 1) | ((uint32_t)(d.z < 0.0f) << 2)) << 21 | m;
    }
    R.skey[i] = key;
    R.sval[i] = val;
}

__global__ void k_rotate(uint32_t* qc) {
    qc[QC_A] = qc[QC_NEXT];
    qc[QC_B] = 0; qc[QC_NEXT] = 0; qc[QC_W] = 0;
    qc[CUR_A] = 0; qc[CUR_W] = 0; qc[CUR_N] = 0; qc[QC_O] = 0; qc[CUR_O] = 0; qc[QC_V] = 0; qc[CUR_V] = 0;
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
int gf_persist_blocks() {
    static int b = 0;
    if (!b) {
        int dev = 0, sms = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        b = (sms > 0 ? sms : 148) * 16;
    }
    return b;
}
static int persist_blocks() { return gf_persist_blocks(); }
static int rec_max_blocks() { return persist_blocks() / 2; }

size_t gf_render_state_bytes(int64_t n, int64_t n_prims, char* base, RenderDev* R, BuildScratch* LS) {
    size_t off = 0;
    auto take = [&](size_t bytes) { char* p = base ? base + off : nullptr; off += (bytes + 255) & ~(size_t)255; return p; };
    const size_t nf = sizeof(float) * (size_t)n, nu = sizeof(uint32_t) * (size_t)n;
    float* ox = (float*)take(nf); float* oy = (float*)take(nf); float* oz = (float*)take(nf);
    float* dx = (float*)take(nf); float* dy = (float*)take(nf); float* dz = (float*)take(nf);
    float* beta = (float*)take(nf); float* L = (float*)take(nf);
    uint32_t* pix = (uint32_t*)take(nu);
    int32_t* ffk = (int32_t*)take(nu);
    double* ffc = (double*)take(sizeof(double) * (size_t)n);
    uint32_t* ffg = (uint32_t*)take(nu);
    float* fkap = (float*)take(nf);
    uint32_t* pmask = (uint32_t*)take(nu);
    float* pw = (float*)take(nf * kMaxGroups);
    uint32_t* skey = (uint32_t*)take(nu); uint32_t* skey2 = (uint32_t*)take(nu); uint32_t* sval = (uint32_t*)take(nu);
    size_t sb = 0;
    if (n > 0)
        cub::DeviceRadixSort::SortPairs(nullptr, sb, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                        (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)n, 0, 24);
    void* sort_temp = take(sb + 256);
    const size_t nw = (size_t)4 * (size_t)std::max<int64_t>(1, std::min<int64_t>((int64_t)rec_max_blocks(), (n + 3) / 4));
    float4* wrec = (float4*)take(sizeof(float4) * 2 * (size_t)kRecCap * nw);
    float4* waux = (float4*)take(sizeof(float4) * (size_t)kRecCap * nw);
    uint32_t* wref = (uint32_t*)take(sizeof(uint32_t) * (size_t)kRefWarp * nw);
    uint32_t* qA = (uint32_t*)take(nu); uint32_t* qB = (uint32_t*)take(nu); uint32_t* qN = (uint32_t*)take(nu);
    uint32_t* qW = (uint32_t*)take(nu); uint32_t* qO = (uint32_t*)take(nu); uint32_t* qV = (uint32_t*)take(nu);
    uint32_t* qc = (uint32_t*)take(sizeof(uint32_t) * 16);
    // light BVH (NEE): nodes, child pairs, primitives in its leaf order, permutation, depth, build scratch
    const size_t np1 = (size_t)std::max<int64_t>(n_prims, 1);
    GNode* lnodes = (GNode*)take(sizeof(GNode) * 2 * np1);
    GNode2* lnodes2 = (GNode2*)take(sizeof(GNode2) * 2 * np1);
    GPrim* lprims = (GPrim*)take(sizeof(GPrim) * np1);
    int32_t* lperm = (int32_t*)take(sizeof(int32_t) * np1);
    uint32_t* ldepth = (uint32_t*)take(sizeof(uint32_t) * 4);
    GNode* cnodes = (GNode*)take(sizeof(GNode) * 2 * np1);  // camera BVH (depth-0 rays)
    GNode2* cnodes2 = (GNode2*)take(sizeof(GNode2) * 2 * np1);
    GPrim* cprims = (GPrim*)take(sizeof(GPrim) * np1);
    int32_t* cperm = (int32_t*)take(sizeof(int32_t) * np1);
    uint32_t* cdepth = (uint32_t*)take(sizeof(uint32_t) * 4);
    const size_t lsb = gf_scratch_layout(n_prims, nullptr).total_bytes;
    char* lscratch = (char*)take(lsb);
    if (LS) *LS = gf_scratch_layout(n_prims, lscratch);
    if (R) {
        R->ox = ox; R->oy = oy; R->oz = oz; R->dx = dx; R->dy = dy; R->dz = dz; R->beta = beta; R->L = L;
        R->pix = pix; R->ffk = ffk; R->ffc = ffc; R->ffg = ffg; R->fkap = fkap; R->pmask = pmask; R->pw = pw;
        R->skey = skey; R->skey2 = skey2; R->sval = sval; R->sort_temp = sort_temp; R->sort_bytes = sb;
        R->wrec = wrec; R->waux = waux; R->rec_cap = kRecCap; R->wref = wref;
        R->qA = qA; R->qB = qB; R->qNext = qN; R->qW = qW; R->qO = qO; R->qV = qV; R->qcount = qc;
        R->lnodes = lnodes; R->lnodes2 = lnodes2; R->lprims = lprims; R->lperm = lperm; R->ldepth = ldepth;
        R->cnodes = cnodes; R->cnodes2 = cnodes2; R->cprims = cprims; R->cperm = cperm; R->cdepth = cdepth;
    }
    return off;
}

static void launch_depth(RenderDev& R, int32_t sample, int d, bool S, bool C, unsigned pgrid, unsigned wgrid,
                         cudaStream_t st, StageTimer& T, bool stoch_nee) {
    cudaEvent_t e;
    const unsigned rgrid = (unsigned)rec_max_blocks();  // kernels with per-warp buffers: one resident wave
    const bool cam = d == 0 && R.camb;  // depth-0 rays from the eye: camera BVH
    // coherent rays under one static mask: packet traversal (camera rays; gf_trace_free_flight packets)
    const bool packet = GF_PACKET && !S && (R.packets == 1 || (R.packets == 0 && d == 0 && R.camb));
    // one-pass kernel for extension rays (records in the warp's buffer); the two-pass kernels for
    // camera packets, and for the rays whose chords overflow a record buffer (queue qO)
    const bool onepass = !packet && R.estimator == 0 && gf_ff_onepass() && R.packets != 2;
    T.pre(STAGE_FFA, st, e);
    if (R.reorder && d > 0 && R.mode == 1 && !packet) {  // extension rays sorted by direction octant and origin
        k_ext_keys<<<(unsigned)((R.n_paths + 255) / 256), 256, 0, st>>>(R);
        size_t tb = R.sort_bytes;
        cub::DeviceRadixSort::SortPairs(R.sort_temp, tb, R.skey, R.skey2, R.sval, R.qA, (int)R.n_paths, 0, 24, st);
    }
    if (S && R.estimator != 1) k_policy<<<(unsigned)((R.n_paths + 127) / 128), 128, 0, st>>>(R, sample, d);
    if (R.estimator == 1) gf_launch_ff_trk(R, sample, d, S, C, st);
    else if (packet) gf_launch_ffa_pkt(R, sample, d, S, C, cam && R.packets == 0, std::min<unsigned>(pgrid, rgrid), st);
    else if (onepass) gf_launch_ff(R, sample, d, S, C, cam, R.qA, QC_A, CUR_A, st);
    else gf_launch_ffa_w(R, sample, d, S, C, cam, R.qA, QC_A, CUR_A, 1, std::min<unsigned>(wgrid, rgrid), st);
    T.post(STAGE_FFA, st, e);
    if (R.estimator == 1 || onepass) {  // record-buffer overflow: passes A + B (timed as stage ffB)
        T.pre(STAGE_FFB, st, e);
        gf_launch_ffa_w(R, sample, d, S, C, cam, R.qO, QC_O, CUR_O, 0, std::min<unsigned>(wgrid, rgrid), st);
        T.post(STAGE_FFB, st, e);
    }
    if (R.estimator != GF_EST_UNIFORM) {
        T.pre(STAGE_FFB, st, e);
        gf_launch_ffb(R, sample, d, S, C, cam && R.ffb_cam, st);
        T.post(STAGE_FFB, st, e);
    }
    if (R.mode == 2) return;  // gf_trace_free_flight: no NEE
    T.pre(STAGE_NEE, st, e);
    if (R.estimator == 1) gf_launch_nee_rt(R, sample, d, stoch_nee, C, st);  // ratio tracking (record buffers)
    else gf_launch_nee_w(R, sample, d, stoch_nee, C, wgrid, st);
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
        gf_launch_tomo(R, sample, stoch_ext, cnt,
                       R.camb && !stoch_ext && !R.fov && GF_PACKET && R.n_paths >= R.tomo_pkt_min, wgrid, st);
        T.post(STAGE_TOMO, st, ev);
    } else {
        T.pre(STAGE_GEN, st, ev);
        if (R.mode == 2) k_gen_rays<<<grid, 128, 0, st>>>(R);
        else k_gen<<<grid, 128, 0, st>>>(R, sample);
        T.post(STAGE_GEN, st, ev);
        const int depths = R.mode == 2 ? 1 : R.max_depth;
        for (int d = 0; d < depths; ++d) {
            launch_depth(R, sample, d, stoch_ext, cnt, pgrid, wgrid, st, T, stoch_nee);
            if (R.mode == 2) break;
            T.pre(STAGE_FINISH, st, ev);
            k_rotate<<<1, 1, 0, st>>>(R.qcount);
            T.post(STAGE_FINISH, st, ev);
            std::swap(R.qA, R.qNext);
        }
    }
    if (R.mode == 2) return cudaGetLastError();
    T.pre(STAGE_FINISH, st, ev);
    k_finish<<<(unsigned)((R.n_paths + 255) / 256), 256, 0, st>>>(R, slot);
    T.post(STAGE_FINISH, st, ev);
    return cudaGetLastError();
}

extern "C" int gf_free_flight_bins(void) { return kNC * kNF; }
