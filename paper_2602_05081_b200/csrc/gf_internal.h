// gf_internal.h -- host-side declarations shared by the library's translation units.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "gf_device.cuh"

struct LoadArgs {
    int64_t n;
    const float *mu, *quat, *scale, *alpha, *omega, *extent;
    const uint8_t *level, *bin;
    int32_t P, K;
    float cutoffs[8];
    float axes[48];
};

struct BuildScratch {
    float* pbox;
    float* center;  // key centre per primitive (frame builds)
    uint32_t* cbounds;
    uint64_t *keys_in, *keys_out;
    uint32_t *vals_in, *vals_out;
    int32_t *left, *right, *parent, *rlo, *rhi;
    float* nbox;
    uint32_t *nmask, *ncount, *nsize, *flags;
    void* sort_temp;
    size_t sort_temp_bytes;
    size_t total_bytes;
};

struct TraceArgs {
    const gfk::GNode* nodes;
    const gfk::GNode2* nodes2;
    uint32_t n_nodes;
    int32_t stk_limit;
    const gfk::GPrim* prims;  // BVH order (sorted) or input order (brute force)
    const uint8_t* group;     // input-order group ids (brute force)
    const int32_t* perm;      // sorted -> input index (candidates)
    int64_t n_prims;
    gfk::PolicyDev pol;
    gfk::SceneDev sc;
    uint64_t seed;
    const float* rays;
    int64_t n;
    float* tau;
    float* T;
    uint32_t* counters;
    int32_t* cand_ids;
    int32_t cand_cap;
    int32_t* cand_count;
    unsigned long long* work;  // gf_stats work counters or null
};

// Stage timing with CUDA events recorded on the launching stream (gf_set_profiling).
enum { STAGE_GEN = 0, STAGE_FFA = 1, STAGE_FFB = 2, STAGE_NEE = 3, STAGE_FINISH = 4, STAGE_TOMO = 5,
       STAGE_TRACE = 6, STAGE_FFAI = 7, N_STAGES = 8 };
struct StageTimer {
    bool on = false;  // record events around every launch
    unsigned long long launches = 0;
    unsigned long long stage_launches[N_STAGES] = {};
    struct Rec { int stage; cudaEvent_t a, b; };
    std::vector<Rec> recs;
    std::vector<cudaEvent_t> pool;
    size_t pool_used = 0;
    cudaEvent_t ev();
    void pre(int stage, cudaStream_t st, cudaEvent_t& a);   // before a kernel launch
    void post(int stage, cudaStream_t st, cudaEvent_t a);   // after it
};

// render launch state (see gf_render.cu)
struct RenderDev {
    const gfk::GNode* nodes;
    const gfk::GNode2* nodes2;
    uint32_t n_nodes;
    int32_t stk_limit;
    const gfk::GPrim* prims;
    gfk::PolicyDev ext, nee;
    gfk::SceneDev sc;
    gfk::CamDev cam;
    float4 root_lo, root_hi;
    int32_t mode, max_depth, jitter, estimator;
    int32_t fov;  // foveated rendering (gf_render_desc.foveation)
    float fov_gaze[2], fov_f0, fov_slope, fov_jitter, fov_lfmax[8];
    int32_t mb;  // motion-blur reference (gf_render_desc.motion_blur)
    float mb_dir[3], mb_m;
    float albedo, hg_g, sun_E, env_L;
    float3 sun;
    uint64_t seed;
    // work decomposition
    int64_t n_paths;           // paths of this chunk of the sample pass (state arrays are per chunk)
    int64_t path_base;         // global index of the chunk's first path
    int64_t n_total;           // paths of the whole pass
    int32_t shard_kind, shard_rank, shard_world;
    int32_t tiles_x, tiles_y;  // 32x32 tiles
    const int32_t* probe;      // probe pixels or null
    int32_t spp_count;
    // per-path state (SoA, n_paths each)
    float *ox, *oy, *oz, *dx, *dy, *dz, *beta, *L;
    double* cum;  // 3 n: tau before the bracketing bin, tau*, tau in the bin
    int32_t* bin;
    uint32_t* pix;
    uint32_t* nhit;  // hits recorded by ffA
    uint2* hits;     // [n_paths][hit_cap]: sorted prim index | group << 24, bin span ka | kb << 8
    int32_t hit_cap;
    float4* wrec;    // [k_ff warp][rec_cap] x 2 float4 hit records (per warp, reused across paths)
    float4* waux;    // [k_ff warp][rec_cap] per-record full integral, amp G(u0), amp cos, -amp sin
    int32_t rec_cap;
    uint32_t* qO;    // record-overflow paths (k_ff redo after k_ff_pkt, else single-pass k_ffA)
    uint32_t* qO2;   // record-overflow paths of the k_ff redo (single-pass k_ffA)
    // light BVH for NEE (built per gf_render call in the frame lf: rows x', y', z' = light direction)
    int32_t light;
    float lf[9];
    gfk::GNode* lnodes;
    gfk::GNode2* lnodes2;
    gfk::GPrim* lprims;
    int32_t* lperm;
    uint32_t* ldepth;
    // camera BVH for depth-0 rays: projective boxes, basis rows r, u, f (cb) at the eye
    int32_t camb;  // camera BVH built for this call
    float cb[9];
    gfk::GNode* cnodes;
    gfk::GNode2* cnodes2;
    gfk::GPrim* cprims;
    int32_t* cperm;
    uint32_t* cdepth;
    uint32_t* qB2;   // record-overflow paths after single-pass ffA (per-thread ffB)
    // queues
    uint32_t *qA, *qB, *qNext;
    uint32_t* qcount;  // [4]: A, B, next, overflow
    unsigned long long* rays;  // [2]
    float* accum;
    unsigned long long* work;  // gf_stats work counters (counting variant) or null
    // (appended last, so the hot kernels' parameter offsets stay as measured)
    int32_t tomo_pkt_min;  // tomography chunks with at least this many paths take k_tomo_pkt
};

cudaError_t gf_launch_load(const LoadArgs& A, void* out, uint8_t* group, uint32_t* err, cudaStream_t st);
size_t gf_sort_temp_bytes(int64_t n);
BuildScratch gf_scratch_layout(int64_t n, char* base);
cudaError_t gf_launch_build(const void* prims, const uint8_t* group, int64_t n, const BuildScratch& S, void* nodes,
                            void* nodes2, void* sorted, int32_t* perm, uint32_t* n_nodes, uint32_t* max_depth,
                            float* root_box, cudaStream_t st);
cudaError_t gf_launch_build_frame(const void* prims, const uint8_t* group, int64_t n, const BuildScratch& S,
                                  const float* F, const float* eye, void* nodes, void* nodes2, void* sorted,
                                  int32_t* perm, uint32_t* depth, cudaStream_t st);
cudaError_t gf_launch_trace(const TraceArgs& A, bool brute, bool count, cudaStream_t st);
cudaError_t gf_launch_candidates(const TraceArgs& A, bool brute, cudaStream_t st);
cudaError_t gf_launch_grad_alpha(const TraceArgs& A, const float* dl, float* grad, cudaStream_t st);
cudaError_t gf_launch_grad_params(const TraceArgs& A, const float* dl, float* acc, bool packets, cudaStream_t st);
cudaError_t gf_launch_grad_finish(const gfk::GPrim* prims, int64_t n, const float* acc, const float* quat, float* grad,
                                  cudaStream_t st);
size_t gf_render_state_bytes(int64_t n_paths, int64_t n_prims, char* base, RenderDev* R, BuildScratch* light_scratch);
cudaError_t gf_launch_render_pass(RenderDev& R, int32_t sample, int32_t sample_slot, cudaStream_t st,
                                  StageTimer& T);
