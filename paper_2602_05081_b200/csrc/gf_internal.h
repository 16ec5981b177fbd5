// gf_internal.h -- host-side declarations shared by the library's translation units.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "gf_device.cuh"

struct LoadArgs {
    int64_t n;
    const float *mu, *quat, *scale, *alpha, *omega, *extent;
    const uint8_t *level, *bin, *band;
    int32_t P, K, n_bands;
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
    int32_t fov;  // foveated rendering mode bits (gf_render_desc.foveation: 1 levels, 2 continuous)
    float fov_gaze[2], fov_f0, fov_slope, fov_jitter, fov_lfmax[8];  // fov_lfmax: gf_scene_info.level_fmax
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
    uint32_t* pix;
    int32_t* ffk;    // free flight: the bin of the first crossing (pass A -> pass B)
    double* ffc;     // free flight: tau before that bin
    uint32_t* ffg;   // free flight: the groups with chords overlapping that bin (pass B's traversal mask)
    float* fkap;     // free flight: kappa at the path's last collision (0: unknown), the next pass A's first cut
    uint32_t* pmask; // stochastic extension masks of the current depth (k_policy) ...
    float* pw;       // ... and their group weights, kMaxGroups per path
    uint32_t *skey, *skey2, *sval;  // extension-ray reordering (R.reorder): keys, sorted keys, path ids
    void* sort_temp;                // CUB temp storage of that sort
    size_t sort_bytes;
    float4* wrec;    // [warp][rec_cap] x 2 float4 hit records (pass-B windows, tracking; reused per path)
    float4* waux;    // [warp][rec_cap] per-record full integral, amp G(u0), amp cos, -amp sin
    int32_t rec_cap;
    uint32_t* wref;  // [warp][kRefWarp] hit lists of pass A (primitive index | group << 27)
    uint32_t* qW;    // paths that collide: pass B queue
    uint32_t* qO;    // paths with more chords than the record buffer (one-pass / tracking -> passes A + B)
    uint32_t* qV;    // pass-B windows with more chords than the record buffer (k_ffb_over)
    // gf_trace_free_flight (mode 2): the caller's rays (n x 8) and output distances, else null
    const float* trays;
    float* tout;
    int32_t packets;  // 0: packets for depth-0 camera rays; 1: always (static masks); 2: never
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
    // queues
    uint32_t *qA, *qB, *qNext;
    uint32_t* qcount;  // [16]: queue counts and work cursors (gf_render.cu QC_* / CUR_*)
    unsigned long long* rays;  // [3]: camera, extension, NEE rays
    float* accum;
    unsigned long long* work;  // gf_stats work counters (counting variant) or null
    // (appended last, so the hot kernels' parameter offsets stay as measured)
    int32_t tomo_pkt_min;  // tomography chunks with at least this many paths take k_tomo_pkt
    int32_t ffb_cam;       // pass B of depth-0 rays walks the camera BVH (1) or the world BVH (0)
    int32_t ff_win;        // pass A of extension rays in windows: 0 one sweep; 1 split at the bin predicted from
                           // kappa at the path's last collision; 2 windows of 1, 2, 4, .. bins on every ray
    int32_t reorder;       // sort extension rays by direction octant and origin before pass A (A/B)
    float win_scale;       // ff_win 1: the split bin is win_scale x the predicted crossing bin
};

cudaError_t gf_launch_load(const LoadArgs& A, void* out, uint8_t* group, uint32_t* err, uint32_t* lfmax_bits,
                           cudaStream_t st);
cudaError_t gf_launch_group_f0(const gfk::GPrim* prims, const uint8_t* group, int64_t n, int P, int K, int G0,
                               const BuildScratch& S, float* f0_dev, cudaStream_t st);
cudaError_t gf_launch_mb_mask(const gfk::GPrim* prims, const uint8_t* group, int64_t n, int32_t G, int32_t G0,
                              const float* dir, float m, float threshold, void* dev_scratch, uint32_t* mask_host,
                              float* att_host, cudaStream_t st);
size_t gf_mb_scratch_bytes();
cudaError_t gf_launch_adaptive_extent(const float* scale, const float* alpha, const float* omega, int64_t n, float eps,
                                      float* out, cudaStream_t st);
cudaError_t gf_launch_hash(const void* data, size_t bytes, unsigned long long* out_dev, cudaStream_t st);
size_t gf_sort_temp_bytes(int64_t n);
BuildScratch gf_scratch_layout(int64_t n, char* base);
// Key prefix of each group in the LBVH keys (prefix << 57 | Morton): the group itself, or its
// (band, level) class (gf_set_bvh_keys)
struct KeyMap {
    uint8_t k[gfk::kMaxGroups];
};
KeyMap gf_keymap(const gfk::SceneDev& sc, int mode);
cudaError_t gf_launch_build(const void* prims, const uint8_t* group, int64_t n, const BuildScratch& S, void* nodes,
                            void* nodes2, void* sorted, int32_t* perm, uint32_t* n_nodes, uint32_t* max_depth,
                            float* root_box, const KeyMap& km, cudaStream_t st);
cudaError_t gf_launch_build_frame(const void* prims, const uint8_t* group, int64_t n, const BuildScratch& S,
                                  const float* F, const float* eye, void* nodes, void* nodes2, void* sorted,
                                  int32_t* perm, uint32_t* depth, const KeyMap& km, cudaStream_t st);
cudaError_t gf_launch_trace(const TraceArgs& A, bool brute, bool count, cudaStream_t st);
cudaError_t gf_launch_candidates(const TraceArgs& A, bool brute, cudaStream_t st);
cudaError_t gf_launch_grad_alpha(const TraceArgs& A, const float* dl, float* grad, cudaStream_t st);
cudaError_t gf_launch_grad_params(const TraceArgs& A, const float* dl, float* acc, bool packets, cudaStream_t st);
cudaError_t gf_launch_grad_finish(const gfk::GPrim* prims, int64_t n, const float* acc, const float* quat, float* grad,
                                  cudaStream_t st);
size_t gf_render_state_bytes(int64_t n_paths, int64_t n_prims, char* base, RenderDev* R, BuildScratch* light_scratch);
cudaError_t gf_launch_render_pass(RenderDev& R, int32_t sample, int32_t sample_slot, cudaStream_t st,
                                  StageTimer& T);
