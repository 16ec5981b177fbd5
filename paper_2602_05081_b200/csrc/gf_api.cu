// gf_api.cu -- the C ABI (include/gf.h): context, validation, workspaces, orchestration.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "gf.h"
#include "gf_internal.h"

using namespace gfk;

struct gf_ctx {
    int device = 0;
    int32_t bvh_keys = GF_BVH_KEYS_LEVEL;  // gf_set_bvh_keys
    std::string err;
    uint32_t* d_err = nullptr;            // [4] load error bits, first bad index
    unsigned long long* d_rays = nullptr;  // [3] dummy ray counters
    uint32_t* d_lfmax = nullptr;           // [8] per-level max |omega_vec| (float bits, F3)
    float* d_f0 = nullptr;                 // [8] per-level representative whitened frequency (C12)
    void* d_mb = nullptr;                  // motion-blur reduction scratch
    unsigned long long* d_hash = nullptr;  // BVH hash
    float lfmax[8] = {};
    bool f0_given = false;
    // scene
    bool loaded = false, built = false;
    int64_t n = 0;
    SceneDev sc{};
    GPrim* prims = nullptr;    // input order (prim_ws)
    uint8_t* group = nullptr;  // input-order group ids (prim_ws, after the records)
    GNode* nodes = nullptr;    // bvh_ws
    GPrim* sorted = nullptr;
    int32_t* perm = nullptr;   // sorted -> input index (bvh_ws, after the nodes)
    GNode2* nodes2 = nullptr;  // children pairs (bvh_ws, after perm)
    uint32_t n_nodes = 0;
    uint32_t max_depth = 0;
    int32_t stk_limit = 0;
    float root[6] = {0, 0, 0, 0, 0, 0};
    // policies
    gf_lod_policy ext{0xFFFFFFFFu, 0, 0.0f, 0, 1.0f}, nee{0xFFFFFFFFu, 0, 0.0f, 0, 1.0f};
    PolicyDev dext{}, dnee{};
    // measurement
    uint32_t prof = 0;
    StageTimer timer;
    unsigned long long* d_work = nullptr;  // [8 stages][kWorkSlots]
    double stage_ms[N_STAGES] = {};
    // scene generation (bumped by load/build) and the frame BVHs gf_render left in a scratch buffer
    uint64_t gen = 0;
    struct FrameCache {
        const char* base = nullptr;   // scratch buffer the BVH was built in
        size_t layout = 0;            // its chunk layout (bytes of the render state)
        uint64_t gen = ~0ull;
        float key[12] = {};
    } light_cache[4], cam_cache[4];  // per scratch buffer (up to 4 in flight, e.g. one per stream)
};

// A gf_render call writes [base, base + layout) of its scratch: drop every cached frame BVH that
// another layout placed inside that range (its nodes are overwritten by this call's per-path state).
static void frame_invalidate(gf_ctx::FrameCache* fcs, const char* base, size_t layout) {
    for (int i = 0; i < 4; ++i) {
        gf_ctx::FrameCache& f = fcs[i];
        if (!f.base || (f.base == base && f.layout == layout)) continue;
        if (f.base < base + layout && base < f.base + f.layout) f = gf_ctx::FrameCache{};
    }
}
// true if the frame BVH of (scratch base, layout, scene generation, key floats) is already there;
// otherwise records it as built now
static bool frame_cached(gf_ctx::FrameCache* fcs, const char* base, size_t layout, uint64_t gen, const float* key,
                         int nkey) {
    frame_invalidate(fcs, base, layout);
    gf_ctx::FrameCache* fc = nullptr;
    for (int i = 0; i < 4 && !fc; ++i)
        if (fcs[i].base == base && fcs[i].layout == layout) fc = fcs + i;
    if (!fc) {  // new scratch buffer: take a free slot, else the first (round robin)
        for (int i = 0; i < 4 && !fc; ++i)
            if (!fcs[i].base) fc = fcs + i;
        if (!fc) {
            for (int i = 0; i < 3; ++i) fcs[i] = fcs[i + 1];
            fc = fcs + 3;
        }
        fc->gen = ~0ull;
    }
    bool same = fc->base == base && fc->layout == layout && fc->gen == gen;
    for (int k = 0; k < nkey && same; ++k) same = fc->key[k] == key[k];
    fc->base = base;
    fc->layout = layout;
    fc->gen = gen;
    for (int k = 0; k < nkey; ++k) fc->key[k] = key[k];
    return same;
}

cudaEvent_t StageTimer::ev() {
    if (pool_used == pool.size()) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        pool.push_back(e);
    }
    return pool[pool_used++];
}
void StageTimer::pre(int stage, cudaStream_t st, cudaEvent_t& a) {
    ++launches;
    ++stage_launches[stage];
    if (!on) return;
    a = ev();
    cudaEventRecord(a, st);
}
void StageTimer::post(int stage, cudaStream_t st, cudaEvent_t a) {
    if (!on) return;
    cudaEvent_t b = ev();
    cudaEventRecord(b, st);
    recs.push_back({stage, a, b});
}

// fold recorded events into per-stage milliseconds (synchronises on the events)
static void harvest(gf_ctx* c) {
    StageTimer& T = c->timer;
    for (auto& r : T.recs) {
        float ms = 0.0f;
        cudaEventSynchronize(r.b);
        cudaEventElapsedTime(&ms, r.a, r.b);
        c->stage_ms[r.stage] += ms;
    }
    T.recs.clear();
    T.pool_used = 0;
}

static gf_status fail(gf_ctx* c, gf_status s, const std::string& msg) {
    if (c) c->err = msg;
    return s;
}
static gf_status cuda_fail(gf_ctx* c, cudaError_t e, const char* where) {
    return fail(c, GF_E_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}
#define GF_CUDA(c, call, where)                              \
    do {                                                     \
        cudaError_t e_ = (call);                             \
        if (e_ != cudaSuccess) return cuda_fail(c, e_, where); \
    } while (0)

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// Test-only overrides (environment, read per call): GF_DEBUG_REC_CAP=n lowers k_ff's record
// capacity so paths take the single-pass fallback; GF_DEBUG_STK_LIMIT=n lowers the warp
// traversal's stack threshold so it runs its depth-first (one node per step) mode.
static int env_int(const char* name, int dflt) {
    const char* v = getenv(name);
    return (v && *v) ? atoi(v) : dflt;
}
static int32_t stk_limit_of(const gf_ctx* c) {
    return std::max(1, std::min<int32_t>(c->stk_limit, env_int("GF_DEBUG_STK_LIMIT", c->stk_limit)));
}

static PolicyDev make_policy_dev(const gf_lod_policy& p, int P) {
    PolicyDev d{};
    d.static_mask = p.static_mask;
    d.ls = p.level_strategy;
    d.os = p.orient_strategy;
    d.delta = p.delta;
    const double om = 1.0 - (double)p.beta;  // same expression as the decision rule
    for (int j = 0; j <= P && j <= kMaxLevels; ++j) d.th[j] = std::pow((double)j / P, om);
    for (int j = 0; j < P && j < kMaxLevels; ++j) {
        d.w_pl[j] = (float)(1.0 / (std::pow((double)(j + 1) / P, om) - std::pow((double)j / P, om)));
        d.w_acc[j] = (float)(1.0 / (1.0 - std::pow((double)j / P, om)));
    }
    if (P > 1) {
        const int Q = P - 1;
        for (int k = 0; k <= Q && k <= kMaxLevels; ++k) d.psi[k] = std::pow((double)k / Q, om);
        for (int k = 0; k < Q && k < kMaxLevels; ++k)
            d.w_plcv[k] = (float)(1.0 / (std::pow((double)(k + 1) / Q, om) - std::pow((double)k / Q, om)));
    }
    return d;
}

static gf_status check_policy(gf_ctx* c, const gf_lod_policy& p) {
    if (p.level_strategy < 0 || p.level_strategy > 5 || p.orient_strategy < 0 || p.orient_strategy > 4)
        return fail(c, GF_E_INVALID_STRATEGY, "unknown strategy");
    if (!(p.beta >= 0.0f && p.beta < 1.0f)) return fail(c, GF_E_INVALID_STRATEGY, "beta must be in [0,1)");
    if (!(p.delta >= 0.0f && p.delta <= 1.0f)) return fail(c, GF_E_INVALID_STRATEGY, "delta must be in [0,1]");
    return GF_OK;
}

static gf_status check_sticky(gf_ctx* c) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(c, e, "pending CUDA error");
    return GF_OK;
}

extern "C" {

int gf_abi_version(void) { return GF_ABI_VERSION; }

gf_status gf_set_bvh_keys(gf_ctx* c, int32_t keys) {
    if (!c) return GF_E_INVALID_ARGUMENT;
    if (keys != GF_BVH_KEYS_GROUP && keys != GF_BVH_KEYS_LEVEL) return fail(c, GF_E_INVALID_ARGUMENT, "bad bvh keys");
    c->bvh_keys = keys;
    return GF_OK;
}

const char* gf_status_string(gf_status s) {
    switch (s) {
    case GF_OK: return "ok";
    case GF_E_INVALID_ARGUMENT: return "invalid argument";
    case GF_E_STATE: return "invalid call order";
    case GF_E_SINGULAR_COVARIANCE: return "singular covariance";
    case GF_E_INVALID_RAY: return "invalid ray";
    case GF_E_INVALID_BOUNDS: return "invalid bounds";
    case GF_E_MASK_OVERFLOW: return "mask overflow";
    case GF_E_INVALID_STRATEGY: return "invalid strategy";
    case GF_E_ASSIGNMENT: return "assignment error";
    case GF_E_CUDA: return "CUDA error";
    case GF_E_OUT_OF_MEMORY: return "workspace too small";
    }
    return "unknown status";
}

gf_status gf_create(int cuda_device, gf_ctx** out) {
    if (!out) return GF_E_INVALID_ARGUMENT;
    *out = nullptr;
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || cuda_device < 0 || cuda_device >= ndev) return GF_E_CUDA;
    if ((e = cudaSetDevice(cuda_device)) != cudaSuccess) return GF_E_CUDA;
    gf_ctx* c = new gf_ctx();
    c->device = cuda_device;
    if (cudaMalloc(&c->d_err, 4 * sizeof(uint32_t)) != cudaSuccess ||
        cudaMalloc(&c->d_rays, 3 * sizeof(unsigned long long)) != cudaSuccess ||
        cudaMalloc(&c->d_lfmax, 8 * sizeof(uint32_t)) != cudaSuccess ||
        cudaMalloc(&c->d_f0, 8 * sizeof(float)) != cudaSuccess ||
        cudaMalloc(&c->d_mb, gf_mb_scratch_bytes()) != cudaSuccess ||
        cudaMalloc(&c->d_hash, sizeof(unsigned long long)) != cudaSuccess ||
        cudaMalloc(&c->d_work, 8 * kWorkSlots * sizeof(unsigned long long)) != cudaSuccess ||
        cudaMemset(c->d_work, 0, 8 * kWorkSlots * sizeof(unsigned long long)) != cudaSuccess) {
        delete c;
        return GF_E_CUDA;
    }
    c->dext = make_policy_dev(c->ext, 4);
    c->dnee = make_policy_dev(c->nee, 4);
    *out = c;
    return GF_OK;
}

void gf_destroy(gf_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    harvest(c);
    for (cudaEvent_t e : c->timer.pool) cudaEventDestroy(e);
    cudaFree(c->d_err);
    cudaFree(c->d_rays);
    cudaFree(c->d_lfmax);
    cudaFree(c->d_f0);
    cudaFree(c->d_mb);
    cudaFree(c->d_hash);
    cudaFree(c->d_work);
    delete c;
}

const char* gf_last_error(const gf_ctx* c) { return c ? c->err.c_str() : "null context"; }

gf_status gf_query_workspace(int64_t n, size_t* prim_bytes, size_t* bvh_bytes, size_t* scratch_bytes) {
    if (n < 0 || n >= (1 << 24)) return GF_E_INVALID_ARGUMENT;
    const size_t n1 = (size_t)std::max<int64_t>(n, 1);
    if (prim_bytes) *prim_bytes = align256(sizeof(GPrim) * n1) + align256(n1);
    if (bvh_bytes)
        *bvh_bytes = align256(sizeof(GPrim) * n1) + align256(sizeof(GNode) * 2 * n1) + align256(sizeof(int32_t) * n1) +
                     align256(sizeof(GNode2) * 2 * n1);
    if (scratch_bytes) {
        if (n > 0) {
            int ndev = 0;
            if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return GF_E_CUDA;
        }
        *scratch_bytes = gf_scratch_layout(n, nullptr).total_bytes;
    }
    return GF_OK;
}

gf_status gf_load_primitives(gf_ctx* c, const gf_prims* p, int64_t n, const gf_pyramid* pyr, void* prim_ws,
                             size_t bytes, gf_stream stream) {
    if (!c) return GF_E_INVALID_ARGUMENT;
    if (!p || !pyr || n < 0) return fail(c, GF_E_INVALID_ARGUMENT, "null argument or n < 0");
    if (n >= (1 << 24)) return fail(c, GF_E_INVALID_ARGUMENT, "n must be < 2^24");
    if (n > 0 && (!p->mu || !p->quat || !p->scale || !p->alpha || !p->omega || !prim_ws))
        return fail(c, GF_E_INVALID_ARGUMENT, "null primitive array");
    const int P = pyr->n_levels, K = pyr->n_bins, B = std::max(1, (int)pyr->n_bands);
    if (P < 1 || P > kMaxLevels || K < 1 || K > 16 || pyr->n_bands < 0)
        return fail(c, GF_E_INVALID_ARGUMENT, "bad n_levels / n_bins / n_bands");
    if (B * (1 + (P - 1) * K) > GF_MAX_GROUPS) return fail(c, GF_E_MASK_OVERFLOW, "n_bands (1 + (P-1) K) > 32 groups");
    if (!pyr->bin_axes) return fail(c, GF_E_INVALID_ARGUMENT, "bin_axes required");
    if (n > 0 && !p->level && P > 2 && !pyr->level_cutoffs)
        return fail(c, GF_E_INVALID_ARGUMENT, "level_cutoffs required when level == NULL");
    size_t need = 0;
    gf_query_workspace(n, &need, nullptr, nullptr);
    if (bytes < need) return fail(c, GF_E_OUT_OF_MEMORY, "prim_ws too small");
    GF_CUDA(c, cudaSetDevice(c->device), "cudaSetDevice");
    if (gf_status s = check_sticky(c)) return s;
    cudaStream_t st = (cudaStream_t)stream;
    c->loaded = c->built = false;
    LoadArgs A{};
    A.n = n; A.mu = p->mu; A.quat = p->quat; A.scale = p->scale; A.alpha = p->alpha; A.omega = p->omega;
    A.extent = p->extent; A.level = p->level; A.bin = p->bin; A.band = p->band; A.P = P; A.K = K; A.n_bands = B;
    for (int i = 0; i < P - 2 && pyr->level_cutoffs; ++i) A.cutoffs[i] = pyr->level_cutoffs[i];
    for (int i = 0; i < 3 * K; ++i) A.axes[i] = pyr->bin_axes[i];
    uint32_t init[4] = {0u, 0xFFFFFFFFu, 0u, 0u};
    GF_CUDA(c, cudaMemcpyAsync(c->d_err, init, sizeof(init), cudaMemcpyHostToDevice, st), "memcpy");
    uint8_t* gptr = (uint8_t*)prim_ws + align256(sizeof(GPrim) * (size_t)std::max<int64_t>(n, 1));
    GF_CUDA(c, cudaMemsetAsync(c->d_lfmax, 0, 8 * sizeof(uint32_t), st), "memset");
    GF_CUDA(c, gf_launch_load(A, prim_ws, gptr, c->d_err, c->d_lfmax, st), "k_load_prims");
    uint32_t herr[4], hlf[8];
    GF_CUDA(c, cudaMemcpyAsync(herr, c->d_err, sizeof(herr), cudaMemcpyDeviceToHost, st), "memcpy");
    GF_CUDA(c, cudaMemcpyAsync(hlf, c->d_lfmax, sizeof(hlf), cudaMemcpyDeviceToHost, st), "memcpy");
    GF_CUDA(c, cudaStreamSynchronize(st), "load sync");
    if (herr[0]) {
        char msg[160];
        snprintf(msg, sizeof(msg), "invalid primitive (first index %u, error bits 0x%x)", herr[1], herr[0]);
        if (herr[0] & 1u) return fail(c, GF_E_SINGULAR_COVARIANCE, msg);
        if (herr[0] & 2u) return fail(c, GF_E_INVALID_BOUNDS, msg);
        if (herr[0] & 12u) return fail(c, GF_E_ASSIGNMENT, msg);
        return fail(c, GF_E_INVALID_ARGUMENT, msg);
    }
    c->n = n;
    c->sc.P = P; c->sc.K = K; c->sc.G0 = 1 + (P - 1) * K; c->sc.n_bands = B; c->sc.G = B * c->sc.G0;
    for (int i = 0; i < 3 * K; ++i) c->sc.axes[i] = pyr->bin_axes[i];
    c->f0_given = pyr->group_f0 != nullptr;  // else medians computed by gf_build_bvh (C12)
    for (int g = 0; g < kMaxGroups; ++g) c->sc.f0[g] = (pyr->group_f0 && g < c->sc.G) ? pyr->group_f0[g] : 0.0f;
    for (int l = 0; l < 8; ++l) { float f; std::memcpy(&f, hlf + l, 4); c->lfmax[l] = f; }
    c->prims = (GPrim*)prim_ws;
    c->group = gptr;
    c->dext = make_policy_dev(c->ext, P);
    c->dnee = make_policy_dev(c->nee, P);
    c->loaded = true;
    ++c->gen;
    return GF_OK;
}

gf_status gf_build_bvh(gf_ctx* c, void* bvh_ws, size_t bvh_bytes, void* scratch, size_t scratch_bytes,
                       gf_stream stream) {
    if (!c) return GF_E_INVALID_ARGUMENT;
    if (!c->loaded) return fail(c, GF_E_STATE, "gf_build_bvh before gf_load_primitives");
    size_t nb = 0, ns = 0;
    if (gf_status s = gf_query_workspace(c->n, nullptr, &nb, &ns)) return fail(c, s, "workspace query failed");
    if (c->n > 0 && (!bvh_ws || !scratch)) return fail(c, GF_E_INVALID_ARGUMENT, "null workspace");
    if (bvh_bytes < nb || scratch_bytes < ns) return fail(c, GF_E_OUT_OF_MEMORY, "bvh_ws or scratch too small");
    GF_CUDA(c, cudaSetDevice(c->device), "cudaSetDevice");
    if (gf_status s = check_sticky(c)) return s;
    cudaStream_t st = (cudaStream_t)stream;
    char* base = (char*)bvh_ws;
    const size_t n1 = (size_t)std::max<int64_t>(c->n, 1);
    c->sorted = (GPrim*)base;
    c->nodes = (GNode*)(base + align256(sizeof(GPrim) * n1));
    c->perm = (int32_t*)(base + align256(sizeof(GPrim) * n1) + align256(sizeof(GNode) * 2 * n1));
    c->nodes2 = (GNode2*)(base + align256(sizeof(GPrim) * n1) + align256(sizeof(GNode) * 2 * n1) +
                          align256(sizeof(int32_t) * n1));
    BuildScratch S = gf_scratch_layout(c->n, (char*)scratch);
    if (!c->f0_given) {  // C12: sqrt(3) x the median omega of each level, on the device (radix sort)
        float f0l[8];
        GF_CUDA(c, gf_launch_group_f0(c->prims, c->group, c->n, c->sc.P, c->sc.K, c->sc.G0, S, c->d_f0, st), "group f0");
        GF_CUDA(c, cudaMemcpyAsync(f0l, c->d_f0, sizeof(f0l), cudaMemcpyDeviceToHost, st), "memcpy");
        GF_CUDA(c, cudaStreamSynchronize(st), "group f0 sync");
        for (int g = 0; g < kMaxGroups; ++g) {
            const int gl = g % c->sc.G0;
            c->sc.f0[g] = (g < c->sc.G && gl > 0) ? f0l[1 + (gl - 1) / c->sc.K] : 0.0f;
        }
    }
    uint32_t nn = 0, md = 0;
    GF_CUDA(c, gf_launch_build(c->prims, c->group, c->n, S, c->nodes, c->nodes2, c->sorted, c->perm, &nn, &md, c->root,
                               gf_keymap(c->sc, c->bvh_keys), st),
            "gf_build_bvh");
    // warp traversal stack bound (gf_device.cuh: warp_traverse)
    if ((int)md + 34 + 64 > kWStk) return fail(c, GF_E_INVALID_ARGUMENT, "BVH deeper than the traversal stack allows");
    c->n_nodes = nn;
    c->max_depth = md;
    c->stk_limit = kWStk - 34 - (int)md;
    c->built = true;
    ++c->gen;
    return GF_OK;
}

gf_status gf_scene_info_get(gf_ctx* c, gf_scene_info* out) {
    if (!c || !out) return GF_E_INVALID_ARGUMENT;
    if (!c->loaded) return fail(c, GF_E_STATE, "gf_scene_info_get before gf_load_primitives");
    GF_CUDA(c, cudaSetDevice(c->device), "cudaSetDevice");
    if (gf_status s = check_sticky(c)) return s;
    std::memset(out, 0, sizeof(*out));
    out->n_prims = c->n;
    out->n_levels = c->sc.P;
    out->n_bins = c->sc.K;
    out->n_bands = c->sc.n_bands;
    out->n_groups = c->sc.G;
    for (int l = 0; l < 8; ++l) out->level_fmax[l] = c->lfmax[l];
    for (int g = 0; g < kMaxGroups; ++g) out->group_f0[g] = c->built || c->f0_given ? c->sc.f0[g] : 0.0f;
    if (c->built) {
        for (int k = 0; k < 3; ++k) { out->root_lo[k] = c->root[k]; out->root_hi[k] = c->root[3 + k]; }
        out->n_nodes = c->n_nodes;
        out->max_depth = c->max_depth;
        // hash of the tree as built: reordered primitives, nodes, permutation (the child pairs are
        // derived from the nodes; unused tails of the workspace are not hashed)
        cudaStream_t st = nullptr;
        GF_CUDA(c, cudaMemsetAsync(c->d_hash, 0, sizeof(unsigned long long), st), "memset");
        unsigned long long h = 0, part = 0;
        const struct { const void* p; size_t b; } parts[3] = {
            {c->sorted, sizeof(GPrim) * (size_t)c->n}, {c->nodes, sizeof(GNode) * (size_t)c->n_nodes},
            {c->perm, sizeof(int32_t) * (size_t)c->n}};
        for (const auto& pt : parts) {
            GF_CUDA(c, gf_launch_hash(pt.p, pt.b, c->d_hash, st), "hash");
            GF_CUDA(c, cudaMemcpy(&part, c->d_hash, sizeof(part), cudaMemcpyDeviceToHost), "memcpy");
            h = h * 0x100000001B3ull + part;
        }
        out->bvh_hash = h;
    }
    return GF_OK;
}

gf_status gf_motion_blur_mask(gf_ctx* c, const float* dir, float m, float threshold, uint32_t* mask_out,
                              float* att_out) {
    if (!c) return GF_E_INVALID_ARGUMENT;
    if (!dir || !mask_out) return fail(c, GF_E_INVALID_ARGUMENT, "null dir / mask_out");
    if (!c->loaded) return fail(c, GF_E_STATE, "gf_motion_blur_mask before gf_load_primitives");
    if (!(m >= 0.0f) || !std::isfinite(m) || !std::isfinite(threshold) ||
        !(std::fabs(dir[0]) + std::fabs(dir[1]) + std::fabs(dir[2]) > 0.0f))
        return fail(c, GF_E_INVALID_ARGUMENT, "motion blur: m >= 0 finite, dir != 0");
    GF_CUDA(c, cudaSetDevice(c->device), "cudaSetDevice");
    if (gf_status s = check_sticky(c)) return s;
    GF_CUDA(c, gf_launch_mb_mask(c->prims, c->group, c->n, c->sc.G, c->sc.G0, dir, m, threshold, c->d_mb, mask_out,
                                 att_out, nullptr),
            "motion-blur mask");
    return GF_OK;
}

gf_status gf_adaptive_extent(gf_ctx* c, const float* scale, const float* alpha, const float* omega, int64_t n, float eps,
                             float* extent_out, gf_stream stream) {
    if (!c) return GF_E_INVALID_ARGUMENT;
    if (n < 0 || (n > 0 && (!scale || !alpha || !omega || !extent_out)))
        return fail(c, GF_E_INVALID_ARGUMENT, "bad adaptive-extent arrays");
    if (!(eps > 0.0f) || !std::isfinite(eps)) return fail(c, GF_E_INVALID_ARGUMENT, "eps must be > 0");
    GF_CUDA(c, cudaSetDevice(c->device), "cudaSetDevice");
    if (gf_status s = check_sticky(c)) return s;
    GF_CUDA(c, gf_launch_adaptive_extent(scale, alpha, omega, n, eps, extent_out, (cudaStream_t)stream),
            "k_adaptive_extent");
    return GF_OK;
}

gf_status gf_set_lod_mask(gf_ctx* c, const gf_lod_policy* ext, const gf_lod_policy* nee) {
    if (!c) return GF_E_INVALID_ARGUMENT;
    if (!ext) return fail(c, GF_E_INVALID_ARGUMENT, "ext policy required");
    if (gf_status s = check_policy(c, *ext)) return s;
    if (nee)
        if (gf_status s = check_policy(c, *nee)) return s;
    c->ext = *ext;
    c->nee = nee ? *nee : *ext;
    const int P = c->loaded ? c->sc.P : 4;
    c->dext = make_policy_dev(c->ext, P);
    c->dnee = make_policy_dev(c->nee, P);
    return GF_OK;
}

static gf_status trace_common(gf_ctx* c, const float* rays, int64_t n, TraceArgs& A, uint32_t flags) {
    if (!c) return GF_E_INVALID_ARGUMENT;
    if (!c->loaded || (!c->built && !(flags & GF_TRACE_BRUTE_FORCE)))
        return fail(c, GF_E_STATE, "trace before gf_load_primitives / gf_build_bvh");
    if (n < 0 || (n > 0 && !rays)) return fail(c, GF_E_INVALID_ARGUMENT, "bad rays");
    if (((uintptr_t)rays & 15u) != 0) return fail(c, GF_E_INVALID_ARGUMENT, "rays must be 16-byte aligned");
    GF_CUDA(c, cudaSetDevice(c->device), "cudaSetDevice");
    if (gf_status s = check_sticky(c)) return s;
    A = TraceArgs{};
    const bool brute = flags & GF_TRACE_BRUTE_FORCE;
    A.nodes = c->nodes;
    A.nodes2 = c->nodes2;
    A.stk_limit = stk_limit_of(c);
    A.n_nodes = c->built ? c->n_nodes : 0;
    A.prims = brute ? c->prims : c->sorted;
    A.group = c->group;
    A.perm = c->perm;
    A.n_prims = c->n;
    A.pol = c->dext;
    A.sc = c->sc;
    A.rays = rays;
    A.n = n;
    return GF_OK;
}

gf_status gf_trace_transmittance_ex(gf_ctx* c, const float* rays, int64_t n, uint64_t seed, uint32_t flags,
                                    float* tau_out, float* T_out, uint32_t* counters, gf_stream stream) {
    TraceArgs A;
    if (gf_status s = trace_common(c, rays, n, A, flags)) return s;
    if (n > 0 && !tau_out) return fail(c, GF_E_INVALID_ARGUMENT, "tau_out required");
    A.seed = seed;
    A.tau = tau_out;
    A.T = T_out;
    A.counters = counters;
    A.work = (c->prof & GF_PROFILE_WORK) ? c->d_work : nullptr;
    cudaEvent_t ev;
    c->timer.pre(STAGE_TRACE, (cudaStream_t)stream, ev);
    GF_CUDA(c, gf_launch_trace(A, flags & GF_TRACE_BRUTE_FORCE, counters != nullptr, (cudaStream_t)stream),
            "k_trace");
    c->timer.post(STAGE_TRACE, (cudaStream_t)stream, ev);
    return GF_OK;
}

gf_status gf_trace_transmittance(gf_ctx* c, const float* rays, int64_t n, uint64_t seed, float* tau_out,
                                 float* T_out, uint32_t* counters, gf_stream stream) {
    return gf_trace_transmittance_ex(c, rays, n, seed, 0u, tau_out, T_out, counters, stream);
}

gf_status gf_trace_grad_alpha(gf_ctx* c, const float* rays, int64_t n, uint64_t seed, const float* dl_dtau,
                              float* grad_alpha, gf_stream stream) {
    TraceArgs A;
    if (gf_status s = trace_common(c, rays, n, A, 0u)) return s;
    if (!c->built) return fail(c, GF_E_STATE, "gf_trace_grad_alpha before gf_build_bvh");
    if (n > 0 && (!dl_dtau || !grad_alpha)) return fail(c, GF_E_INVALID_ARGUMENT, "null gradient buffers");
    A.seed = seed;
    GF_CUDA(c, gf_launch_grad_alpha(A, dl_dtau, grad_alpha, (cudaStream_t)stream), "k_grad_alpha");
    return GF_OK;
}

gf_status gf_trace_grad_params(gf_ctx* c, const float* rays, int64_t n, uint64_t seed, uint32_t flags,
                               const float* dl_dtau, float* accum, gf_stream stream) {
    TraceArgs A;
    if (flags & ~GF_TRACE_PACKETS) return fail(c, GF_E_INVALID_ARGUMENT, "bad gf_trace_grad_params flags");
    if (gf_status s = trace_common(c, rays, n, A, 0u)) return s;
    if (!c->built) return fail(c, GF_E_STATE, "gf_trace_grad_params before gf_build_bvh");
    if (n > 0 && (!dl_dtau || !accum)) return fail(c, GF_E_INVALID_ARGUMENT, "null gradient buffers");
    if (((uintptr_t)accum & 15u) != 0) return fail(c, GF_E_INVALID_ARGUMENT, "accum must be 16-byte aligned");
    A.seed = seed;
    GF_CUDA(c, gf_launch_grad_params(A, dl_dtau, accum, (flags & GF_TRACE_PACKETS) != 0, (cudaStream_t)stream),
            "k_grad_params");
    return GF_OK;
}

gf_status gf_grad_params_finish(gf_ctx* c, const float* accum, const float* quat, float* grad, gf_stream stream) {
    if (!c) return GF_E_INVALID_ARGUMENT;
    if (!c->loaded) return fail(c, GF_E_STATE, "gf_grad_params_finish before gf_load_primitives");
    if (c->n > 0 && (!accum || !quat || !grad)) return fail(c, GF_E_INVALID_ARGUMENT, "null gradient buffers");
    if (((uintptr_t)quat & 15u) != 0) return fail(c, GF_E_INVALID_ARGUMENT, "quat must be 16-byte aligned");
    GF_CUDA(c, cudaSetDevice(c->device), "cudaSetDevice");
    GF_CUDA(c, gf_launch_grad_finish(c->prims, c->n, accum, quat, grad, (cudaStream_t)stream), "k_grad_finish");
    return GF_OK;
}

gf_status gf_trace_candidates(gf_ctx* c, const float* rays, int64_t n, uint32_t flags, int32_t* ids,
                              int32_t capacity, int32_t* count, gf_stream stream) {
    TraceArgs A;
    if (gf_status s = trace_common(c, rays, n, A, flags)) return s;
    if (capacity < 0 || (n > 0 && (!count || (capacity > 0 && !ids))))
        return fail(c, GF_E_INVALID_ARGUMENT, "bad candidate buffers");
    A.cand_ids = ids;
    A.cand_cap = capacity;
    A.cand_count = count;
    GF_CUDA(c, gf_launch_candidates(A, flags & GF_TRACE_BRUTE_FORCE, (cudaStream_t)stream), "k_candidates");
    return GF_OK;
}

#ifndef GF_CHUNK_LOG2
#define GF_CHUNK_LOG2 20
#endif
static constexpr int64_t kRenderChunk = 1ll << GF_CHUNK_LOG2;  // paths per wavefront chunk (per-path state ~50 MB at 2^20)

static int64_t render_paths(const gf_render_desc* d) {
    if (d->probe_pixels) return d->n_probe;
    const int64_t tx = (d->width + 31) / 32, ty = (d->height + 31) / 32, tiles = tx * ty;
    if (d->shard_kind == GF_SHARD_TILES) {
        const int64_t mine = tiles > d->shard_rank ? (tiles - d->shard_rank + d->shard_world - 1) / d->shard_world : 0;
        return mine * 1024;
    }
    return tiles * 1024;
}

static gf_status check_desc(gf_ctx* c, const gf_render_desc* d) {
    if (!d) return fail(c, GF_E_INVALID_ARGUMENT, "null desc");
    if (d->mode != GF_MODE_TOMOGRAPHY && d->mode != GF_MODE_SCATTER) return fail(c, GF_E_INVALID_ARGUMENT, "bad mode");
    if (d->width <= 0 || d->height <= 0 || (int64_t)d->width * d->height >= (1ll << 31))
        return fail(c, GF_E_INVALID_ARGUMENT, "bad image size");
    if (d->mode == GF_MODE_SCATTER && (d->max_depth < 1 || d->max_depth > 1024))
        return fail(c, GF_E_INVALID_ARGUMENT, "max_depth must be in [1,1024]");
    if (d->spp_count < 0 || d->spp_begin < 0) return fail(c, GF_E_INVALID_ARGUMENT, "bad spp range");
    if (d->shard_kind < 0 || d->shard_kind > 2) return fail(c, GF_E_INVALID_ARGUMENT, "bad shard kind");
    if (d->shard_kind != GF_SHARD_NONE && (d->shard_world < 1 || d->shard_rank < 0 || d->shard_rank >= d->shard_world))
        return fail(c, GF_E_INVALID_ARGUMENT, "bad shard rank/world");
    if (d->probe_pixels && (d->n_probe < 0 || d->shard_kind == GF_SHARD_TILES))
        return fail(c, GF_E_INVALID_ARGUMENT, "probe mode: n_probe >= 0 and no tile sharding");
    if (!(d->hg_g > -1.0f && d->hg_g < 1.0f)) return fail(c, GF_E_INVALID_ARGUMENT, "hg_g must be in (-1,1)");
    if (d->estimator != GF_EST_ANALYTIC && d->estimator != GF_EST_TRACKING && d->estimator != GF_EST_UNIFORM)
        return fail(c, GF_E_INVALID_ARGUMENT, "bad estimator");
    if (d->motion_blur && !(d->mb_m >= 0.0f && std::isfinite(d->mb_m)))
        return fail(c, GF_E_INVALID_ARGUMENT, "motion blur: mb_m must be finite and >= 0");
    if (d->foveation < 0 || d->foveation > 3) return fail(c, GF_E_INVALID_ARGUMENT, "foveation: mode bits 0..3");
    if (d->foveation && !(d->fov_f0 >= 0.0f && d->fov_slope >= 0.0f && d->fov_jitter >= 0.0f && d->fov_jitter < 1.0f))
        return fail(c, GF_E_INVALID_ARGUMENT, "foveation: f0, slope >= 0 and jitter in [0,1)");
    return GF_OK;
}

gf_status gf_render_scratch_bytes(gf_ctx* c, const gf_render_desc* d, size_t* bytes) {
    if (!c || !bytes) return GF_E_INVALID_ARGUMENT;
    if (gf_status s = check_desc(c, d)) return s;
    *bytes = gf_render_state_bytes(std::min<int64_t>(std::max<int64_t>(render_paths(d), 1), kRenderChunk), c->n,
                                   nullptr, nullptr, nullptr);
    return GF_OK;
}

gf_status gf_render(gf_ctx* c, const gf_render_desc* d, float* accum, void* scratch, size_t scratch_bytes,
                    uint64_t* ray_counts, gf_stream stream) {
    if (!c) return GF_E_INVALID_ARGUMENT;
    if (gf_status s = check_desc(c, d)) return s;
    if (!c->loaded || !c->built) return fail(c, GF_E_STATE, "render before gf_load_primitives / gf_build_bvh");
    const int64_t np = render_paths(d);
    const int64_t chunk = std::min<int64_t>(std::max<int64_t>(np, 1), kRenderChunk);
    size_t need = gf_render_state_bytes(chunk, c->n, nullptr, nullptr, nullptr);
    if (scratch_bytes < need || !scratch) return fail(c, GF_E_OUT_OF_MEMORY, "render scratch too small");
    if (!accum && np > 0) return fail(c, GF_E_INVALID_ARGUMENT, "accum required");
    GF_CUDA(c, cudaSetDevice(c->device), "cudaSetDevice");
    if (gf_status s = check_sticky(c)) return s;
    RenderDev R{};
    BuildScratch LS;
    gf_render_state_bytes(chunk, c->n, (char*)scratch, &R, &LS);
    // this call writes [scratch, scratch + need): frame BVHs another layout left there are gone
    frame_invalidate(c->light_cache, (const char*)scratch, need);
    frame_invalidate(c->cam_cache, (const char*)scratch, need);
    R.rec_cap = std::max(0, std::min(R.rec_cap, env_int("GF_DEBUG_REC_CAP", R.rec_cap)));
    R.nodes = c->nodes;
    R.nodes2 = c->nodes2;
    R.stk_limit = stk_limit_of(c);
    R.n_nodes = c->n_nodes;
    R.prims = c->sorted;
    R.ext = c->dext;
    R.nee = c->dnee;
    R.sc = c->sc;
    for (int k = 0; k < 3; ++k) {
        R.cam.pos[k] = d->cam_pos[k]; R.cam.fwd[k] = d->cam_fwd[k];
        R.cam.right[k] = d->cam_right[k]; R.cam.up[k] = d->cam_up[k];
    }
    R.cam.W = d->width;
    R.cam.H = d->height;
    R.root_lo = make_float4(c->root[0], c->root[1], c->root[2], 0.0f);
    R.root_hi = make_float4(c->root[3], c->root[4], c->root[5], 0.0f);
    R.mode = d->mode;
    R.max_depth = d->mode == GF_MODE_SCATTER ? d->max_depth : 1;
    R.jitter = d->jitter;
    R.estimator = d->estimator;
    R.fov = d->foveation;
    R.fov_gaze[0] = d->fov_gaze[0]; R.fov_gaze[1] = d->fov_gaze[1];
    R.fov_f0 = d->fov_f0; R.fov_slope = d->fov_slope; R.fov_jitter = d->fov_jitter;
    for (int k = 0; k < 8; ++k) R.fov_lfmax[k] = c->lfmax[k];  // F3: the library's per-level maxima
    R.mb = d->motion_blur != 0;
    for (int k = 0; k < 3; ++k) R.mb_dir[k] = d->mb_dir[k];
    R.mb_m = d->mb_m;
    R.albedo = d->albedo; R.hg_g = d->hg_g; R.sun_E = d->sun_E; R.env_L = d->env_L;
    R.sun = make_float3(d->sun_dir[0], d->sun_dir[1], d->sun_dir[2]);
    R.seed = d->seed;
    R.n_total = np;
    R.shard_kind = d->shard_kind;
    R.shard_rank = d->shard_rank;
    R.shard_world = std::max(1, d->shard_world);
    R.tiles_x = (d->width + 31) / 32;
    R.tiles_y = (d->height + 31) / 32;
    R.probe = d->probe_pixels;
    R.spp_count = d->spp_count;
    R.rays = ray_counts ? (unsigned long long*)ray_counts : c->d_rays;
    R.accum = accum;
    R.work = (c->prof & GF_PROFILE_WORK) ? c->d_work : nullptr;
    cudaStream_t st = (cudaStream_t)stream;
    // NEE light BVH: a second tree over the primitives with boxes in a frame whose third axis is
    // the light direction (shadow rays become axis-parallel); rebuilt per call, asynchronously
    R.light = d->mode == GF_MODE_SCATTER && d->estimator != GF_EST_TRACKING && c->n > 0 &&
              env_int("GF_DEBUG_NO_LIGHT_BVH", 0) == 0;
    if (R.light) {
        double z[3] = {d->sun_dir[0], d->sun_dir[1], d->sun_dir[2]};
        const double zn = std::sqrt(z[0] * z[0] + z[1] * z[1] + z[2] * z[2]);
        for (double& v : z) v /= zn;
        const double a[3] = {std::fabs(z[0]) < 0.9 ? 1.0 : 0.0, std::fabs(z[0]) < 0.9 ? 0.0 : 1.0, 0.0};
        double x[3] = {a[1] * z[2] - a[2] * z[1], a[2] * z[0] - a[0] * z[2], a[0] * z[1] - a[1] * z[0]};
        const double xn = std::sqrt(x[0] * x[0] + x[1] * x[1] + x[2] * x[2]);
        for (double& v : x) v /= xn;
        const double y[3] = {z[1] * x[2] - z[2] * x[1], z[2] * x[0] - z[0] * x[2], z[0] * x[1] - z[1] * x[0]};
        for (int k = 0; k < 3; ++k) {
            R.lf[k] = (float)x[k]; R.lf[3 + k] = (float)y[k]; R.lf[6 + k] = (float)z[k];
        }
        if (!frame_cached(c->light_cache, (const char*)scratch, need, c->gen, R.lf, 9) || !d->reuse_accel) {
            GF_CUDA(c, gf_launch_build_frame(c->prims, c->group, c->n, LS, R.lf, nullptr, R.lnodes, R.lnodes2,
                                             R.lprims, R.lperm, R.ldepth, gf_keymap(c->sc, c->bvh_keys), st),
                    "light BVH build");
            c->timer.launches += 7;  // k_bounds, k_keys, k_karras, k_refit, k_layout, k_pair_dev, k_gather (+ CUB)
        }
    }
    // camera BVH for the depth-0 packet kernel (static ext mask, analytic): projective boxes at the eye
    R.camb = (d->mode == GF_MODE_TOMOGRAPHY || d->estimator != GF_EST_TRACKING) && c->n > 0 && !d->motion_blur &&
             env_int("GF_DEBUG_NO_CAMERA_BVH", 0) == 0;  // (motion blur moves the eye per sample)
    // packets pay off once the chunk fills the GPU (small images: one warp per pixel, k_tomo_w)
    R.tomo_pkt_min = env_int("GF_DEBUG_TOMO_PKT_MIN", 1 << 16);
    R.ffb_cam = env_int("GF_FFB_CAM", 1);
    R.ff_win = env_int("GF_FF_WIN", 1);
    R.reorder = env_int("GF_REORDER", 0);
    R.win_scale = 0.1f * (float)env_int("GF_FF_WIN_SCALE10", 12);
    if (R.camb) {
        const float* axes[3] = {d->cam_right, d->cam_up, d->cam_fwd};
        for (int a = 0; a < 3; ++a) {
            const double nn = std::sqrt((double)axes[a][0] * axes[a][0] + (double)axes[a][1] * axes[a][1] +
                                        (double)axes[a][2] * axes[a][2]);
            for (int k = 0; k < 3; ++k) R.cb[3 * a + k] = (float)(axes[a][k] / nn);
        }
        float key[12];
        for (int k = 0; k < 9; ++k) key[k] = R.cb[k];
        for (int k = 0; k < 3; ++k) key[9 + k] = d->cam_pos[k];
        if (!frame_cached(c->cam_cache, (const char*)scratch, need, c->gen, key, 12) || !d->reuse_accel) {
            GF_CUDA(c, gf_launch_build_frame(c->prims, c->group, c->n, LS, R.cb, d->cam_pos, R.cnodes, R.cnodes2,
                                             R.cprims, R.cperm, R.cdepth, gf_keymap(c->sc, c->bvh_keys), st),
                    "camera BVH build");
            c->timer.launches += 7;
        }
    }
    for (int32_t k = 0; k < d->spp_count; ++k) {
        const int32_t s = d->spp_begin + k;
        if (d->shard_kind == GF_SHARD_SAMPLES && (s % R.shard_world) != d->shard_rank) continue;
        for (int64_t base = 0; base < np; base += chunk) {  // bounded scratch: chunks of <= 1M paths
            R.path_base = base;
            R.n_paths = std::min<int64_t>(chunk, np - base);
            GF_CUDA(c, gf_launch_render_pass(R, s, k, st, c->timer), "render pass");
        }
    }
    if (c->timer.recs.size() > 4096) harvest(c);  // bound the event pool
    return GF_OK;
}

gf_status gf_free_flight_scratch_bytes(gf_ctx* c, int64_t n, size_t* bytes) {
    if (!c || !bytes || n < 0) return GF_E_INVALID_ARGUMENT;
    *bytes = gf_render_state_bytes(std::min<int64_t>(std::max<int64_t>(n, 1), kRenderChunk), 0, nullptr, nullptr, nullptr);
    return GF_OK;
}

gf_status gf_trace_free_flight(gf_ctx* c, const float* rays, int64_t n, uint64_t seed, uint32_t flags, float* t_out,
                               void* scratch, size_t scratch_bytes, gf_stream stream) {
    if (!c) return GF_E_INVALID_ARGUMENT;
    if (flags & ~(GF_TRACE_PACKETS | GF_FF_UNIFORM)) return fail(c, GF_E_INVALID_ARGUMENT, "bad gf_trace_free_flight flags");
    if (!c->loaded || !c->built) return fail(c, GF_E_STATE, "free flight before gf_load_primitives / gf_build_bvh");
    if (n < 0 || (n > 0 && (!rays || !t_out || !scratch))) return fail(c, GF_E_INVALID_ARGUMENT, "bad buffers");
    if (((uintptr_t)rays & 15u) != 0) return fail(c, GF_E_INVALID_ARGUMENT, "rays must be 16-byte aligned");
    const int64_t chunk = std::min<int64_t>(std::max<int64_t>(n, 1), kRenderChunk);
    const size_t need = gf_render_state_bytes(chunk, 0, nullptr, nullptr, nullptr);
    if (scratch_bytes < need) return fail(c, GF_E_OUT_OF_MEMORY, "free-flight scratch too small");
    GF_CUDA(c, cudaSetDevice(c->device), "cudaSetDevice");
    if (gf_status s = check_sticky(c)) return s;
    RenderDev R{};
    gf_render_state_bytes(chunk, 0, (char*)scratch, &R, nullptr);
    frame_invalidate(c->light_cache, (const char*)scratch, need);
    frame_invalidate(c->cam_cache, (const char*)scratch, need);
    R.rec_cap = std::max(0, std::min(R.rec_cap, env_int("GF_DEBUG_REC_CAP", R.rec_cap)));
    R.nodes = c->nodes;
    R.nodes2 = c->nodes2;
    R.stk_limit = stk_limit_of(c);
    R.n_nodes = c->n_nodes;
    R.prims = c->sorted;
    R.ext = c->dext;
    R.nee = c->dnee;
    R.sc = c->sc;
    R.root_lo = make_float4(c->root[0], c->root[1], c->root[2], 0.0f);
    R.root_hi = make_float4(c->root[3], c->root[4], c->root[5], 0.0f);
    R.mode = 2;
    R.max_depth = 1;
    R.seed = seed;
    R.n_total = n;
    R.rays = c->d_rays;
    R.work = (c->prof & GF_PROFILE_WORK) ? c->d_work : nullptr;
    R.trays = rays;
    R.tout = t_out;
    R.packets = (flags & GF_TRACE_PACKETS) ? 1 : 2;
    R.estimator = (flags & GF_FF_UNIFORM) ? GF_EST_UNIFORM : GF_EST_ANALYTIC;
    cudaStream_t st = (cudaStream_t)stream;
    for (int64_t base = 0; base < n; base += chunk) {
        R.path_base = base;
        R.n_paths = std::min<int64_t>(chunk, n - base);
        GF_CUDA(c, gf_launch_render_pass(R, 0, 0, st, c->timer), "free flight");
    }
    if (c->timer.recs.size() > 4096) harvest(c);
    return GF_OK;
}

gf_status gf_set_profiling(gf_ctx* c, uint32_t flags) {
    if (!c) return GF_E_INVALID_ARGUMENT;
    if (flags & ~(GF_PROFILE_TIMING | GF_PROFILE_WORK)) return fail(c, GF_E_INVALID_ARGUMENT, "bad flags");
    GF_CUDA(c, cudaSetDevice(c->device), "cudaSetDevice");
    c->prof = flags;
    c->timer.on = (flags & GF_PROFILE_TIMING) != 0;
    return GF_OK;
}

gf_status gf_get_stats(gf_ctx* c, gf_stats* out, int32_t reset) {
    if (!c || !out) return GF_E_INVALID_ARGUMENT;
    GF_CUDA(c, cudaSetDevice(c->device), "cudaSetDevice");
    GF_CUDA(c, cudaDeviceSynchronize(), "sync");
    harvest(c);
    std::memset(out, 0, sizeof(*out));
    out->launches = c->timer.launches;
    for (int s = 0; s < N_STAGES; ++s) {
        out->stage_launches[s] = c->timer.stage_launches[s];
        out->stage_ms[s] = c->stage_ms[s];
    }
    unsigned long long w[8 * kWorkSlots];
    GF_CUDA(c, cudaMemcpy(w, c->d_work, sizeof(w), cudaMemcpyDeviceToHost), "memcpy");
    for (int i = 0; i < 8 * kWorkSlots; ++i) out->work[i / kWorkSlots][i % kWorkSlots] = w[i];
    if (reset) {
        c->timer.launches = 0;
        for (int s = 0; s < N_STAGES; ++s) { c->timer.stage_launches[s] = 0; c->stage_ms[s] = 0.0; }
        GF_CUDA(c, cudaMemset(c->d_work, 0, sizeof(w)), "memset");
    }
    return GF_OK;
}

int32_t gf_shard_pixel_owner(int32_t px, int32_t py, int32_t width, int32_t height, int32_t world) {
    if (px < 0 || py < 0 || px >= width || py >= height || world < 1) return -1;
    const int32_t tx = (width + 31) / 32;
    const int64_t tile = (int64_t)(py / 32) * tx + (px / 32);
    return (int32_t)(tile % world);
}

int64_t gf_shard_paths(int32_t width, int32_t height, int32_t kind, int32_t rank, int32_t world) {
    if (width <= 0 || height <= 0 || kind < 0 || kind > 2 || world < 1 || rank < 0 || rank >= world) return -1;
    gf_render_desc d{};
    d.width = width; d.height = height; d.shard_kind = kind; d.shard_rank = rank; d.shard_world = world;
    return render_paths(&d);
}

int32_t gf_shard_path_pixel(int64_t p, int32_t width, int32_t height, int32_t kind, int32_t rank, int32_t world) {
    if (width <= 0 || height <= 0 || world < 1 || rank < 0 || rank >= world) return -1;
    return shard_path_pixel(p, width, height, kind, rank, world);
}

int32_t gf_shard_sample_owner(int32_t s, int32_t world) {
    if (s < 0 || world < 1) return -1;
    return s % world;
}

}  // extern "C"
