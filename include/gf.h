/*
 * gf.h -- C ABI of the B200-native Gabor Fields hot path (arXiv 2602.05081).
 *
 * One shared library, libgf.so (paper_2602_05081_b200/libgf.so), hand-written
 * sm_100a CUDA kernels behind plain C entry points: no torch types, only
 * pointers, sizes and a CUDA stream handle.  Citations "P:Lnnn" are lines of
 * PAPER.md; "C<n>" are the readings listed in DESIGN.md §3.
 *
 * Conventions (all entry points):
 *  - Memory ownership: the CALLER allocates every buffer (the library never
 *    calls cudaMalloc after gf_create).  Pointers documented as "device" must
 *    be device (or managed) memory of the context's device; "host" pointers are
 *    read during the call only.  The context keeps non-owning pointers to the
 *    workspaces passed to gf_load_primitives / gf_build_bvh; they must outlive
 *    the context or the next gf_load_primitives.
 *  - Streams: every call enqueues asynchronously on `stream` (a cudaStream_t,
 *    NULL = legacy default stream).  Only gf_load_primitives and gf_build_bvh
 *    synchronise the stream (to surface data errors found on the device).
 *  - Errors: a non-GF_OK status is returned synchronously for argument / state
 *    errors; gf_last_error(ctx) then holds a message.  Asynchronous CUDA faults
 *    surface as GF_E_CUDA at the next call.  No exception or abort crosses the ABI.
 *  - Thread safety: one context per device and per host thread at a time;
 *    distinct contexts are independent.
 *  - Determinism: results are bitwise deterministic for a given (scene, rays,
 *    policies, seed, shard layout).
 */
#ifndef GF_H
#define GF_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GF_ABI_VERSION 8
#define GF_MAX_GROUPS 32  /* 32-bit ray/group masks (C24); the paper's OptiX masks are 8-bit */
#define GF_MAX_LEVELS 8

typedef enum {
    GF_OK = 0,
    GF_E_INVALID_ARGUMENT = 1,    /* null/ill-sized argument, n < 0, bad enum value              */
    GF_E_STATE = 2,               /* call order: trace/render before load + build               */
    GF_E_SINGULAR_COVARIANCE = 3, /* scale <= 0, non-finite, or cond(S) > 1e6           */
    GF_E_INVALID_RAY = 4,         /* (reserved: rays are not validated on the hot path)           */
    GF_E_INVALID_BOUNDS = 5,      /* extent E <= 0 or non-finite                                  */
    GF_E_MASK_OVERFLOW = 6,       /* G = 1 + (P-1) K > 32 groups (C24)                             */
    GF_E_INVALID_STRATEGY = 7,    /* beta not in [0,1), delta not in [0,1], unknown strategy      */
    GF_E_ASSIGNMENT = 8,          /* level >= P or bin >= K in the input, bad quaternion norm     */
    GF_E_CUDA = 9,                /* CUDA runtime error (message in gf_last_error)                */
    GF_E_OUT_OF_MEMORY = 10       /* a caller workspace is smaller than the queried size          */
} gf_status;

typedef struct gf_ctx gf_ctx;   /* opaque, one per CUDA device */
typedef void *gf_stream;        /* cudaStream_t */

/* ---- context ------------------------------------------------------------ */
int gf_abi_version(void);
const char *gf_status_string(gf_status s);
/* Create a context on CUDA device `cuda_device`.  Allocates its small
 * internal state (error flag, counters) once. */
gf_status gf_create(int cuda_device, gf_ctx **out);
void gf_destroy(gf_ctx *ctx);
/* message of the last non-OK status returned for this context ("" if none) */
const char *gf_last_error(const gf_ctx *ctx);

/* ---- sizes -------------------------------------------------------------- */
/* Bytes the caller must provide for n primitives: prim_bytes for
 * gf_load_primitives, bvh_bytes + scratch_bytes for gf_build_bvh.  Pure
 * host computation except the radix-sort temp size (needs a CUDA device). */
gf_status gf_query_workspace(int64_t n_prims, size_t *prim_bytes, size_t *bvh_bytes, size_t *scratch_bytes);

/* ---- a1: primitive ingest + pyramid partition ----------- */
/* Primitive arrays, DEVICE pointers, structure of arrays, fp32:
 *   mu[3n] kernel means; quat[4n] unit quaternions (x,y,z,w), |q| = 1 +- 1e-5;
 *   scale[3n] principal standard deviations s (> 0, max/min <= 1e6);
 *   alpha[n] kernel weights (Eq. 1, >= 0); omega[n] modulation scalar (P:L183:
 *   omega_vec = R S^-1 (omega,omega,omega)^T, >= 0; 0 = Gaussian);
 *   extent[n] whitened truncation radius E (C7/C8), NULL -> 3 (the 3 sigma bound);
 *   level[n] pyramid level (0 = Gaussians), NULL -> derived from level_cutoffs (C10);
 *   bin[n] orientation bin, NULL or 255 -> derived: argmax_k |omega_vec . o_k| in fp32 (C11);
 *   band[n] spatial band (e.g. the distance band of an instance, config 5, fig:army_bunny
 *     P:L606-L617), < gf_pyramid.n_bands, NULL -> 0.  Group id = band * G0 + g(level, bin). */
typedef struct {
    const float *mu, *quat, *scale, *alpha, *omega, *extent;
    const uint8_t *level, *bin, *band;
} gf_prims;

/* Pyramid description, HOST pointers:
 *   n_levels P (1..8), n_bins K (>= 1), G0 = 1 + (P-1) K groups per band,
 *   n_bands B (0 or 1: no bands), G = B G0 <= 32 groups;
 *   group id g(0,*) = 0, g(l,b) = 1 + (l-1) K + b, plus band * G0  (C24);
 *   bin_axes[3K] unit axes o_k (C11);
 *   level_cutoffs[P-2] ascending world peak frequencies f0 = |omega_vec| separating
 *     Gabor levels 1..P-1 (used only when prims.level == NULL; may be NULL otherwise);
 *   group_f0[G] representative whitened frequency per group for the Importance
 *     orientation strategy (C12); NULL -> computed by gf_build_bvh on the device:
 *     sqrt(3) x the median omega of the group's level (even count: fp32 mean of the
 *     two middle values), the same for every bin and band of the level. */
typedef struct {
    int32_t n_levels;
    int32_t n_bins;
    const float *bin_axes;
    const float *level_cutoffs;
    const float *group_f0;
    int32_t n_bands;
} gf_pyramid;

/* Convert n primitives into the 64-byte device records (W = S^-1 R^T whitening,
 * c = alpha/(2 pi s1 s2 s3), E^2, group) stored in prim_ws (device, >= prim_bytes),
 * and derive the per-level maximum world frequency max |omega_vec| (reading F3, used by
 * foveated rendering; gf_scene_info).  Validates on the device and synchronises
 * `stream`; returns the first error class found (GF_E_SINGULAR_COVARIANCE,
 * GF_E_INVALID_BOUNDS, GF_E_ASSIGNMENT: level/bin/band out of range or |q| != 1).
 * n == 0 is valid (empty scene: every ray has tau = 0). Invalidates the BVH. */
gf_status gf_load_primitives(gf_ctx *ctx, const gf_prims *prims, int64_t n, const gf_pyramid *pyr,
                             void *prim_ws, size_t prim_ws_bytes, gf_stream stream);

/* ---- a2: bounds + LBVH build ------------------------------- */
/* Conservative world AABBs of the ellipsoids, 64-bit keys (group or level class << 57 |
 * Morton57 of the centre, gf_set_bvh_keys), radix sort (CUB), Karras hierarchy, bottom-up refit with group
 * masks, collapse to leaves of <= 3 single-group primitives, depth-first layout
 * with escape links.  Class bits are the top key bits, so the top of the tree
 * routes by level (or group): one tree playing the role of the paper's per-level GAS +
 * masked TLAS.  bvh_ws (device, >= bvh_bytes) holds the nodes and the reordered
 * primitives and must stay alive; scratch (device, >= scratch_bytes) may be
 * reused after the call.  Synchronises `stream`. */
gf_status gf_build_bvh(gf_ctx *ctx, void *bvh_ws, size_t bvh_ws_bytes, void *scratch, size_t scratch_bytes,
                       gf_stream stream);
/* Key prefix of the BVHs built after this call (gf_build_bvh, and the light / camera BVHs of gf_render):
 * GF_BVH_KEYS_LEVEL (default) = (distance band, level): one spatial subtree per level and band, the
 * paper's per-level acceleration structures, orientation bins mixed below it (leaves stay
 * single-group, node masks prune); GF_BVH_KEYS_GROUP = the full group (level x bin x band): subtrees
 * per orientation bin too -- for stochastic orientation masks (Table B2 Importance / Uniform), which
 * then prune whole subtrees.  Results are identical either way; only traversal cost differs.
 * GF_E_INVALID_ARGUMENT for another value.  Synchronous, no device work. */
#define GF_BVH_KEYS_GROUP 0
#define GF_BVH_KEYS_LEVEL 1
gf_status gf_set_bvh_keys(gf_ctx *ctx, int32_t keys);

/* Scene-derived quantities (synchronous; after gf_load_primitives, the BVH fields after
 * gf_build_bvh).  bvh_hash: a 64-bit hash of the whole BVH workspace (nodes, child pairs,
 * reordered primitives, permutation), equal on every rank that built the same scene -- the
 * multi-GPU replica check; 0 before gf_build_bvh. */
typedef struct {
    int64_t n_prims;
    int32_t n_levels, n_bins, n_bands, n_groups;
    float level_fmax[8];    /* max |omega_vec| per level (F3); [0] = 0 (Gaussians)          */
    float group_f0[32];     /* the Importance strategy's f0 per group (C12), as used        */
    float root_lo[3], root_hi[3];
    uint32_t n_nodes, max_depth;
    uint64_t bvh_hash;
} gf_scene_info;
gf_status gf_scene_info_get(gf_ctx *ctx, gf_scene_info *out);

/* Accelerated motion blur (readings M1-M3): for a blur of
 * length m along dir (host float[3], normalised here), per group the mean of its members'
 * omega_vec (signs aligned with the member of largest |omega_vec|) -> k = |mean . dir| -> box-filter
 * attenuation |sin(m k/2) / (m k/2)|; *mask_out (host) = the groups with attenuation >= threshold
 * (level-0 and empty groups always kept), att_out (host, n_groups floats, nullable) the
 * attenuations.  Device reductions over the loaded primitives; synchronous. */
gf_status gf_motion_blur_mask(gf_ctx *ctx, const float *dir, float m, float threshold, uint32_t *mask_out,
                              float *att_out);

/* Adaptive clamping (Eq. 15; reading C8'): per primitive the whitened extent
 *   E = min(3, sqrt(max(0, -2 ln(eps 2 pi s1 s2 s3 / (alpha s_max)) - 3 omega^2))), floored at 1e-3,
 * beyond which the worst-case untruncated line integral is below eps.  scale[3n], alpha[n],
 * omega[n]: device inputs as for gf_load_primitives; extent_out: device n floats (the `extent`
 * input of a later gf_load_primitives).  Asynchronous on `stream`. */
gf_status gf_adaptive_extent(gf_ctx *ctx, const float *scale, const float *alpha, const float *omega, int64_t n,
                             float eps, float *extent_out, gf_stream stream);

/* ---- a3: LOD policy (Tables B1/B2) ------------- */
typedef enum {
    GF_LEVEL_DETERMINISTIC = 0, GF_LEVEL_UNIFORM = 1, GF_LEVEL_POWERLAW = 2, GF_LEVEL_UNIFORM_CV = 3,
    GF_LEVEL_POWERLAW_CV = 4, GF_LEVEL_POWERLAW_CV_ACCUM = 5
} gf_level_strategy;
typedef enum {
    GF_ORIENT_DETERMINISTIC = 0, GF_ORIENT_THRESHOLD_CULL = 1, GF_ORIENT_UNIFORM = 2,
    GF_ORIENT_IMPORTANCE = 3, GF_ORIENT_THRESHOLD_UNIFORM = 4
} gf_orient_strategy;

/* Per ray segment: mask = (stochastic level x orientation draw) & static_mask;
 * group weight w_g = w_level * w_bin (reciprocal probabilities, readings C13-C15).
 * Deterministic/Deterministic with static_mask = the static LOD masks. */
typedef struct {
    uint32_t static_mask;
    int32_t level_strategy;   /* gf_level_strategy */
    float beta;               /* power-law shape, [0,1) */
    int32_t orient_strategy;  /* gf_orient_strategy */
    float delta;              /* alignment threshold, [0,1] */
} gf_lod_policy;

/* Set the policy of camera/extension segments (`ext`) and of next-event /
 * shadow segments (`nee`, NULL -> same as ext; "Zero NEE" = static_mask 1,
 * P:L365).  Host pointers; takes effect for later calls. */
gf_status gf_set_lod_mask(gf_ctx *ctx, const gf_lod_policy *ext, const gf_lod_policy *nee);

/* ---- a4-a7: masked traversal + fused line integral + transmittance -------- */
/* rays: device, 16-byte aligned, n x 8 fp32 (ox,oy,oz,tmin, dx,dy,dz,tmax), |d| = 1, tmin < tmax,
 * tmax may be +inf.  tau_out: device n fp32 optical depth tau = sum_i w_g alpha_i
 * int_tmin^tmax K_i (Eq. 2, App. A closed form, C3-C5), accumulated in fp64.
 * T_out: device n fp32 exp(-tau) (Eq. 3) or NULL.  The `ext` policy applies;
 * stochastic strategies draw uniforms (seed, pixel = ray index, sample 0,
 * depth 0, stream 0).  counters_out: device n x 3 uint32
 * (nodes visited, primitives tested, hits) or NULL. */
gf_status gf_trace_transmittance(gf_ctx *ctx, const float *rays, int64_t n, uint64_t seed, float *tau_out,
                                 float *T_out, uint32_t *counters_out, gf_stream stream);

#define GF_TRACE_BRUTE_FORCE 1u   /* test path: test every primitive, no BVH */
/* As gf_trace_transmittance with flags (GF_TRACE_BRUTE_FORCE). */
gf_status gf_trace_transmittance_ex(gf_ctx *ctx, const float *rays, int64_t n, uint64_t seed, uint32_t flags,
                                    float *tau_out, float *T_out, uint32_t *counters_out, gf_stream stream);

/* Backward of the optical depth w.r.t. the opacities (the alpha part of
 * d tau / d(mu, q, s, alpha, omega); tomographic regression P:L370-L470):
 *   grad_alpha[i] += sum_r dl_dtau[r] * d tau_r / d alpha_i,  d tau_r / d alpha_i = w_g(i) tau_ri / alpha_i
 * (tau is linear in alpha).  rays as gf_trace_transmittance (same ext policy and draws); dl_dtau:
 * device n fp32; grad_alpha: device n_prims fp32 in input order, accumulated (caller zeroes). */
gf_status gf_trace_grad_alpha(gf_ctx *ctx, const float *rays, int64_t n, uint64_t seed, const float *dl_dtau,
                              float *grad_alpha, gf_stream stream);

/* Backward of the optical depth w.r.t. every primitive parameter (SURVEY §8(f) rank 4:
 * d tau / d(mu, q, s, alpha, omega)), in two calls.
 *
 * gf_trace_grad_params accumulates, per primitive, the derivative of sum_r dl_dtau[r] tau_r
 * w.r.t. the primitive's mean, whitening matrix W = S^-1 R^T, omega and alpha,
 * each hit in closed form (the App. A moments J0..J2 by integration by parts, plus the terms of the
 * chord ends that move with the ellipsoid, C7) -- rays, policy and draws as
 * gf_trace_transmittance.  flags: 0 (one warp per ray) or GF_TRACE_PACKETS (32 consecutive rays walk
 * the BVH together and sum each primitive's terms across the warp before one set of atomics: faster
 * for coherent rays, correct for any; E_INVALID_ARGUMENT for other bits).  accum: device n_prims x 16 fp32 (16-byte aligned), input order, caller-zeroed,
 * accumulated across calls: [0..2] d/dmu, [3..11] d/dW (row-major), [12] d/domega, [13] d/dalpha,
 * [14] sum dl tau_ri (the |det W| part), [15] unused.
 *
 * gf_grad_params_finish converts accum to the load parameters by the chain rule through
 * W = S^-1 R(q / |q|)^T and |det W| = 1/(s_x s_y s_z): grad: device n_prims x 12 fp32
 * (mu_x, mu_y, mu_z, q_x, q_y, q_z, q_w, s_x, s_y, s_z, omega, alpha), overwritten.  quat: the
 * device n_prims x 4 quaternion array given to gf_load_primitives (16-byte aligned).
 * tau is not differentiable where a chord appears or vanishes (grazing rays, r2 = E^2): the
 * moving-end terms grow like 1/h there. */
#define GF_TRACE_PACKETS 2u  /* rays come in coherent groups of 32 (e.g. 8x4 pixel blocks): packet walk */
gf_status gf_trace_grad_params(gf_ctx *ctx, const float *rays, int64_t n, uint64_t seed, uint32_t flags,
                               const float *dl_dtau, float *accum, gf_stream stream);
gf_status gf_grad_params_finish(gf_ctx *ctx, const float *accum, const float *quat, float *grad, gf_stream stream);

/* Free-flight distance sampling of single rays (a8, Eq. 5; test / measurement path of
 * the kernels gf_render uses): for ray i, xi = uniform (seed, pixel = i, sample 0, depth 0, stream 0,
 * k = 0), tau* = -ln(1 - xi), and t_out[i] = the first t in [tmin, tmax] at which the
 * optical depth of the `ext`-masked field reaches tau* (C17: the first of the gf_free_flight_bins()
 * equal t-bins of the ray's scene interval -- the root box within [tmin, tmax] -- whose right edge
 * reaches tau*, then the root inside it), +inf if no bin edge reaches tau* (escape).  rays as gf_trace_transmittance (tmax = +inf allowed); t_out: device n floats.
 * flags: 0, or GF_TRACE_PACKETS (32 consecutive rays walk the BVH together, as gf_render's camera
 * rays do), | GF_FF_UNIFORM (the GF_EST_UNIFORM estimator: t* uniform in the crossing bin, u from
 * stream 8 of (pixel = i, sample 0, depth 0)).  scratch: device, >= gf_free_flight_scratch_bytes(n). */
#define GF_FF_UNIFORM 4u
gf_status gf_trace_free_flight(gf_ctx *ctx, const float *rays, int64_t n, uint64_t seed, uint32_t flags,
                               float *t_out, void *scratch, size_t scratch_bytes, gf_stream stream);
/* Number of t-bins of the free-flight pass A (reading C17: t* is the root inside the first of these
 * equal bins of the ray's scene interval whose right edge reaches tau*). */
int gf_free_flight_bins(void);
/* Device scratch gf_trace_free_flight needs for n rays (per-path state of <= 2^20 rays at a time). */
gf_status gf_free_flight_scratch_bytes(gf_ctx *ctx, int64_t n, size_t *bytes);

/* Candidate sets (test path, C21): for each ray, the ORIGINAL indices of the
 * primitives accepted by the fp32 ellipsoid predicate (traversal order),
 * ids[r * capacity + k], count[r] = total (may exceed capacity: truncated). */
gf_status gf_trace_candidates(gf_ctx *ctx, const float *rays, int64_t n, uint32_t flags, int32_t *ids,
                              int32_t capacity, int32_t *count, gf_stream stream);

/* ---- a8-a10: free flight + scatter loop + accumulation -------------------- */
typedef enum { GF_MODE_TOMOGRAPHY = 0, GF_MODE_SCATTER = 1 } gf_render_mode;
typedef enum { GF_SHARD_NONE = 0, GF_SHARD_TILES = 1, GF_SHARD_SAMPLES = 2 } gf_shard_kind;

/* Camera: pinhole; for pixel (px,py) and jitter (jx,jy) in [0,1):
 *   sx = (px+jx) (2/W) - 1, sy = 1 - (py+jy)(2/H), d = normalize(fwd + sx right + sy up)
 * with right/up pre-scaled by tan(vfov/2) (*aspect), evaluated in fp32 with
 * correctly rounded operations.  jitter = 0 -> pixel centres.
 * TOMOGRAPHY: per sample tau-hat of the camera ray.
 * SCATTER: free flight (Eq. 5, C17: tau integrated exactly into the gf_free_flight_bins() t-bins of
 *   the ray's scene interval, escape if no bin edge reaches tau*, else the root of tau(t) = tau*
 *   inside the first bin whose right edge does, by safeguarded Halley / bisection), NEE to the
 *   directional light (sun_dir towards the light, irradiance sun_E) with the
 *   nee policy, Henyey-Greenstein phase (g), grey albedo, constant env_L on
 *   escape, max_depth vertices (1 = single scattering), no Russian roulette (C19).
 * RNG: Philox4x32-10, key = seed, counter = (pixel, sample, depth, stream<<16 | k>>2).
 * estimator (a9, SURVEY §8 a9 alternative): GF_EST_ANALYTIC = closed-form tau, free flight by the
 *   root of tau(t) = tau*, NEE T = exp(-tau); GF_EST_TRACKING = null-collision delta tracking for
 *   free flight and ratio tracking for NEE against a per-ray piecewise-constant majorant (64 bins
 *   of the summed per-primitive density bounds); unbiased only where kappa >= 0 (C18); tracking
 *   step j of a segment uses Philox block k = 4j of stream 4 (free flight: u0 distance, u1
 *   acceptance) or stream 5 (NEE: u0 distance).  GF_EST_UNIFORM = the paper's biased alternative
 *   ("uniform sampling along the candidate segment containing a path vertex"), reading
 *   U1: the candidate segment is the crossing t-bin of C17 (found exactly, as above) and t* is uniform
 *   in it, u = Philox stream 8, k = 0 -- no root finding; NEE as GF_EST_ANALYTIC. */
typedef enum { GF_EST_ANALYTIC = 0, GF_EST_TRACKING = 1, GF_EST_UNIFORM = 2 } gf_estimator;
#define GF_FOV_LEVELS 1u
#define GF_FOV_CONTINUOUS 2u
typedef struct {
    int32_t mode;               /* gf_render_mode */
    int32_t width, height;
    int32_t max_depth;          /* >= 1 (SCATTER) */
    int32_t jitter;             /* 0 = pixel centres */
    int32_t spp_begin, spp_count;
    int32_t shard_kind;         /* gf_shard_kind */
    int32_t shard_rank, shard_world;
    const int32_t *probe_pixels; /* device, n_probe pixel indices (y*W+x) or NULL = full image */
    int64_t n_probe;
    float cam_pos[3], cam_fwd[3], cam_right[3], cam_up[3];
    float albedo, hg_g, sun_dir[3], sun_E, env_L;
    uint64_t seed;
    int32_t estimator;          /* gf_estimator (SCATTER) */
    int32_t reuse_accel;        /* 1: reuse the light / camera BVHs left in scratch by the previous
                                   call (see gf_render); 0: rebuild them */
    /* Foveated rendering (readings F1-F5): foveation != 0
     * gives every path of pixel (px, py) the frequency threshold
     *   f_max = max(0, fov_f0 - fov_slope e) (1 + fov_jitter (2u - 1)),
     *   e = |(px + 0.5, py + 0.5) - fov_gaze| / max(W, H),  u = uniform of stream 6, k = 0, depth 0;
     * mode bit 0 (GF_FOV_LEVELS): Gabor levels whose maximum frequency (gf_scene_info.level_fmax)
     * exceeds f_max are masked (level 0 never); bit 1 (GF_FOV_CONTINUOUS): a primitive whose
     * frequency along the ray |omega_vec . d| exceeds f_max is not integrated.  3 = both. */
    int32_t foveation;
    float fov_gaze[2];          /* gaze point in pixels */
    float fov_f0, fov_slope, fov_jitter;
    /* Motion-blur reference (readings M1-M3):
     * motion_blur = 1 renders the field moving along mb_dir by mb_m during the exposure, a box
     * filter of length mb_m: each (pixel, sample) draws u (stream 7, k = 0, depth 0) and the field
     * is shifted by s = mb_m (u - 1/2) mb_dir, i.e. the camera by -s.  (The accelerated version
     * culls orientation/frequency groups with inputs.motion_blur_mask -> a static mask.) */
    int32_t motion_blur;
    float mb_dir[3];
    float mb_m;
} gf_render_desc;

/* Device scratch needed by gf_render for `desc`. */
gf_status gf_render_scratch_bytes(gf_ctx *ctx, const gf_render_desc *desc, size_t *bytes);

/* Render.  accum (device fp32):
 *   full image (probe_pixels == NULL): H*W*2, accum[2p] += sum of estimates,
 *     accum[2p+1] += sum of squared estimates over this call's samples of pixel p
 *     (only the shard's pixels/samples are touched; caller zeroes it);
 *   probes: n_probe * spp_count, accum[i*spp_count + k] = estimate of sample
 *     spp_begin + k at probe i (overwritten).
 * ray_counts: device uint64[3] or NULL, += (camera rays, extension rays, NEE rays).
 * scratch also holds two acceleration structures gf_render builds on the stream: the light BVH
 *   (boxes in the light's frame, for NEE) and, for static camera masks, the camera BVH
 *   (projective boxes at the eye, for the camera rays).  With desc->reuse_accel = 1 they are
 *   reused when this call has the same scratch pointer, scene (no gf_load_primitives /
 *   gf_build_bvh in between), light and camera as the one that built them: the caller
 *   guarantees that scratch was not written in between by anything but gf_render calls of this
 *   context (a gf_render call with a different chunk layout of the same scratch invalidates them). */
gf_status gf_render(gf_ctx *ctx, const gf_render_desc *desc, float *accum, void *scratch, size_t scratch_bytes,
                    uint64_t *ray_counts, gf_stream stream);

/* ---- measurement (bench.py roofline / launch counts) ---------------------- */
#define GF_PROFILE_TIMING 1u  /* record CUDA events around every kernel launch (on its stream)   */
#define GF_PROFILE_WORK 2u    /* use the counting kernel variants (work[] below; slower)          */
/* Stages: 0 gen (camera rays), 1 ffA (free flight pass A: tau of the whole ray into 32 exact t-bins,
 * escape test, the bin of the first crossing), 2 ffB (pass B: that bin's chords -> root of tau(t) = tau*),
 * 3 nee (shadow rays + phase sampling), 4 finish (queue rotation + accumulation), 5 tomo,
 * 6 trace (gf_trace_transmittance), 7 unused.  work[s][0] counts node box tests (the warp traversal
 * tests both children of a popped node). */
typedef struct {
    uint64_t launches;           /* kernels launched by the library since the last reset        */
    uint64_t stage_launches[8];
    double stage_ms[8];          /* summed event time per stage (GF_PROFILE_TIMING)             */
    uint64_t work[8][12];        /* GF_PROFILE_WORK, per stage: nodes visited, primitives tested,
                                    hits, complex-erf endpoint evaluations (Eq. 13 series), real
                                    erf evaluations (Omega = 0), Gauss-Legendre fallbacks, pass-B
                                    window halvings, root-finder evaluations, paths/rays, 3 spare */
} gf_stats;
gf_status gf_set_profiling(gf_ctx *ctx, uint32_t flags);
/* Synchronises the context's device, fills *out, optionally resets the counters. */
gf_status gf_get_stats(gf_ctx *ctx, gf_stats *out, int32_t reset);

/* ---- e: multi-GPU shard assignment (host only, no device) ---------------- */
/* Owner rank of pixel (px,py) under tile-interleaved sharding (32x32 tiles, tile t -> rank t mod world). */
int32_t gf_shard_pixel_owner(int32_t px, int32_t py, int32_t width, int32_t height, int32_t world);
/* Owner rank of sample s under sample-interleaved sharding (s mod world). */
int32_t gf_shard_sample_owner(int32_t s, int32_t world);
/* Number of paths of one sample pass of a shard (gf_render's work items), -1 on bad args. */
int64_t gf_shard_paths(int32_t width, int32_t height, int32_t kind, int32_t rank, int32_t world);
/* Pixel (y*W+x) rendered by path p of a shard's pass, -1 for padding paths: the exact map the
 * kernels use (8x4-pixel warps inside 32x32 tiles). */
int32_t gf_shard_path_pixel(int64_t p, int32_t width, int32_t height, int32_t kind, int32_t rank, int32_t world);

#ifdef __cplusplus
}
#endif
#endif /* GF_H */
