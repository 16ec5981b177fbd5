"""Thin ctypes binding of libgf.so (include/gf.h) -- argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; this module only
allocates the caller-owned workspaces with torch, passes device pointers and the
current CUDA stream, and turns non-OK statuses into exceptions.  There is no CPU
fallback: if libgf.so is missing or CUDA is unavailable, calls raise.
"""
import ctypes
import os
import re

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GF_LIB", os.path.join(HERE, "libgf.so"))  # GF_LIB: tuning variants only
HEADER = os.path.join(os.path.dirname(HERE), "include", "gf.h")
_lib = None

GF_OK = 0
MODE_TOMOGRAPHY, MODE_SCATTER = 0, 1
SHARD_NONE, SHARD_TILES, SHARD_SAMPLES = 0, 1, 2
TRACE_BRUTE_FORCE = 1
TRACE_PACKETS = 2
FF_UNIFORM = 4  # gf_trace_free_flight: GF_EST_UNIFORM (t uniform in the crossing bin)
BVH_KEYS_GROUP, BVH_KEYS_LEVEL = 0, 1  # gf_set_bvh_keys


class GFError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"gf status {status}: {msg}")
        self.status = status


class Prims(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in ("mu", "quat", "scale", "alpha", "omega", "extent", "level", "bin",
                                               "band")]


class Pyramid(ctypes.Structure):
    _fields_ = [("n_levels", ctypes.c_int32), ("n_bins", ctypes.c_int32), ("bin_axes", ctypes.c_void_p),
                ("level_cutoffs", ctypes.c_void_p), ("group_f0", ctypes.c_void_p), ("n_bands", ctypes.c_int32)]


class SceneInfo(ctypes.Structure):
    _fields_ = [("n_prims", ctypes.c_int64), ("n_levels", ctypes.c_int32), ("n_bins", ctypes.c_int32),
                ("n_bands", ctypes.c_int32), ("n_groups", ctypes.c_int32), ("level_fmax", ctypes.c_float * 8),
                ("group_f0", ctypes.c_float * 32), ("root_lo", ctypes.c_float * 3), ("root_hi", ctypes.c_float * 3),
                ("n_nodes", ctypes.c_uint32), ("max_depth", ctypes.c_uint32), ("bvh_hash", ctypes.c_uint64)]


class LodPolicy(ctypes.Structure):
    _fields_ = [("static_mask", ctypes.c_uint32), ("level_strategy", ctypes.c_int32), ("beta", ctypes.c_float),
                ("orient_strategy", ctypes.c_int32), ("delta", ctypes.c_float)]


class Stats(ctypes.Structure):
    _fields_ = [("launches", ctypes.c_uint64), ("stage_launches", ctypes.c_uint64 * 8),
                ("stage_ms", ctypes.c_double * 8), ("work", (ctypes.c_uint64 * 12) * 8)]


STAGES = ("gen", "ffA", "ffB", "nee", "finish", "tomo", "trace", "unused")
WORK = ("nodes", "tests", "hits", "erf_complex", "erf_real", "gl_fallbacks", "window_splits", "root_evals", "paths")
PROFILE_TIMING, PROFILE_WORK = 1, 2


class RenderDesc(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int32), ("width", ctypes.c_int32), ("height", ctypes.c_int32),
                ("max_depth", ctypes.c_int32), ("jitter", ctypes.c_int32), ("spp_begin", ctypes.c_int32),
                ("spp_count", ctypes.c_int32), ("shard_kind", ctypes.c_int32), ("shard_rank", ctypes.c_int32),
                ("shard_world", ctypes.c_int32), ("probe_pixels", ctypes.c_void_p), ("n_probe", ctypes.c_int64),
                ("cam_pos", ctypes.c_float * 3), ("cam_fwd", ctypes.c_float * 3), ("cam_right", ctypes.c_float * 3),
                ("cam_up", ctypes.c_float * 3), ("albedo", ctypes.c_float), ("hg_g", ctypes.c_float),
                ("sun_dir", ctypes.c_float * 3), ("sun_E", ctypes.c_float), ("env_L", ctypes.c_float),
                ("seed", ctypes.c_uint64), ("estimator", ctypes.c_int32), ("reuse_accel", ctypes.c_int32),
                ("foveation", ctypes.c_int32), ("fov_gaze", ctypes.c_float * 2), ("fov_f0", ctypes.c_float),
                ("fov_slope", ctypes.c_float), ("fov_jitter", ctypes.c_float),
                ("motion_blur", ctypes.c_int32), ("mb_dir", ctypes.c_float * 3), ("mb_m", ctypes.c_float)]


def header_symbols():
    """Function names declared in include/gf.h."""
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(gf_[a-z_]+)\s*\(", txt)))


def lib():
    """Load libgf.so (built by paper_2602_05081_b200.build). Raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run `python -m paper_2602_05081_b200.build`")
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, i64, u32, u64, sz = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, ctypes.c_uint64,
                                  ctypes.c_size_t)
    L.gf_abi_version.restype = ctypes.c_int
    L.gf_status_string.restype = ctypes.c_char_p
    L.gf_status_string.argtypes = [ctypes.c_int]
    L.gf_create.argtypes = [ctypes.c_int, ctypes.POINTER(vp)]
    L.gf_destroy.argtypes = [vp]
    L.gf_last_error.restype = ctypes.c_char_p
    L.gf_last_error.argtypes = [vp]
    L.gf_query_workspace.argtypes = [i64, ctypes.POINTER(sz), ctypes.POINTER(sz), ctypes.POINTER(sz)]
    L.gf_load_primitives.argtypes = [vp, ctypes.POINTER(Prims), i64, ctypes.POINTER(Pyramid), vp, sz, vp]
    L.gf_build_bvh.argtypes = [vp, vp, sz, vp, sz, vp]
    L.gf_set_bvh_keys.argtypes = [vp, ctypes.c_int32]
    L.gf_set_lod_mask.argtypes = [vp, ctypes.POINTER(LodPolicy), ctypes.POINTER(LodPolicy)]
    L.gf_trace_transmittance.argtypes = [vp, vp, i64, u64, vp, vp, vp, vp]
    L.gf_trace_transmittance_ex.argtypes = [vp, vp, i64, u64, u32, vp, vp, vp, vp]
    L.gf_trace_candidates.argtypes = [vp, vp, i64, u32, vp, i32, vp, vp]
    L.gf_trace_free_flight.argtypes = [vp, vp, i64, u64, u32, vp, vp, sz, vp]
    L.gf_free_flight_scratch_bytes.argtypes = [vp, i64, ctypes.POINTER(sz)]
    L.gf_free_flight_bins.restype = ctypes.c_int
    L.gf_scene_info_get.argtypes = [vp, ctypes.POINTER(SceneInfo)]
    L.gf_motion_blur_mask.argtypes = [vp, vp, ctypes.c_float, ctypes.c_float, vp, vp]
    L.gf_adaptive_extent.argtypes = [vp, vp, vp, vp, i64, ctypes.c_float, vp, vp]
    L.gf_trace_grad_alpha.argtypes = [vp, vp, i64, u64, vp, vp, vp]
    L.gf_trace_grad_params.argtypes = [vp, vp, i64, u64, u32, vp, vp, vp]
    L.gf_grad_params_finish.argtypes = [vp, vp, vp, vp, vp]
    L.gf_render_scratch_bytes.argtypes = [vp, ctypes.POINTER(RenderDesc), ctypes.POINTER(sz)]
    L.gf_render.argtypes = [vp, ctypes.POINTER(RenderDesc), vp, vp, sz, vp, vp]
    L.gf_set_profiling.argtypes = [vp, u32]
    L.gf_get_stats.argtypes = [vp, ctypes.POINTER(Stats), i32]
    L.gf_shard_pixel_owner.restype = i32
    L.gf_shard_pixel_owner.argtypes = [i32, i32, i32, i32, i32]
    L.gf_shard_sample_owner.restype = i32
    L.gf_shard_sample_owner.argtypes = [i32, i32]
    L.gf_shard_paths.restype = i64
    L.gf_shard_paths.argtypes = [i32, i32, i32, i32, i32]
    L.gf_shard_path_pixel.restype = i32
    L.gf_shard_path_pixel.argtypes = [i64, i32, i32, i32, i32, i32]
    _lib = L
    return L


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream():
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def make_policy(p=None):
    p = p or {}
    return LodPolicy(p.get("static_mask", 0xFFFFFFFF) & 0xFFFFFFFF, p.get("level_strategy", 0), p.get("beta", 0.0),
                     p.get("orient_strategy", 0), p.get("delta", 1.0))


class GaborField:
    """A scene on one GPU: primitives, LBVH, LOD policies; trace and render entry points."""

    def __init__(self, device=0):
        import torch
        self.torch = torch
        self.device = torch.device("cuda", device)
        self.L = lib()
        self.ctx = ctypes.c_void_p()
        st = self.L.gf_create(device, ctypes.byref(self.ctx))
        if st != GF_OK:
            raise GFError(st, "gf_create failed (no CUDA device?)")
        self.n = 0
        self._keep = {}

    def __del__(self):
        if getattr(self, "ctx", None) and self.ctx.value:
            self.L.gf_destroy(self.ctx)
            self.ctx = ctypes.c_void_p()

    def _check(self, st):
        if st != GF_OK:
            raise GFError(st, self.L.gf_last_error(self.ctx).decode())

    def _buf(self, nbytes):
        return self.torch.empty(max(int(nbytes), 1), dtype=self.torch.uint8, device=self.device)

    # -------------------------------------------------------------- a1, a2
    def load_primitives(self, scene, level_cutoffs=None, group_f0=None):
        """scene: dict of arrays (numpy or torch) as produced by paper_2602_05081_b200.inputs."""
        torch = self.torch
        n = int(scene["n"])
        P, K = int(scene["P"]), int(scene["K"])

        def dev(key, dtype):
            a = scene.get(key)
            if a is None:
                return None
            t = torch.as_tensor(np.ascontiguousarray(a) if isinstance(a, np.ndarray) else a)
            return t.to(device=self.device, dtype=dtype).contiguous()

        arrs = {k: dev(k, torch.float32) for k in ("mu", "quat", "scale", "alpha", "omega", "extent")}
        arrs["level"] = dev("level", torch.uint8)
        arrs["bin"] = dev("bin", torch.uint8)
        arrs["band"] = dev("band", torch.uint8)
        prims = Prims(*[_ptr(arrs[k]) for k in ("mu", "quat", "scale", "alpha", "omega", "extent", "level", "bin",
                                                 "band")])
        axes = np.ascontiguousarray(scene["bin_axes"], np.float32)
        cut = None if level_cutoffs is None else np.ascontiguousarray(level_cutoffs, np.float32)
        f0 = None if group_f0 is None else np.ascontiguousarray(group_f0, np.float32)
        nb = int(scene.get("n_bands", 1))
        pyr = Pyramid(P, K, axes.ctypes.data, None if cut is None else cut.ctypes.data,
                      None if f0 is None else f0.ctypes.data, nb)
        pb, bb, sb = ctypes.c_size_t(), ctypes.c_size_t(), ctypes.c_size_t()
        self._check(self.L.gf_query_workspace(n, ctypes.byref(pb), ctypes.byref(bb), ctypes.byref(sb)))
        self.prim_ws = self._buf(pb.value)
        self._check(self.L.gf_load_primitives(self.ctx, ctypes.byref(prims), n, ctypes.byref(pyr),
                                              _ptr(self.prim_ws), pb.value, _stream()))
        self._sizes = (bb.value, sb.value)
        self.n, self.P, self.K, self.G = n, P, K, nb * (1 + (P - 1) * K)
        self._quat = arrs["quat"]  # kept for gf_grad_params_finish (the quaternions as loaded)
        return self

    def set_bvh_keys(self, keys):
        """gf_set_bvh_keys: BVH_KEYS_LEVEL (default) or BVH_KEYS_GROUP for the BVHs built afterwards."""
        self._check(self.L.gf_set_bvh_keys(self.ctx, int(keys)))
        return self

    def build_bvh(self):
        bb, sb = self._sizes
        self.bvh_ws = self._buf(bb)
        scratch = self._buf(sb)
        self._check(self.L.gf_build_bvh(self.ctx, _ptr(self.bvh_ws), bb, _ptr(scratch), sb, _stream()))
        del scratch
        return self

    def scene_info(self):
        """gf_scene_info_get: level_fmax (F3), group_f0 (C12), root box, node count, BVH hash."""
        si = SceneInfo()
        self._check(self.L.gf_scene_info_get(self.ctx, ctypes.byref(si)))
        return {"n_prims": si.n_prims, "n_levels": si.n_levels, "n_bins": si.n_bins, "n_bands": si.n_bands,
                "n_groups": si.n_groups, "level_fmax": np.array(si.level_fmax[:], np.float32),
                "group_f0": np.array(si.group_f0[:si.n_groups], np.float32),
                "root_lo": list(si.root_lo), "root_hi": list(si.root_hi), "n_nodes": si.n_nodes,
                "max_depth": si.max_depth, "bvh_hash": int(si.bvh_hash)}

    def motion_blur_mask(self, direction, m, threshold):
        """gf_motion_blur_mask (readings M1-M3): (32-bit group mask, attenuation per group)."""
        d = np.ascontiguousarray(direction, np.float32).reshape(3)
        mask = ctypes.c_uint32()
        att = np.zeros(32, np.float32)
        self._check(self.L.gf_motion_blur_mask(self.ctx, d.ctypes.data, ctypes.c_float(m), ctypes.c_float(threshold),
                                               ctypes.byref(mask), att.ctypes.data))
        return int(mask.value), att[:self.G]

    def adaptive_extent(self, scene, eps):
        """gf_adaptive_extent (Eq. 15, C8'): per-primitive extents for threshold eps (device tensor)."""
        torch = self.torch
        t = {k: torch.as_tensor(np.ascontiguousarray(scene[k], np.float32)).to(self.device).contiguous()
             for k in ("scale", "alpha", "omega")}
        n = int(scene["n"])
        out = torch.empty(max(n, 1), dtype=torch.float32, device=self.device)
        self._check(self.L.gf_adaptive_extent(self.ctx, _ptr(t["scale"]), _ptr(t["alpha"]), _ptr(t["omega"]), n,
                                              ctypes.c_float(eps), _ptr(out), _stream()))
        return out[:n]

    # -------------------------------------------------------------- a3
    def set_lod_mask(self, ext=None, nee=None):
        e = make_policy(ext)
        n = make_policy(nee) if nee is not None else None
        self._check(self.L.gf_set_lod_mask(self.ctx, ctypes.byref(e), None if n is None else ctypes.byref(n)))
        return self

    # -------------------------------------------------------------- a4-a7
    def trace_transmittance(self, rays, seed=0, want_T=True, counters=False, brute_force=False, out=None):
        torch = self.torch
        rays = torch.as_tensor(rays).to(device=self.device, dtype=torch.float32).contiguous().view(-1, 8)
        n = rays.shape[0]
        tau = out if out is not None else torch.empty(n, dtype=torch.float32, device=self.device)
        T = torch.empty(n, dtype=torch.float32, device=self.device) if want_T else None
        cnt = torch.zeros((n, 3), dtype=torch.int32, device=self.device) if counters else None
        flags = TRACE_BRUTE_FORCE if brute_force else 0
        self._check(self.L.gf_trace_transmittance_ex(self.ctx, _ptr(rays), n, seed & 0xFFFFFFFFFFFFFFFF, flags,
                                                     _ptr(tau), _ptr(T), _ptr(cnt), _stream()))
        return tau, T, cnt

    def trace_free_flight(self, rays, seed=0, packets=False, uniform=False):
        """gf_trace_free_flight: first t with tau(tmin, t) = tau* per ray (+inf: escape); uniform: the
        GF_EST_UNIFORM estimator (t uniform in the crossing bin)."""
        torch = self.torch
        rays = torch.as_tensor(rays).to(device=self.device, dtype=torch.float32).contiguous().view(-1, 8)
        n = rays.shape[0]
        t = torch.empty(max(n, 1), dtype=torch.float32, device=self.device)
        nb = ctypes.c_size_t()
        self._check(self.L.gf_free_flight_scratch_bytes(self.ctx, n, ctypes.byref(nb)))
        scratch = self._buf(nb.value)
        self._check(self.L.gf_trace_free_flight(self.ctx, _ptr(rays), n, seed & 0xFFFFFFFFFFFFFFFF,
                                                (TRACE_PACKETS if packets else 0) | (FF_UNIFORM if uniform else 0),
                                                _ptr(t), _ptr(scratch), nb.value,
                                                _stream()))
        return t[:n]

    def trace_grad_alpha(self, rays, dl_dtau, seed=0, out=None):
        """d(sum_r dl_dtau[r] tau_r) / d alpha (input order, fp32)."""
        torch = self.torch
        rays = torch.as_tensor(rays).to(device=self.device, dtype=torch.float32).contiguous().view(-1, 8)
        dl = torch.as_tensor(dl_dtau).to(device=self.device, dtype=torch.float32).contiguous()
        grad = out if out is not None else torch.zeros(self.n, dtype=torch.float32, device=self.device)
        self._check(self.L.gf_trace_grad_alpha(self.ctx, _ptr(rays), rays.shape[0], seed,
                                               _ptr(dl), _ptr(grad), _stream()))
        return grad

    def trace_grad_params(self, rays, dl_dtau, seed=0, accum=None, finish=True, packets=False):
        """d(sum_r dl_dtau[r] tau_r) / d(mu, q, s, omega, alpha): (n_prims, 12) fp32 in input order
        (gf_trace_grad_params + gf_grad_params_finish).  accum (n_prims, 16) fp32 accumulates across
        calls when given; finish=False returns it raw."""
        torch = self.torch
        rays = torch.as_tensor(rays).to(device=self.device, dtype=torch.float32).contiguous().view(-1, 8)
        dl = torch.as_tensor(dl_dtau).to(device=self.device, dtype=torch.float32).contiguous()
        acc = accum if accum is not None else torch.zeros((self.n, 16), dtype=torch.float32, device=self.device)
        self._check(self.L.gf_trace_grad_params(self.ctx, _ptr(rays), rays.shape[0], seed,
                                                TRACE_PACKETS if packets else 0, _ptr(dl), _ptr(acc), _stream()))
        if not finish:
            return acc
        grad = torch.empty((self.n, 12), dtype=torch.float32, device=self.device)
        self._check(self.L.gf_grad_params_finish(self.ctx, _ptr(acc), _ptr(self._quat), _ptr(grad), _stream()))
        return grad

    def trace_candidates(self, rays, capacity=2048, brute_force=False):
        torch = self.torch
        rays = torch.as_tensor(rays).to(device=self.device, dtype=torch.float32).contiguous().view(-1, 8)
        n = rays.shape[0]
        ids = torch.full((n, capacity), -1, dtype=torch.int32, device=self.device)
        count = torch.zeros(n, dtype=torch.int32, device=self.device)
        self._check(self.L.gf_trace_candidates(self.ctx, _ptr(rays), n, TRACE_BRUTE_FORCE if brute_force else 0,
                                               _ptr(ids), capacity, _ptr(count), _stream()))
        return ids, count

    # -------------------------------------------------------------- a8-a10
    def render_desc(self, desc, spp_begin=0, spp_count=1, shard=(SHARD_NONE, 0, 1), probes=None):
        d = RenderDesc()
        d.mode = desc["mode"]
        d.width, d.height = desc["width"], desc["height"]
        d.max_depth = desc.get("max_depth", 1)
        d.jitter = int(desc.get("jitter", 1))
        d.spp_begin, d.spp_count = spp_begin, spp_count
        d.shard_kind, d.shard_rank, d.shard_world = shard
        d.probe_pixels = None if probes is None else probes.data_ptr()
        d.n_probe = 0 if probes is None else probes.numel()
        for k in ("cam_pos", "cam_fwd", "cam_right", "cam_up", "sun_dir"):
            getattr(d, k)[:] = [float(x) for x in np.asarray(desc[k], np.float32)]
        d.albedo, d.hg_g = desc.get("albedo", 1.0), desc.get("hg_g", 0.0)
        d.sun_E, d.env_L = desc.get("sun_E", 0.0), desc.get("env_L", 0.0)
        d.seed = desc["seed"] & 0xFFFFFFFFFFFFFFFF
        d.estimator = int(desc.get("estimator", 0))
        d.reuse_accel = int(desc.get("reuse_accel", 0))
        fov = desc.get("foveation")
        if fov:
            d.foveation = int(fov.get("mode", 3))
            d.fov_gaze[:] = [float(x) for x in fov["gaze"]]
            d.fov_f0, d.fov_slope, d.fov_jitter = float(fov["f0"]), float(fov["slope"]), float(fov.get("jitter", 0.0))
        mb = desc.get("motion_blur")
        if mb:
            d.motion_blur = 1
            d.mb_dir[:] = [float(x) for x in np.asarray(mb["dir"], np.float32)]
            d.mb_m = float(np.float32(mb["m"]))
        return d

    def render(self, desc, spp_begin=0, spp_count=1, shard=(SHARD_NONE, 0, 1), probes=None, accum=None,
               ray_counts=None, scratch=None):
        """Render; returns (accum, ray_counts).  Policies come from desc['ext'] / desc['nee'] if
        present (set via gf_set_lod_mask), else from the last set_lod_mask call."""
        torch = self.torch
        if "ext" in desc:
            self.set_lod_mask(desc["ext"], desc.get("nee"))
        if probes is not None:
            probes = torch.as_tensor(probes).to(device=self.device, dtype=torch.int32).contiguous()
        d = self.render_desc(desc, spp_begin, spp_count, shard, probes)
        nb = ctypes.c_size_t()
        self._check(self.L.gf_render_scratch_bytes(self.ctx, ctypes.byref(d), ctypes.byref(nb)))
        if scratch is None or scratch.numel() < nb.value:
            scratch = self._buf(nb.value)
        if accum is None:
            size = probes.numel() * spp_count if probes is not None else desc["width"] * desc["height"] * 2
            accum = torch.zeros(size, dtype=torch.float32, device=self.device)
        if ray_counts is None:
            ray_counts = torch.zeros(3, dtype=torch.int64, device=self.device)  # camera, extension, NEE
        self._check(self.L.gf_render(self.ctx, ctypes.byref(d), _ptr(accum), _ptr(scratch), scratch.numel(),
                                     _ptr(ray_counts), _stream()))
        self._last_scratch = scratch
        return accum, ray_counts

    # -------------------------------------------------------------- measurement
    def set_profiling(self, timing=False, work=False):
        self._check(self.L.gf_set_profiling(self.ctx, (PROFILE_TIMING if timing else 0) |
                                            (PROFILE_WORK if work else 0)))

    def stats(self, reset=True):
        s = Stats()
        self._check(self.L.gf_get_stats(self.ctx, ctypes.byref(s), int(reset)))
        return {"launches": int(s.launches),
                "stage_launches": {STAGES[i]: int(s.stage_launches[i]) for i in range(8)},
                "stage_ms": {STAGES[i]: float(s.stage_ms[i]) for i in range(8)},
                "work": {STAGES[j]: {WORK[i]: int(s.work[j][i]) for i in range(len(WORK))} for j in range(8)}}

    def render_scratch(self, desc, spp_count=1, shard=(SHARD_NONE, 0, 1), probes=None):
        d = self.render_desc(desc, 0, spp_count, shard, probes)
        nb = ctypes.c_size_t()
        self._check(self.L.gf_render_scratch_bytes(self.ctx, ctypes.byref(d), ctypes.byref(nb)))
        return self._buf(nb.value)


def shard_pixel_owner(px, py, width, height, world):
    return lib().gf_shard_pixel_owner(px, py, width, height, world)


def shard_sample_owner(s, world):
    return lib().gf_shard_sample_owner(s, world)


def shard_paths(width, height, kind, rank, world):
    return lib().gf_shard_paths(width, height, kind, rank, world)


def shard_path_pixel(p, width, height, kind, rank, world):
    return lib().gf_shard_path_pixel(p, width, height, kind, rank, world)
