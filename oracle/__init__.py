"""CPU double-precision oracle for the Gabor Fields hot path -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product package
``paper_2602_05081_b200`` never imports it, and the two share no code: the only
common module is ``paper_2602_05081_b200.inputs`` (seeded input generators,
none of the method's arithmetic).

The arithmetic lives in ``gf_oracle.c`` (plain C, fp64, brute force over all
primitives); this module only marshals numpy arrays through ctypes.
"""
import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gf_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force=False):
    """Compile liboracle.so with gcc (no contraction, so fp32 decisions match C11 semantics)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=gnu11", "-ffp-contract=off", "-fPIC", "-shared",
               "-o", _LIB, _SRC, "-lm", "-lpthread"]
        subprocess.check_call(cmd)
    return _LIB


class Policy(ctypes.Structure):
    _fields_ = [("static_mask", ctypes.c_uint32), ("level_strategy", ctypes.c_int32),
                ("beta", ctypes.c_float), ("orient_strategy", ctypes.c_int32),
                ("delta", ctypes.c_float)]


class RenderDesc(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int32), ("width", ctypes.c_int32), ("height", ctypes.c_int32),
                ("max_depth", ctypes.c_int32), ("jitter", ctypes.c_int32),
                ("cam_pos", ctypes.c_float * 3), ("cam_fwd", ctypes.c_float * 3),
                ("cam_right", ctypes.c_float * 3), ("cam_up", ctypes.c_float * 3),
                ("albedo", ctypes.c_float), ("hg_g", ctypes.c_float), ("sun_dir", ctypes.c_float * 3),
                ("sun_E", ctypes.c_float), ("env_L", ctypes.c_float), ("seed", ctypes.c_uint64),
                ("ext", Policy), ("nee", Policy), ("group_f0", ctypes.c_void_p),
                ("foveation", ctypes.c_int32), ("fov_gaze", ctypes.c_float * 2), ("fov_f0", ctypes.c_float),
                ("fov_slope", ctypes.c_float), ("fov_jitter", ctypes.c_float),
                ("motion_blur", ctypes.c_int32), ("mb_dir", ctypes.c_float * 3), ("mb_m", ctypes.c_float)]


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        vp, i32, i64, u32, u64, dbl = (ctypes.c_void_p, ctypes.c_int, ctypes.c_long, ctypes.c_uint32,
                                       ctypes.c_uint64, ctypes.c_double)
        L.or_scene_create.restype = vp
        L.or_scene_create.argtypes = [i32, vp, vp, vp, vp, vp, vp, vp, vp, i32, i32, vp, vp, i32]
        L.or_scene_info.argtypes = [vp, vp, vp]
        L.or_motion_blur_mask.argtypes = [vp, vp, ctypes.c_float, ctypes.c_float, vp, vp]
        L.or_adaptive_extent.argtypes = [i64, vp, vp, vp, ctypes.c_float, vp]
        L.or_fov_fmax.restype = ctypes.c_float
        L.or_fov_fmax.argtypes = [vp, u32, u32]
        L.or_free_flight_diag.argtypes = [vp, vp, u32, vp, dbl, dbl, vp]
        L.or_scene_destroy.argtypes = [vp]
        L.or_scene_groups.argtypes = [vp, vp, vp]
        L.or_eval_kernel.restype = dbl
        L.or_eval_kernel.argtypes = [vp, i32, vp, i32]
        L.or_erf_parts.argtypes = [dbl, dbl, vp]
        L.or_prim_integral.restype = dbl
        L.or_prim_integral.argtypes = [vp, i32, vp, vp, dbl, dbl]
        L.or_prim_integral_infinite.restype = dbl
        L.or_prim_integral_infinite.argtypes = [vp, i32, vp, vp]
        L.or_trace.argtypes = [vp, vp, i64, u32, vp, vp, vp, vp, vp, i32]
        L.or_grad_alpha.argtypes = [vp, vp, i64, u32, vp, vp, vp]
        L.or_grad_params.argtypes = [vp, vp, vp, i64, u32, vp, vp, vp, vp, i32]
        L.or_candidates.restype = i32
        L.or_candidates.argtypes = [vp, vp, u32, vp, i32, vp]
        L.or_pair_r2_rel.restype = dbl
        L.or_pair_r2_rel.argtypes = [vp, i32, vp]
        L.or_philox.argtypes = [vp, vp, vp]
        L.or_uniform.restype = ctypes.c_float
        L.or_uniform.argtypes = [u64, u32, u32, u32, u32, u32]
        L.or_policy_eval.argtypes = [vp, vp, vp, ctypes.c_float, vp, vp, vp, vp]
        L.or_policy_eval_batch.argtypes = [vp, vp, vp, vp, vp, vp, i64, vp, vp]
        L.or_free_flight_f.restype = i32
        L.or_free_flight_f.argtypes = [vp, vp, u32, vp, dbl, vp]
        L.or_render_probes.argtypes = [vp, vp, vp, i64, i32, i32, vp, vp, i32]
        L.or_camera_ray.argtypes = [vp, i32, i32, ctypes.c_float, ctypes.c_float, vp, vp]
        L.or_hg_eval.restype = dbl
        L.or_hg_eval.argtypes = [dbl, dbl]
        L.or_hg_sample.argtypes = [dbl, vp, dbl, dbl, vp]
        L.or_sizeof_render_desc.restype = ctypes.c_size_t
        L.or_sizeof_policy.restype = ctypes.c_size_t
        assert L.or_sizeof_render_desc() == ctypes.sizeof(RenderDesc)
        assert L.or_sizeof_policy() == ctypes.sizeof(Policy)
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _f32(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float32)


def default_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


class Scene:
    """Oracle view of a scene (dict from paper_2602_05081_b200.inputs)."""

    def __init__(self, scene):
        L = lib()
        self.n = int(scene["n"])
        self.P = int(scene["P"])
        self.K = int(scene["K"])
        self.G = 1 + (self.P - 1) * self.K
        self.n_bands = int(scene.get("n_bands", 1))
        self.G0 = self.G
        self.G = self.G0 * self.n_bands
        self._keep = [_f32(scene["mu"]), _f32(scene["quat"]), _f32(scene["scale"]), _f32(scene["alpha"]),
                      _f32(scene["omega"]), _f32(scene.get("extent")),
                      None if scene.get("level") is None else np.ascontiguousarray(scene["level"], np.uint8),
                      None if scene.get("bin") is None else np.ascontiguousarray(scene["bin"], np.uint8),
                      _f32(scene["bin_axes"]),
                      None if scene.get("band") is None else np.ascontiguousarray(scene["band"], np.uint8)]
        k = self._keep
        self.h = L.or_scene_create(self.n, _p(k[0]), _p(k[1]), _p(k[2]), _p(k[3]), _p(k[4]), _p(k[5]),
                                   _p(k[6]), _p(k[7]), self.P, self.K, _p(k[8]), _p(k[9]), self.n_bands)
        if not self.h:
            raise ValueError("oracle rejected scene")

    def __del__(self):
        if getattr(self, "h", None):
            lib().or_scene_destroy(self.h)
            self.h = None

    def groups(self):
        g = np.zeros(max(self.n, 1), np.int32)
        b = np.zeros(max(self.n, 1), np.int32)
        lib().or_scene_groups(self.h, _p(g), _p(b))
        return g[:self.n], b[:self.n]

    def info(self):
        """(level_fmax[8], group_f0[32]): the scene-derived policy parameters (readings F3, C12)."""
        lf = np.zeros(8, np.float32)
        f0 = np.zeros(32, np.float32)
        lib().or_scene_info(self.h, _p(lf), _p(f0))
        return lf, f0[:self.G]

    def motion_blur_mask(self, direction, m, threshold):
        """Accelerated motion blur (readings M1-M3): (32-bit group mask, attenuation per group)."""
        d = _f32(direction).reshape(3)
        mask = np.zeros(1, np.uint32)
        att = np.zeros(32, np.float32)
        lib().or_motion_blur_mask(self.h, _p(d), ctypes.c_float(m), ctypes.c_float(threshold), _p(mask), _p(att))
        return int(mask[0]), att[:self.G]

    def free_flight_diag(self, ray, xi, t_q, mask=0xFFFFFFFF, weights=None):
        """(tau(t0, t_q), max cumulative tau at event points before t_q, tau*) -- C17 root checks."""
        ray = _f32(ray).reshape(8)
        out = np.zeros(3, np.float64)
        w = _f32(weights)
        lib().or_free_flight_diag(self.h, _p(ray), mask & 0xFFFFFFFF, _p(w), float(xi), float(t_q), _p(out))
        return out

    def eval_kernel(self, i, x, truncated=True):
        x = np.ascontiguousarray(x, np.float64)
        return lib().or_eval_kernel(self.h, i, _p(x), int(truncated))

    def prim_integral(self, i, o, v, t0, t1):
        o, v = _f32(o), _f32(v)
        return lib().or_prim_integral(self.h, i, _p(o), _p(v), float(t0), float(t1))

    def prim_integral_infinite(self, i, o, v):
        o, v = _f32(o), _f32(v)
        return lib().or_prim_integral_infinite(self.h, i, _p(o), _p(v))

    def trace(self, rays, mask=0xFFFFFFFF, weights=None, nthreads=None, want_groups=False):
        rays = _f32(rays).reshape(-1, 8)
        n = rays.shape[0]
        tau = np.zeros(n, np.float64)
        A = np.zeros(n, np.float64)
        nh = np.zeros(n, np.int32)
        grp = np.zeros((n, self.G), np.float64) if want_groups else None
        w = _f32(weights)
        lib().or_trace(self.h, _p(rays), n, mask & 0xFFFFFFFF, _p(w), _p(tau), _p(A), _p(grp), _p(nh),
                       nthreads or default_threads())
        out = {"tau": tau, "A": A, "nhits": nh}
        if want_groups:
            out["groups"] = grp
        return out

    def grad_alpha(self, rays, dl_dtau, mask=0xFFFFFFFF, weights=None):
        """d(sum_r dl[r] tau_r)/d alpha_i for every primitive (input order)."""
        rays = _f32(rays).reshape(-1, 8)
        dl = np.ascontiguousarray(dl_dtau, np.float64)
        g = np.zeros(self.n, np.float64)
        w = _f32(weights)
        lib().or_grad_alpha(self.h, _p(rays), rays.shape[0], mask & 0xFFFFFFFF, _p(w), _p(dl), _p(g))
        return g

    def grad_params(self, rays, dl_dtau, mask=0xFFFFFFFF, weights=None, nthreads=None):
        """d(sum_r dl[r] tau_r)/d theta_i, theta = (mu[3], q[4], s[3], omega, alpha) per primitive
        (input order), by Richardson central differences of the closed form (or_grad_params).
        Returns (grad, gabs): n x 12 each, gabs the sum of |per-ray terms| (a tolerance scale)."""
        rays = _f32(rays).reshape(-1, 8)
        dl = np.ascontiguousarray(dl_dtau, np.float64)
        k = self._keep
        theta = np.ascontiguousarray(np.concatenate(
            [k[0].reshape(-1, 3), k[1].reshape(-1, 4), k[2].reshape(-1, 3), k[4].reshape(-1, 1),
             k[3].reshape(-1, 1)], axis=1), np.float32)
        g = np.zeros((self.n, 12), np.float64)
        ga = np.zeros((self.n, 12), np.float64)
        w = _f32(weights)
        lib().or_grad_params(self.h, _p(theta), _p(rays), rays.shape[0], mask & 0xFFFFFFFF, _p(w), _p(dl), _p(g),
                             _p(ga), nthreads or default_threads())
        return g, ga

    def candidates(self, ray, mask=0xFFFFFFFF):
        ray = _f32(ray).reshape(8)
        cap = max(self.n, 1)
        ids = np.zeros(cap, np.int32)
        r2 = np.zeros(cap, np.float64)
        m = lib().or_candidates(self.h, _p(ray), mask & 0xFFFFFFFF, _p(ids), cap, _p(r2))
        return ids[:m], r2[:m]

    def r2_rel(self, i, ray):
        ray = _f32(ray).reshape(8)
        return lib().or_pair_r2_rel(self.h, int(i), _p(ray))

    def free_flight(self, ray, xi, mask=0xFFFFFFFF, weights=None):
        ray = _f32(ray).reshape(8)
        t = np.zeros(1, np.float64)
        w = _f32(weights)
        hit = lib().or_free_flight_f(self.h, _p(ray), mask & 0xFFFFFFFF, _p(w), float(xi), _p(t))
        return (float(t[0]) if hit else None)

    def policy_eval(self, policy, direction, ul, uo, group_f0=None):
        pol = make_policy(**policy) if isinstance(policy, dict) else policy
        d = _f32(direction).reshape(3)
        uo = _f32(np.asarray(uo, np.float32).reshape(-1) if len(uo) else np.zeros(1, np.float32))
        f0 = _f32(group_f0)
        m = np.zeros(1, np.uint32)
        w = np.zeros(self.G, np.float32)
        lib().or_policy_eval(self.h, ctypes.byref(pol), _p(d), ctypes.c_float(ul), _p(uo), _p(f0), _p(m), _p(w))
        return int(m[0]), w

    def policy_eval_batch(self, policy, dirs, ul, uo, group_f0=None):
        pol = make_policy(**policy) if isinstance(policy, dict) else policy
        dirs = _f32(dirs).reshape(-1, 3)
        n = dirs.shape[0]
        ul = _f32(ul).reshape(n)
        uo = _f32(uo).reshape(n, max(self.P - 1, 1))
        f0 = _f32(group_f0)
        m = np.zeros(n, np.uint32)
        w = np.zeros((n, self.G), np.float32)
        lib().or_policy_eval_batch(self.h, ctypes.byref(pol), _p(dirs), _p(ul), _p(uo), _p(f0), n, _p(m), _p(w))
        return m, w

    def render_probes(self, desc, probes, spp_begin, spp_count, nthreads=None):
        """desc: dict (see paper_2602_05081_b200.inputs.render_desc). Returns (values[n_probe, spp], nrays)."""
        d, keep = make_render_desc(desc)
        probes = np.ascontiguousarray(probes, np.int32)
        out = np.zeros(len(probes) * spp_count, np.float64)
        nr = np.zeros(len(probes) * spp_count, np.int32)
        lib().or_render_probes(self.h, ctypes.byref(d), _p(probes), len(probes), spp_begin, spp_count,
                               _p(out), _p(nr), nthreads or default_threads())
        del keep
        return out.reshape(len(probes), spp_count), nr.reshape(len(probes), spp_count)


def make_policy(static_mask=0xFFFFFFFF, level_strategy=0, beta=0.0, orient_strategy=0, delta=1.0):
    return Policy(static_mask & 0xFFFFFFFF, level_strategy, beta, orient_strategy, delta)


def make_render_desc(desc):
    d = RenderDesc()
    d.mode = desc["mode"]
    d.width, d.height = desc["width"], desc["height"]
    d.max_depth = desc.get("max_depth", 1)
    d.jitter = int(desc.get("jitter", 1))
    for name in ("cam_pos", "cam_fwd", "cam_right", "cam_up", "sun_dir"):
        getattr(d, name)[:] = [float(x) for x in np.asarray(desc[name], np.float32)]
    d.albedo = desc.get("albedo", 1.0)
    d.hg_g = desc.get("hg_g", 0.0)
    d.sun_E = desc.get("sun_E", 0.0)
    d.env_L = desc.get("env_L", 0.0)
    d.seed = desc["seed"] & 0xFFFFFFFFFFFFFFFF
    d.ext = make_policy(**desc.get("ext", {}))
    d.nee = make_policy(**desc.get("nee", desc.get("ext", {})))
    fov = desc.get("foveation")
    if fov:
        d.foveation = int(fov.get("mode", 3))
        d.fov_gaze[:] = [float(x) for x in np.asarray(fov["gaze"], np.float32)]
        d.fov_f0, d.fov_slope = float(np.float32(fov["f0"])), float(np.float32(fov["slope"]))
        d.fov_jitter = float(np.float32(fov.get("jitter", 0.0)))
    mb = desc.get("motion_blur")
    if mb:
        d.motion_blur = 1
        d.mb_dir[:] = [float(x) for x in np.asarray(mb["dir"], np.float32)]
        d.mb_m = float(np.float32(mb["m"]))
    f0 = desc.get("group_f0")
    keep = None
    if f0 is not None:
        keep = np.ascontiguousarray(f0, np.float32)
        d.group_f0 = keep.ctypes.data
    return d, keep


def philox(ctr, key):
    c = np.ascontiguousarray(ctr, np.uint32)
    k = np.ascontiguousarray(key, np.uint32)
    o = np.zeros(4, np.uint32)
    lib().or_philox(_p(c), _p(k), _p(o))
    return o


def uniform(seed, pix, smp, depth, stream, k):
    return lib().or_uniform(seed & 0xFFFFFFFFFFFFFFFF, pix, smp, depth, stream, k)


def erf(z):
    """complex erf by the oracle's Maclaurin series (Eq. 13)."""
    out = np.zeros(2, np.float64)
    lib().or_erf_parts(float(z.real), float(z.imag), _p(out))
    return complex(out[0], out[1])


def camera_ray(desc, px, py, jx=0.5, jy=0.5):
    d, keep = make_render_desc(desc)
    o = np.zeros(3, np.float32)
    v = np.zeros(3, np.float32)
    lib().or_camera_ray(ctypes.byref(d), px, py, ctypes.c_float(jx), ctypes.c_float(jy), _p(o), _p(v))
    return o, v


def adaptive_extent(scene, eps):
    """Adaptive clamping (Eq. 15, reading C8'): per-primitive extents E for threshold eps."""
    sc, al, om = _f32(scene["scale"]), _f32(scene["alpha"]), _f32(scene["omega"])
    n = int(scene["n"])
    out = np.zeros(max(n, 1), np.float32)
    lib().or_adaptive_extent(n, _p(sc), _p(al), _p(om), ctypes.c_float(eps), _p(out))
    return out[:n]


def fov_fmax(desc, pix, smp):
    """Foveation threshold of (pixel, sample) (readings F1, F2, F5)."""
    d, keep = make_render_desc(desc)
    return float(lib().or_fov_fmax(ctypes.byref(d), pix, smp))


def hg_eval(g, cost):
    return lib().or_hg_eval(g, cost)


def hg_sample(g, v, u1, u2):
    v = np.ascontiguousarray(v, np.float64)
    out = np.zeros(3, np.float64)
    lib().or_hg_sample(g, _p(v), u1, u2, _p(out))
    return out
