"""Seeded synthetic inputs shared by the CUDA path and the oracle.

This module holds NONE of the method's arithmetic (no kernel, integral,
whitening, bin/group derivation, mask sampling or RNG of the method): it only
draws primitive parameters, rays and camera frames with numpy's seeded
generators, following the recipe of DESIGN.md §6.  Both the
product path (bench.py, tests) and the oracle (tests) consume its output.

Scene dict keys (SoA, fp32 unless stated):
  n, P (pyramid levels, level 0 = Gaussians), K (orientation bins per Gabor level),
  mu[n,3], quat[n,4] (x,y,z,w, unit), scale[n,3] (>0), alpha[n] (>=0), omega[n] (>=0),
  extent[n] (whitened radius E, 3 = the paper's 3 sigma bound), level u8[n],
  bin u8[n] (255 = let each side derive it), bin_axes[K,3]; optionally band u8[n] and n_bands
  (spatial bands folded into the group id, config 5).
"""
import math

import numpy as np

P_DEFAULT = 4
K_DEFAULT = 3
SCENE_SEED = 0x5EED0000
RENDER_SEED = 0xC0FFEE00
TWO_PI_32 = (2.0 * math.pi) ** 1.5  # (2 pi)^(3/2): peak density -> alpha conversion of Eq. 6's normalisation


def bin_axes(K):
    """Representative orientation axes o_k (reading C11): K=3 -> x,y,z; K=6 -> icosahedral axes."""
    if K == 3:
        return np.eye(3, dtype=np.float32)
    if K == 6:
        p = (1.0 + 5 ** 0.5) / 2.0
        v = np.array([[0, 1, p], [0, -1, p], [1, p, 0], [-1, p, 0], [p, 0, 1], [-p, 0, 1]], np.float64)
        return (v / np.linalg.norm(v, axis=1, keepdims=True)).astype(np.float32)
    if K == 1:
        return np.array([[0, 0, 1]], np.float32)
    raise ValueError("K must be 1, 3 or 6")


def random_quats(rng, n):
    """Uniform random unit quaternions (Shoemake 1992), (x,y,z,w)."""
    u1, u2, u3 = rng.random(n), rng.random(n), rng.random(n)
    a, b = np.sqrt(1 - u1), np.sqrt(u1)
    q = np.stack([a * np.sin(2 * np.pi * u2), a * np.cos(2 * np.pi * u2),
                  b * np.sin(2 * np.pi * u3), b * np.cos(2 * np.pi * u3)], axis=1)
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    return q.astype(np.float32)


def _alpha_from_peak(peak, scale):
    """alpha such that the peak of alpha*K_i is `peak` (K_i's own normalisation, Eq. 6)."""
    return (peak * TWO_PI_32 * np.prod(scale.astype(np.float64), axis=1)).astype(np.float32)


def _finish(mu, quat, scale, peak, omega, level, P=P_DEFAULT, K=K_DEFAULT, extent=3.0, name=""):
    n = mu.shape[0]
    scale = scale.astype(np.float32)
    return {
        "name": name, "n": n, "P": P, "K": K,
        "mu": np.ascontiguousarray(mu, np.float32),
        "quat": np.ascontiguousarray(quat, np.float32),
        "scale": np.ascontiguousarray(scale, np.float32),
        "alpha": _alpha_from_peak(np.asarray(peak, np.float64), scale),
        "omega": np.ascontiguousarray(omega, np.float32),
        "extent": np.full(n, extent, np.float32),
        "level": np.ascontiguousarray(level, np.uint8),
        "bin": np.full(n, 255, np.uint8),
        "bin_axes": bin_axes(K),
    }


def scene_cfg1(seed=SCENE_SEED + 1, n=1000, density=1.1):
    """Config 1: 1k random primitives in [-1,1]^3; 20% Gaussians, Gabors in 3 scale bands."""
    rng = np.random.default_rng(seed)
    n0 = n // 5
    level = np.concatenate([np.zeros(n0, np.uint8), rng.integers(1, 4, n - n0).astype(np.uint8)])
    band = {0: (0.12, 0.2), 1: (0.12, 0.2), 2: (0.08, 0.12), 3: (0.05, 0.08)}
    lo = np.array([band[int(l)][0] for l in level])
    hi = np.array([band[int(l)][1] for l in level])
    base = np.exp(rng.uniform(np.log(lo), np.log(hi)))
    scale = base[:, None] * np.exp(rng.normal(0, 0.25, (n, 3)))
    mu = rng.uniform(-1, 1, (n, 3))
    omega = np.where(level == 0, 0.0, rng.uniform(0.7, 1.5, n))
    amp = np.array([1.0, 0.5, 0.35, 0.25])[level]
    peak = density * np.where(level == 0, rng.uniform(0.5, 1.0, n), amp)
    return _finish(mu, random_quats(rng, n), scale, peak, omega, level, name="cfg1")


def scene_cfg1p(seed=SCENE_SEED + 101, n_pairs=500, density=1.5):
    """Config 1p: paired-positive scene (reading C18): each Gabor gets a level-0 Gaussian with
    identical mu, q, s, E and alpha_G >= alpha_gabor, so kappa >= 0 for masks containing level 0."""
    rng = np.random.default_rng(seed)
    level_g = rng.integers(1, 4, n_pairs).astype(np.uint8)
    band = {1: (0.12, 0.2), 2: (0.08, 0.12), 3: (0.05, 0.08)}
    lo = np.array([band[int(l)][0] for l in level_g])
    hi = np.array([band[int(l)][1] for l in level_g])
    base = np.exp(rng.uniform(np.log(lo), np.log(hi)))
    scale = base[:, None] * np.exp(rng.normal(0, 0.25, (n_pairs, 3)))
    mu = rng.uniform(-1, 1, (n_pairs, 3))
    quat = random_quats(rng, n_pairs)
    omega = rng.uniform(0.7, 1.5, n_pairs)
    peak_gabor = density * np.array([0, 0.5, 0.35, 0.25])[level_g]
    peak_gauss = peak_gabor * rng.uniform(1.0, 1.5, n_pairs)
    return _finish(np.concatenate([mu, mu]), np.concatenate([quat, quat]), np.concatenate([scale, scale]),
                   np.concatenate([peak_gauss, peak_gabor]), np.concatenate([np.zeros(n_pairs), omega]),
                   np.concatenate([np.zeros(n_pairs, np.uint8), level_g]), name="cfg1p")


# --- config 2: "bunny-like" union of ellipsoids ---------------------------------------------
_BUNNY = [  # (centre, radii)
    ((0.0, -0.2, 0.0), (0.6, 0.5, 0.45)),    # body
    ((0.45, 0.25, 0.0), (0.3, 0.28, 0.28)),  # head
    ((0.5, 0.7, 0.1), (0.08, 0.3, 0.06)),    # ear
    ((0.5, 0.7, -0.1), (0.08, 0.3, 0.06)),   # ear
    ((-0.6, -0.1, 0.0), (0.12, 0.12, 0.12)),  # tail
]


def _bunny_f(x):
    """approximate signed distance to the union of the bunny ellipsoids (shape function, not the method)."""
    f = np.full(x.shape[0], np.inf)
    for c, r in _BUNNY:
        c, r = np.asarray(c), np.asarray(r)
        f = np.minimum(f, (np.linalg.norm((x - c) / r, axis=1) - 1.0) * r.min())
    return f


def _sample_where(rng, n, pred, lo, hi):
    out = []
    need = n
    while need > 0:
        x = rng.uniform(lo, hi, (max(4 * need, 1024), 3))
        x = x[pred(x)]
        out.append(x[:need])
        need -= len(out[-1])
    return np.concatenate(out)[:n]


def scene_bunny(seed=SCENE_SEED + 2, counts=(1500, 10500, 28000, 60000),
                s_levels=(0.09, 0.03, 0.015, 0.0075), name="cfg2", density=2.2):
    """Config 2 (and the config-5 asset): L0 Gaussians inside the union, Gabor levels 1..3 in a
    surface shell |f| < 6 s_l."""
    rng = np.random.default_rng(seed)
    lo, hi = np.array([-0.9, -0.85, -0.6]), np.array([0.9, 1.1, 0.6])
    mus, scales, levels, peaks, omegas = [], [], [], [], []
    for l, cnt in enumerate(counts):
        s_l = s_levels[l]
        if l == 0:
            pts = _sample_where(rng, cnt, lambda x: _bunny_f(x) < -0.5 * s_l, lo, hi)
        else:
            pts = _sample_where(rng, cnt, lambda x, s=s_l: np.abs(_bunny_f(x)) < 6 * s, lo - 0.1, hi + 0.1)
        mus.append(pts)
        scales.append(s_l * np.exp(rng.normal(0, 0.25, (cnt, 3))))
        levels.append(np.full(cnt, l, np.uint8))
        if l == 0:
            peaks.append(density * rng.uniform(0.5, 1.0, cnt))
            omegas.append(np.zeros(cnt))
        else:
            peaks.append(density * np.full(cnt, (0.5, 0.35, 0.25)[l - 1]))
            omegas.append(rng.uniform(0.7, 1.5, cnt))
    n = sum(counts)
    return _finish(np.concatenate(mus), random_quats(rng, n), np.concatenate(scales), np.concatenate(peaks),
                   np.concatenate(omegas), np.concatenate(levels), name=name)


def scene_cfg2(seed=SCENE_SEED + 2):
    return scene_bunny(seed=seed)


def _maxwell(rng, a, n):
    """Maxwell-distributed samples with scale a (norm of a 3D normal vector of std a)."""
    return a * np.linalg.norm(rng.normal(size=(n, 3)), axis=1)


def scene_cfg3(seed=SCENE_SEED + 3, n_clouds=100, depth=3, children=5, density=5.0):
    """Config 3: procedural clouds (§6.3): each cloud is a chunk tree (depth 3, 5 children
    per chunk -> 156 chunks); a chunk is one Gaussian core (sigma = r/3) plus 20 Gabors placed at a
    random position inside each cell of a 4x5 latitude-longitude grid on its surface sphere, scales
    Maxwell(r/12), omega ~ U[0.7,1.5], random orientation; child chunks sit uniformly at random on
    the parent's surface with Maxwell(0.25 r_parent) radii.  100 clouds in [-20,20]x[0,6]x[-20,20].
    Gabor levels by scale tertile (smaller -> higher level)."""
    rng = np.random.default_rng(seed)
    cores, core_r = [], []
    for _ in range(n_clouds):
        c0 = rng.uniform([-20, 0, -20], [20, 6, 20])
        frontier = [(c0, rng.uniform(1.0, 2.0))]
        for lvl in range(depth + 1):
            nxt = []
            for c, r in frontier:
                cores.append(c)
                core_r.append(r)
                if lvl < depth:
                    d = rng.normal(size=(children, 3))
                    d /= np.linalg.norm(d, axis=1, keepdims=True)
                    rc = np.maximum(_maxwell(rng, 0.25 * r / np.sqrt(3), children), 0.05 * r)
                    nxt += [(c + r * d[k], rc[k]) for k in range(children)]
            frontier = nxt
    cores, core_r = np.array(cores), np.array(core_r)
    nc = len(cores)
    # 20 Gabors per chunk on a jittered 4 (lat) x 5 (lon) grid over the chunk's surface sphere
    lat = (np.arange(4)[None, :, None] + rng.random((nc, 4, 5))) / 4.0  # cos(theta) cells
    lon = (np.arange(5)[None, None, :] + rng.random((nc, 4, 5))) / 5.0
    ct = 1 - 2 * lat
    st = np.sqrt(1 - ct ** 2)
    ph = 2 * np.pi * lon
    dirs = np.stack([st * np.cos(ph), ct, st * np.sin(ph)], -1).reshape(nc, 20, 3)
    gmu = (cores[:, None, :] + core_r[:, None, None] * dirs).reshape(-1, 3)
    gr = np.repeat(core_r, 20)
    gs = np.maximum(_maxwell(rng, gr / 12 / np.sqrt(3), len(gr)), 0.02 * gr)
    gscale = gs[:, None] * np.exp(rng.normal(0, 0.15, (len(gs), 3)))
    rel = gs / gr
    q1, q2 = np.quantile(rel, [1 / 3, 2 / 3])
    glevel = np.where(rel >= q2, 1, np.where(rel >= q1, 2, 3)).astype(np.uint8)
    cscale = (core_r / 3.0)[:, None] * np.exp(rng.normal(0, 0.1, (nc, 3)))
    mu = np.concatenate([cores, gmu])
    scale = np.concatenate([cscale, gscale])
    level = np.concatenate([np.zeros(nc, np.uint8), glevel])
    omega = np.concatenate([np.zeros(nc), rng.uniform(0.7, 1.5, len(gmu))])
    peak = density * np.concatenate([rng.uniform(0.5, 1.0, nc), np.array([0, 0.5, 0.35, 0.25])[glevel]])
    n = len(mu)
    return _finish(mu, random_quats(rng, n), scale, peak, omega, level, name="cfg3")


def scene_cfg4(seed=SCENE_SEED + 4, counts=(12000, 48000, 192000, 748000), s_levels=(0.075, 0.025, 0.0125, 0.00625),
               density=0.26):
    """Config 4: 'dense asset' -- a volume-filling pyramid in the cube [-1,1]^3, levels 0..3 with
    12k/48k/192k/748k primitives (N = 1,000,000) at scales 0.075/0.025/0.0125/0.00625."""
    rng = np.random.default_rng(seed)
    mus, scales, levels, peaks, omegas = [], [], [], [], []
    for l, cnt in enumerate(counts):
        mus.append(rng.uniform(-1, 1, (cnt, 3)))
        scales.append(s_levels[l] * np.exp(rng.normal(0, 0.25, (cnt, 3))))
        levels.append(np.full(cnt, l, np.uint8))
        peaks.append(density * (rng.uniform(0.5, 1.0, cnt) if l == 0 else np.full(cnt, (0.5, 0.35, 0.25)[l - 1])))
        omegas.append(np.zeros(cnt) if l == 0 else rng.uniform(0.7, 1.5, cnt))
    n = sum(counts)
    return _finish(np.concatenate(mus), random_quats(rng, n), np.concatenate(scales), np.concatenate(peaks),
                   np.concatenate(omegas), np.concatenate(levels), name="cfg4")


CFG5_EYE = (0.0, 6.0, 22.0)


def scene_cfg5(seed=SCENE_SEED + 5, copies=120, grid=(12, 10), spacing=2.2, n_bands=3):
    """Config 5: 'army' -- 120 yawed, scaled copies of a 33,280-primitive bunny-like asset (config-2
    generator at 500/3,494/9,318/19,968) on a 12 x 10 ground grid: N = 3,993,600.  Every primitive
    carries the distance band of its copy (`fig:army_bunny` P:L606-L617): the
    copies ranked by the distance of their grid position from the config-5 eye, split into n_bands
    equal groups (near / mid / far), folded into the group id as band * 10 + g(l, b)."""
    base = scene_bunny(seed=seed, counts=(500, 3494, 9318, 19968), name="cfg5-asset")
    rng = np.random.default_rng(seed + 1)
    nb = base["n"]
    out = {k: [] for k in ("mu", "quat", "scale", "alpha")}
    for c in range(copies):
        gx, gz = c % grid[0], c // grid[0]
        yaw = rng.uniform(0, 2 * np.pi)
        sc = rng.uniform(0.8, 1.2)
        cy, sy = np.cos(yaw), np.sin(yaw)
        Ry = np.array([[cy, 0, sy], [0, 1, 0], [-sy, 0, cy]])
        off = np.array([(gx - (grid[0] - 1) / 2) * spacing, 0.0, (gz - (grid[1] - 1) / 2) * spacing])
        out["mu"].append(base["mu"].astype(np.float64) @ Ry.T * sc + off)
        qy = np.array([0.0, np.sin(yaw / 2), 0.0, np.cos(yaw / 2)])  # (x,y,z,w)
        q = base["quat"].astype(np.float64)
        x1, y1, z1, w1 = qy
        x2, y2, z2, w2 = q[:, 0], q[:, 1], q[:, 2], q[:, 3]
        out["quat"].append(np.stack([w1 * x2 + x1 * w2 + y1 * z2 - z1 * y2, w1 * y2 - x1 * z2 + y1 * w2 + z1 * x2,
                                     w1 * z2 + x1 * y2 - y1 * x2 + z1 * w2, w1 * w2 - x1 * x2 - y1 * y2 - z1 * z2], 1))
        out["scale"].append(base["scale"].astype(np.float64) * sc)
        out["alpha"].append(base["alpha"].astype(np.float64) * sc ** 2)  # keeps peak density (alpha ~ s^3 / s)
    n = nb * copies
    pos = np.array([[(c % grid[0] - (grid[0] - 1) / 2) * spacing, 0.0, (c // grid[0] - (grid[1] - 1) / 2) * spacing]
                    for c in range(copies)])
    rank = np.argsort(np.argsort(np.linalg.norm(pos - np.asarray(CFG5_EYE), axis=1), kind="stable"), kind="stable")
    copy_band = (rank * n_bands // copies).astype(np.uint8)
    q = np.concatenate(out["quat"])
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    return {"name": "cfg5", "n": n, "P": base["P"], "K": base["K"],
            "mu": np.concatenate(out["mu"]).astype(np.float32), "quat": q.astype(np.float32),
            "scale": np.concatenate(out["scale"]).astype(np.float32),
            "alpha": np.concatenate(out["alpha"]).astype(np.float32),
            "omega": np.tile(base["omega"], copies), "extent": np.full(n, 3.0, np.float32),
            "level": np.tile(base["level"], copies), "bin": np.full(n, 255, np.uint8),
            "bin_axes": base["bin_axes"], "band": np.repeat(copy_band, nb), "n_bands": n_bands}


def empty_scene(P=P_DEFAULT, K=K_DEFAULT):
    z = np.zeros((0, 3), np.float32)
    return _finish(z, np.zeros((0, 4), np.float32), z, np.zeros(0), np.zeros(0), np.zeros(0, np.uint8), P, K,
                   name="empty")


def scene_column(seed=SCENE_SEED + 9, n=1500, density=0.02):
    """Stress case (not a paper workload): n small primitives strung along the x axis in [-1, 1]
    (80% Gaussians, 20% Gabors), so a ray along the axis overlaps all of them -- more hit records
    than the free-flight record buffer holds (1024), exercising the single-pass fallback."""
    rng = np.random.default_rng(seed)
    mu = np.stack([np.linspace(-1, 1, n), rng.normal(0, 0.002, n), rng.normal(0, 0.002, n)], 1)
    scale = 0.02 * np.exp(rng.normal(0, 0.2, (n, 3)))
    level = np.where(rng.random(n) < 0.8, 0, rng.integers(1, 4, n)).astype(np.uint8)
    omega = np.where(level == 0, 0.0, rng.uniform(0.7, 1.5, n))
    peak = density * rng.uniform(0.5, 1.0, n)
    return _finish(mu, random_quats(rng, n), scale, peak, omega, level, name="column")


def foveation(gaze, f0, slope, jitter=0.0, mode=3):
    """Foveated-rendering parameters (gf_render_desc foveation fields): gaze point in pixels, threshold
    at the fovea, slope per unit eccentricity, jitter; mode bit 0 = level masking, bit 1 = the
    continuous per-primitive check (3 = both, the paper's full method)."""
    return {"gaze": [float(gaze[0]), float(gaze[1])], "f0": float(f0), "slope": float(slope),
            "jitter": float(jitter), "mode": int(mode)}


def motion_blur(direction, m):
    """Motion-blur reference parameters (gf_render_desc motion_blur fields): unit direction, length."""
    d = np.asarray(direction, np.float64)
    return {"dir": (d / np.linalg.norm(d)).astype(np.float32).tolist(), "m": float(m)}


def level_mask(levels, P=P_DEFAULT, K=K_DEFAULT, n_bands=1, bands=None):
    """32-bit group mask selecting whole pyramid levels: level 0 -> bit 0, Gabor level l ->
    bits 1+(l-1)K .. (l)K of each spatial band (group numbering band * G0 + g(l,b) of DESIGN.md §5;
    paper V_l = 2^l).  bands: the bands to select (default all)."""
    G0 = 1 + (P - 1) * K
    m = 0
    for l in levels:
        if l == 0:
            m |= 1
        else:
            for b in range(K):
                m |= 1 << (1 + (l - 1) * K + b)
    out = 0
    for bd in (range(n_bands) if bands is None else bands):
        out |= m << (bd * G0)
    return out


# --- rays and cameras ---------------------------------------------------------------------
def camera(eye, look, up, vfov_deg, width, height):
    """Pinhole frame as fp32 vectors (pos, fwd, right*tan*aspect, up*tan) -- the numbers both sides
    consume, so that their fp32 camera rays are bit-identical."""
    eye, look, up = (np.asarray(a, np.float64) for a in (eye, look, up))
    fwd = look - eye
    fwd /= np.linalg.norm(fwd)
    right = np.cross(fwd, up)
    right /= np.linalg.norm(right)
    upv = np.cross(right, fwd)
    th = math.tan(math.radians(vfov_deg) / 2)
    return {"cam_pos": eye.astype(np.float32), "cam_fwd": fwd.astype(np.float32),
            "cam_right": (right * th * width / height).astype(np.float32),
            "cam_up": (upv * th).astype(np.float32), "width": width, "height": height}


def policy(static_mask=0xFFFFFFFF, level_strategy=0, beta=0.0, orient_strategy=0, delta=1.0):
    return {"static_mask": static_mask & 0xFFFFFFFF, "level_strategy": level_strategy, "beta": beta,
            "orient_strategy": orient_strategy, "delta": delta}


SUN = (np.array([1.0, 1.0, 0.5]) / np.linalg.norm([1.0, 1.0, 0.5])).astype(np.float32)


def render_desc_cfg1(width=64, height=64, seed=RENDER_SEED + 1):
    d = camera((0, 0, 4), (0, 0, 0), (0, 1, 0), 40.0, width, height)
    d.update(mode=0, max_depth=1, jitter=0, albedo=1.0, hg_g=0.0, sun_dir=SUN, sun_E=0.0, env_L=0.0, seed=seed,
             ext=policy(), nee=policy())
    return d


CFG2_LOD_LEVELS = ([0], [0, 1], [0, 1, 2], [0, 1, 2, 3])


def render_desc_cfg2(mask_index=3, width=1024, height=1024, seed=RENDER_SEED + 2):
    """Config 2: single scattering, one of the 4 static LOD masks (levels {0},{0,1},{0..2},{0..3})."""
    d = camera((0, 0.3, 3.2), (0, 0.05, 0), (0, 1, 0), 40.0, width, height)
    m = level_mask(CFG2_LOD_LEVELS[mask_index])
    d.update(mode=1, max_depth=1, jitter=1, albedo=0.8, hg_g=0.0, sun_dir=SUN, sun_E=3.0, env_L=0.2,
             seed=seed + 0x100 * mask_index, ext=policy(static_mask=m), nee=policy(static_mask=m))
    return d


def render_desc_cfg3(width=1024, height=1024, seed=RENDER_SEED + 3):
    """Config 3: multiple scattering, depth 8, albedo 0.95, HG g = 0.6, full mask (4 spp per frame)."""
    d = camera((0, 4, 34), (0, 2, 0), (0, 1, 0), 60.0, width, height)
    d.update(mode=1, max_depth=8, jitter=1, albedo=0.95, hg_g=0.6, sun_dir=SUN, sun_E=3.0, env_L=0.2, seed=seed,
             ext=policy(), nee=policy())
    return d


def render_desc_cfg4(width=2048, height=2048, seed=RENDER_SEED + 4):
    """Config 4: multiple scattering depth 8 with stochastic per-recursion masks: extension rays
    PL+CV(Accum.) beta = 0.2 x orientation Importance, NEE 'Zero NEE' (level 0 only)."""
    d = camera((0, 0, 4), (0, 0, 0), (0, 1, 0), 40.0, width, height)
    d.update(mode=1, max_depth=8, jitter=1, albedo=0.8, hg_g=0.3, sun_dir=SUN, sun_E=3.0, env_L=0.2, seed=seed,
             ext=policy(level_strategy=5, beta=0.2, orient_strategy=3), nee=policy(static_mask=1))
    return d


CFG5_BANDED_LEVELS = ((0, 1, 2, 3), (0, 1, 2), (0, 1))  # near / mid / far (fig:army_bunny)


def render_desc_cfg5(mask_levels=(0, 1, 2, 3), width=4096, height=4096, seed=RENDER_SEED + 5, n_bands=3):
    """Config 5: multiple scattering depth 8 over the army, one static LOD mask: the levels
    `mask_levels` in every distance band, or mask_levels = "banded": levels 0..3 near, 0..2 mid,
    0..1 far (the distance-dependent LOD of fig:army_bunny)."""
    d = camera(CFG5_EYE, (0, 0, 0), (0, 1, 0), 50.0, width, height)
    if isinstance(mask_levels, str) and mask_levels == "banded":
        m = 0
        for bd, lv in enumerate(CFG5_BANDED_LEVELS[:n_bands]):
            m |= level_mask(lv, n_bands=n_bands, bands=[bd])
    else:
        m = level_mask(mask_levels, n_bands=n_bands)
    d.update(mode=1, max_depth=8, jitter=1, albedo=0.8, hg_g=0.0, sun_dir=SUN, sun_E=3.0, env_L=0.2, seed=seed,
             ext=policy(static_mask=m), nee=policy(static_mask=m))
    return d


def camera_rays_f64(desc, px, py, jx=0.5, jy=0.5):
    """Camera rays computed in float64 numpy from the fp32 frame (for picking test rays; the
    kernels and the oracle each compute their own fp32 camera rays)."""
    px, py = np.asarray(px, np.float64), np.asarray(py, np.float64)
    sx = 2 * (px + jx) / desc["width"] - 1
    sy = 1 - 2 * (py + jy) / desc["height"]
    d = (desc["cam_fwd"][None].astype(np.float64) + sx[:, None] * desc["cam_right"][None]
         + sy[:, None] * desc["cam_up"][None])
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    o = np.broadcast_to(desc["cam_pos"].astype(np.float64), d.shape)
    return o, d


def rays_through_box(seed, n, lo=-1.0, hi=1.0, dist=4.0, tmin=0.0, tmax=np.inf):
    """n rays (n x 8 fp32) from a sphere of radius `dist` aimed at random points in the box."""
    rng = np.random.default_rng(seed)
    tgt = rng.uniform(lo, hi, (n, 3))
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    o = tgt - dist * d
    return pack_rays(o, d, tmin, tmax)


def pack_rays(o, d, tmin=0.0, tmax=np.inf):
    n = o.shape[0]
    d = np.asarray(d, np.float64)
    d = d / np.linalg.norm(d, axis=1, keepdims=True)
    r = np.zeros((n, 8), np.float32)
    r[:, 0:3] = o
    r[:, 3] = tmin
    r[:, 4:7] = d
    r[:, 7] = tmax
    return r


def far_origin_pairs(seed, n, ratio, s_lo=0.005, s_hi=0.05):
    """Far-origin stress set: single primitives of scale s in [s_lo,s_hi] placed at
    random, rays starting |o-mu|/s = ratio away, passing within the 3-sigma ellipsoid."""
    rng = np.random.default_rng(seed)
    s = np.exp(rng.uniform(np.log(s_lo), np.log(s_hi), n))
    scale = s[:, None] * np.exp(rng.normal(0, 0.25, (n, 3)))
    mu = rng.uniform(-1, 1, (n, 3))
    quat = random_quats(rng, n)
    omega = rng.uniform(0.7, 1.5, n)
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    off = rng.normal(size=(n, 3))
    off -= (off * d).sum(1, keepdims=True) * d
    off /= np.linalg.norm(off, axis=1, keepdims=True)
    off *= (rng.uniform(0, 2.0, n) * s)[:, None]  # perpendicular miss distance, world units
    o = mu + off - (ratio * s)[:, None] * d
    return {"mu": mu, "quat": quat, "scale": scale, "omega": omega, "rays": pack_rays(o, d)}
