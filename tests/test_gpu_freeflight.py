"""GPU free-flight distance sampling (a8, Eq. 5) per sample, against the oracle.

gf_trace_free_flight runs the render's free-flight kernels (pass A: the ray's tau integrated exactly
into gf_free_flight_bins() t-bins, the first bin whose right edge reaches tau*; pass B: the root inside
that bin) on arbitrary rays, with xi drawn from the same Philox stream the oracle uses (pixel = ray
index).  Reading C17: the oracle brackets the first crossing by the first event segment whose end
reaches tau* (event resolution), the kernels by the first bin edge (bin resolution); the two differ
only where tau(t) rises above tau* and falls back inside one bin (negative Gabor lobes).

Per sample: a "flip" is an escape/collision mismatch or |t_gpu - t_or| > 1e-4 (1 + |t_or|).  At most
0.5 % of the samples may flip, and every flipped sample must satisfy C17 by the oracle's own arithmetic
(or_free_flight_diag): the GPU's t* a root, tau(t*) = tau* within the conditioning floor, in the first
bin whose right-edge tau reaches tau*; a GPU escape must have no bin edge reaching tau*.
"""
import math

import numpy as np
import pytest

from paper_2602_05081_b200 import inputs as I

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def gfm():
    from paper_2602_05081_b200 import build as B
    B.build()
    from paper_2602_05081_b200 import gf
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    return gf


@pytest.fixture(autouse=True, params=["0", "2"], ids=["one_sweep", "windows"])
def windows(request, monkeypatch):
    """Pass A of the warp kernel in one sweep, and in front-to-back windows of 1, 2, 4, .. bins on every ray
    (each window's chords clipped to it, a decision after each): the same first crossings."""
    monkeypatch.setenv("GF_FF_WIN", request.param)
    return request.param


def field(gfm, scene):
    f = gfm.GaborField(0)
    f.load_primitives(scene)
    f.build_bvh()
    return f


def _bin_edges(ray, lo, hi, nb):
    """The ray's scene interval (root box within [tmin, tmax]) and its nb equal bin edges, in double."""
    o, d = ray[:3].astype(np.float64), ray[4:7].astype(np.float64)
    with np.errstate(divide="ignore", invalid="ignore"):
        t1, t2 = (np.asarray(lo) - o) / d, (np.asarray(hi) - o) / d
    ta = max(float(ray[3]), float(np.nanmax(np.minimum(t1, t2))))
    tb = min(float(ray[7]), float(np.nanmin(np.maximum(t1, t2))))
    if not tb >= ta:
        return None
    return ta + (tb - ta) * np.arange(1, nb + 1) / nb


def _check_free_flight(gfm, orc, sc, rays, seed, policy=None, packets=False, what="", flip_tol=0.005):
    """Per-sample comparison; a flipped sample must still be what reading C17 defines: the GPU's t* a
    root (tau(t*) = tau* by the oracle) inside the first bin whose right edge reaches tau* (oracle tau at
    the bin edges), or, for a GPU escape, no bin edge reaching tau*."""
    f = field(gfm, sc)
    if policy is not None:
        f.set_lod_mask(policy)
    info = f.scene_info()
    nb = f.L.gf_free_flight_bins()
    t_g = f.trace_free_flight(rays, seed=seed, packets=packets).cpu().numpy().astype(np.float64)
    S = orc.Scene(sc)
    _, f0 = S.info()
    pol = dict(I.policy(), **(policy or {}))
    n = len(rays)
    flips, bad, not_first = 0, [], 0
    ncol = 0
    for i in range(n):
        xi = orc.uniform(seed, i, 0, 0, 0, 0)
        m, w = pol["static_mask"], None
        if pol["level_strategy"] or pol["orient_strategy"]:
            ul = orc.uniform(seed, i, 0, 0, 0, 1)
            uo = [orc.uniform(seed, i, 0, 0, 0, 2 + l) for l in range(sc["P"] - 1)]
            m, w = S.policy_eval(pol, rays[i, 4:7], ul, uo, f0)
        t_o = S.free_flight(rays[i], xi, m, w)
        tg = t_g[i]
        col_o, col_g = t_o is not None, np.isfinite(tg)
        ncol += col_o
        if col_o == col_g and (not col_o or abs(tg - t_o) <= 1e-4 * (1 + abs(t_o))):
            continue
        flips += 1
        A = S.trace(rays[i:i + 1], mask=m, weights=w, nthreads=1)["A"][0]
        floor = 1e-5 * (1.0 + A)
        tstar = -math.log1p(-xi)
        edges = _bin_edges(rays[i], info["root_lo"], info["root_hi"], nb)
        tau_e = np.array([S.free_flight_diag(rays[i], xi, e, m, w)[0] for e in edges]) if edges is not None else []
        if col_g:
            tau_t, before, _ = S.free_flight_diag(rays[i], xi, tg, m, w)
            kb = int(np.searchsorted(edges, tg))  # the GPU's bin
            ok = abs(tau_t - tstar) <= floor and np.all(tau_e[:kb] < tstar + floor)
            not_first += before >= tstar + floor  # an earlier crossing inside the bin (bin resolution)
        else:
            ok = np.all(np.asarray(tau_e) < tstar + floor)
        if not ok:
            bad.append((i, tg, t_o))
    assert ncol > n // 10, (what, ncol)
    assert not bad, f"{what}: {len(bad)} flipped samples violate C17, e.g. {bad[:3]}"
    assert flips <= flip_tol * n, (what, flips, n)
    print(f"{what}: {flips} flips / {n}, {not_first} roots after an earlier in-bin crossing")
    return flips


def test_free_flight_negative_lobes_per_sample(gfm, orc):
    """Config 1 (unpaired Gabors: kappa < 0 in places, 5 % of rays with tau < 0): 4096 camera rays
    and 1024 random rays, warp-per-ray kernels."""
    sc = I.scene_cfg1()
    desc = I.render_desc_cfg1()
    o, d = I.camera_rays_f64(desc, np.arange(64 * 64) % 64, np.arange(64 * 64) // 64)
    rays = np.concatenate([I.pack_rays(o, d), I.rays_through_box(3, 1024)])
    _check_free_flight(gfm, orc, sc, rays, 0xF1F1, what="cfg1 warp")


def test_free_flight_packets_per_sample(gfm, orc):
    """The packet kernel (32 coherent rays per warp, world slabs) on the same camera rays, and a ragged
    tail (4095 rays)."""
    sc = I.scene_cfg1()
    desc = I.render_desc_cfg1()
    idx = np.arange(64 * 64 - 1)
    o, d = I.camera_rays_f64(desc, idx % 64, idx // 64)
    _check_free_flight(gfm, orc, sc, I.pack_rays(o, d), 0xF1F2, packets=True, what="cfg1 packets")


def test_free_flight_paired_positive_is_exact(gfm, orc):
    """kappa >= 0 (paired-positive scene, C18): tau(t) is monotone, the root unique -- no flips beyond
    the fp32 decisions at tau_total ~ tau*."""
    sc = I.scene_cfg1p()
    rays = I.rays_through_box(5, 2048)
    flips = _check_free_flight(gfm, orc, sc, rays, 0xF1F3, what="cfg1p", flip_tol=0.002)
    assert flips <= 4


@pytest.mark.parametrize("pol", [dict(level_strategy=5, beta=0.2, orient_strategy=3),
                                 dict(static_mask=I.level_mask([0, 2]))])
def test_free_flight_masks_per_sample(gfm, orc, pol):
    """Stochastic (PL+CV Accum. x Importance, weights != 1) and static masks: the masked, reweighted
    field's first crossing."""
    sc = I.scene_cfg1(seed=91)
    rays = I.rays_through_box(6, 1536)
    _check_free_flight(gfm, orc, sc, rays, 0xF1F4, policy=pol, what=str(pol))


def test_free_flight_bunny_surface(gfm, orc):
    """A scaled-down config-2 bunny (surface shell of Gabors over Gaussian interior): camera rays, both
    kernels; clipped [tmin, tmax] ranges on a third of the rays."""
    sc = I.scene_bunny(counts=(300, 2100, 5600, 12000))
    desc = I.render_desc_cfg2(3, 48, 48)
    idx = np.arange(48 * 48)
    o, d = I.camera_rays_f64(desc, idx % 48, idx // 48)
    rays = I.pack_rays(o, d)
    rays[::3, 3] = 2.9
    rays[1::3, 7] = 3.4
    for packets in (False, True):
        _check_free_flight(gfm, orc, sc, rays, 0xF1F5, packets=packets, what=f"bunny packets={packets}")


def test_free_flight_window_halving(gfm, orc, monkeypatch):
    """Pass-B windows with more chords than the record buffer are halved by the exact tau of their left
    half: a 3-record buffer forces that on nearly every ray; same first roots."""
    monkeypatch.setenv("GF_DEBUG_REC_CAP", "3")
    sc = I.scene_cfg1()
    _check_free_flight(gfm, orc, sc, I.rays_through_box(8, 512), 0xF1F6, what="halving")


def test_free_flight_edge_cases(gfm, orc):
    """Empty scene (escape everywhere), rays missing the scene, a zero-length range, and xi = 0 giving
    tau* = 0: collision at tmin (C16)."""
    f = field(gfm, I.empty_scene())
    t = f.trace_free_flight(I.rays_through_box(1, 40)).cpu().numpy()
    assert np.all(np.isinf(t))
    sc = I.scene_cfg1(n=200)
    f = field(gfm, sc)
    miss = I.pack_rays(np.tile([[10.0, 10.0, 10.0]], (33, 1)), np.tile([[1.0, 0, 0]], (33, 1)))
    assert np.all(np.isinf(f.trace_free_flight(miss).cpu().numpy()))
    rays = I.rays_through_box(2, 64)
    rays[:, 7] = rays[:, 3]  # tmax == tmin: nothing to integrate
    assert np.all(np.isinf(f.trace_free_flight(rays).cpu().numpy()))


@pytest.mark.parametrize("packets", [False, True])
def test_free_flight_uniform_in_bin(gfm, orc, packets):
    """GF_EST_UNIFORM (reading U1, the paper's biased alternative): the crossing bin is
    the exact one of C17 and t* = e_{k-1} + u (e_k - e_{k-1}) with u = Philox stream 8 -- per sample,
    from the oracle's tau at the bin edges and the oracle's own Philox.  A flip (different bin or
    escape decision) is allowed only where the deciding edge's tau is within the fp32 floor of tau*."""
    sc = I.scene_cfg1()
    desc = I.render_desc_cfg1()
    idx = np.arange(64 * 64)
    o, d = I.camera_rays_f64(desc, idx % 64, idx // 64)
    rays = np.concatenate([I.pack_rays(o, d), I.rays_through_box(4, 1024)]) if not packets else I.pack_rays(o, d)
    seed = 0xF1F7
    f = field(gfm, sc)
    info = f.scene_info()
    nb = f.L.gf_free_flight_bins()
    t_g = f.trace_free_flight(rays, seed=seed, packets=packets, uniform=True).cpu().numpy().astype(np.float64)
    S = orc.Scene(sc)
    m = I.policy()["static_mask"]
    # the oracle's tau(tmin, e) at every bin edge of every ray, in one batch (rays cut at the edges)
    E = [_bin_edges(r, info["root_lo"], info["root_hi"], nb) for r in rays]
    cut = np.repeat(rays, nb, axis=0)
    cut[:, 7] = np.concatenate([e if e is not None else np.full(nb, r[3]) for e, r in zip(E, rays)])
    tr = S.trace(cut, mask=m)
    tau_all, A_all = tr["tau"].reshape(-1, nb), tr["A"].reshape(-1, nb)[:, -1]
    flips, ncol = 0, 0
    for i in range(len(rays)):
        edges = E[i]
        if edges is None:
            assert np.isinf(t_g[i])
            continue
        tstar = -math.log1p(-orc.uniform(seed, i, 0, 0, 0, 0))
        tau_e = tau_all[i]
        floor = 1e-5 * (1.0 + A_all[i])
        reach = np.nonzero(tau_e >= tstar)[0]
        if len(reach) == 0:
            if np.isinf(t_g[i]):
                continue
            flips += 1
            assert np.max(tau_e) >= tstar - floor, (i, t_g[i])
            continue
        k = int(reach[0])
        ncol += 1
        lo = edges[k - 1] if k > 0 else edges[0] - (edges[-1] - edges[0]) / (nb - 1)  # (k = 0: t_lo)
        u = orc.uniform(seed, i, 0, 0, 8, 0)
        t_exp = lo + u * (edges[k] - lo)
        span = edges[-1] - edges[0] + (edges[1] - edges[0])
        if np.isfinite(t_g[i]) and abs(t_g[i] - t_exp) <= 1e-5 * span + 1e-6:
            continue
        flips += 1  # a neighbouring bin decided in fp32: its deciding edge must be at tau* within the floor
        assert np.min(np.abs(tau_e - tstar)) <= floor, (i, t_g[i], t_exp, k)
    assert ncol > len(rays) // 10
    assert flips <= 0.005 * len(rays), flips
    print(f"uniform-in-bin packets={packets}: {flips} flips / {len(rays)}")
