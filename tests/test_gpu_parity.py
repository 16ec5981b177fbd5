"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded inputs.

Tolerances (DESIGN.md §3 C20/C21, north star): deterministic tau within
|tau_gpu - tau_or| <= 1e-4 |tau_or| + 1e-6 A_or + 1e-7 (A = sum |tau_i|) and T within 1e-4
relative; candidate sets bit-exact between the BVH and brute-force kernels, equal to the
oracle's up to grazing pairs; stochastic estimates with identical Philox streams agree in
per-pixel mean within 3 standard errors.
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


def field(gfm, scene, **kw):
    f = gfm.GaborField(0)
    f.load_primitives(scene, **kw)
    f.build_bvh()
    return f


def assert_tau_parity(tau_g, tau_o, A_o, T_g=None, what=""):
    tau_g = np.asarray(tau_g, np.float64)
    err = np.abs(tau_g - tau_o)
    tol = 1e-4 * np.abs(tau_o) + 1e-6 * A_o + 1e-7
    bad = np.nonzero(err > tol)[0]
    assert bad.size == 0, f"{what}: {bad.size} rays out of tolerance, worst {err[bad].max():.3e} e.g. ray {bad[0]}: " \
                          f"gpu {tau_g[bad[0]]} oracle {tau_o[bad[0]]} A {A_o[bad[0]]}"
    if T_g is not None:
        T_o = np.exp(-tau_o)
        assert np.all(np.abs(np.asarray(T_g, np.float64) - T_o) <= 1e-4 * T_o + 1e-7), what


def camera_rays(desc, n=None, seed=0):
    W, H = desc["width"], desc["height"]
    if n is None:
        idx = np.arange(W * H)
    else:
        idx = np.random.default_rng(seed).integers(0, W * H, n)
    o, d = I.camera_rays_f64(desc, idx % W, idx // W)
    return I.pack_rays(o, d)


# ------------------------------------------------------------------------------ a1
def test_load_groups_match_oracle(gfm, orc):
    sc = I.scene_cfg1()
    f = field(gfm, sc)
    # prim_ws layout: n x 64-byte records, then (256-aligned) n group ids
    off = (64 * sc["n"] + 255) // 256 * 256
    g_gpu = f.prim_ws[off: off + sc["n"]].cpu().numpy().astype(np.int64)
    g_or, _ = orc.Scene(sc).groups()
    assert np.array_equal(g_gpu, g_or)


def test_invalid_inputs_rejected(gfm):
    sc = I.scene_cfg1(n=50)
    bad = dict(sc, scale=sc["scale"].copy())
    bad["scale"][7, 1] = 0.0
    f = gfm.GaborField(0)
    with pytest.raises(gfm.GFError) as e:
        f.load_primitives(bad)
    assert e.value.status == 3  # GF_E_SINGULAR_COVARIANCE
    bad = dict(sc, level=sc["level"].copy())
    bad["level"][3] = 9
    with pytest.raises(gfm.GFError) as e:
        f.load_primitives(bad)
    assert e.value.status == 8
    with pytest.raises(gfm.GFError) as e:
        f.trace_transmittance(np.zeros((1, 8), np.float32))
    assert e.value.status == 2  # GF_E_STATE
    with pytest.raises(gfm.GFError) as e:
        f.set_lod_mask({"level_strategy": 2, "beta": 1.0})
    assert e.value.status == 7


# ------------------------------------------------------------------------------ a4-a7
@pytest.mark.parametrize("brute", [False, True])
def test_cfg1_camera_tau_parity(gfm, orc, brute):
    sc = I.scene_cfg1()
    desc = I.render_desc_cfg1()
    rays = camera_rays(desc)
    f = field(gfm, sc)
    tau, T, _ = f.trace_transmittance(rays, brute_force=brute)
    r = orc.Scene(sc).trace(rays)
    assert_tau_parity(tau.cpu().numpy(), r["tau"], r["A"], T.cpu().numpy(), "cfg1 camera")


def test_random_rays_and_ragged_sizes(gfm, orc):
    sc = I.scene_cfg1(seed=77)
    f = field(gfm, sc)
    S = orc.Scene(sc)
    for n in (1, 31, 129, 1000):
        rays = I.rays_through_box(n, n, tmin=0.0)
        rays[::3, 3] = 2.5   # clipped starts
        rays[::5, 7] = 4.7   # clipped ends
        tau, T, _ = f.trace_transmittance(rays)
        r = S.trace(rays)
        assert_tau_parity(tau.cpu().numpy(), r["tau"], r["A"], T.cpu().numpy(), f"n={n}")


def test_empty_scene_and_misses(gfm):
    f = field(gfm, I.empty_scene())
    tau, T, _ = f.trace_transmittance(I.rays_through_box(1, 64))
    assert torch.all(tau == 0) and torch.all(T == 1)
    f2 = field(gfm, I.scene_cfg1(n=100))
    miss = I.pack_rays(np.tile([[10.0, 10.0, 10.0]], (8, 1)), np.tile([[1.0, 0, 0]], (8, 1)))
    tau, T, _ = f2.trace_transmittance(miss)
    assert torch.all(tau == 0)


@pytest.mark.parametrize("keys", ["level", "group"])
def test_candidate_sets_bvh_equal_brute_force(gfm, orc, keys):
    """C21: BVH candidate sets == brute-force kernel sets bit-exactly (same fp32 predicate), and ==
    the double oracle's up to grazing pairs (|r^2/E^2 - 1| <= 1e-5) -- with (band, level) key classes
    (orientation bins mixed below them) and with per-group subtrees (gf_set_bvh_keys)."""
    for sc, masks in ((I.scene_cfg1(), (0xFFFFFFFF, I.level_mask([0, 2]), 1 << 5)),
                      (I.scene_cfg2(), (0xFFFFFFFF, I.level_mask([0, 1]))),
                      (I.scene_cfg5(copies=4, grid=(2, 2)), (0xFFFFFFFF, I.level_mask([0, 1], n_bands=3)))):
        f = gfm.GaborField(0)
        f.set_bvh_keys(gfm.BVH_KEYS_GROUP if keys == "group" else gfm.BVH_KEYS_LEVEL)
        f.load_primitives(sc)
        f.build_bvh()
        S = orc.Scene(sc)
        if "band" in sc:  # 4 army copies, 3 distance bands: rays through the scene's root box
            info = f.scene_info()
            lo, hi = np.asarray(info["root_lo"], np.float64), np.asarray(info["root_hi"], np.float64)
            rng = np.random.default_rng(5)
            tgt = lo + (hi - lo) * rng.random((300, 3))
            org = (lo + hi) / 2 + np.linalg.norm(hi - lo) * rng.normal(size=(300, 3))
            rays = I.pack_rays(org, tgt - org)
        else:
            desc = I.render_desc_cfg1() if sc["n"] == 1000 else I.render_desc_cfg2(3, 256, 256)
            rays = camera_rays(desc, 300, seed=5)
            rays[::4] = I.rays_through_box(9, len(rays[::4]))
        for m in masks:
            f.set_lod_mask({"static_mask": m})
            ids_b, cnt_b = f.trace_candidates(rays, 4096)
            ids_f, cnt_f = f.trace_candidates(rays, 4096, brute_force=True)
            ids_b, cnt_b, ids_f, cnt_f = (t.cpu().numpy() for t in (ids_b, cnt_b, ids_f, cnt_f))
            assert np.array_equal(cnt_b, cnt_f)
            grazing = 0
            for k in range(len(rays)):
                sb = set(ids_b[k, :cnt_b[k]].tolist())
                assert sb == set(ids_f[k, :cnt_f[k]].tolist())
                so = set(S.candidates(rays[k], m)[0].tolist())
                for i in sb ^ so:
                    assert abs(S.r2_rel(i, rays[k]) - 1.0) <= 1e-5, (k, i)
                    grazing += 1
            assert grazing <= 2


def test_static_masks_parity(gfm, orc):
    sc = I.scene_cfg1()
    f = field(gfm, sc)
    S = orc.Scene(sc)
    rays = camera_rays(I.render_desc_cfg1(), 512, seed=3)
    for levels in ([0], [0, 1], [0, 1, 2], [1, 3]):
        m = I.level_mask(levels)
        f.set_lod_mask({"static_mask": m})
        tau, _, _ = f.trace_transmittance(rays)
        r = S.trace(rays, mask=m)
        assert_tau_parity(tau.cpu().numpy(), r["tau"], r["A"], None, f"mask {levels}")


@pytest.mark.parametrize("pol", [dict(level_strategy=5, beta=0.2, orient_strategy=3),
                                 dict(level_strategy=1), dict(level_strategy=4, beta=0.5, orient_strategy=4,
                                                              delta=0.5),
                                 dict(orient_strategy=2), dict(level_strategy=3, orient_strategy=1, delta=0.7)])
def test_stochastic_mask_parity(gfm, orc, pol):
    """Per-ray stochastic policy with identical Philox uniforms: same mask and weights on both sides
    (DESIGN.md §5), so tau-hat agrees per ray to the deterministic tolerance."""
    sc = I.scene_cfg1()
    f = field(gfm, sc)  # group f0: the library's medians (C12)
    f.set_lod_mask(pol)
    rays = camera_rays(I.render_desc_cfg1(), 256, seed=11)
    seed = 0xABCDEF12345
    tau, _, _ = f.trace_transmittance(rays, seed=seed)
    S = orc.Scene(sc)
    f0 = S.info()[1]
    P = sc["P"]
    tau_o, A_o = np.zeros(len(rays)), np.zeros(len(rays))
    for i in range(len(rays)):
        ul = orc.uniform(seed, i, 0, 0, 0, 1)
        uo = [orc.uniform(seed, i, 0, 0, 0, 2 + l) for l in range(P - 1)]
        m, w = S.policy_eval(dict(I.policy(), **pol), rays[i, 4:7], ul, uo, f0)
        r = S.trace(rays[i:i + 1], mask=m, weights=w, nthreads=1)
        tau_o[i], A_o[i] = r["tau"][0], r["A"][0]
    assert_tau_parity(tau.cpu().numpy(), tau_o, A_o, None, str(pol))


@pytest.mark.parametrize("ratio", [30.0, 300.0, 3000.0])
def test_far_origin_stress(gfm, orc, ratio):
    """rays starting |o-mu|/s in {30,300,3000} from primitives of s in [0.005,0.05]."""
    fo = I.far_origin_pairs(int(ratio), 2000, ratio)
    n = len(fo["rays"])
    sc = {"n": n, "P": 4, "K": 3, "mu": fo["mu"].astype(np.float32), "quat": fo["quat"],
          "scale": fo["scale"].astype(np.float32), "alpha": np.ones(n, np.float32),
          "omega": fo["omega"].astype(np.float32), "extent": np.full(n, 3.0, np.float32),
          "level": np.ones(n, np.uint8), "bin": np.zeros(n, np.uint8), "bin_axes": I.bin_axes(3)}
    f = field(gfm, sc)
    tau, _, _ = f.trace_transmittance(fo["rays"])
    r = orc.Scene(sc).trace(fo["rays"])
    assert_tau_parity(tau.cpu().numpy(), r["tau"], r["A"], None, f"far origin {ratio}")


def test_cfg2_sampled_rays(gfm, orc):
    sc = I.scene_cfg2()
    f = field(gfm, sc)
    desc = I.render_desc_cfg2(3)
    rays = camera_rays(desc, 600, seed=21)
    S = orc.Scene(sc)
    for li, levels in enumerate(I.CFG2_LOD_LEVELS):
        m = I.level_mask(levels)
        f.set_lod_mask({"static_mask": m})
        tau, T, cnt = f.trace_transmittance(rays, counters=True)
        r = S.trace(rays, mask=m)
        assert_tau_parity(tau.cpu().numpy(), r["tau"], r["A"], T.cpu().numpy(), f"cfg2 mask {levels}")
        assert np.array_equal(cnt.cpu().numpy()[:, 2], r["nhits"])


# ------------------------------------------------------------------------------ render
def test_render_tomography_cfg1_full_image(gfm, orc):
    """Config 1 exactly as the bench runs it: 64x64, pixel centres, 1 spp, full LOD, gf_render."""
    sc = I.scene_cfg1()
    desc = I.render_desc_cfg1()
    f = field(gfm, sc)
    acc, rc = f.render(desc)
    acc = acc.view(-1, 2).cpu().numpy()
    S = orc.Scene(sc)
    pix = np.arange(64 * 64)
    vals, _ = S.render_probes(desc, pix, 0, 1)
    r = S.trace(camera_rays(desc))
    assert_tau_parity(acc[:, 0], vals[:, 0], r["A"], None, "cfg1 tomo")
    assert int(rc[0]) == 64 * 64


@pytest.mark.parametrize("wh", [(37, 29), (64, 64)])
def test_render_tomography_packets_forced(gfm, orc, monkeypatch, wh):
    """k_tomo_pkt (camera-BVH packets, lane-local integrals) forced on small images, a ragged
    37x29 one included (last packet partly empty): every pixel against the oracle."""
    monkeypatch.setenv("GF_DEBUG_TOMO_PKT_MIN", "0")
    sc = I.scene_cfg1()
    W, H = wh
    desc = I.render_desc_cfg1(W, H)
    f = field(gfm, sc)
    acc, rc = f.render(desc)
    acc = acc.view(-1, 2).cpu().numpy()
    S = orc.Scene(sc)
    vals, _ = S.render_probes(desc, np.arange(W * H), 0, 1)
    r = S.trace(camera_rays(desc))
    assert_tau_parity(acc[:, 0], vals[:, 0], r["A"], None, f"packet tomo {wh}")
    assert int(rc[0]) == W * H
    # incoherent packets (random probe pixels) and an empty mask
    probes = np.random.default_rng(9).integers(0, W * H, 77).astype(np.int32)
    vg, _ = f.render(desc, probes=probes)
    assert_tau_parity(vg.cpu().numpy().reshape(-1), vals[probes, 0], r["A"][probes], None, "packet tomo probes")
    acc0, _ = f.render(dict(desc, ext=I.policy(static_mask=0)))
    assert np.all(acc0.view(-1, 2).cpu().numpy()[:, 0] == 0.0)


def test_render_tomography_cfg2_full_size_sampled(gfm, orc):
    """The bench's --tomography variant of config 2 (1024x1024, jittered, 4 LOD masks) in its launch
    configuration (k_tomo_pkt): 256 sampled pixels per mask against the oracle."""
    sc = I.scene_cfg2()
    f = field(gfm, sc)
    S = orc.Scene(sc)
    rng = np.random.default_rng(10)
    for i in range(4):
        desc = dict(I.render_desc_cfg2(i), mode=0, max_depth=1)
        acc, rc = f.render(desc)
        acc = acc.view(-1, 2).cpu().numpy()
        assert int(rc[0]) == 1024 * 1024
        pix = rng.integers(0, 1024 * 1024, 256).astype(np.int32)
        vo, _ = S.render_probes(desc, pix, 0, 1)
        d = np.abs(acc[pix, 0] - vo[:, 0])
        assert np.all(d <= 1e-4 * np.maximum(1.0, np.abs(vo[:, 0]))), (i, d.max())


def test_render_tomography_packets_two_chunks_jittered(gfm, orc):
    """k_tomo_pkt across the 1M-path chunk boundary (2048x1024 = two chunks), jittered, 2 samples
    (spp_begin 3): sampled pixels, both samples, against the oracle's identical Philox draws."""
    sc = I.scene_cfg2()
    f = field(gfm, sc)
    desc = dict(I.render_desc_cfg2(2, 2048, 1024), mode=0, max_depth=1, jitter=1)
    acc, rc = f.render(desc, 3, 2)
    acc = acc.view(-1, 2).cpu().numpy().astype(np.float64)
    assert int(rc[0]) == 2 * 2048 * 1024
    rng = np.random.default_rng(13)
    # pixels near the chunk boundary (path index 2^20 = tile-ordered) and random ones
    pix = np.concatenate([rng.integers(0, 2048 * 1024, 200), np.arange(1024 * 512 - 40, 1024 * 512 + 40)]).astype(np.int32)
    vo, _ = orc.Scene(sc).render_probes(desc, pix, 3, 2)
    d = np.abs(acc[pix, 0] - vo.sum(axis=1))
    assert np.all(d <= 1e-4 * np.maximum(1.0, np.abs(vo.sum(axis=1)))), d.max()


def _probe_compare(gfm, orc, sc, desc, probes, spp, what, frac_tol=0.02, f=None):
    f = f or field(gfm, sc)  # group f0 on both sides: the scene's medians (C12)
    vg, rc = f.render(desc, 0, spp, probes=probes)
    vg = vg.view(len(probes), spp).cpu().numpy().astype(np.float64)
    vo, nr = orc.Scene(sc).render_probes(desc, probes, 0, spp)
    diff = np.abs(vg - vo)
    flips = np.mean(diff > 1e-3 * (np.abs(vo) + 1e-2))
    se = vo.std() / math.sqrt(vo.size)
    assert abs(vg.mean() - vo.mean()) <= 3 * se + 1e-6, (what, vg.mean(), vo.mean(), se)
    assert flips <= frac_tol, (what, flips)
    per_pix_se = vo.std(1) / math.sqrt(spp) + 1e-9
    assert np.mean(np.abs(vg.mean(1) - vo.mean(1)) <= 3 * per_pix_se + 1e-6) >= 0.98
    return vg, vo, int(rc.sum())


def test_render_single_scatter_probes_paired(gfm, orc):
    sc = I.scene_cfg1p()
    desc = I.render_desc_cfg2(3, 64, 64)
    desc.update(**I.camera((0, 0, 4), (0, 0, 0), (0, 1, 0), 40.0, 64, 64))
    desc["ext"] = desc["nee"] = I.policy()
    probes = np.random.default_rng(1).integers(0, 64 * 64, 48)
    _probe_compare(gfm, orc, sc, desc, probes, 16, "single scatter cfg1p")


def test_render_multi_scatter_probes(gfm, orc):
    sc = I.scene_cfg1p()
    desc = I.render_desc_cfg2(3, 32, 32)
    desc.update(**I.camera((0, 0, 4), (0, 0, 0), (0, 1, 0), 40.0, 32, 32))
    desc.update(max_depth=6, albedo=0.95, hg_g=0.6, ext=I.policy(), nee=I.policy())
    probes = np.random.default_rng(2).integers(0, 32 * 32, 24)
    _probe_compare(gfm, orc, sc, desc, probes, 16, "multi scatter", frac_tol=0.05)


def test_render_stochastic_masks_probes(gfm, orc):
    """Config-4 style policies: PL+CV(Accum.) beta=0.2 x orientation Importance on extension
    rays, Zero NEE, multiple scattering, identical Philox streams."""
    sc = I.scene_cfg1()
    desc = I.render_desc_cfg2(3, 32, 32)
    desc.update(**I.camera((0, 0, 4), (0, 0, 0), (0, 1, 0), 40.0, 32, 32))
    desc.update(max_depth=4, albedo=0.9, ext=I.policy(level_strategy=5, beta=0.2, orient_strategy=3),
                nee=I.policy(static_mask=1))
    probes = np.random.default_rng(3).integers(0, 32 * 32, 24)
    _probe_compare(gfm, orc, sc, desc, probes, 16, "stochastic", frac_tol=0.05)


def test_render_tomography_stochastic_probes(gfm, orc):
    sc = I.scene_cfg1()
    desc = I.render_desc_cfg1(32, 32)
    desc.update(jitter=1, ext=I.policy(level_strategy=2, beta=0.5, orient_strategy=2))
    probes = np.random.default_rng(4).integers(0, 32 * 32, 32)
    vg, vo, _ = _probe_compare(gfm, orc, sc, desc, probes, 32, "stochastic tomography", frac_tol=0.0)


def test_render_record_fallback_paths(gfm, orc, monkeypatch):
    """Free-flight windows with more chords than the pass-B record buffer are halved by the exact
    tau of their left half until they fit: a 4-record buffer routes nearly every path there."""
    monkeypatch.setenv("GF_DEBUG_REC_CAP", "4")
    sc = I.scene_cfg1p()
    desc = I.render_desc_cfg2(3, 32, 32)
    desc.update(**I.camera((0, 0, 4), (0, 0, 0), (0, 1, 0), 40.0, 32, 32))
    desc.update(max_depth=3, albedo=0.9, ext=I.policy(), nee=I.policy())
    probes = np.random.default_rng(6).integers(0, 32 * 32, 24)
    _probe_compare(gfm, orc, sc, desc, probes, 16, "record fallback", frac_tol=0.05)


def _mean_parity(vg, vo, what, pix_frac=0.95):
    """Different estimators of the same pixel values: global and per-pixel means within 3 combined SE."""
    n = vg.shape[1]
    se = math.sqrt(vg.var() / vg.size + vo.var() / vo.size)
    assert abs(vg.mean() - vo.mean()) <= 3 * se + 1e-6, (what, vg.mean(), vo.mean(), se)
    se_pix = np.sqrt(vg.var(1) / n + vo.var(1) / n) + 1e-9
    ok = np.abs(vg.mean(1) - vo.mean(1)) <= 3 * se_pix + 1e-6
    assert ok.mean() >= pix_frac, (what, ok.mean())


@pytest.mark.parametrize("max_depth", [1, 3])
def test_render_tracking_estimators_mean_parity(gfm, orc, max_depth):
    """SURVEY §8 a9 alternative: delta tracking (free flight) + ratio tracking (NEE) against the
    oracle's analytic estimator on a kappa >= 0 (paired-positive, C18) scene: same pixel means."""
    sc = I.scene_cfg1p()
    desc = I.render_desc_cfg2(3, 32, 32)
    desc.update(**I.camera((0, 0, 4), (0, 0, 0), (0, 1, 0), 40.0, 32, 32))
    desc.update(max_depth=max_depth, albedo=0.9, hg_g=0.3, ext=I.policy(), nee=I.policy())
    probes = np.random.default_rng(7).integers(0, 32 * 32, 40)
    spp = 96
    f = field(gfm, sc)
    vg, _ = f.render(dict(desc, estimator=1), 0, spp, probes=probes)
    vg = vg.view(len(probes), spp).cpu().numpy().astype(np.float64)
    vo, _ = orc.Scene(sc).render_probes(desc, probes, 0, spp)
    _mean_parity(vg, vo, f"tracking depth {max_depth}")
    va, _ = f.render(desc, 0, spp, probes=probes)  # analytic on the GPU: same means too
    _mean_parity(vg, va.view(len(probes), spp).cpu().numpy().astype(np.float64), "tracking vs analytic gpu")


@pytest.mark.parametrize("rec_cap", [None, "16"])
def test_column_more_hits_than_record_buffer(gfm, orc, monkeypatch, rec_cap):
    """1500 primitives along one axis: rays along it overlap all of them.  With a 16-record buffer the
    free-flight windows overflow and are halved (pass B); with the default buffer they fit.
    Transmittance parity, then free flight through the column vs the oracle."""
    if rec_cap:
        monkeypatch.setenv("GF_DEBUG_REC_CAP", rec_cap)
    sc = I.scene_column()
    f = field(gfm, sc)
    S = orc.Scene(sc)
    o = np.array([[-1.5, 0.0005 * k, -0.0003 * k] for k in range(8)])
    d = np.tile([[1.0, 0.0, 0.0]], (8, 1))
    rays = I.pack_rays(o, d)
    tau, T, cnt = f.trace_transmittance(rays, counters=True)
    r = S.trace(rays)
    assert_tau_parity(tau.cpu().numpy(), r["tau"], r["A"], T.cpu().numpy(), "column")
    assert cnt.cpu().numpy()[:, 2].min() > 1024
    desc = I.render_desc_cfg2(3, 16, 16)
    desc.update(**I.camera((-1.5, 0, 0), (0, 0, 0), (0, 1, 0), 1.0, 16, 16))
    desc.update(max_depth=2, albedo=0.9, ext=I.policy(), nee=I.policy())
    probes = np.arange(16 * 16)[::8]
    _probe_compare(gfm, orc, sc, desc, probes, 8, "column free flight", frac_tol=0.05)


@pytest.mark.parametrize("which", ["LIGHT", "CAMERA"])
@pytest.mark.parametrize("stoch", [False, True])
def test_view_bvhs_same_hits(gfm, monkeypatch, stoch, which):
    """NEE traverses the light BVH (boxes in the light's frame), the camera rays the camera BVH
    (projective boxes at the eye).  Each must find exactly the hits of the world BVH: same hit
    counts, same image (static masks: packet kernel; stochastic: warp-per-ray kernels)."""
    sc = I.scene_cfg2()
    f = field(gfm, sc)
    desc = I.render_desc_cfg2(3, 64, 64)
    desc.update(max_depth=3, albedo=0.9, hg_g=0.3)
    if stoch:
        desc.update(ext=I.policy(level_strategy=5, beta=0.2, orient_strategy=3),
                    nee=I.policy(level_strategy=2, beta=0.5, orient_strategy=2))
    stage = "nee" if which == "LIGHT" else "ffA"
    # (pass A in windows stops at the first crossing, at a split that depends on the last collision's kappa:
    # the hit counts compare one full sweep per ray)
    monkeypatch.setenv("GF_FF_WIN", "0")
    out = []
    for off in ("0", "1"):
        monkeypatch.setenv(f"GF_DEBUG_NO_{which}_BVH", off)
        f.set_profiling(work=True)
        acc, _ = f.render(desc, 0, 2)
        st = f.stats(reset=True)
        f.set_profiling()
        out.append((acc.cpu().numpy(), st["work"][stage]))
    # the same chords: equal hit counts up to the few grazing chords of bounces whose origins moved by an
    # ulp (the two free-flight kernels sum the same integrals in different orders)
    assert abs(out[0][1]["hits"] - out[1][1]["hits"]) <= 1e-5 * out[0][1]["hits"] and out[0][1]["hits"] > 0
    assert abs(out[0][1]["paths"] - out[1][1]["paths"]) <= 1e-4 * out[0][1]["paths"]
    np.testing.assert_allclose(out[0][0], out[1][0], rtol=1e-4, atol=1e-5)


def test_reused_view_bvhs(gfm):
    """gf_render reuse_accel: the light / camera BVHs kept in scratch are reused only for the same
    scene, light and camera; results equal those of fresh builds, also after a camera change."""
    sc = I.scene_cfg2()
    f = field(gfm, sc)
    d1 = I.render_desc_cfg2(3, 64, 64)
    d2 = dict(d1, **I.camera((0.3, 0.2, 3.0), (0, 0.05, 0), (0, 1, 0), 40.0, 64, 64))
    scratch = f.render_scratch(d1, 1)
    ref1, _ = f.render(d1, 0, 1)
    ref2, _ = f.render(d2, 0, 1)
    a1, _ = f.render(dict(d1, reuse_accel=1), 0, 1, scratch=scratch)
    b1, _ = f.render(dict(d1, reuse_accel=1), 0, 1, scratch=scratch)
    a2, _ = f.render(dict(d2, reuse_accel=1), 0, 1, scratch=scratch)
    for x, y in ((a1, ref1), (b1, ref1), (a2, ref2)):
        assert torch.equal(x, y)


def test_reused_view_bvhs_probe_and_full_layouts(gfm):
    """a probe render, a full-image render and the probe render again on ONE scratch with
    reuse_accel = 1.  The two calls lay the scratch out differently (per-path arrays sized by their path
    counts), so the full render overwrites the probe call's view BVHs; the cache is keyed on the layout
    and must rebuild -- every result equals a fresh build's."""
    sc = I.scene_cfg2()
    f = field(gfm, sc)
    d = I.render_desc_cfg2(3, 96, 96)
    rng = np.random.default_rng(3)
    probes = rng.choice(96 * 96, 200, replace=False).astype(np.int32)
    scratch = f.render_scratch(d, 1)
    ref_p, _ = f.render(d, 0, 2, probes=probes)
    ref_f, _ = f.render(d, 0, 1)
    seq = [("p", f.render(dict(d, reuse_accel=1), 0, 2, probes=probes, scratch=scratch)[0]),
           ("f", f.render(dict(d, reuse_accel=1), 0, 1, scratch=scratch)[0]),
           ("p", f.render(dict(d, reuse_accel=1), 0, 2, probes=probes, scratch=scratch)[0]),
           ("f", f.render(dict(d, reuse_accel=1), 0, 1, scratch=scratch)[0])]
    for kind, x in seq:
        assert torch.equal(x, ref_p if kind == "p" else ref_f), kind


def test_warp_traversal_depth_first_mode(gfm, orc, monkeypatch):
    """The warp traversal pops one node per step above its stack threshold (bounded stack);
    forcing that mode everywhere gives the same hits and transmittance."""
    sc = I.scene_cfg2()
    f = field(gfm, sc)
    rays = camera_rays(I.render_desc_cfg2(3), 300, seed=23)
    tau0, _, c0 = f.trace_transmittance(rays, counters=True)
    monkeypatch.setenv("GF_DEBUG_STK_LIMIT", "1")
    tau1, _, c1 = f.trace_transmittance(rays, counters=True)
    assert torch.equal(c0[:, 1:], c1[:, 1:])
    r = orc.Scene(sc).trace(rays)
    assert_tau_parity(tau1.cpu().numpy(), r["tau"], r["A"], None, "depth-first mode")
    assert np.array_equal(c1.cpu().numpy()[:, 2], r["nhits"])


@pytest.mark.parametrize("mode", [0, 1])
def test_render_foveation_probes(gfm, orc, mode):
    """Foveated rendering: per-pixel frequency threshold linear in
    the eccentricity with stochastic smoothing, level masking and the per-primitive check along the
    ray; identical Philox streams.  Tomography and multiple scattering vs the oracle."""
    sc = I.scene_cfg1p() if mode else I.scene_cfg1()
    f = field(gfm, sc)
    lf = f.scene_info()["level_fmax"]
    np.testing.assert_allclose(lf, orc.Scene(sc).info()[0], rtol=1e-6)
    fov = I.foveation((10.0, 20.0), float(lf[1:4].max()) * 1.05, float(lf[1:4].max()) * 1.6, 0.3)
    if mode == 0:
        desc = dict(I.render_desc_cfg1(32, 32), jitter=1, foveation=fov)
    else:
        desc = I.render_desc_cfg2(3, 32, 32)
        desc.update(**I.camera((0, 0, 4), (0, 0, 0), (0, 1, 0), 40.0, 32, 32))
        desc.update(max_depth=3, albedo=0.9, hg_g=0.3, ext=I.policy(), nee=I.policy(), foveation=fov)
    probes = np.random.default_rng(8).integers(0, 32 * 32, 40)
    _probe_compare(gfm, orc, sc, desc, probes, 8, f"foveation mode {mode}", frac_tol=0.03, f=f)
    for fm in (1, 2):  # level masking only, continuous check only
        d = dict(desc, foveation=dict(fov, mode=fm))
        _probe_compare(gfm, orc, sc, d, probes, 8, f"foveation mode {mode} bits {fm}", frac_tol=0.03, f=f)


@pytest.mark.parametrize("mode", [0, 1])
def test_render_motion_blur_reference_probes(gfm, orc, mode):
    """Motion-blur reference: per-sample exposure time, field shifted
    along the motion (camera shifted back), identical Philox streams; plus the accelerated version
    (culled groups) is just a static mask: both vs the oracle."""
    sc = I.scene_cfg1p() if mode else I.scene_cfg1()
    mb = I.motion_blur((1.0, 0.2, 0.0), 0.3)
    if mode == 0:
        desc = dict(I.render_desc_cfg1(32, 32), jitter=1, motion_blur=mb)
    else:
        desc = I.render_desc_cfg2(3, 32, 32)
        desc.update(**I.camera((0, 0, 4), (0, 0, 0), (0, 1, 0), 40.0, 32, 32))
        desc.update(max_depth=2, albedo=0.9, hg_g=0.3, ext=I.policy(), nee=I.policy(), motion_blur=mb)
    probes = np.random.default_rng(9).integers(0, 32 * 32, 40)
    f = field(gfm, sc)
    _probe_compare(gfm, orc, sc, desc, probes, 8, f"motion blur mode {mode}", frac_tol=0.03, f=f)
    mask, att = f.motion_blur_mask(mb["dir"], mb["m"], 0.6)  # the library's culling (M3)
    mask_o, att_o = orc.Scene(sc).motion_blur_mask(mb["dir"], mb["m"], 0.6)
    np.testing.assert_allclose(att, att_o, rtol=1e-5, atol=1e-6)
    assert mask == mask_o and 0 < bin(mask).count("1") < 10
    culled = dict(desc, ext=I.policy(static_mask=mask), nee=I.policy(static_mask=mask))
    culled.pop("motion_blur")
    _probe_compare(gfm, orc, sc, culled, probes, 8, f"motion blur culled mode {mode}", frac_tol=0.03, f=f)


def test_adaptive_extent_parity(gfm, orc):
    """Adaptive clamping (Eq. 15, reading C8'): per-primitive extents are inputs of both sides; the
    transmittance parity holds and the clamped field is cheaper (fewer hits) than the 3-sigma one."""
    sc = I.scene_cfg2()
    f3 = field(gfm, sc)
    ext = f3.adaptive_extent(sc, 1e-3).cpu().numpy()  # the library's extents (gf_adaptive_extent)
    ext_o = orc.adaptive_extent(sc, 1e-3)
    np.testing.assert_allclose(ext, ext_o, rtol=2e-7)
    sca = dict(sc, extent=ext)
    assert np.all(sca["extent"] <= 3.0) and np.mean(sca["extent"]) < 3.0
    rays = camera_rays(I.render_desc_cfg2(3), 300, seed=31)
    f = field(gfm, sca)
    tau, T, cnt = f.trace_transmittance(rays, counters=True)
    r = orc.Scene(sca).trace(rays)
    assert_tau_parity(tau.cpu().numpy(), r["tau"], r["A"], T.cpu().numpy(), "adaptive extent")
    assert np.array_equal(cnt.cpu().numpy()[:, 2], r["nhits"])
    _, _, c3 = f3.trace_transmittance(rays, counters=True)
    assert cnt[:, 2].sum() < c3[:, 2].sum()


@pytest.mark.parametrize("stoch", [False, True])
def test_grad_alpha_parity(gfm, orc, stoch):
    """Opacity gradient (the alpha part) vs the oracle's plain double loops:
    per primitive within 1e-4 relative + 1e-6 of the largest |gradient|."""
    sc = I.scene_cfg1(seed=21)
    f = field(gfm, sc)
    pol = I.policy(level_strategy=5, beta=0.2, orient_strategy=3) if stoch else I.policy(static_mask=I.level_mask([0, 2, 3]))
    f.set_lod_mask(pol)
    rays = I.rays_through_box(4, 500)
    dl = np.random.default_rng(7).normal(size=500).astype(np.float32)
    g = f.trace_grad_alpha(rays, dl, seed=5).cpu().numpy().astype(np.float64)
    S = orc.Scene(sc)
    if stoch:
        go = np.zeros(sc["n"])
        f0 = S.info()[1]
        for r in range(len(rays)):  # per-ray masks and weights (same draws as gf_trace_transmittance)
            ul = orc.uniform(5, r, 0, 0, 0, 1)
            uo = [orc.uniform(5, r, 0, 0, 0, 2 + l) for l in range(sc["P"] - 1)]
            m, w = S.policy_eval(dict(I.policy(), **pol), rays[r, 4:7], ul, uo, f0)
            go += S.grad_alpha(rays[r:r + 1], dl[r:r + 1].astype(np.float64), m, w)
    else:
        go = S.grad_alpha(rays, dl.astype(np.float64), pol["static_mask"])
    tol = 1e-4 * np.abs(go) + 1e-6 * np.abs(go).max()
    assert np.all(np.abs(g - go) <= tol), np.max(np.abs(g - go) - tol)
    assert np.count_nonzero(go) > 100


def _bench_frames(f, descs, spp_begin=0):
    """The frames of one bench step, in bench.py's launch configuration: two CUDA streams, one render
    scratch each, view BVHs reused (reuse_accel); returns the accumulators (frames x H*W*2)."""
    H, W = descs[0]["height"], descs[0]["width"]
    streams = [torch.cuda.current_stream(), torch.cuda.Stream()]
    scr = [f.render_scratch(descs[0], 1) for _ in streams]
    acc = torch.zeros((len(descs), H * W * 2), dtype=torch.float32, device="cuda")
    rays = torch.zeros(3, dtype=torch.int64, device="cuda")
    for rep in range(2):  # the second pass reuses the view BVHs the first built
        acc.zero_()
        rays.zero_()
        streams[1].wait_stream(streams[0])
        for i, d in enumerate(descs):
            with torch.cuda.stream(streams[i % 2]):
                f.render(dict(d, reuse_accel=1), spp_begin, 1, accum=acc[i], ray_counts=rays, scratch=scr[i % 2])
        streams[0].wait_stream(streams[1])
    torch.cuda.synchronize()
    return acc.view(len(descs), -1, 2).cpu().numpy().astype(np.float64), rays


def _sampled_parity(orc, sc, desc, acc, pix, what, max_flips):
    """Sampled pixels of a 1-spp full-image render vs the oracle's paths with identical Philox streams:
    per-sample flips (fp32 / fp64 branch decisions along the path) bounded, and the sample mean within 3
    standard errors."""
    vo, _ = orc.Scene(sc).render_probes(desc, pix, 0, 1)
    vo = vo[:, 0]
    vg = acc[pix, 0]
    flips = int(np.sum(np.abs(vg - vo) > 1e-3 * (np.abs(vo) + 1e-2)))
    se = vo.std() / math.sqrt(len(vo))
    assert flips <= max_flips, (what, flips)
    assert abs(vg.mean() - vo.mean()) <= 3 * se + 1e-6, (what, vg.mean(), vo.mean(), se)
    assert np.all(np.abs(acc[pix, 1] - vg * vg) <= 1e-6 * (vg * vg) + 1e-12)  # 1 spp: sum of squares


def test_cfg2_bench_configuration_sampled(gfm, orc):
    """Config 2 at full size in the launch configuration bench.py times (1024^2, 1 spp per LOD mask,
    single scattering, 2 streams, reused view BVHs): 128 sampled pixels per mask vs the oracle's paths."""
    sc = I.scene_cfg2()
    f = field(gfm, sc)
    descs = [I.render_desc_cfg2(i) for i in range(4)]
    acc, rays = _bench_frames(f, descs)
    assert int(rays[0]) == 4 * 1024 * 1024 and int(rays[1]) == 0  # single scattering: camera rays only
    rng = np.random.default_rng(5)
    for mi in (0, 3):
        pix = rng.integers(0, 1024 * 1024, 128).astype(np.int32)
        _sampled_parity(orc, sc, descs[mi], acc[mi], pix, f"cfg2 mask {mi}", 2)


def test_cfg4_full_size_four_chunks(gfm, orc):
    """Config 4 at 2048^2 (4 chunks of 2^20 paths) as the bench renders it: multiple scattering depth 8,
    stochastic per-recursion masks, Zero NEE; 64 sampled pixels vs the oracle."""
    sc = I.scene_cfg4()
    f = field(gfm, sc)
    desc = I.render_desc_cfg4()
    acc, rays = _bench_frames(f, [desc])
    assert int(rays[0]) == 2048 * 2048 and int(rays[1]) > 0
    pix = np.random.default_rng(44).integers(0, 2048 * 2048, 64).astype(np.int32)
    pix[:8] = [gfm.shard_path_pixel((1 << 20) - 4 + k, 2048, 2048, 0, 0, 1) for k in range(8)]  # chunk boundary
    _sampled_parity(orc, sc, desc, acc[0], pix, "cfg4 2048^2", 3)


def test_cfg5_full_size_sixteen_chunks(gfm, orc):
    """Config 5 at 4096^2 (16 chunks) as the bench renders it: the banded LOD mask (near all levels,
    mid 0..2, far 0..1) and the full mask, multiple scattering depth 8; 48 sampled pixels each."""
    sc = I.scene_cfg5()
    f = field(gfm, sc)
    descs = [I.render_desc_cfg5("banded"), I.render_desc_cfg5((0, 1, 2, 3))]
    acc, rays = _bench_frames(f, descs)
    assert int(rays[0]) == 2 * 4096 * 4096
    rng = np.random.default_rng(55)
    for i, d in enumerate(descs):
        pix = rng.integers(0, 4096 * 4096, 48).astype(np.int32)
        _sampled_parity(orc, sc, d, acc[i], pix, f"cfg5 frame {i}", 3)


# ------------------------------------------------------------------------------ configs 3-5
def test_cfg3_clouds_sampled(gfm, orc):
    """Config 3 (procedural clouds, 327,600 primitives): camera-ray tau parity at sampled pixels and
    multiple-scattering (depth 8, g = 0.6) probe paths with identical Philox streams."""
    sc = I.scene_cfg3()
    f = field(gfm, sc)
    S = orc.Scene(sc)
    desc = I.render_desc_cfg3()
    rays = camera_rays(desc, 400, seed=31)
    tau, T, _ = f.trace_transmittance(rays)
    r = S.trace(rays)
    assert_tau_parity(tau.cpu().numpy(), r["tau"], r["A"], T.cpu().numpy(), "cfg3 camera")
    # probes on cloud pixels (tau > 0) so the paths scatter
    W = desc["width"]
    idx = np.random.default_rng(31).integers(0, W * W, 400)
    probes = idx[r["tau"] > 0.2][:24].astype(np.int32)
    _probe_compare(gfm, orc, sc, desc, probes, 4, "cfg3 multi scatter", frac_tol=0.08)


def test_cfg4_dense_sampled(gfm, orc):
    """Config 4 (1M primitives, dense cube): tau parity at sampled camera rays (full mask and a
    static LOD mask) and stochastic per-recursion masks (PL+CV Accum. beta 0.2 x Importance, Zero
    NEE) in multiple scattering at probe pixels."""
    sc = I.scene_cfg4()
    f = field(gfm, sc)
    S = orc.Scene(sc)
    desc = I.render_desc_cfg4()
    rays = camera_rays(desc, 64, seed=41)
    for m in (0xFFFFFFFF, I.level_mask([0, 1])):
        f.set_lod_mask({"static_mask": m})
        tau, T, _ = f.trace_transmittance(rays)
        r = S.trace(rays, mask=m)
        assert_tau_parity(tau.cpu().numpy(), r["tau"], r["A"], T.cpu().numpy(), f"cfg4 mask {m:#x}")
    probes = np.random.default_rng(41).integers(0, desc["width"] * desc["height"], 12).astype(np.int32)
    d = dict(desc, max_depth=4)
    _probe_compare(gfm, orc, sc, d, probes, 4, "cfg4 stochastic multi scatter", frac_tol=0.1, f=f)


def test_cfg5_army_primary_tau(gfm, orc):
    """Config 5 (3,993,600 primitives, 30 banded groups): primary-ray tau parity under the full, a
    coarse global and the banded LOD mask (24-bit primitive indices exercised at 4M)."""
    sc = I.scene_cfg5()
    assert sc["n"] == 3993600
    f = field(gfm, sc)
    S = orc.Scene(sc)
    desc = I.render_desc_cfg5()
    rays = camera_rays(desc, 32, seed=51)
    for m in (0xFFFFFFFF, I.level_mask([0, 1], n_bands=3), I.render_desc_cfg5("banded")["ext"]["static_mask"]):
        f.set_lod_mask({"static_mask": m})
        tau, T, _ = f.trace_transmittance(rays)
        r = S.trace(rays, mask=m)
        assert_tau_parity(tau.cpu().numpy(), r["tau"], r["A"], T.cpu().numpy(), f"cfg5 mask {m:#x}")


def _non_grazing_rays(S, sc, rays, band=0.01):
    """rays none of whose chords is near-grazing (|r2/E^2 - 1| > band): tau is not differentiable
    where a chord appears (gf_trace_grad_params contract)."""
    keep = []
    for r in range(len(rays)):
        rel = np.array([S.r2_rel(i, rays[r]) for i in range(sc["n"])])
        if not np.any(np.abs(rel - 1.0) <= band):
            keep.append(r)
    return rays[keep]


@pytest.mark.parametrize("packets", [False, True])
@pytest.mark.parametrize("stoch", [False, True])
def test_grad_params_parity(gfm, orc, stoch, packets):
    """Full parameter gradient: d(sum_r dl_r tau_r)/d(mu, q, s, omega, alpha) per
    primitive, closed-form moments + moving chord ends + chain rule on the GPU, against the oracle's
    Richardson central differences of the fp64 closed form.  Tolerance: 1e-3 of the sum of |per-ray
    terms| (fp32 moments: J2 and the W-gradient cancel across the chord) + 1e-6 of the column's
    largest."""
    sc = I.scene_cfg1(seed=23, n=300)
    f = field(gfm, sc)
    S = orc.Scene(sc)
    pol = I.policy(level_strategy=5, beta=0.2, orient_strategy=3) if stoch else I.policy(static_mask=I.level_mask([0, 1, 3]))
    f.set_lod_mask(pol)
    rays = _non_grazing_rays(S, sc, I.rays_through_box(6, 300))
    assert len(rays) > 60
    dl = np.random.default_rng(8).normal(size=len(rays)).astype(np.float32)
    g = f.trace_grad_params(rays, dl, seed=5, packets=packets).cpu().numpy().astype(np.float64)
    if stoch:
        go = np.zeros((sc["n"], 12)); ga = np.zeros((sc["n"], 12))
        f0 = S.info()[1]
        for r in range(len(rays)):
            ul = orc.uniform(5, r, 0, 0, 0, 1)
            uo = [orc.uniform(5, r, 0, 0, 0, 2 + l) for l in range(sc["P"] - 1)]
            m, w = S.policy_eval(dict(I.policy(), **pol), rays[r, 4:7], ul, uo, f0)
            a, b = S.grad_params(rays[r:r + 1], dl[r:r + 1].astype(np.float64), m, w)
            go += a; ga += b
    else:
        go, ga = S.grad_params(rays, dl.astype(np.float64), pol["static_mask"])
    tol = 1e-3 * ga + 1e-6 * ga.max(axis=0, keepdims=True)
    err = np.abs(g - go)
    print("max err/gabs per param", np.max(err / (ga + 1e-30), axis=0), "worst/tol", np.max(err / tol))
    assert np.all(err <= tol), (np.unravel_index(np.argmax(err / tol), err.shape), np.max(err / tol))
    assert np.count_nonzero(go[:, 0]) > 50
