"""GPU tests of the scene-derived quantities, distance bands, sharding, accumulation channels and the
special integration branches, each against the oracle (or an exact identity of the library itself).
"""
import math

import numpy as np
import pytest

from paper_2602_05081_b200 import inputs as I
from tests import refmath as RM

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


def tau_ok(tau_g, r, what):
    tau_g = np.asarray(tau_g, np.float64)
    err = np.abs(tau_g - r["tau"])
    tol = 1e-4 * np.abs(r["tau"]) + 1e-6 * r["A"] + 1e-7
    assert np.all(err <= tol), (what, int(np.sum(err > tol)), float(np.max(err - tol)))


def _subsample(sc, step):
    out = {k: (v[::step] if isinstance(v, np.ndarray) and v.ndim and len(v) == sc["n"] else v) for k, v in sc.items()}
    out["n"] = len(out["mu"])
    return out


# ------------------------------------------------------------------------------ scene-derived parameters
def test_scene_info_matches_oracle(gfm, orc):
    """F3 level maxima (k_load_prims atomics) and C12 group f0 medians (device radix sort) against the
    oracle's independent C, for configs 1, 2 and a banded config-5 subset; an explicit group_f0 input
    is used as given."""
    for sc in (I.scene_cfg1(), I.scene_cfg2(), _subsample(I.scene_cfg5(), 53)):
        f = field(gfm, sc)
        info = f.scene_info()
        lf_o, f0_o = orc.Scene(sc).info()
        np.testing.assert_allclose(info["level_fmax"], lf_o, rtol=1e-6)
        np.testing.assert_array_equal(info["group_f0"], f0_o)
        assert info["n_groups"] == len(f0_o) == 10 * int(sc.get("n_bands", 1))
    sc = I.scene_cfg1()
    given = np.linspace(0.1, 1.0, 10).astype(np.float32)
    f = field(gfm, sc, group_f0=given)
    np.testing.assert_array_equal(f.scene_info()["group_f0"], given)


def test_bvh_hash_replica_check(gfm):
    """independent builds of the same scene (two contexts, as two ranks would) hash
    equal; another scene hashes differently."""
    sc = I.scene_cfg2()
    h1 = field(gfm, sc).scene_info()["bvh_hash"]
    h2 = field(gfm, sc).scene_info()["bvh_hash"]
    sc2 = dict(sc, alpha=sc["alpha"] * np.float32(1.0001))
    h3 = field(gfm, sc2).scene_info()["bvh_hash"]
    assert h1 == h2 != 0 and h3 != h1


def test_motion_blur_mask_library_vs_oracle(gfm, orc):
    """gf_motion_blur_mask (M1-M3) against the oracle for several directions and lengths on configs 1
    and 2: attenuations within fp32 noise, identical masks away from the threshold."""
    for sc in (I.scene_cfg1(), I.scene_cfg2()):
        f = field(gfm, sc)
        S = orc.Scene(sc)
        for d, m in (((1, 0, 0), 0.2), ((0.3, 1, 0.2), 0.05), ((0, 0, 1), 1.0)):
            mask, att = f.motion_blur_mask(d, m, 0.6)
            mask_o, att_o = S.motion_blur_mask(d, m, 0.6)
            np.testing.assert_allclose(att, att_o, rtol=2e-5, atol=1e-6)
            near = np.abs(att_o - 0.6) < 1e-4
            sel = ~near
            assert np.array_equal([(mask >> g) & 1 for g in np.flatnonzero(sel)],
                                  [(mask_o >> g) & 1 for g in np.flatnonzero(sel)])


def test_level_cutoffs_partition(gfm, orc):
    """C10: with no level input the loader assigns Gabor levels from f0 = omega |S^-1 (1,1,1)| against the
    cutoffs (last level open); the group ids equal the oracle's for levels derived here in numpy."""
    sc = I.scene_cfg1()
    s = sc["scale"].astype(np.float64)
    f0 = sc["omega"].astype(np.float64) * np.sqrt((1.0 / s ** 2).sum(1))
    cut = np.quantile(f0[sc["omega"] > 0], [1 / 3, 2 / 3]).astype(np.float32)
    lev = np.where(sc["omega"] == 0, 0, 1 + (f0 >= cut[0]) + (f0 >= cut[1])).astype(np.uint8)
    nolev = dict(sc)
    nolev.pop("level")
    f = field(gfm, nolev, level_cutoffs=cut)
    off = (64 * sc["n"] + 255) // 256 * 256
    g_gpu = f.prim_ws[off: off + sc["n"]].cpu().numpy().astype(np.int64)
    g_or, _ = orc.Scene(dict(sc, level=lev)).groups()
    near = np.abs(f0[:, None] - cut[None, :].astype(np.float64)).min(1) <= 1e-6 * f0
    assert np.array_equal(g_gpu[~near], g_or[~near])
    assert len(set((g_gpu[g_gpu > 0] - 1) // 3)) == 3


# ------------------------------------------------------------------------------ distance bands (cfg5)
def test_banded_masks_parity(gfm, orc):
    """Config 5's distance bands (fig:army_bunny): primary-ray tau under the banded LOD mask
    (near all levels, mid 0..2, far 0..1) and a one-band mask, vs the oracle on a subset of the army."""
    sc = _subsample(I.scene_cfg5(), 11)
    f = field(gfm, sc)
    S = orc.Scene(sc)
    desc = I.render_desc_cfg5("banded", 256, 256)
    idx = np.random.default_rng(3).integers(0, 256 * 256, 200)
    o, d = I.camera_rays_f64(desc, idx % 256, idx // 256)
    rays = I.pack_rays(o, d)
    for m in (desc["ext"]["static_mask"], I.level_mask((0, 1, 2, 3), n_bands=3, bands=[2]), 0xFFFFFFFF):
        f.set_lod_mask({"static_mask": m})
        tau, _, _ = f.trace_transmittance(rays)
        tau_ok(tau.cpu().numpy(), S.trace(rays, mask=m), f"band mask {m:#x}")
    pol = I.policy(level_strategy=5, beta=0.2, orient_strategy=3)
    probes = idx[:16].astype(np.int32)
    d5 = dict(desc, max_depth=3, ext=pol)
    vg, _ = f.render(d5, 0, 4, probes=probes)
    vo, _ = S.render_probes(d5, probes, 0, 4)
    vg = vg.view(16, 4).cpu().numpy().astype(np.float64)
    assert np.mean(np.abs(vg - vo) > 1e-3 * (np.abs(vo) + 1e-2)) <= 2 / 64


# ------------------------------------------------------------------------------ special integration branches
def test_gauss_legendre_and_midpoint_branches(gfm, orc):
    """C5/C9: high-frequency Gabors (omega in [2, 3], |z|^2 > 8 on parallel rays) take the Gauss-Legendre
    fallback; sub-1e-4 whitened pieces (rays clipped to 1e-6 inside primitives) the midpoint rule.
    Both against the oracle's exact closed form, with the branch counters > 0."""
    rng = np.random.default_rng(17)
    n = 400
    sc = I._finish(rng.uniform(-1, 1, (n, 3)), I.random_quats(rng, n), np.exp(rng.normal(-2.0, 0.2, (n, 3))),
                   np.full(n, 0.5), rng.uniform(2.0, 3.0, n), np.ones(n, np.uint8), name="hf")
    f = field(gfm, sc)
    S = orc.Scene(sc)
    rays = I.rays_through_box(4, 1500)
    f.set_profiling(work=True)
    tau, _, _ = f.trace_transmittance(rays)
    st = f.stats(reset=True)
    f.set_profiling()
    tau_ok(tau.cpu().numpy(), S.trace(rays), "gauss-legendre")
    assert st["work"]["trace"]["gl_fallbacks"] > 0
    # midpoint: rays starting inside primitives, [tmin, tmin + 1e-6]
    k = rng.integers(0, n, 300)
    d = rng.normal(size=(300, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    short = I.pack_rays(sc["mu"][k] - 0.5 * np.exp(-2.0) * d, d, tmin=0.4 * np.exp(-2.0))
    short[:, 7] = short[:, 3] + 1e-6
    tau, _, _ = f.trace_transmittance(short)
    r = S.trace(short)
    assert np.count_nonzero(r["tau"]) > 100
    tau_ok(tau.cpu().numpy(), r, "midpoint")


# ------------------------------------------------------------------------------ accumulation channels
def test_accumulator_sum_and_square_channels(gfm, orc):
    """a10: the full-image accumulators hold the sum and the sum of squares of the per-sample estimates
    (the same (pixel, sample) paths the probe mode returns one by one), and match the oracle's."""
    sc = I.scene_cfg1p()
    f = field(gfm, sc)
    desc = I.render_desc_cfg2(3, 40, 24)
    desc.update(**I.camera((0, 0, 4), (0, 0, 0), (0, 1, 0), 40.0, 40, 24))
    desc.update(max_depth=3, albedo=0.9, ext=I.policy(), nee=I.policy())
    acc, _ = f.render(desc, 2, 4)
    acc = acc.view(-1, 2).cpu().numpy()
    pix = np.arange(40 * 24, dtype=np.int32)
    vg, _ = f.render(desc, 2, 4, probes=pix)
    vg = vg.view(-1, 4).cpu().numpy()
    s1 = np.zeros(len(pix), np.float32)
    s2 = np.zeros(len(pix), np.float32)
    for k in range(4):  # k_finish: acc += v; acc2 = fma(v, v, acc2) (one rounding)
        s1 += vg[:, k]
        s2 = (s2.astype(np.float64) + vg[:, k].astype(np.float64) ** 2).astype(np.float32)
    np.testing.assert_array_equal(acc[:, 0], s1)
    np.testing.assert_array_equal(acc[:, 1], s2)
    vo, _ = orc.Scene(sc).render_probes(desc, pix[::7], 2, 4)
    so = (vo ** 2).sum(1)
    close = np.abs(acc[::7, 1] - so) <= 1e-3 * (so + 1e-2)
    assert close.mean() >= 0.97


# ------------------------------------------------------------------------------ multi-GPU sharding (§8(e))
@pytest.mark.parametrize("world", [2, 3, 8])
def test_tile_and_sample_sharding_every_rank(gfm, world):
    """Every rank r of world N renders its shard on this one GPU (no rank waits on another): tile
    sharding (32x32 tiles, tile t -> rank t mod N) -- the ranks' images add up to the unsharded one bit
    for bit; sample sharding (s -> rank s mod N) -- the sum matches within fp32 reassociation."""
    sc = I.scene_bunny(counts=(300, 2100, 5600, 12000))
    f = field(gfm, sc)
    desc = dict(I.render_desc_cfg2(3, 100, 70), max_depth=3, albedo=0.9)
    ref, _ = f.render(desc, 0, 2)
    tiles = torch.zeros_like(ref)
    for r in range(world):
        a, _ = f.render(desc, 0, 2, shard=(gfm.SHARD_TILES, r, world))
        own = torch.from_numpy(np.array([[gfm.shard_pixel_owner(x, y, 100, 70, world) == r for x in range(100)]
                                         for y in range(70)]).reshape(-1)).to(a.device)
        assert torch.all(a.view(-1, 2)[~own] == 0)
        tiles += a
    assert torch.equal(tiles, ref)
    ref8, _ = f.render(desc, 0, 2 * world)
    samples = torch.zeros_like(ref8)
    for r in range(world):
        a, _ = f.render(desc, 0, 2 * world, shard=(gfm.SHARD_SAMPLES, r, world))
        samples += a
    torch.testing.assert_close(samples, ref8, rtol=1e-5, atol=1e-6)


# ------------------------------------------------------------------------------ view-BVH reuse
def test_reuse_accel_alternating_layouts(gfm):
    """reuse_accel with one scratch shared by renders of different chunk layouts (probes, full image,
    probes again): the later call must not reuse view BVHs the full-image call overwrote."""
    sc = I.scene_cfg2()
    f = field(gfm, sc)
    small = I.render_desc_cfg2(3, 64, 64)
    big = I.render_desc_cfg2(3, 256, 256)
    probes = np.arange(0, 64 * 64, 5, dtype=np.int32)
    scratch = f.render_scratch(big, 1)
    ref_p, _ = f.render(small, 0, 1, probes=probes)
    ref_b, _ = f.render(big, 0, 1)
    for _ in range(2):
        p1, _ = f.render(dict(small, reuse_accel=1), 0, 1, probes=probes, scratch=scratch)
        b1, _ = f.render(dict(big, reuse_accel=1), 0, 1, scratch=scratch)
        p2, _ = f.render(dict(small, reuse_accel=1), 0, 1, probes=probes, scratch=scratch)
        assert torch.equal(p1, ref_p) and torch.equal(p2, ref_p) and torch.equal(b1, ref_b)


def test_misaligned_rays_rejected(gfm):
    """The ABI requires 16-byte aligned ray arrays (float4 loads): an offset view is rejected with
    GF_E_INVALID_ARGUMENT instead of faulting the context."""
    f = field(gfm, I.scene_cfg1(n=64))
    buf = torch.zeros(8 * 4 + 1, dtype=torch.float32, device="cuda")
    with pytest.raises(gfm.GFError) as e:
        f.trace_transmittance(buf[1:].view(4, 8))
    assert e.value.status == 1
    tau, _, _ = f.trace_transmittance(torch.from_numpy(I.rays_through_box(1, 4)).cuda())
    assert torch.isfinite(tau).all()
