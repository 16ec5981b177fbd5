"""Pins of the CPU oracle against what the paper and mathematics fix (no GPU).

Each test names the passage (P:Lnnn of PAPER.md) or the DESIGN.md reading it
checks.  References come from *outside* the oracle: closed forms written out
here, scipy.special.erf, adaptive quadrature of Eq. 6 (tests/refmath.py),
published test vectors, and statistical identities.
"""
import math

import numpy as np
import pytest
from scipy import special

from paper_2602_05081_b200 import inputs as I
from tests import refmath as RM

TWO_PI = 2.0 * math.pi


def make_scene(prims, P=4, K=3, level=None):
    """scene dict from a list of (mu, q, s, omega, alpha, E)."""
    n = len(prims)
    mu = np.array([p[0] for p in prims], np.float32).reshape(n, 3)
    q = np.array([p[1] for p in prims], np.float32).reshape(n, 4)
    s = np.array([p[2] for p in prims], np.float32).reshape(n, 3)
    om = np.array([p[3] for p in prims], np.float32)
    al = np.array([p[4] for p in prims], np.float32)
    E = np.array([p[5] for p in prims], np.float32)
    lev = np.array(level if level is not None else [0 if o == 0 else 1 for o in om], np.uint8)
    return {"n": n, "P": P, "K": K, "mu": mu, "quat": q, "scale": s, "alpha": al, "omega": om, "extent": E,
            "level": lev, "bin": np.full(n, 255, np.uint8), "bin_axes": I.bin_axes(K)}


ID = (0.0, 0.0, 0.0, 1.0)


# ---------------------------------------------------------------- complex erf (Eq. 13)
@pytest.mark.parametrize("z", [0.5, 1.0, 0.5 + 0.5j, 2.1 - 1.8j, -1.3 + 2.6j / math.sqrt(2), 3 / math.sqrt(2) - 1.3j])
def test_erf_series_matches_library(orc, z):
    """Eq. 13 Maclaurin series vs scipy's Faddeeva-based erf; S:L85/S:L91 examples."""
    got = orc.erf(complex(z))
    ref = complex(special.erf(complex(z)))
    assert abs(got - ref) <= 1e-13 * max(1.0, abs(ref))


def test_erf_printed_values(orc):
    assert abs(orc.erf(0.5).real - 0.520500) < 5e-7     # S:L91 example
    assert abs(orc.erf(1.0).real - 0.842701) < 5e-7     # S:L85 example
    assert orc.erf(0.0) == 0.0


# ---------------------------------------------------------------- golden line integrals
def test_golden_G1_G2_gaussian_through_centre(orc):
    """G1: iso sigma=1, omega=0, through centre: untruncated 1/(2 pi); G2: truncated at E=3
    keeps erf(3/sqrt2) of it (C7)."""
    S = orc.Scene(make_scene([((0, 0, 0), ID, (1, 1, 1), 0.0, 1.0, 3.0)]))
    o, v = (-10, 0, 0), (1, 0, 0)
    assert abs(S.prim_integral_infinite(0, o, v) - 1 / TWO_PI) < 1e-15
    assert abs(S.prim_integral(0, o, v, -np.inf, np.inf) - math.erf(3 / math.sqrt(2)) / TWO_PI) < 1e-14


def test_golden_G3_parallel_attenuation(orc):
    """G3: omega=1, ray parallel to k_W=(1,1,1) through the centre: Omega=sqrt3, untruncated
    K e^{-Omega^2/2} = e^{-1.5}/(2 pi) (P:L306 'reduces the contribution by K exp(-f0^2/2)')."""
    S = orc.Scene(make_scene([((0, 0, 0), ID, (1, 1, 1), 1.0, 1.0, 3.0)]))
    v = np.array([1, 1, 1]) / math.sqrt(3)
    o = -5 * v
    assert abs(S.prim_integral_infinite(0, o, v) - math.exp(-1.5) / TWO_PI) < 2e-8  # fp32 ray input
    # truncated: symmetric chord u in [-3,3]: J = e^{-Omega^2/2} cos(phi) Re erf((3 - i Omega)/sqrt2), phi=0
    trunc = math.exp(-1.5) * special.erf(complex(3, -math.sqrt(3)) / math.sqrt(2)).real / TWO_PI
    got = S.prim_integral(0, o.astype(np.float32), v.astype(np.float32), -np.inf, np.inf)
    assert abs(got - trunc) < 2e-8  # fp32 ray input
    assert abs(trunc - 0.0351960712051) < 1e-11


def test_golden_G4_perpendicular_equals_gaussian(orc):
    """G4: ray perpendicular to k_W through the centre: Omega=0, phase 0 -> equals the Gaussian G2."""
    S = orc.Scene(make_scene([((0, 0, 0), ID, (1, 1, 1), 1.0, 1.0, 3.0)]))
    v = np.array([1, -1, 0]) / math.sqrt(2)
    got = S.prim_integral(0, (-5 * v).astype(np.float32), v.astype(np.float32), -np.inf, np.inf)
    assert abs(got - math.erf(3 / math.sqrt(2)) / TWO_PI) < 2e-8


@pytest.mark.parametrize("case", ["G5", "G6"])
def test_golden_quadrature(orc, case):
    """G5/G6: off-centre Gabor and anisotropic primitive vs quadrature of Eq. 6."""
    if case == "G5":
        prim = ((0, 0, 0), ID, (1, 1, 1), 1.0, 1.0, 3.0)
        o, v, golden_full, golden_trunc = (-5, 0, 1), (1, 0, 0), 0.0316346089808, 0.0318696002871
    else:
        prim = ((0, 0, 0), ID, (2, 1, 0.5), 0.8, 1.0, 3.0)
        o, v, golden_full, golden_trunc = (-10, 0.3, 0.2), (1, 0, 0), None, 0.173438166432
    S = orc.Scene(make_scene([prim]))
    p = RM.Prim(*prim)
    o32 = np.asarray(o, np.float32).astype(np.float64)
    q = p.line_integral(o32, v)
    got = S.prim_integral(0, o, v, -np.inf, np.inf)
    assert abs(got - q) <= 1e-10 * abs(q)
    # golden values are for the exact decimal inputs; fp32 input rounding moves them by ~1e-8
    assert abs(got - golden_trunc) < 5e-8 * golden_trunc
    if golden_full is not None:
        assert abs(S.prim_integral_infinite(0, o, v) - golden_full) < 5e-8 * golden_full
        assert abs(p.line_integral(o32, v, truncated=False) - S.prim_integral_infinite(0, o, v)) < 1e-10


def test_closed_form_vs_quadrature_random(orc):
    """North-star pin: App. A closed form vs adaptive quadrature of the plain
    definition (Eq. 6) on random anisotropic primitives and random segments, 1e-9 relative."""
    rng = np.random.default_rng(7)
    prims = []
    for _ in range(30):
        prims.append((tuple(rng.uniform(-1, 1, 3)), tuple(I.random_quats(rng, 1)[0]),
                      tuple(np.exp(rng.uniform(np.log(0.05), np.log(0.5), 3))), float(rng.uniform(0, 1.5)),
                      1.0, 3.0))
    S = orc.Scene(make_scene(prims))
    checked = 0
    for i, pr in enumerate(prims):
        p = RM.Prim(*pr)
        for _ in range(4):
            tgt = p.mu + rng.normal(size=3) * np.array(pr[2]) * 1.5
            v = rng.normal(size=3)
            v /= np.linalg.norm(v)
            o = (tgt - 3 * v).astype(np.float32)
            v = v.astype(np.float32)
            t0, t1 = sorted(rng.uniform(0, 6, 2))
            q = p.line_integral(o.astype(np.float64), v.astype(np.float64), t0, t1)
            got = S.prim_integral(i, o, v, t0, t1)
            scale = p.line_integral(o.astype(np.float64), v.astype(np.float64)) if q != 0 else 1.0
            assert abs(got - q) <= 1e-9 * max(abs(q), 1e-3 * abs(scale)) + 1e-14, (i, got, q)
            checked += q != 0
    assert checked > 40


def test_misprinted_eq9_is_not_used(orc):
    """Reading C3: Eq. 9 as printed (no 1/2, cos-only) disagrees with quadrature; the oracle follows
    App. A.  Guard: for an asymmetric segment the printed form is off by a large factor."""
    prim = ((0, 0, 0), ID, (1, 1, 1), 1.0, 1.0, 3.0)
    S = orc.Scene(make_scene([prim]))
    p = RM.Prim(*prim)
    o, v = np.array([-5.0, 0.3, 0.2], np.float32).astype(np.float64), np.array([1.0, 0.0, 0.0])
    q = p.line_integral(o, v, 4.2, 5.9)
    got = S.prim_integral(0, o.astype(np.float32), v.astype(np.float32), 4.2, 5.9)
    assert abs(got - q) < 1e-12
    # printed Eq. 9: K e^{-(c-b^2+Om^2)/2} cos(d - Om b) [erf(z1) - erf(z0)] (real part)
    pW, vW, kW = o - 0, v.copy(), np.ones(3)
    b, c, Om, d = pW @ vW, pW @ pW, kW @ vW, kW @ pW
    Kc = 1 / (TWO_PI)
    z1, z0 = (5.9 + b - 1j * Om) / math.sqrt(2), (4.2 + b - 1j * Om) / math.sqrt(2)
    printed = (Kc * math.exp(-0.5 * (c - b * b + Om * Om)) * math.cos(d - Om * b) *
               (special.erf(z1) - special.erf(z0))).real
    assert abs(printed - q) > 0.2 * abs(q)


def test_zero_frequency_reduces_to_gaussian(orc):
    """omega=0 Gabor = Gaussian; J reduces to a real erf difference (scipy)."""
    rng = np.random.default_rng(3)
    for _ in range(20):
        pr = (tuple(rng.uniform(-1, 1, 3)), tuple(I.random_quats(rng, 1)[0]),
              tuple(np.exp(rng.uniform(-3, -0.5, 3))), 0.0, 1.0, 3.0)
        S = orc.Scene(make_scene([pr]))
        p = RM.Prim(*pr)
        v = rng.normal(size=3)
        v /= np.linalg.norm(v)
        o = p.mu - 2 * v + rng.normal(size=3) * 0.3 * np.array(pr[2])
        o32, v32 = o.astype(np.float32), v.astype(np.float32)
        o, v = o32.astype(np.float64), v32.astype(np.float64)
        a = v @ p.Sinv @ v
        beta = v @ p.Sinv @ (o - p.mu)
        gam = (o - p.mu) @ p.Sinv @ (o - p.mu)
        ch = p.chord(o, v, 0, 10)
        if ch is None:
            continue
        t0, t1 = ch
        gauss = (p.norm * math.sqrt(math.pi / (2 * a)) * math.exp(-0.5 * (gam - beta * beta / a)) *
                 (math.erf(math.sqrt(a / 2) * (t1 + beta / a)) - math.erf(math.sqrt(a / 2) * (t0 + beta / a))))
        got = S.prim_integral(0, o32, v32, 0, 10)
        assert abs(got - gauss) <= 1e-12 * abs(gauss) + 1e-15


def test_segment_limit_and_additivity(orc):
    """S:L74 (+-20 sigma proxy = full integral) and S:L120 additivity over split segments."""
    # E = 6 whitened units: the erf(6/sqrt2) tail is 2e-9 (series domain |z|^2 <= 24, oracle header)
    pr = ((0.1, -0.2, 0.3), (0.1, 0.2, 0.3, 0.927), (0.2, 0.1, 0.3), 0.3, 1.0, 6.0)
    S = orc.Scene(make_scene([pr]))
    o, v = np.array([-3, 0, 0], np.float32), np.array([1, 0, 0], np.float32)
    full = S.prim_integral_infinite(0, o, v)
    assert abs(S.prim_integral(0, o, v, -np.inf, np.inf) - full) < 2e-8 * abs(full)
    S3 = orc.Scene(make_scene([pr[:5] + (3.0,)]))
    a = S3.prim_integral(0, o, v, 0, 3.05)
    b = S3.prim_integral(0, o, v, 3.05, 9)
    ab = S3.prim_integral(0, o, v, 0, 9)
    assert abs(a + b - ab) < 1e-13
    assert S3.prim_integral(0, o, v, 3.0, 3.0) == 0.0   # empty interval


def test_eval_kernel_examples(orc):
    """S:L47 peak (2 pi)^{-3/2}; cosine zero crossing; dense Eq. 6 match."""
    S = orc.Scene(make_scene([((0, 0, 0), ID, (1, 1, 1), 0.0, 1.0, 3.0), ((0, 0, 0), ID, (1, 1, 1), 1.0, 1.0, 3.0),
                              ((0.2, 0.1, -0.3), (0.3, -0.1, 0.2, 0.927), (0.3, 0.2, 0.5), 0.9, 1.0, 3.0)]))
    assert abs(S.eval_kernel(0, [0, 0, 0]) - (TWO_PI) ** -1.5) < 1e-16
    x = np.array([1, 1, 1]) * (math.pi / 2) / 3.0  # omega_vec . x = pi/2
    assert abs(S.eval_kernel(1, x)) < 1e-16
    p = RM.Prim((0.2, 0.1, -0.3), (0.3, -0.1, 0.2, 0.927), (0.3, 0.2, 0.5), 0.9)
    for x in np.random.default_rng(1).normal(size=(10, 3)) * 0.4:
        assert abs(S.eval_kernel(2, x) - p.K(x)) < 1e-13


def test_rotation_equivariance(orc):
    """rotating scene and ray by the same rotation leaves tau unchanged."""
    sc = I.scene_cfg1(n=60)
    rays = I.rays_through_box(5, 20)
    S = orc.Scene(sc)
    t0 = S.trace(rays)["tau"]
    Rq = np.array([0.2, -0.3, 0.1, 0.927])
    Rq /= np.linalg.norm(Rq)
    R = RM.quat_R(Rq)
    sc2 = dict(sc)
    sc2["mu"] = (sc["mu"].astype(np.float64) @ R.T).astype(np.float32)
    # compose quaternions: q' = Rq * q
    x1, y1, z1, w1 = Rq
    q = sc["quat"].astype(np.float64)
    x2, y2, z2, w2 = q[:, 0], q[:, 1], q[:, 2], q[:, 3]
    sc2["quat"] = np.stack([w1 * x2 + x1 * w2 + y1 * z2 - z1 * y2, w1 * y2 - x1 * z2 + y1 * w2 + z1 * x2,
                            w1 * z2 + x1 * y2 - y1 * x2 + z1 * w2, w1 * w2 - x1 * x2 - y1 * y2 - z1 * z2],
                           1).astype(np.float32)
    sc2["bin"] = np.zeros(sc["n"], np.uint8)  # groups irrelevant for the full mask
    rays2 = rays.copy()
    rays2[:, 0:3] = rays[:, 0:3].astype(np.float64) @ R.T
    rays2[:, 4:7] = rays[:, 4:7].astype(np.float64) @ R.T
    t1 = orc.Scene(sc2).trace(rays2)["tau"]
    # fp32 rounding of the rotated inputs is the only difference
    assert np.allclose(t0, t1, rtol=2e-5, atol=2e-6)


# ---------------------------------------------------------------- brute-force tau vs quadrature
def test_trace_matches_quadrature_small_scene(orc):
    """Eq. 1-3: tau of a ray through a 12-primitive scene = sum of quadratures of the plain
    truncated definition (kernels bounded by an ellipsoid)."""
    sc = I.scene_cfg1(n=12, seed=11)
    sc["mu"] *= 0.3
    S = orc.Scene(sc)
    prims = [RM.Prim.from_scene(sc, i) for i in range(sc["n"])]
    rays = I.rays_through_box(12, 6, -0.3, 0.3)
    r = S.trace(rays)
    for k in range(len(rays)):
        o, v = rays[k, 0:3].astype(np.float64), rays[k, 4:7].astype(np.float64)
        q = RM.tau_quad(prims, o, v, 0.0, np.inf)
        assert abs(r["tau"][k] - q) <= 1e-9 * max(abs(q), r["A"][k]) + 1e-13


def test_far_origin_oracle_accuracy(orc):
    """Reading C25 / SURVEY §0 finding 7: the oracle stays exact for |o-mu|/s up to 3000."""
    fo = I.far_origin_pairs(9, 12, 3000.0)
    for i in range(12):
        pr = (fo["mu"][i], fo["quat"][i], fo["scale"][i], float(fo["omega"][i]), 1.0, 3.0)
        S = orc.Scene(make_scene([pr]))
        p = RM.Prim(*pr)
        ray = fo["rays"][i]
        o, v = ray[0:3].astype(np.float64), ray[4:7].astype(np.float64)
        q = p.line_integral(o, v, 0, np.inf)
        env = p.line_integral(o, v, 0, np.inf) if q else 0
        got = S.prim_integral(0, ray[0:3], ray[4:7], 0, np.inf)
        ch = p.chord(o, v, 0, np.inf)
        if ch is None:
            continue
        mag = p.norm * (ch[1] - ch[0])  # envelope magnitude bound of the chord
        assert abs(got - q) <= 1e-8 * mag, (i, got, q, env)


# ---------------------------------------------------------------- masks
def test_level_mask_algebra():
    """V_l = 2^l generalised to (level, bin) groups: g(0)=0, g(l,b)=1+(l-1)K+b (C24)."""
    assert I.level_mask([0]) == 1
    assert I.level_mask([0, 1]) == 0b1111
    assert I.level_mask([3]) == 0b1110000000
    assert I.level_mask([0, 1, 2, 3]) == 0x3FF
    assert I.level_mask([]) == 0


def test_masking_removes_only_targeted_groups(orc):
    """North-star pin: full mask = unmasked field; tau(mask) = sum of the per-group tau of the
    groups in the mask (masking removes only the targeted bands)."""
    sc = I.scene_cfg1(n=300, seed=21)
    S = orc.Scene(sc)
    rays = I.rays_through_box(22, 40)
    full = S.trace(rays, mask=0xFFFFFFFF, want_groups=True)
    allg = S.trace(rays, mask=(1 << S.G) - 1)
    assert np.array_equal(full["tau"], allg["tau"])
    assert np.allclose(full["groups"].sum(1), full["tau"], rtol=1e-12, atol=1e-14)
    rng = np.random.default_rng(2)
    for _ in range(6):
        m = int(rng.integers(1, 1 << S.G))
        sub = S.trace(rays, mask=m)["tau"]
        ref = full["groups"][:, [g for g in range(S.G) if (m >> g) & 1]].sum(1)
        assert np.allclose(sub, ref, rtol=1e-12, atol=1e-14)
    # mask correctness: masked render == render of the visible sub-field
    g, _ = S.groups()
    m = I.level_mask([0, 2])
    keep = ((m >> g) & 1).astype(bool)
    sub = {k: (v[keep] if isinstance(v, np.ndarray) and v.shape[:1] == (sc["n"],) else v) for k, v in sc.items()}
    sub["n"] = int(keep.sum())
    sub["bin"] = np.zeros(sub["n"], np.uint8)
    Ssub = orc.Scene(sub)
    assert np.allclose(S.trace(rays, mask=m)["tau"], Ssub.trace(rays)["tau"], rtol=1e-13, atol=1e-15)


def test_transmittance_bounds_and_monotone_on_paired_positive(orc):
    """T in [0,1] and non-increasing in t_max on paired-positive scenes (reading C18)."""
    sc = I.scene_cfg1p(n_pairs=150)
    S = orc.Scene(sc)
    base = I.rays_through_box(31, 30)
    prev = None
    for tmax in (2.0, 3.0, 3.5, 4.0, 5.0, np.inf):
        r = base.copy()
        r[:, 7] = tmax
        for m in (I.level_mask([0]), I.level_mask([0, 1]), I.level_mask([0, 1, 2, 3])):
            tau = S.trace(r, mask=m)["tau"]
            assert (tau >= -1e-15).all()
        tau = S.trace(r)["tau"]
        T = np.exp(-tau)
        assert ((T >= 0) & (T <= 1 + 1e-15)).all()
        if prev is not None:
            assert (T <= prev + 1e-15).all()
        prev = T


# ---------------------------------------------------------------- Philox KAT
def test_philox_kat(orc):
    """Random123 Philox4x32-10 known-answer vectors."""
    assert [f"{x:08x}" for x in orc.philox([0, 0, 0, 0], [0, 0])] == ["6627e8d5", "e169c58d", "bc57ac4c", "9b00dbd8"]
    assert [f"{x:08x}" for x in orc.philox([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2)] == \
        ["408f276d", "41c83b0e", "a20bc7c6", "6d5451fd"]
    assert [f"{x:08x}" for x in orc.philox([0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344],
                                           [0xa4093822, 0x299f31d0])] == ["d16cfe09", "94fdcceb", "5001e420", "24126ea1"]


def test_uniform_mapping(orc):
    """C16: u = (x >> 8) 2^-24 in [0,1), exactly representable."""
    for k in range(8):
        u = orc.uniform(123, 5, 7, 1, 0, k)
        w = orc.philox([5, 7, 1, (0 << 16) | (k >> 2)], [123, 0])[k & 3]
        assert u == (int(w) >> 8) / 16777216.0
        assert 0.0 <= u < 1.0


# ---------------------------------------------------------------- strategies (Tables B1/B2)
LEVEL_STRATS = [(1, 0.0), (2, 0.0), (2, 0.2), (2, 0.5), (3, 0.0), (4, 0.2), (4, 0.9), (5, 0.0), (5, 0.2), (5, 0.5),
                (5, 0.9)]
ORIENT_STRATS = [(2, 1.0), (3, 1.0), (4, 0.5), (4, 0.2)]


def _draws(S, pol, n, seed, dirs=None):
    rng = np.random.default_rng(seed)
    if dirs is None:
        dirs = rng.normal(size=(n, 3))
        dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    ul = (rng.integers(0, 1 << 24, n) / 16777216.0).astype(np.float32)
    uo = (rng.integers(0, 1 << 24, (n, S.P - 1)) / 16777216.0).astype(np.float32)
    f0 = np.array([0] + [1.2 * math.sqrt(3)] * 3 + [0.9 * math.sqrt(3)] * 3 + [1.1 * math.sqrt(3)] * 3, np.float32)
    return S.policy_eval_batch(pol, dirs, ul, uo, f0)


@pytest.mark.parametrize("ls,beta", LEVEL_STRATS)
def test_level_strategies_unbiased(orc, ls, beta):
    """Table B1 rows with readings C13/C14: E[reweighted group indicator] = 1 +- 4 SE."""
    S = orc.Scene(I.scene_cfg1(n=20))
    masks, w = _draws(S, orc.make_policy(level_strategy=ls, beta=beta), 200000, 100 + ls)
    mean, se = w.mean(0), w.std(0) / math.sqrt(len(w))
    assert np.all(np.abs(mean - 1.0) <= 4 * se + 1e-6), (mean, se)
    # weights are positive and finite where selected, zero elsewhere
    sel = ((masks[:, None] >> np.arange(S.G)[None]) & 1).astype(bool)
    assert np.all((w > 0) == sel) and np.all(np.isfinite(w))


@pytest.mark.parametrize("os_,delta", ORIENT_STRATS)
def test_orientation_strategies_unbiased(orc, os_, delta):
    """Table B2 rows jointly with Deterministic levels (C15): unbiased where the
    strategy is, Gaussians always weight 1."""
    S = orc.Scene(I.scene_cfg1(n=20))
    masks, w = _draws(S, orc.make_policy(orient_strategy=os_, delta=delta), 200000, 200 + os_)
    assert np.all(w[:, 0] == 1.0)
    mean, se = w.mean(0), w.std(0) / math.sqrt(len(w))
    assert np.all(np.abs(mean - 1.0) <= 4 * se + 1e-6), (mean, se)


def test_joint_level_orientation_unbiased(orc):
    S = orc.Scene(I.scene_cfg1(n=20))
    masks, w = _draws(S, orc.make_policy(level_strategy=5, beta=0.2, orient_strategy=3), 300000, 77)
    mean, se = w.mean(0), w.std(0) / math.sqrt(len(w))
    assert np.all(np.abs(mean - 1.0) <= 4 * se + 1e-6)


def test_strategy_examples(orc):
    """S:L232 (Uniform P=4 u=0.6 -> level 2 weight 4), Deterministic -> all weight 1,
    ThresholdCull(delta=1) == Deterministic, Importance with one bin -> weight 1,
    w(a=1,f0=2)=e^-2 via the importance weight ratio."""
    S = orc.Scene(I.scene_cfg1(n=20))
    m, w = S.policy_eval({"level_strategy": 1}, [0, 0, 1], 0.6, [0.1, 0.2, 0.3])
    assert m == I.level_mask([2]) and np.all(w[[4, 5, 6]] == 4.0) and w.sum() == 12.0
    m, w = S.policy_eval({}, [0, 0, 1], 0.3, [0.1, 0.2, 0.3])
    assert m == 0x3FF and np.all(w == 1.0)
    m2, w2 = S.policy_eval({"orient_strategy": 1, "delta": 1.0}, [0.3, 0.4, 0.866], 0.3, [0.1, 0.2, 0.3])
    assert m2 == m and np.array_equal(w2, w)
    S1 = orc.Scene(dict(I.scene_cfg1(n=20), K=1, bin_axes=I.bin_axes(1)))
    m, w = S1.policy_eval({"orient_strategy": 3}, [0, 0, 1], 0.3, [0.1, 0.2, 0.3], np.full(S1.G, 2.0, np.float32))
    assert np.all(w[1:] == 1.0)
    # importance with K=3: dir along x, f0=2: w_x = e^{-2}, w_y = w_z = 1 -> P(x) = e^-2/(2+e^-2)
    f0 = np.full(S.G, 2.0, np.float32)
    masks, wts = _draws(S, orc.make_policy(orient_strategy=3), 100000, 5,
                        dirs=np.tile([1.0, 0.0, 0.0], (100000, 1)))
    masks, wts = S.policy_eval_batch(orc.make_policy(orient_strategy=3), np.tile([1.0, 0, 0], (100000, 1)),
                                     np.full(100000, 0.5, np.float32),
                                     np.random.default_rng(1).random((100000, 3)).astype(np.float32), f0)
    px = ((masks >> 1) & 1).mean()
    pe = math.exp(-2) / (2 + math.exp(-2))
    assert abs(px - pe) < 4 * math.sqrt(pe * (1 - pe) / 100000)
    sel = (masks >> 1) & 1 == 1
    assert np.allclose(wts[sel, 1], (2 + math.exp(-2)) / math.exp(-2), rtol=1e-6)


def test_spec_accum_reading_is_biased():
    """Reading C14: SPEC's S:L270 attribution (the sampled level's weight on every level) is biased;
    the per-level weight 1/(1-(j/P)^(1-beta)) is not (pure-probability check, P=4, beta=0.2)."""
    P, beta = 4, 0.2
    th = [(j / P) ** (1 - beta) for j in range(P + 1)]
    p_k = [th[k + 1] - th[k] for k in range(P)]
    ours = [sum(p_k[k] for k in range(j, P)) / (1 - th[j]) for j in range(P)]
    assert np.allclose(ours, 1.0)
    spec = [sum(p_k[k] / (1 - th[k]) for k in range(j, P)) if j > 0 else 1.0 for j in range(P)]
    assert max(abs(s - 1) for s in spec) > 0.4


# ---------------------------------------------------------------- free flight (Eq. 5)
def test_free_flight_G7_symmetric(orc):
    """G7: single truncated Gaussian with tau_total = 2; xi = 1-e^-1 -> t* = centre (symmetry)."""
    alpha = 2.0 / (math.erf(3 / math.sqrt(2)) / TWO_PI)
    assert abs(alpha - 12.6003890952) < 1e-9
    S = orc.Scene(make_scene([((0, 0, 0), ID, (1, 1, 1), 0.0, alpha, 3.0)]))
    ray = I.pack_rays(np.array([[-5.0, 0, 0]]), np.array([[1.0, 0, 0]]))[0]
    t = S.free_flight(ray, 1 - math.exp(-1))
    assert abs(t - 5.0) < 1e-7  # alpha is fp32: tau_total = 2 (1 + O(3e-8))
    half = 0.5 * float(np.float32(alpha)) * math.erf(3 / math.sqrt(2)) / TWO_PI  # exact half of fp32 scene
    assert abs(S.free_flight(ray, -math.expm1(-half)) - 5.0) < 1e-9
    assert S.free_flight(ray, 1 - math.exp(-2.5)) is None   # escape: tau* > tau_total
    assert S.free_flight(ray, 0.0) == 0.0                    # tau* = 0 -> t_min


def test_free_flight_inverts_quadrature_cdf(orc):
    """Eq. 5: the sampled t* satisfies tau(t_min, t*) = -ln(1-xi) with tau from QUADRATURE of the
    plain definition (independent of the oracle's closed form), incl. negative-density lobes."""
    sc = I.scene_cfg1(n=14, seed=5)   # unpaired: Gabor lobes make kappa < 0 in places
    sc["mu"] = sc["mu"] * 0.2
    sc["alpha"] = sc["alpha"] * 6
    S = orc.Scene(sc)
    prims = [RM.Prim.from_scene(sc, i) for i in range(sc["n"])]
    rays = I.rays_through_box(6, 8, -0.15, 0.15)
    rng = np.random.default_rng(4)
    n_coll = 0
    for r in rays:
        o, v = r[0:3].astype(np.float64), r[4:7].astype(np.float64)
        total = RM.tau_quad(prims, o, v, 0, np.inf)
        for xi in rng.random(4):
            t = S.free_flight(r, xi)
            ts = -math.log1p(-xi)
            if t is None:
                assert total < ts + 1e-9
            else:
                n_coll += 1
                assert abs(RM.tau_quad(prims, o, v, 0, t) - ts) < 1e-8
    assert n_coll > 5


# ---------------------------------------------------------------- camera / phase function
def test_camera_ray_matches_f64(orc):
    d = I.render_desc_cfg2(3, 64, 48)
    for px, py in [(0, 0), (63, 47), (10, 30), (32, 24)]:
        o, v = orc.camera_ray(d, px, py, 0.25, 0.75)
        o64, v64 = I.camera_rays_f64(d, np.array([px]), np.array([py]), 0.25, 0.75)
        assert np.allclose(v, v64[0], atol=2e-7) and np.allclose(o, o64[0])


def test_hg_phase_function(orc):
    """Reading C19: HG normalised over the sphere; samples follow the density (chi^2)."""
    from scipy import integrate, stats
    for g in (0.0, 0.6, -0.3):
        val, _ = integrate.quad(lambda c: orc.hg_eval(g, c) * 2 * math.pi, -1, 1)
        assert abs(val - 1) < 1e-10
    g = 0.6
    rng = np.random.default_rng(0)
    v = np.array([0.3, -0.4, 0.866])
    v /= np.linalg.norm(v)
    cs = np.array([orc.hg_sample(g, v, *rng.random(2)) @ v for _ in range(20000)])
    edges = np.linspace(-1, 1, 21)
    obs, _ = np.histogram(cs, edges)
    exp_ = np.array([integrate.quad(lambda c: orc.hg_eval(g, c) * 2 * math.pi, a, b)[0]
                     for a, b in zip(edges[:-1], edges[1:])]) * len(cs)
    assert stats.chisquare(obs, exp_).pvalue > 1e-3


# ---------------------------------------------------------------- estimators
def _tiny_desc(mode, **kw):
    d = I.camera((0, 0, 2.0), (0, 0, 0), (0, 1, 0), 20.0, 8, 8)
    d.update(mode=mode, max_depth=1, jitter=0, albedo=0.8, hg_g=0.3, sun_dir=I.SUN, sun_E=3.0, env_L=0.2,
             seed=99, ext=I.policy(), nee=I.policy())
    d.update(kw)
    return d


def _tiny_scene():
    sc = I.scene_cfg1p(n_pairs=10, seed=8)
    sc["mu"] = sc["mu"] * 0.25
    return sc


def test_tomography_estimator_unbiased(orc):
    """P:L363 / P:L317: per-segment tau-hat is unbiased under stochastic level+orientation masks;
    mean over samples = deterministic tau (+-4 SE)."""
    sc = _tiny_scene()
    S = orc.Scene(sc)
    det = S.render_probes(_tiny_desc(0), [27, 36], 0, 1)[0][:, 0]
    d = _tiny_desc(0, ext=I.policy(level_strategy=5, beta=0.2, orient_strategy=3))  # scene-default f0 (C12)
    vals, nr = S.render_probes(d, [27, 36], 0, 4000)
    mean, se = vals.mean(1), vals.std(1) / math.sqrt(vals.shape[1])
    assert np.all(np.abs(mean - det) <= 4 * se + 1e-12), (mean, det, se)
    assert np.all(nr == 1)


def test_single_scattering_matches_quadrature(orc):
    """Single scattering has a deterministic reference: L = int kappa(t) T(0,t)
    albedo p(theta) T_sun(x_t) E_sun dt + T(0,inf) L_env, with T and kappa by quadrature."""
    from scipy import integrate
    sc = _tiny_scene()
    S = orc.Scene(sc)
    prims = [RM.Prim.from_scene(sc, i) for i in range(sc["n"])]
    d = _tiny_desc(1)
    pix = 3 * 8 + 4
    o, v = orc.camera_ray(d, pix % 8, pix // 8)
    o, v = o.astype(np.float64), v.astype(np.float64)
    sun = I.SUN.astype(np.float64)
    kappa = lambda t: sum(p.alpha * p.K(o + t * v) for p in prims)
    ts = sorted(c for p in prims for c in (p.chord(o, v, 0, np.inf) or ()))
    lo, hi = ts[0], ts[-1]
    # tabulate T(0,t) by cumulative quadrature on a fine grid
    grid = np.linspace(lo, hi, 801)
    kv = np.array([kappa(t) for t in grid])
    tau_cum = integrate.cumulative_trapezoid(kv, grid, initial=0)
    cost = float(v @ sun)
    ph = orc.hg_eval(0.3, cost)
    tsun = np.array([math.exp(-RM.tau_quad(prims, o + t * v, sun, 0, np.inf)) if kv[k] != 0 else 0.0
                     for k, t in enumerate(grid)])
    L_ref = integrate.trapezoid(kv * np.exp(-tau_cum) * 0.8 * ph * tsun * 3.0, grid) + math.exp(-tau_cum[-1]) * 0.2
    vals, nr = S.render_probes(d, [pix], 0, 20000)
    mean, se = vals.mean(), vals.std() / math.sqrt(vals.size)
    assert abs(mean - L_ref) <= 4 * se + 2e-4 * abs(L_ref), (mean, L_ref, se)


def test_albedo_zero_and_white_furnace(orc):
    """Albedo 0 => pixel = L_env T(camera ray) in expectation; white furnace (albedo 1, L_env=1, no
    sun, deep paths, kappa >= 0) => every path returns 1 unless the depth cap is hit."""
    sc = _tiny_scene()
    S = orc.Scene(sc)
    prims = [RM.Prim.from_scene(sc, i) for i in range(sc["n"])]
    d = _tiny_desc(1, albedo=0.0, sun_E=0.0, env_L=0.7, max_depth=4)
    pix = 27
    o, v = orc.camera_ray(d, pix % 8, pix // 8)
    T = math.exp(-RM.tau_quad(prims, o.astype(np.float64), v.astype(np.float64), 0, np.inf))
    vals, _ = S.render_probes(d, [pix], 0, 20000)
    mean, se = vals.mean(), vals.std() / math.sqrt(vals.size)
    assert abs(mean - 0.7 * T) <= 4 * se
    d = _tiny_desc(1, albedo=1.0, sun_E=0.0, env_L=1.0, max_depth=64, hg_g=0.0)
    vals, nr = S.render_probes(d, [27, 28, 36], 0, 300)
    assert abs(vals.mean() - 1.0) < 0.02
    assert set(np.unique(vals)) <= {0.0, 1.0}


# ---------------------------------------------------------------- foveation
def test_foveation_limits_reduce_to_plain_renders(orc):
    """P:L624-L634, readings F1-F5: a threshold above every frequency changes nothing; a threshold of
    0 keeps exactly level 0 (the Gaussians, frequency 0): both reduce to renders without foveation
    (static masks all / {0}), sample for sample, for tomography and single scattering."""
    sc = I.scene_cfg1()
    S = orc.Scene(sc)
    pix = list(range(0, 64, 3))
    for mode in (0, 1):
        base = _tiny_desc(mode, jitter=1)
        plain = S.render_probes(base, pix, 0, 6)[0]
        lvl0 = S.render_probes(dict(base, ext=I.policy(static_mask=1), nee=I.policy(static_mask=1)), pix, 0, 6)[0]
        hi = S.render_probes(dict(base, foveation=I.foveation((4, 4), 1e30, 0.0, 0.3)), pix, 0, 6)[0]
        zero = S.render_probes(dict(base, foveation=I.foveation((4, 4), 0.0, 0.0, 0.3)), pix, 0, 6)[0]
        assert np.array_equal(hi, plain)
        assert np.array_equal(zero, lvl0)
        assert not np.array_equal(plain, lvl0)


def test_foveation_primitive_check_follows_definition(orc):
    """F4: a primitive is integrated iff its frequency along the ray |omega_vec . d| does not
    exceed f_max, omega_vec = R S^-1 (omega, omega, omega) computed here independently in
    numpy from the primitive's quaternion and scales; thresholds 1 % either side of it."""
    rng = np.random.default_rng(12)
    n = 1
    mu = np.zeros((1, 3))
    quat = I.random_quats(rng, 1)
    scale = np.array([[0.3, 0.2, 0.25]])
    sc = I._finish(mu, quat, scale, np.array([1.0]), np.array([1.2]), np.array([1], np.uint8), name="one")
    S = orc.Scene(sc)
    d = _tiny_desc(0)
    x, y, z, w = (float(v) for v in sc["quat"][0])
    nq = math.sqrt(x * x + y * y + z * z + w * w)
    x, y, z, w = x / nq, y / nq, z / nq, w / nq
    R = np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                  [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                  [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])
    wvec = R @ (float(sc["omega"][0]) / sc["scale"][0].astype(np.float64))
    pix = [27, 28, 35, 36]
    _, dirs = I.camera_rays_f64(d, np.array(pix) % 8, np.array(pix) // 8)
    full = S.render_probes(d, pix, 0, 1)[0][:, 0]
    assert np.all(np.abs(full) > 1e-6)
    for k, p in enumerate(pix):
        f = abs(float(dirs[k] @ wvec))
        # continuous mode only (foveation mode 2: the per-primitive check without level masking)
        above = dict(d, foveation=I.foveation((0, 0), f * 1.01, 0.0, 0.0, mode=2))
        below = dict(d, foveation=I.foveation((0, 0), f * 0.99, 0.0, 0.0, mode=2))
        assert S.render_probes(above, [p], 0, 1)[0][0, 0] == full[k]
        assert S.render_probes(below, [p], 0, 1)[0][0, 0] == 0.0


# ---------------------------------------------------------------- motion blur
def test_motion_blur_zero_magnitude_is_plain(orc):
    """M1: a box filter of length 0 leaves every sample unchanged."""
    sc = I.scene_cfg1()
    S = orc.Scene(sc)
    pix = list(range(0, 64, 5))
    for mode in (0, 1):
        base = _tiny_desc(mode, jitter=1)
        plain = S.render_probes(base, pix, 0, 4)[0]
        mb = S.render_probes(dict(base, motion_blur=I.motion_blur((1, 2, 0.5), 0.0)), pix, 0, 4)[0]
        assert np.array_equal(plain, mb)


def test_motion_blur_is_the_box_filtered_field(orc):
    """M1/M2: the estimate over exposure times is the optical depth of the field convolved with
    a box of length m along d: the sample mean matches the shift average of the closed form computed
    here by Gauss-Legendre quadrature over the shift (one Gabor, one ray), within 4 SE."""
    rng = np.random.default_rng(3)
    sc = I._finish(np.zeros((1, 3)), I.random_quats(rng, 1), np.array([[0.3, 0.2, 0.25]]), np.array([1.0]),
                   np.array([1.3]), np.array([1], np.uint8), name="one")
    S = orc.Scene(sc)
    d = _tiny_desc(0)
    mdir, m = np.array([0.6, 0.0, 0.8]), 0.4
    pix = 27
    o, v = I.camera_rays_f64(d, np.array([pix % 8]), np.array([pix // 8]))
    xs, ws = np.polynomial.legendre.leggauss(64)
    ref = 0.0
    for x, wgt in zip(xs, ws):  # shift s = m (u - 1/2), u = (x + 1) / 2
        sft = m * 0.5 * x * mdir
        ray = I.pack_rays(o - sft, v)[0]
        ref += 0.5 * wgt * float(orc.lib().or_prim_integral(S.h, 0, orc._p(ray[:3]), orc._p(ray[4:7]), 0.0, np.inf))
    ref *= float(sc["alpha"][0])
    vals = S.render_probes(dict(d, motion_blur=I.motion_blur(mdir, m)), [pix], 0, 20000)[0][0]
    se = vals.std() / math.sqrt(vals.size)
    assert abs(vals.mean() - ref) <= 4 * se + 1e-9, (vals.mean(), ref, se)
    assert vals.std() > 0


def test_motion_blur_mask_attenuation(orc):
    """M3: a group is culled iff |sin(m k/2)/(m k/2)| of its mean frequency along d is
    below the threshold, k from the sign-aligned group means computed here independently in numpy
    (tests/refmath.py); level 0 is never culled; m = 0 culls nothing."""
    sc = I.scene_cfg1()
    S = orc.Scene(sc)
    mask0, att0 = S.motion_blur_mask((1, 0, 0), 0.0, 0.99)
    assert mask0 == (1 << 10) - 1 and np.all(att0 == 1.0)
    groups, _ = S.groups()
    k = RM.motion_blur_group_k(sc, groups, (1, 0, 0))
    mask, att = S.motion_blur_mask((1, 0, 0), 0.2, 0.6)
    assert mask & 1 and att[0] == 1.0
    for g in range(1, 10):
        x = 0.5 * 0.2 * k[g]
        assert att[g] == pytest.approx(abs(math.sin(x) / x), rel=1e-6)
        assert bool(mask >> g & 1) == (att[g] >= 0.6)
    assert 0 < bin(mask).count("1") < 10


@pytest.mark.parametrize("mk", [1.0, 2.5, 5.0])
def test_motion_blur_attenuation_is_the_box_filter_response(orc, mk):
    """M2 pinned to the physics it stands for: for a Gabor whose envelope is wide against
    the blur length (s = 40, m = 0.08), the box-filtered optical depth (shift average of the closed
    form over s = m (u - 1/2) d, 64-node Gauss-Legendre) divided by the unblurred one equals the signed
    sinc(m k / 2), k = omega_vec . d -- for a ray through the centre across d, so the envelope barely
    moves.  The oracle's attenuation for that one-member group must be its magnitude."""
    s_ = 40.0
    m = 0.08
    k = mk / m  # omega_vec . d with omega_vec along d = x: |omega_vec| = omega sqrt(3) / s for R = I?
    # omega_vec = R S^-1 (w, w, w): with R = I and isotropic s it is (w/s)(1,1,1); choose d along it
    w = k * s_ / math.sqrt(3.0)
    sc = make_scene([((0, 0, 0), ID, (s_, s_, s_), w, 1.0, 3.0)])
    S = orc.Scene(sc)
    d = np.ones(3) / math.sqrt(3.0)
    v = np.array([1.0, -1.0, 0.0]) / math.sqrt(2.0)  # ray across the motion direction, through the centre
    o = -300.0 * v
    xs, ws = np.polynomial.legendre.leggauss(64)
    blur = 0.0
    for x, wgt in zip(xs, ws):
        ray = I.pack_rays((o - m * 0.5 * x * d)[None], v[None])[0]
        blur += 0.5 * wgt * S.prim_integral(0, ray[:3], ray[4:7], 0.0, np.inf)
    plain = S.prim_integral(0, o, v, 0.0, np.inf)
    ratio = blur / plain
    sinc = math.sin(0.5 * m * k) / (0.5 * m * k)
    assert ratio == pytest.approx(sinc, abs=2e-4), (ratio, sinc)
    _, att = S.motion_blur_mask(d, m, 0.0)
    assert att[1] == pytest.approx(abs(ratio), abs=2e-4)


# ---------------------------------------------------------------- scene-derived parameters (C11, C12, F3, C8')
def test_orientation_bins_match_independent_argmax(orc):
    """C11: bin = argmax_k |d . o_k|, d = R S^-1 (1,1,1), ties -> lower k.  The oracle's fp32 decision
    equals a float64 numpy argmax (tests/refmath.py) wherever the best two scores differ by more than
    1e-5 relative, for K = 3 and K = 6; constructed exact ties go to the lower bin."""
    rng = np.random.default_rng(21)
    for K in (3, 6):
        n = 800
        sc = I._finish(rng.uniform(-1, 1, (n, 3)), I.random_quats(rng, n), np.exp(rng.normal(-3, 0.6, (n, 3))),
                       np.ones(n), np.full(n, 1.0), np.ones(n, np.uint8), K=K, name="bins")
        _, b = orc.Scene(sc).groups()
        ref = RM.bins_f64(sc)
        ok = ref >= 0
        assert ok.mean() > 0.98
        assert np.array_equal(b[ok], ref[ok])
        assert len(set(b.tolist())) == K
    ties = [((1, 1, 1), 0), ((2, 1, 1), 1), ((1, 2, 2), 0), ((3, 3, 1), 2), ((1, 2, 1), 0)]
    sc = make_scene([((0, 0, 0), ID, s, 1.0, 1.0, 3.0) for s, _ in ties])
    _, b = orc.Scene(sc).groups()
    assert list(b) == [t for _, t in ties]


def test_level_fmax_is_the_level_maximum(orc):
    """F3: the per-level bound the foveation level mask compares with is the maximum of
    |omega_vec| over the level; pinned by the rotation-invariant form w |S^-1 (1,1,1)| (no R)."""
    for sc in (I.scene_cfg1(), I.scene_bunny(counts=(50, 300, 600, 900))):
        lf, _ = orc.Scene(sc).info()
        ref = RM.level_fmax_invariant(sc)
        assert lf[0] == 0.0
        np.testing.assert_allclose(lf, ref, rtol=1e-6)
        assert np.all(lf[1:4] > 0)


def test_group_f0_is_the_level_median(orc):
    """C12: the representative whitened frequency of a group is sqrt(3) x the median omega of its level
    (numpy's median), shared by every bin (and band) of the level; level 0 gets 0."""
    for sc in (I.scene_cfg1(), I.scene_bunny(counts=(50, 301, 600, 900))):
        _, f0 = orc.Scene(sc).info()
        np.testing.assert_allclose(f0, RM.group_f0_median(sc), rtol=1e-6)
    sc = I.scene_cfg5()
    sub = {k: (v[::97] if isinstance(v, np.ndarray) and v.ndim and len(v) == sc["n"] else v) for k, v in sc.items()}
    sub["n"] = len(sub["mu"])
    _, f0 = orc.Scene(sub).info()
    assert len(f0) == 30
    np.testing.assert_allclose(f0, RM.group_f0_median(sub), rtol=1e-6)


def test_adaptive_extent_level_set(orc):
    """C8' (Eq. 15): E is the whitened distance at which the worst-case untruncated line
    integral alpha s_max /(2 pi s1 s2 s3) e^{-(E^2 + 3 w^2)/2} equals eps.  Pinned by the oracle's own
    closed-form integral (itself pinned to quadrature above) on rays that realise the worst case:
    a Gaussian (w = 0) crossed along its major axis, and an isotropic Gabor crossed along k_W at
    a closest point with zero phase (Omega^2 = 3 w^2, cos = 1)."""
    eps = 1e-3
    # anisotropic Gaussian, major axis x
    s = (0.3, 0.1, 0.15)
    sc = make_scene([((0, 0, 0), ID, s, 0.0, 0.005, 3.0)])
    E = float(orc.adaptive_extent(sc, eps)[0])
    assert 1e-3 < E < 3.0
    # whitened perpendicular distance E along y: world offset E * s_y
    o = np.array([-5.0, E * 0.1, 0.0])
    val = float(sc["alpha"][0]) * orc.Scene(dict(sc, extent=np.array([50.0], np.float32))).prim_integral_infinite(
        0, o, np.array([1.0, 0.0, 0.0]))
    assert val == pytest.approx(eps, rel=1e-5)
    # isotropic Gabor, ray along (1,1,1)/sqrt3 (k_W direction), offset along (1,-1,0)/sqrt2 (phase 0)
    s0, w = 0.2, 0.9
    sc = make_scene([((0, 0, 0), ID, (s0, s0, s0), w, 0.05, 3.0)])
    E = float(orc.adaptive_extent(sc, eps)[0])
    assert 1e-3 < E < 3.0
    v = np.ones(3) / math.sqrt(3.0)
    off = np.array([1.0, -1.0, 0.0]) / math.sqrt(2.0) * E * s0
    o = off - 4.0 * v
    val = float(sc["alpha"][0]) * orc.Scene(dict(sc, extent=np.array([50.0], np.float32))).prim_integral_infinite(
        0, o, v)
    assert val == pytest.approx(eps, rel=1e-5)
    # clamps: huge alpha -> 3, tiny alpha -> the 1e-3 floor
    big = make_scene([((0, 0, 0), ID, s, 0.0, 1e9, 3.0), ((0, 0, 0), ID, s, 0.0, 1e-12, 3.0)])
    assert list(orc.adaptive_extent(big, eps)) == [3.0, np.float32(1e-3)]


def test_foveation_threshold_closed_forms(orc):
    """F1/F2/F5 at points where the threshold has a closed form: at the gaze pixel centre
    e = 0 so f_max = f0 (1 + sigma (2u - 1)) with u the stream-6 uniform; along a row the threshold
    falls linearly, f0 - slope |dx| / max(W, H); beyond e = f0 / slope it is 0."""
    d = _tiny_desc(0)
    W = d["width"]
    f0, slope, sig = 2.0, 3.0, 0.25
    gaze = (3.5, 2.5)  # the centre of pixel (3, 2)
    fov = I.foveation(gaze, f0, slope, sig)
    dd = dict(d, foveation=fov)
    for smp in range(4):
        u = orc.uniform(d["seed"], 2 * W + 3, smp, 0, 6, 0)
        assert orc.fov_fmax(dd, 2 * W + 3, smp) == pytest.approx(f0 * (1 + sig * (2 * u - 1)), rel=1e-6)
    dn = dict(d, foveation=I.foveation(gaze, f0, slope, 0.0))
    for px in range(W):
        e = abs(px + 0.5 - gaze[0]) / W
        assert orc.fov_fmax(dn, 2 * W + px, 0) == pytest.approx(max(0.0, f0 - slope * e), rel=1e-6, abs=1e-7)
    far = dict(d, foveation=I.foveation((0.0, 0.0), 0.5, 10.0, 0.3))
    assert orc.fov_fmax(far, 7 * W + 7, 1) == 0.0


# ---------------------------------------------------------------- backward (alpha part)
def test_grad_alpha_matches_finite_differences(orc):
    """tau is linear in the opacities (Eq. 1-2), so the opacity gradient of sum_r dl_r tau_r equals the
    finite difference of the oracle's own forward trace (one primitive's alpha doubled), to rounding."""
    sc = I.scene_cfg1(n=60, seed=5)
    S = orc.Scene(sc)
    rays = I.rays_through_box(3, 40)
    dl = np.random.default_rng(2).normal(size=40)
    g = S.grad_alpha(rays, dl)
    base = S.trace(rays)["tau"]
    for i in (0, 7, 33, 59):
        sc2 = dict(sc, alpha=sc["alpha"].copy())
        sc2["alpha"][i] *= 2.0
        d = (orc.Scene(sc2).trace(rays)["tau"] - base) @ dl / float(sc["alpha"][i])
        assert abs(d - g[i]) <= 1e-9 * (1 + abs(g[i])), (i, d, g[i])
    assert np.count_nonzero(g) > 10


# ---------------------------------------------------------------- parameter gradient (§8(f) rank 4)
def _R_of_q(q):
    """rotation matrix of the quaternion (x, y, z, w), normalised; complex-safe (complex-step pins)."""
    x, y, z, w = q / np.sqrt(np.sum(q * q))
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


def _tau_full_line(th, o, v):
    """App. A boxed infinite-limit integral times alpha, written out here:
    alpha (8 pi^3 |S|)^-1/2 sqrt(2 pi / a) e^{-(gamma - beta^2/a)/2} e^{-B^2/2a} cos(delta - beta B / a)."""
    mu, q, s, om, al = th[0:3], th[3:7], th[7:10], th[10], th[11]
    R = _R_of_q(q)
    Si = R @ np.diag(1.0 / s ** 2) @ R.T
    wv = R @ (om / s)
    d = o - mu
    a, b, g = v @ Si @ v, v @ Si @ d, d @ Si @ d
    B, dl = wv @ v, wv @ d
    norm = 1.0 / np.sqrt(8 * np.pi ** 3 * np.prod(s) ** 2)
    return al * norm * np.sqrt(2 * np.pi / a) * np.exp(-0.5 * (g - b * b / a)) * np.exp(-B * B / (2 * a)) * \
        np.cos(dl - b * B / a)


def _one_prim_scene(th, E):
    return make_scene([(th[0:3], th[3:7], th[7:10], th[10], th[11], E)])


@pytest.mark.parametrize("omega", [0.0, 0.8])
def test_grad_params_full_line_complex_step(orc, omega):
    """d tau / d(mu, q, s, omega, alpha) of one primitive whose truncation is negligible (E = 6:
    e^{-18}) on a ray covering its whole chord, against the complex-step derivative (exact to
    rounding) of the full-line closed form written out above -- pins the oracle's finite
    differences, its parameter order and its q/s/omega chain (a transposed R or a wrong s power
    fails)."""
    rng = np.random.default_rng(11)
    for trial in range(4):
        q = rng.normal(size=4)
        q /= np.linalg.norm(q)
        th = np.concatenate([rng.uniform(-0.3, 0.3, 3), q, rng.uniform(0.15, 0.35, 3), [omega], [0.7]])
        th = th.astype(np.float32).astype(np.float64)
        o = np.array([-2.0, rng.uniform(-0.1, 0.1), rng.uniform(-0.1, 0.1)])
        v = np.array([1.0, 0.1 * rng.normal(), 0.1 * rng.normal()])
        v /= np.linalg.norm(v)
        ray = np.array([*o, -20.0, *v, 20.0], np.float32)
        o, v = ray[0:3].astype(np.float64), ray[4:7].astype(np.float64)
        S = orc.Scene(_one_prim_scene(th, 6.0))
        g, _ = S.grad_params(ray[None, :], np.array([1.0]))
        ref = np.array([(_tau_full_line(th + 1e-30j * np.eye(12)[k], o, v)).imag / 1e-30 for k in range(12)])
        scale = np.abs(ref).max()
        assert np.all(np.abs(g[0] - ref) <= 1e-6 * scale), (trial, g[0], ref)
        # alpha enters linearly; q's norm does not matter (gradient orthogonal to q)
        assert abs(g[0, 11] * th[11] - _tau_full_line(th, o, v)) <= 1e-7 * abs(g[0, 11] * th[11]) + 1e-12
        assert abs(g[0, 3:7] @ th[3:7]) <= 1e-6 * scale


def test_grad_params_truncated_leibniz(orc):
    """Truncated kernel (E = 3, C7), chord strictly inside the ray's range: d tau / d mu and d tau /
    d omega by Leibniz's rule written out here -- adaptive quadrature (scipy) of dg/dmu, dg/domega
    of Eq. 6 along the chord plus the moving-endpoint terms g(x_e) dt_e/dmu, dt_e/dmu =
    S^-1 d_e / (v . S^-1 d_e) -- against the oracle's finite differences; and the translation
    invariance v . d tau / d mu = 0."""
    from scipy import integrate
    rng = np.random.default_rng(12)
    for trial in range(4):
        q = rng.normal(size=4)
        q /= np.linalg.norm(q)
        th = np.concatenate([rng.uniform(-0.2, 0.2, 3), q, rng.uniform(0.15, 0.35, 3), [1.1], [0.9]])
        th = th.astype(np.float32).astype(np.float64)
        ray = np.array([-2.0, 0.05 * rng.normal(), 0.05 * rng.normal(), 0.0, 1.0, 0.0, 0.0, 10.0], np.float32)
        o, v = ray[0:3].astype(np.float64), ray[4:7].astype(np.float64)
        S = orc.Scene(_one_prim_scene(th, 3.0))
        g, _ = S.grad_params(ray[None, :], np.array([1.0]))
        mu, R, s, om, al = th[0:3], _R_of_q(th[3:7]), th[7:10], th[10], th[11]
        Si = R @ np.diag(1.0 / s ** 2) @ R.T
        wv = R @ (om / s)
        norm = 1.0 / np.sqrt(8 * np.pi ** 3 * np.prod(s) ** 2)
        d0 = o - mu
        a, b, c = v @ Si @ v, v @ Si @ d0, d0 @ Si @ d0 - 9.0
        disc = b * b - a * c
        assert disc > 0.05 * b * b
        t0, t1 = (-b - np.sqrt(disc)) / a, (-b + np.sqrt(disc)) / a

        def gk(t):
            d = o + t * v - mu
            return norm * np.exp(-0.5 * d @ Si @ d), d

        dmu = np.zeros(3)
        for k in range(3):
            f = lambda t: (lambda e, d: e * ((Si @ d)[k] * np.cos(wv @ d) + wv[k] * np.sin(wv @ d)))(*gk(t))
            dmu[k] = al * integrate.quad(f, t0, t1, epsabs=1e-13, epsrel=1e-10, limit=200)[0]
        for te, sgn in ((t1, 1.0), (t0, -1.0)):
            e, d = gk(te)
            dmu += sgn * al * e * np.cos(wv @ d) * (Si @ d) / (v @ Si @ d)
        fo = lambda t: (lambda e, d: -e * np.sin(wv @ d) * (wv @ d) / om)(*gk(t))
        dom = al * integrate.quad(fo, t0, t1, epsabs=1e-13, epsrel=1e-10, limit=200)[0]
        scale = np.abs(dmu).max()
        assert np.all(np.abs(g[0, 0:3] - dmu) <= 1e-6 * scale), (trial, g[0, 0:3], dmu)
        assert abs(g[0, 10] - dom) <= 1e-6 * max(abs(dom), scale), (trial, g[0, 10], dom)
        assert abs(g[0, 0:3] @ v) <= 1e-6 * scale


def test_distance_bands_fold_into_groups(orc):
    """Config 5's distance bands (C24, fig:army_bunny P:L606-L617): group = band * 10 + g(l, b); a mask
    selecting one band's groups gives exactly the optical depth of that band's primitives (per-group
    sums), and a stochastic policy draws once and applies the same weights to every band's copy."""
    sc = I.scene_cfg5()
    keep = np.flatnonzero(np.isin(np.arange(sc["n"]) // 33280, [0, 60, 119]))[::40]
    sub = {k: (v[keep] if isinstance(v, np.ndarray) and v.ndim and len(v) == sc["n"] else v) for k, v in sc.items()}
    sub["n"] = len(keep)
    assert set(np.unique(sub["band"]).tolist()) == {0, 1, 2}
    S = orc.Scene(sub)
    g, _ = S.groups()
    np.testing.assert_array_equal(g // 10, sub["band"])
    rng = np.random.default_rng(5)
    tgt = sub["mu"][rng.integers(0, sub["n"], 24)]
    rays = I.pack_rays(tgt - 30 * np.array([0.1, 0.3, 0.95]), np.tile([0.1, 0.3, 0.95], (24, 1)))
    full = S.trace(rays, want_groups=True)
    for bd in range(3):
        m = I.level_mask((0, 1, 2, 3), n_bands=3, bands=[bd])
        r = S.trace(rays, mask=m)
        np.testing.assert_allclose(r["tau"], full["groups"][:, 10 * bd:10 * bd + 10].sum(1), rtol=1e-12, atol=1e-15)
    pol = I.policy(level_strategy=5, beta=0.2, orient_strategy=3)
    m, w = S.policy_eval(pol, np.array([0.0, 0.6, 0.8]), 0.7, [0.3, 0.5, 0.9], group_f0=S.info()[1])
    assert m == (m & 0x3FF) * (1 | 1 << 10 | 1 << 20)
    np.testing.assert_array_equal(w[:10], w[10:20])
    np.testing.assert_array_equal(w[:10], w[20:30])
