"""Test-side independent reference pieces (numpy/scipy), used to PIN the oracle.

Nothing here is shared with the oracle or the CUDA path: Eq. 6 is evaluated in its
dense world-space matrix form and line integrals are taken by adaptive quadrature
(scipy.integrate.quad), i.e. by the plain definition, not by any closed form.
"""
import math

import numpy as np
from scipy import integrate


def quat_R(q):
    x, y, z, w = (float(a) for a in q)
    n = math.sqrt(x * x + y * y + z * z + w * w)
    x, y, z, w = x / n, y / n, z / n, w / n
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


class Prim:
    """One primitive in the paper's parameterisation: Sigma = R S S^T R^T,
    omega_vec = R S^-1 (w,w,w)^T."""

    def __init__(self, mu, q, s, omega, alpha=1.0, E=3.0):
        # inputs are rounded to fp32 exactly as the scene arrays are (reading C25: the input
        # rounding is shared, the arithmetic is not)
        f = lambda a: np.asarray(np.asarray(a, np.float32), np.float64)
        mu, q, s, omega, alpha, E = f(mu), f(q), f(s), float(f(omega)), float(f(alpha)), float(f(E))
        self.mu = np.asarray(mu, np.float64)
        self.R = quat_R(q)
        self.s = np.asarray(s, np.float64)
        self.Sigma = self.R @ np.diag(self.s ** 2) @ self.R.T
        self.Sinv = np.linalg.inv(self.Sigma)
        self.wvec = self.R @ (float(omega) / self.s)
        self.alpha = float(alpha)
        self.E = float(E)
        self.norm = 1.0 / math.sqrt(8 * math.pi ** 3 * np.linalg.det(self.Sigma))

    @classmethod
    def from_scene(cls, sc, i):
        return cls(sc["mu"][i], sc["quat"][i], sc["scale"][i], sc["omega"][i], sc["alpha"][i], sc["extent"][i])

    def K(self, x, truncated=True):
        """Eq. 6, optionally truncated at the ellipsoid ||W(x-mu)|| <= E (C7)."""
        d = np.asarray(x, np.float64) - self.mu
        q = d @ self.Sinv @ d
        if truncated and q > self.E ** 2:
            return 0.0
        return self.norm * math.exp(-0.5 * q) * math.cos(self.wvec @ d)

    def chord(self, o, v, t0=-np.inf, t1=np.inf):
        """[t_in, t_out] of the ellipsoid along o + t v, clipped; None if empty (quadratic roots)."""
        o, v = np.asarray(o, np.float64), np.asarray(v, np.float64)
        d = o - self.mu
        a = v @ self.Sinv @ v
        b = v @ self.Sinv @ d
        c = d @ self.Sinv @ d - self.E ** 2
        disc = b * b - a * c
        if disc <= 0:
            return None
        r = math.sqrt(disc)
        ta, tb = (-b - r) / a, (-b + r) / a
        ta, tb = max(ta, t0), min(tb, t1)
        return (ta, tb) if tb > ta else None

    def line_integral(self, o, v, t0=-np.inf, t1=np.inf, truncated=True):
        """int K(o + t v) dt by adaptive quadrature of the plain definition."""
        o, v = np.asarray(o, np.float64), np.asarray(v, np.float64)
        if truncated:
            ch = self.chord(o, v, t0, t1)
            if ch is None:
                return 0.0
            a, b = ch
        else:
            # untruncated: integrate over +-40 envelope widths around the closest approach
            a_ = v @ self.Sinv @ v
            tc = -(v @ self.Sinv @ (o - self.mu)) / a_
            w = 40.0 / math.sqrt(a_)
            a, b = max(t0, tc - w), min(t1, tc + w)
        f = lambda t: self.K(o + t * v, truncated=False)
        val, err = integrate.quad(f, a, b, epsabs=1e-15, epsrel=1e-12, limit=400)
        return val


def tau_quad(prims, o, v, t0, t1, weights=None):
    """alpha-weighted optical depth (Eq. 2) of a list of Prims by quadrature."""
    tot = 0.0
    for k, p in enumerate(prims):
        w = 1.0 if weights is None else weights[k]
        tot += w * p.alpha * p.line_integral(o, v, t0, t1)
    return tot


# ---------------------------------------------------------------- scene-derived policy parameters
def omega_vectors(scene):
    """World frequency vectors omega_vec = R S^-1 (omega, omega, omega), float64 [n, 3]."""
    return np.array([quat_R(q) @ (float(w) / np.asarray(s, np.float64))
                     for q, s, w in zip(scene["quat"], scene["scale"], scene["omega"])]).reshape(-1, 3)


def bins_f64(scene, margin=1e-5):
    """Orientation bin argmax_k |d . o_k| (C11) in float64 from the quaternion, d = R S^-1 (1,1,1);
    -1 where the two best scores are within `margin` (relative): ties decided by rounding."""
    K = scene["K"]
    axes = np.asarray(scene["bin_axes"], np.float64).reshape(K, 3)
    out = []
    for q, s in zip(scene["quat"], scene["scale"]):
        d = quat_R(q) @ (1.0 / np.asarray(s, np.float64))
        a = np.abs(axes @ d)
        o = np.sort(a)[::-1]
        out.append(-1 if K > 1 and o[0] - o[1] <= margin * o[0] else int(np.argmax(a)))
    return np.array(out)


def level_fmax_invariant(scene):
    """Maximum |omega_vec| per level from the rotation-invariant form |R S^-1 (w,w,w)| = w |S^-1 (1,1,1)|
    (R orthogonal), i.e. without forming R."""
    s = np.asarray(scene["scale"], np.float64)
    f = np.asarray(scene["omega"], np.float64) * np.sqrt((1.0 / s ** 2).sum(1))
    out = np.zeros(8)
    for l in range(1, scene["P"]):
        sel = np.asarray(scene["level"]) == l
        if sel.any():
            out[l] = f[sel].max()
    return out


def group_f0_median(scene):
    """Reading C12: sqrt(3) x the median omega of each Gabor level (numpy's median), for every bin and
    band of the level."""
    P, K, nb = scene["P"], scene["K"], int(scene.get("n_bands", 1))
    G0 = 1 + (P - 1) * K
    out = np.zeros(G0 * nb)
    for l in range(1, P):
        sel = np.asarray(scene["level"]) == l
        if not sel.any():
            continue
        med = float(np.median(np.asarray(scene["omega"], np.float32)[sel])) * math.sqrt(3.0)
        for bd in range(nb):
            for b in range(K):
                out[bd * G0 + 1 + (l - 1) * K + b] = med
    return out


def motion_blur_group_k(scene, groups, direction):
    """Reading M3: per group |mean omega_vec . d| with each member's sign aligned to the group's member
    of largest |omega_vec| (first index on ties); nan for empty groups."""
    d = np.asarray(direction, np.float64)
    d = d / np.linalg.norm(d)
    wv = omega_vectors(scene)
    G = int(groups.max()) + 1 if len(groups) else 0
    out = np.full(G, np.nan)
    for g in range(G):
        sel = np.flatnonzero(groups == g)
        if not len(sel):
            continue
        v = wv[sel]
        ref = v[np.argmax(np.linalg.norm(v, axis=1))]
        v = np.where((v @ ref)[:, None] < 0, -v, v)
        out[g] = abs(float(v.mean(0) @ d))
    return out
