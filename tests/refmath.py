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
