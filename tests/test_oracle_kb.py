"""Pins of the oracle's Kaiser-Bessel window path.

Remark rmk::PWindow names the KB window and builds polynomial approximations of the
windows by Chebyshev interpolation; Section 5.1 (Fig. 5(a)) compares it with the
Gaussian at equal support.  These pins check the oracle's KB pieces against quadrature, the
window's definition, the SOG-exact sums, Ewald2D and the paper's Fig. 5(a) ordering.
"""
import math

import numpy as np
import pytest
from numpy.polynomial import chebyshev as npcheb
from scipy.integrate import quad
from scipy.special import i0

from oracle import plan as P
from oracle import sog, sog_exact, ewald2d
from synth import config_system


def _kb(x, H, beta):
    """Kaiser (1980) window written out independently of the oracle."""
    return i0(beta * math.sqrt(1.0 - (x / H) ** 2)) / i0(beta) if abs(x) <= H else 0.0


@pytest.mark.parametrize("H,beta", [(1.0, 10.0), (2.5, 18.9), (4.0, 31.5)])
def test_kb_window_fourier_transform(H, beta):
    """The closed-form KB transform (both the sinh and the sin branch, kH <> beta) equals the
    quadrature of the truncated window; a slip in the sqrt(beta^2 - (kH)^2) argument fails this."""
    for kH in (0.0, 0.3 * beta, 0.99 * beta, beta, 1.01 * beta, 1.7 * beta, 3.3 * beta):
        k = kH / H
        ref = quad(lambda x: _kb(x, H, beta) * math.cos(k * x), -H, H, limit=400, epsabs=1e-15, epsrel=1e-13)[0]
        scale = quad(lambda x: _kb(x, H, beta), -H, H, limit=400)[0]
        assert abs(sog.kb_window_hat(k, H, beta) - ref) < 1e-11 * scale


def test_kb_polynomials_interpolate_the_window():
    """R6-KB: the degree-nu polynomial of stencil point j equals W_KB(j - p - u) (h = 1, H = P/2) at the
    nu+1 first-kind Chebyshev points of u in [-1/2, 1/2] and approximates it between them to the
    plan's window accuracy; the stencil's W and dW agree with the window / finite differences."""
    for Pw, beta, nu, acc in ((7, 14.7, 10, 1e-6), (9, 18.9, 12, 1e-8), (15, 31.5, 18, 1e-13)):
        p = (Pw - 1) // 2
        C = sog.kb_stencil_polys(Pw, beta, nu)
        tn = np.cos((np.arange(nu + 1) + 0.5) * math.pi / (nu + 1))
        for j in range(Pw):
            exact = np.array([_kb(j - p - 0.5 * t, 0.5 * Pw, beta) for t in tn])
            assert np.allclose(npcheb.chebval(tn, C[j]), exact, rtol=0, atol=1e-14)
            tt = np.linspace(-1, 1, 101)
            exact = np.array([_kb(j - p - 0.5 * t, 0.5 * Pw, beta) for t in tt])
            assert np.max(np.abs(npcheb.chebval(tt, C[j]) - exact)) < acc
    # stencil(): weights against the window at the particle offsets; derivative by differences
    h, I, Pw, beta, nu = 0.5, 20, 9, 18.9, 14
    x = np.array([-4.9, -0.01, 0.0, 0.26, 1.13, 4.99])
    g, W, dW = sog.stencil(x, I, h, Pw, beta, True, "kb", nu)
    g0 = np.floor(x / h + I / 2 + 0.5).astype(int)
    d = (g0[:, None] + np.arange(-4, 5)[None, :] - I / 2) * h - x[:, None]
    ref = np.array([[_kb(v, 4.5 * h, beta) for v in row] for row in d])
    assert np.max(np.abs(W - ref)) < 1e-9
    e = 1e-6
    Wp = sog.stencil(x + e, I, h, Pw, beta, True, "kb", nu)[1]
    Wm = sog.stencil(x - e, I, h, Pw, beta, True, "kb", nu)[1]
    assert np.allclose((Wp - Wm) / (2 * e), dW, atol=1e-7)


def test_kb_plan_rule():
    """R6-KB: P = smallest odd >= 5 with 10^(0.4 - 0.92 P) <= eps_w, beta = 2.2 P, nu = P + 3, and
    the mesh at the Nyquist bound; support below the Gaussian's at every tolerance (Fig. 5(a))."""
    for tol in (1e-4, 1e-6, 1e-8, 1e-10, 1e-12):
        g = P.make_plan(1000, 10.0, 10.0, 10.0, tol)
        k = P.make_plan(1000, 10.0, 10.0, 10.0, tol, window="kb")
        assert k.window == "kb" and k.P % 2 == 1 and k.P >= 5
        assert k.S == pytest.approx(2.2 * k.P) and k.nu == k.P + 3 and k.nul == k.Pl + 3
        assert k.P <= g.P and k.Pl <= g.Pl
        assert k.P < g.P or tol >= 1e-4


def test_kb_beats_gaussian_at_equal_support():
    """Fig. 5(a): at equal support P and grid, with S = 0.455 pi P (Gaussian) and
    beta = 2.5 P, nu = 10 (KB), the KB window's mid-range error is the smaller one."""
    xyz, q, L = config_system("c1", N=200)
    t = np.arange(10)
    base = P.make_plan(len(q), *L, 1e-10)
    x = sog.canonicalize(xyz, base)
    ex = sog_exact.mid_exact(base, x, q, t)[0]
    for Pw in (5, 7, 9):
        g = P.make_plan(len(q), *L, 1e-10, P=Pw, S=0.455 * math.pi * Pw)
        k = P.make_plan(len(q), *L, 1e-10, window="kb", P=Pw, S=2.5 * Pw, nu=10)
        assert (g.Ix, g.Iy, g.Izs) == (k.Ix, k.Iy, k.Izs)
        eg = np.max(np.abs(sog.mid_range(g, x, q, t)[0] - ex))
        ek = np.max(np.abs(sog.mid_range(k, x, q, t)[0] - ex))
        assert ek < eg


@pytest.mark.parametrize("tol", [1e-4, 1e-6, 1e-8, 1e-10, 1e-12])
def test_kb_mid_long_converge_to_exact(tol):
    """Algorithms 1 and 2 with the KB window -> the SOG-exact mid and long sums within the plan's
    tolerance (the error estimate is expected to follow Thms 4.2/4.3)."""
    xyz, q, L = config_system("c1", N=300)
    t = np.arange(12)
    p = P.make_plan(len(q), *L, tol, window="kb")
    x = sog.canonicalize(xyz, p)
    for spec, exact in ((sog.mid_range, sog_exact.mid_exact), (sog.long_range, sog_exact.long_exact)):
        sp, ex = spec(p, x, q, t), exact(p, x, q, t)
        assert np.max(np.abs(sp[0] - ex[0])) < 10 * tol
        assert np.max(np.abs(sp[1] - ex[1])) < 100 * tol


@pytest.mark.parametrize("name,N,tol", [("c1", 1000, 1e-6), ("c2", 1500, 1e-8), ("c4", 3000, 1e-6)])
def test_kb_total_vs_ewald2d(name, N, tol):
    """epsilon_r <= tol with the KB window; forces relative L2 <= 10 tol."""
    xyz, q, L = config_system(name, N=N)
    t = np.arange(24)
    p = P.make_plan(len(q), *L, tol, window="kb")
    phi, F = sog.evaluate(p, xyz, q, targets=t)
    ref, g = ewald2d.ewald2d(xyz, q, L, targets=t)
    Fref = -q[t, None] * g
    assert np.max(np.abs(phi - ref)) / np.max(np.abs(ref)) < tol
    assert np.linalg.norm(F - Fref) / np.linalg.norm(Fref) < 10 * tol


# ------------------------------------------------------------------ ES window (R6-ES)
def _es(x, H, beta):
    return math.exp(beta * (math.sqrt(1.0 - (x / H) ** 2) - 1.0)) if abs(x) <= H else 0.0


@pytest.mark.parametrize("H,beta", [(2.5, 11.5), (4.5, 20.7), (7.5, 34.5)])
def test_es_window_fourier_transform(H, beta):
    """The oracle's ES transform (quadrature in theta, x = H sin theta) equals the direct x-integral
    of the window written out independently."""
    for kH in (0.0, 0.5, 2.0, 0.5 * math.pi * 2 * H, 1.3 * beta):
        k = kH / H
        ref = quad(lambda x: _es(x, H, beta) * math.cos(k * x), -H, H, limit=800, epsabs=1e-15, epsrel=1e-12)[0]
        scale = quad(lambda x: _es(x, H, beta), -H, H, limit=800)[0]
        assert abs(sog.es_window_hat(k, H, beta) - ref) < 1e-10 * scale


def test_es_polynomials_interpolate_the_window():
    for Pw, nu, acc in ((7, 10, 1e-6), (11, 14, 1e-9), (15, 18, 1e-12)):
        beta = 2.3 * Pw
        p = (Pw - 1) // 2
        C = sog.kb_stencil_polys(Pw, beta, nu, "es")
        tt = np.linspace(-1, 1, 101)
        for j in range(Pw):
            exact = np.array([_es(j - p - 0.5 * t, 0.5 * Pw, beta) for t in tt])
            assert np.max(np.abs(npcheb.chebval(tt, C[j]) - exact)) < acc


@pytest.mark.parametrize("tol", [1e-4, 1e-8, 1e-12])
def test_es_mid_long_converge_to_exact(tol):
    xyz, q, L = config_system("c1", N=300)
    t = np.arange(12)
    p = P.make_plan(len(q), *L, tol, window="es")
    assert p.S == pytest.approx(2.3 * p.P)
    x = sog.canonicalize(xyz, p)
    for spec, exact in ((sog.mid_range, sog_exact.mid_exact), (sog.long_range, sog_exact.long_exact)):
        sp, ex = spec(p, x, q, t), exact(p, x, q, t)
        assert np.max(np.abs(sp[0] - ex[0])) < 10 * tol
        assert np.max(np.abs(sp[1] - ex[1])) < 100 * tol


def test_es_total_vs_ewald2d():
    xyz, q, L = config_system("c1", N=1000)
    t = np.arange(24)
    p = P.make_plan(len(q), *L, 1e-6, window="es")
    phi, F = sog.evaluate(p, xyz, q, targets=t)
    ref, g = ewald2d.ewald2d(xyz, q, L, targets=t)
    assert np.max(np.abs(phi - ref)) / np.max(np.abs(ref)) < 1e-6
    assert np.linalg.norm(F + q[t, None] * g) / np.linalg.norm(q[t, None] * g) < 1e-5
