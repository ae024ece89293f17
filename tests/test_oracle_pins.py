"""Pins of the CPU oracle against the paper and the mathematics (not against itself).

Each test names the passage it pins.  These run without a GPU.
"""
import math

import numpy as np
import pytest
from scipy.integrate import quad
from scipy.special import factorial

from oracle import plan as P
from oracle import sog, sog_exact, ewald2d
from synth import uniform_system, config_system


# ------------------------------------------------------------------ SOG decomposition
def F1(b, omega, r, M=None):
    """F_b^1(r) with sigma = 1 and M -> infinity (Table 1's rows are the M->inf solution)."""
    M = M or int(60 / math.log10(b))          # s_M ~ 1e60: the tail is below rounding
    w, s = P.sog_nodes_weights(b, 1.0, omega, M)
    e = np.exp(-(r / s) ** 2)
    return float(np.sum(w * e)), float(np.sum(w * e * (-2.0 * r / s ** 2)))


def test_table1_rows_solve_c0_c1(golden):
    """Table 1: r0 F(r0) = 1 and r0^2 F'(r0) = -1 (Eqs. 2.20, 2.22 via eq::2.35z).
    A wrong weight (missing log b, omega on the wrong term, sqrt(2) slip) fails this."""
    for b, r0, om, *_ in golden("table1.txt"):
        F, dF = F1(b, om, r0)
        assert abs(r0 * F - 1.0) < 2e-14
        assert abs(r0 * r0 * dF + 1.0) < 3e-14


def test_weight_closed_forms():
    """w_0(b=2, sigma=1, omega=1) = sqrt(2/pi) ln 2 = 0.55305143373... (SPEC S:111 quotes
    0.5530843701, whose 5th digit is wrong: 0.7978845608 x 0.6931471806 = 0.5530514337)."""
    w, s = P.sog_nodes_weights(2.0, 1.0, 1.0, 5)
    assert abs(w[0] - 0.5530514337328164) < 1e-15
    assert abs(s[0] - math.sqrt(2.0)) < 1e-15
    w, s = P.sog_nodes_weights(1.3, 0.7, 1.01, 30)
    assert np.allclose(s[1:] / s[:-1], 1.3, rtol=1e-15)
    assert np.allclose(w[2:] / w[1:-1], 1 / 1.3, rtol=1e-15)
    assert abs(w[0] / w[1] - 1.01 * 1.3) < 1e-14          # omega on w_0 only


def test_bsa_pointwise_error_bound(golden):
    """Eq. eq::pointwiseerror: |1 - r F(r)| <~ 2 sqrt2 exp(-pi^2/(2 ln b)) for s_0 << r << s_M.
    The maximum over r must sit at the bound (0.3x..1.2x): a wrong exponent or base fails."""
    for b, r0, om, *_ in golden("table1.txt")[:5]:
        bound = 2 * math.sqrt(2) * math.exp(-math.pi ** 2 / (2 * math.log(b)))
        Mb = int(30 / math.log10(b))
        w, s = P.sog_nodes_weights(b, 1.0, 1.0, Mb)
        # include l<0 terms so the series is bilateral (Eq. BSA)
        ell = np.arange(1, Mb + 1)
        wneg = (math.pi / 2) ** -0.5 * b ** ell * math.log(b)
        sneg = math.sqrt(2) * b ** (-ell)
        r = np.geomspace(10.0, 1e4, 400)
        Fr = (np.exp(-(r[:, None] / s) ** 2) * w).sum(1) + (np.exp(-(r[:, None] / sneg) ** 2) * wneg).sum(1)
        err = np.max(np.abs(1 - r * Fr))
        assert 0.3 * bound < err < 1.2 * bound, (b, err, bound)


def test_near_kernel_c0_c1_and_identity():
    """N(r_c) = 0, N'(r_c) = 0 (C0/C1) for any sigma; N + F = 1/r inside r_c."""
    for tol in (1e-4, 1e-6, 1e-8, 1e-12):
        p = P.make_plan(1000, 10.0, 10.0, 10.0, tol)
        rc = p.rc
        N, dN = sog.near_kernel(p, np.array([rc * (1 - 1e-15)]))
        # with finite M the residual at r_c is exactly the omitted tail sum_{l>M} w_l e^{-rc^2/s_l^2}
        wt, st = P.sog_nodes_weights(p.b, p.sigma, p.omega, p.M + 400)
        tail = np.sum((wt * np.exp(-(rc / st) ** 2))[p.M + 1:])
        dtail = np.sum((wt * np.exp(-(rc / st) ** 2) * (-2 * rc / st ** 2))[p.M + 1:])
        assert abs(N[0] - tail) < 1e-13 / p.sigma and abs(dN[0] - dtail) < 1e-13 / p.sigma ** 2
        r = np.linspace(0.05, rc * 0.999, 50)
        N, _ = sog.near_kernel(p, r)
        w, s = p.weights()
        F = (w * np.exp(-(r[:, None] / s) ** 2)).sum(1)
        assert np.allclose(N + F, 1 / r, rtol=1e-14, atol=0)
        assert np.all(sog.near_kernel(p, np.array([rc, 2 * rc]))[0] == 0.0)
        assert abs(sog.self_coefficient(p) - w.sum()) == 0.0


# ------------------------------------------------------------------ Chebyshev
def test_theorem_3_1_values(golden):
    """Thm 3.1 bound 1/(sqrt(P!) (2 sqrt2 eta)^P) gives the digits quoted at P:422, and the
    actual interpolation error of exp(-z^2/s^2), s = eta Lz, is within 1.1x the bound."""
    for eta, Pn, digits in golden("thm31.txt"):
        Pn = int(Pn)
        bound = 1.0 / (math.sqrt(factorial(Pn)) * (2 * math.sqrt(2) * eta) ** Pn)
        assert 10 ** (-digits - 1) < bound < 10 ** (-digits + 1)
    # eta = 1, P = 6: measured error sits at the bound (7.42e-5 vs 7.28e-5)
    Lz, s, Pn = 2.0, 2.0, 6
    za = cheb_z = 0.5 * Lz * P.cheb_nodes(Pn)
    xt = np.linspace(-1, 1, 2001)
    approx = P.lagrange_matrix(xt, Pn) @ np.exp(-(cheb_z / s) ** 2)
    err = np.max(np.abs(approx - np.exp(-(0.5 * Lz * xt / s) ** 2)))
    bound = 1.0 / (math.sqrt(factorial(Pn)) * (2 * math.sqrt(2) * 1.0) ** Pn)
    assert 0.9 * bound < err < 1.1 * bound


def test_chebyshev_basis_identities():
    """Nodes x_i = cos((i-1/2) pi/P); L(x) = T(x) V^-1: L_a(x_b) = delta_ab,
    sum_a L_a = 1, exact on polynomials of degree < P; dL/dz matches finite differences."""
    for Pn in (2, 5, 16, 28):
        x = P.cheb_nodes(Pn)
        assert np.all(np.diff(x) < 0)
        Lm = P.lagrange_matrix(x, Pn)
        assert np.allclose(Lm, np.eye(Pn), atol=1e-12)
        xt = np.linspace(-1, 1, 37)
        Lt = P.lagrange_matrix(xt, Pn)
        assert np.allclose(Lt.sum(1), 1.0, atol=1e-12)
        poly = lambda t: 0.3 - t + 2 * t ** (Pn - 1)
        assert np.allclose(Lt @ poly(x), poly(xt), atol=1e-11)
    p = P.make_plan(1000, 10.0, 10.0, 10.0, 1e-6)
    z = np.linspace(-4.9, 4.9, 11)
    La, dLa = sog.long_basis(p, z)
    d = 1e-6
    fd = (sog.long_basis(p, z + d)[0] - sog.long_basis(p, z - d)[0]) / (2 * d)
    assert np.allclose(dLa, fd, atol=1e-7)


# ------------------------------------------------------------------ windows
def test_gaussian_window_fourier_transform(golden):
    """W_hat of Eq. eq::GS equals the quadrature of the (untruncated) Gaussian window."""
    for S, H, k in golden("window_gauss.txt"):
        val = quad(lambda x: math.exp(-S * (x / H) ** 2) * math.cos(k * x), -np.inf, np.inf)[0]
        assert abs(sog.gaussian_window_hat(k, H, S) - val) < 1e-12


def test_stencil_geometry():
    """R6 stencil: P consecutive points centred at the nearest grid point of x_g=(g-I/2)h."""
    x = np.array([-5.0, -0.01, 0.0, 0.26, 4.99])
    g, W, dW = sog.stencil(x, 20, 0.5, 5, 8.0, True)
    g0 = np.rint(x / 0.5 + 10).astype(int)
    assert np.all(g[:, 2] == g0 % 20)
    xg = (g0 - 10) * 0.5
    d = xg - x
    H = 1.0
    assert np.allclose(W[:, 2], np.exp(-8.0 * (d / H) ** 2))
    # derivative of W(x_i - x_g) w.r.t. x_i by finite differences
    h = 1e-6
    Wp = sog.stencil(x + h, 20, 0.5, 5, 8.0, True)[1]
    Wm = sog.stencil(x - h, 20, 0.5, 5, 8.0, True)[1]
    ok = np.abs(((x + h) / 0.5 + 10.5) % 1 - 0.5) < 0.49      # away from stencil switch points
    assert np.allclose(((Wp - Wm) / (2 * h))[ok], dW[ok], atol=1e-7)


# ------------------------------------------------------------------ near sum
def test_near_cell_list_equals_brute_force():
    """Neighbour-searched near sum == O(N^2) min-image double loop."""
    xyz, q = uniform_system(600, (8.0, 9.0, 7.0), 11)
    p = P.make_plan(600, 8.0, 9.0, 7.0, 1e-6)
    x = sog.canonicalize(xyz, p)
    a = sog.near_field(p, x, q, brute_force=True)
    b = sog.near_field(p, x, q, brute_force=False)
    assert np.allclose(a[0], b[0], rtol=0, atol=1e-13)
    assert np.allclose(a[1], b[1], rtol=0, atol=1e-13)


def test_near_single_pair_closed_form():
    """Two charges +-1 at distance d < r_c straddling the x boundary: phi_1 = -N(d), grad by hand."""
    p = P.make_plan(2, 20.0, 20.0, 20.0, 1e-6, rc=3.0)
    xyz = np.array([[9.5, 0.0, 0.0], [-9.3, 0.4, -0.2]])     # min-image dx = -1.2
    q = np.array([1.0, -1.0])
    x = sog.canonicalize(xyz, p)
    phi, grad = sog.near_field(p, x, q, brute_force=True)
    dvec = np.array([-1.2, -0.4, 0.2])
    d = np.linalg.norm(dvec)
    w, s = p.weights()
    N = 1 / d - np.sum(w * np.exp(-(d / s) ** 2))
    dN = -1 / d ** 2 + np.sum(w * np.exp(-(d / s) ** 2) * 2 * d / s ** 2)
    assert abs(phi[0] - (-N)) < 1e-14 and abs(phi[1] - (+N)) < 1e-14
    assert np.allclose(grad[0], -dN * dvec / d, atol=1e-14)


# ------------------------------------------------------------------ Ewald2D (the oracle's own oracle)
def test_ewald2d_alpha_independence_and_force():
    """Ewald2D is independent of the splitting alpha (exactness of the textbook form);
    its gradient equals the finite difference of its potential field."""
    xyz, q = uniform_system(40, (3.0, 4.0, 2.0), 5)
    t = np.arange(6)
    a = ewald2d.ewald2d(xyz, q, (3.0, 4.0, 2.0), targets=t, alpha=0.8)
    b = ewald2d.ewald2d(xyz, q, (3.0, 4.0, 2.0), targets=t, alpha=2.0)
    assert np.allclose(a[0], b[0], rtol=0, atol=1e-13 * np.abs(a[0]).max())
    assert np.allclose(a[1], b[1], rtol=0, atol=1e-12 * np.abs(a[1]).max())
    # FD: move target 0 (its own images stay excluded only at n=0, so compare field of others)
    i = 0
    h = 1e-5
    for d in range(3):
        xp = xyz.copy(); xp[i, d] += h
        xm = xyz.copy(); xm[i, d] -= h
        # potential at r_i due to the others == phi_i  (self image terms also move, cancel in FD
        # only for the k-space/self parts; they are independent of r_i, so use full phi)
        pp = ewald2d.ewald2d(xp, q, (3.0, 4.0, 2.0), targets=[i], alpha=1.2)[0][0]
        pm = ewald2d.ewald2d(xm, q, (3.0, 4.0, 2.0), targets=[i], alpha=1.2)[0][0]
        # d phi_i / d x_i includes the (r_i-independent) self-image sum -> FD equals gradient
        assert abs((pp - pm) / (2 * h) - a[1][i, d]) < 1e-6


def test_ewald2d_dilute_limit_is_coulomb():
    """A neutral cluster of size ~1 in a 400x400 periodic cell: Ewald2D -> free-space Coulomb
    (image and sheet terms are O(a^2/L^3)); pins every Ewald2D term's sign and prefactor."""
    rng = np.random.default_rng(3)
    xyz = rng.random((8, 3)) - 0.5
    q = np.array([1, -1, 1, -1, 2, -2, 0.5, -0.5], dtype=float)
    L = (400.0, 400.0, 2.0)
    phi, grad = ewald2d.ewald2d(xyz, q, L, alpha=0.02)
    d = xyz[:, None, :] - xyz[None, :, :]
    r = np.linalg.norm(d, axis=-1)
    np.fill_diagonal(r, np.inf)
    coul = (q[None, :] / r).sum(1)
    gc = (-q[None, :, None] * d / r[..., None] ** 3).sum(1)
    assert np.allclose(phi, coul, atol=2e-6)
    assert np.allclose(grad, gc, atol=2e-6)


def test_ewald2d_c_loops_equal_numpy():
    """The C-loop Ewald2D used at full BASELINE sizes (ewald2d_targets) is the same sum as the pinned
    NumPy ewald2d: equal at small N for two alphas, and alpha-independent on a c5-shaped box."""
    L = (6.0, 7.0, 5.0)
    xyz, q = uniform_system(300, L, 3)
    t = np.arange(0, 300, 7)
    p0, g0 = ewald2d.ewald2d(xyz, q, L, targets=t)
    for alpha in (None, 0.3, 1.1):
        p1, g1 = ewald2d.ewald2d_targets(xyz, q, L, t, tol=1e-16, alpha=alpha)
        assert np.abs(p1 - p0).max() <= 2e-14 * np.abs(p0).max()
        assert np.abs(g1 - g0).max() <= 2e-14 * np.abs(g0).max()
    xyz, q, L = config_system("c5", N=20000)
    t = np.arange(5) * 101
    a = ewald2d.ewald2d_targets(xyz, q, L, t, tol=1e-13, alpha=0.05)
    b = ewald2d.ewald2d_targets(xyz, q, L, t, tol=1e-13, alpha=0.12)
    assert np.abs(a[0] - b[0]).max() <= 1e-11 * np.abs(a[0]).max()
    assert np.abs(a[1] - b[1]).max() <= 1e-11 * np.abs(a[1]).max()


def test_mid_spread_loops_equals_add_at():
    """The C-loop gridding used at full BASELINE sizes (mid_spread_loops) is the sum of
    mid_spread (np.add.at): equal to rounding at c1 and on a c5-shaped box, every window."""
    for name, N, window in (("c1", 1000, "gs"), ("c5", 6000, "gs"), ("c1", 1000, "kb"), ("c4", 3000, "es")):
        xyz, q, L = config_system(name, N=N)
        p = P.make_plan(len(q), *L, 1e-6, window=window)
        x = sog.canonicalize(xyz, p)
        a = sog.mid_spread(p, x, q)
        b = sog.mid_spread_loops(p, x, q)
        assert a.shape == b.shape
        assert np.abs(a - b).max() <= 1e-14 * np.abs(a).max(), (name, window)


def test_long_spread_dense_equals_add_at():
    """The dense-row long anterpolation used at full BASELINE sizes (long_spread_dense) is the sum
    of long_spread (np.add.at), every window."""
    for name, N, window in (("c1", 1000, "gs"), ("c5", 6000, "gs"), ("c5", 6000, "kb"), ("c4", 3000, "es")):
        xyz, q, L = config_system(name, N=N)
        p = P.make_plan(len(q), *L, 1e-6, window=window)
        x = sog.canonicalize(xyz, p)
        a = sog.long_spread(p, x, q)
        b = sog.long_spread_dense(p, x, q, chunk=1777)
        assert np.abs(a - b).max() <= 1e-14 * np.abs(a).max(), (name, window)


def test_c1_solve_reproduces_table1_simple_roots():
    """NEXT #4: the general-b C^1 solve returns Table 1's printed (r0, omega) for the rows
    whose r0 is a simple root (b = 2 and b = 1.4878...; rows 2, 4, 5 are tangential roots of the
    system, which a sign-change solve does not bracket), each at that row's force error as tol."""
    for k in (0, 2):
        b, r0, om, _, _, ferr, _ = P.TABLE1[k]
        r, w = P.c1_solve(b, ferr)
        assert abs(r - r0) <= 1e-11 * r0, (k, r, r0)
        assert abs(w - om) <= 1e-12, (k, w, om)


def test_c1_solve_general_b_satisfies_the_continuity_system():
    """For a non-table b (Table 4's 1.17; and 1.25, 1.4) the solved (r0, omega) make the SOG
    sum C^0 and C^1 at r_c: r0 F(r0) = 1 and r0^2 F'(r0) = -1 with M -> infinity, evaluated
    by plain summation of the sog_nodes_weights Gaussians (sigma = 1) in double precision."""
    for b, tol in ((1.17, 1e-12), (1.25, 1e-8), (1.4, 1e-5)):
        r0, om = P.c1_solve(b, tol)
        w, s = P.sog_nodes_weights(b, 1.0, om, int(60.0 / math.log(b)))
        F = float(np.sum(w * np.exp(-(r0 / s) ** 2)))
        dF = float(np.sum(w * np.exp(-(r0 / s) ** 2) * (-2.0 * r0 / s ** 2)))
        assert abs(r0 * F - 1.0) < 5e-15 and abs(r0 * r0 * dF + 1.0) < 5e-14, (b, r0 * F - 1, r0 * r0 * dF + 1)
        assert r0 > 1.0 and abs(om - 1.0) < 0.05


def test_general_b_total_vs_ewald2d():
    """A Table-4-like plan with the general b = 1.17 at tol 1e-12 reaches tol vs Ewald2D."""
    xyz, q, L = config_system("c1", N=400)
    p = P.make_plan(len(q), *L, 1e-12, b=1.17)
    assert p.b == 1.17
    t = np.arange(16)
    phi, F = sog.evaluate(p, xyz, q, targets=t)
    ref, g = ewald2d.ewald2d(xyz, q, L, targets=t)
    assert np.max(np.abs(phi - ref)) / np.max(np.abs(ref)) < 1e-12
    assert np.linalg.norm(F + q[t, None] * g) / np.linalg.norm(q[t, None] * g) < 1e-11


# ------------------------------------------------------------------ spectral components vs SOG-exact
@pytest.fixture(scope="module")
def small_system():
    xyz, q, L = config_system("c1", N=400)
    return xyz, q, L


def test_sog_exact_vs_ewald_decomposition_error(small_system):
    """SOG-exact (near + mid + long image sums - self) vs Ewald2D isolates the decomposition error:
    below tol with Table 1 rows b_4, b_5, b_6 and R3 M."""
    xyz, q, L = small_system
    t = np.arange(12)
    ref = ewald2d.ewald2d(xyz, q, L, targets=t)[0]
    for tol, bound in ((1e-6, 1e-6), (1e-8, 1e-8), (1e-12, 1e-12)):
        p = P.make_plan(len(q), *L, tol)
        x = sog.canonicalize(xyz, p)
        ex = sog_exact.sog_exact(p, x, q, t)[0]
        assert np.max(np.abs(ex - ref)) / np.max(np.abs(ref)) < bound


def test_mid_spectral_converges_to_exact(small_system):
    """Algorithm 1 output -> the SOG-exact mid sum; error within the plan's tolerance and
    decreasing with the window support / grid (Thms 4.1-4.3)."""
    xyz, q, L = small_system
    t = np.arange(12)
    errs = []
    for tol in (1e-4, 1e-7, 1e-10):
        p = P.make_plan(len(q), *L, tol)
        x = sog.canonicalize(xyz, p)
        ex = sog_exact.mid_exact(p, x, q, t)
        sp = sog.mid_range(p, x, q, t)
        e = np.max(np.abs(sp[0] - ex[0]))
        errs.append(e)
        assert e < 10 * tol
        assert np.max(np.abs(sp[1] - ex[1])) < 100 * tol
    assert errs[0] > errs[1] > errs[2]


def test_long_spectral_converges_to_exact(small_system):
    """Algorithm 2 (two-sided proxies, R9/R10) -> the SOG-exact long sum (Eq. eq::trun2)."""
    xyz, q, L = small_system
    t = np.arange(12)
    for tol in (1e-4, 1e-7, 1e-10, 1e-12):
        p = P.make_plan(len(q), *L, tol)
        x = sog.canonicalize(xyz, p)
        ex = sog_exact.long_exact(p, x, q, t)
        sp = sog.long_range(p, x, q, t)
        assert np.max(np.abs(sp[0] - ex[0])) < 10 * tol
        assert np.max(np.abs(sp[1] - ex[1])) < 100 * tol


def test_long_chebyshev_rate():
    """Fig. 4(b) with R19: the long error falls like C^-P / sqrt(P!), C = 2 sqrt2 s_{m+1}/L_z;
    the measured ratio err(16)/err(6) must match the predicted ratio within 3x."""
    xyz, q, L = config_system("c1", N=200)
    t = np.arange(6)
    p = P.make_plan(len(q), *L, 1e-12)
    x = sog.canonicalize(xyz, p)
    ex = sog_exact.long_exact(p, x, q, t)[0]
    import dataclasses
    e6 = np.max(np.abs(sog.long_range(dataclasses.replace(p, Pc=6), x, q, t)[0] - ex))
    e16 = np.max(np.abs(sog.long_range(dataclasses.replace(p, Pc=16), x, q, t)[0] - ex))
    C = 2 * math.sqrt(2) * p.sigma * math.sqrt(2) * p.b ** (p.m + 1) / p.Lz
    pred = C ** -10 * math.sqrt(factorial(6) / factorial(16))
    assert pred / 3 < e16 / e6 < 3 * pred


# ------------------------------------------------------------------ total vs Ewald2D
@pytest.mark.parametrize("name,N,tol", [("c1", 1000, 1e-6), ("c1", 1000, 1e-4), ("c2", 1500, 1e-8),
                                        ("c3", 3000, 1e-6), ("c4", 3000, 1e-6)])
def test_total_vs_ewald2d(name, N, tol):
    """epsilon_r = relative L-inf potential error vs Ewald2D <= tol, target-subsampled
    (forces: relative L2 <= 10 tol)."""
    xyz, q, L = config_system(name, N=N)
    t = np.arange(24)
    p = P.make_plan(len(q), *L, tol)
    phi, F = sog.evaluate(p, xyz, q, targets=t)
    ref, g = ewald2d.ewald2d(xyz, q, L, targets=t)
    Fref = -q[t, None] * g
    assert np.max(np.abs(phi - ref)) / np.max(np.abs(ref)) < tol
    assert np.linalg.norm(F - Fref) / np.linalg.norm(Fref) < 10 * tol


# ------------------------------------------------------------------ symmetries / invariants
@pytest.fixture(scope="module")
def sym_case():
    xyz, q = uniform_system(300, (8.0, 8.0, 6.0), 21)
    p = P.make_plan(300, 8.0, 8.0, 6.0, 1e-8)
    phi, F = sog.evaluate(p, xyz, q)
    return xyz, q, p, phi, F


def test_invariance_period_and_permutation(sym_case):
    xyz, q, p, phi, F = sym_case
    s = xyz.copy(); s[:, 0] += 8.0; s[:, 1] -= 16.0
    phi2, F2 = sog.evaluate(p, s, q)
    assert np.allclose(phi2, phi, atol=1e-13 * np.abs(phi).max(), rtol=0)
    perm = np.random.default_rng(0).permutation(len(q))
    phi3, F3 = sog.evaluate(p, xyz[perm], q[perm])
    assert np.allclose(phi3, phi[perm], atol=1e-13 * np.abs(phi).max(), rtol=0)
    phi4, F4 = sog.evaluate(p, xyz, 2.5 * q)
    assert np.allclose(phi4, 2.5 * phi, atol=1e-13 * np.abs(phi).max(), rtol=0)


def test_reflection_symmetry(sym_case):
    """Grids and Chebyshev nodes are symmetric: z -> -z leaves phi invariant and flips F_z."""
    xyz, q, p, phi, F = sym_case
    r = xyz.copy(); r[:, 2] *= -1
    phi2, F2 = sog.evaluate(p, r, q)
    assert np.allclose(phi2, phi, atol=1e-12 * np.abs(phi).max(), rtol=0)
    assert np.allclose(F2[:, 2], -F[:, 2], atol=1e-11 * np.abs(F).max(), rtol=0)
    assert np.allclose(F2[:, :2], F[:, :2], atol=1e-11 * np.abs(F).max(), rtol=0)


def test_translation_and_total_force(sym_case):
    """Arbitrary x/y translation changes U by <= tol (north_star); sum_i F_i ~ 0 (neutral)."""
    xyz, q, p, phi, F = sym_case
    U = sog.energy(q, phi)
    s = xyz.copy(); s[:, 0] += 0.3171; s[:, 1] += 1.234
    U2 = sog.energy(q, sog.evaluate(p, s, q)[0])
    assert abs(U2 - U) < 10 * p.tol * abs(U)
    assert np.linalg.norm(F.sum(0)) < 10 * p.tol * np.abs(F).max() * math.sqrt(len(q))


def test_forces_are_gradient_of_discrete_energy():
    """R11: spread/gather are adjoint and mult, K symmetric, so F_i = -dU/dr_i exactly for the
    discrete scheme (central difference, away from stencil switch points)."""
    xyz, q = uniform_system(60, (7.0, 7.0, 5.0), 31)
    p = P.make_plan(60, 7.0, 7.0, 5.0, 1e-8)
    phi, F = sog.evaluate(p, xyz, q)
    i, h = 3, 1e-6
    for d in range(3):
        xp = xyz.copy(); xp[i, d] += h
        xm = xyz.copy(); xm[i, d] -= h
        Up = sog.energy(q, sog.evaluate(p, xp, q)[0])
        Um = sog.energy(q, sog.evaluate(p, xm, q)[0])
        assert abs(-(Up - Um) / (2 * h) - F[i, d]) < 1e-7 * max(1.0, abs(F[i, d]))


def test_validation_errors():
    p = P.make_plan(4, 5.0, 5.0, 5.0, 1e-6)
    with pytest.raises(ValueError):
        sog.canonicalize(np.array([[0, 0, 2.6]]), p)
    with pytest.raises(ValueError):
        sog.canonicalize(np.array([[np.nan, 0, 0]]), p)
    with pytest.raises(ValueError):
        sog.evaluate(p, np.zeros((2, 3)) + [[0, 0, 0], [1, 1, 1]], np.array([1.0, 0.5]))
    with pytest.raises(ValueError):
        P.make_plan(10, 5.0, 5.0, 5.0, 1e-15)
    x = sog.canonicalize(np.array([[3.0, -2.6, 0.1], [-2.5, 2.5, 2.5]]), p)
    assert np.allclose(x, [[-2.0, 2.4, 0.1], [-2.5, -2.5, 2.5]])


# ------------------------------------------------------------------ App. C Taylor form (NEXT #3)
def test_taylor_variant_kernel_within_lagrange_bound():
    """App. C: sum_p A_p(kdot) ((z_a - z_b)/L_z)^{2p} -> K_ab(kdot) (the two-sided
    kernel, R9/R10) with the Lagrange remainder of Lemma lemma::Taylor (Eq. eq::Taylor2) over
    z_a - z_b in [-L_z, L_z] (R23)."""
    p = P.make_plan(300, 20.0, 20.0, 4.0, 1e-10)
    assert p.m >= 0
    K = sog.long_kernel(p)
    za = 0.5 * p.Lz * P.cheb_nodes(p.Pc)
    d = (za[:, None] - za[None, :]) / p.Lz
    errs = []
    for Q in (16, 24, 32, 40):
        A = sog.long_coeff_taylor(p, Q)
        KT = sum(A[k][None, None] * (d ** (2 * k))[:, :, None, None] for k in range(Q))
        err = np.max(np.abs(KT - K)) / np.max(np.abs(K))
        assert err <= sog.taylor_bound(p, Q)
        errs.append(err)
    assert errs[-1] < 1e-9 and errs[0] > 1e3 * errs[-1]         # converging, not constant


def test_taylor_variant_converges_to_exact(small_system):
    """App. C's one-sided Taylor form of Alg. 2 -> the SOG-exact long sum (Eq. eq::trun2);
    with a Q whose Lagrange bound is below tol the error is that of the plan."""
    xyz, q, L = small_system
    t = np.arange(12)
    for tol in (1e-6, 1e-10):
        p = P.make_plan(len(q), *L, tol)
        x = sog.canonicalize(xyz, p)
        ex = sog_exact.long_exact(p, x, q, t)
        Q = next(k for k in range(1, 200) if sog.taylor_bound(p, k) < 0.01 * tol)
        phi, grad = sog.long_range_taylor(p, x, q, Q, t)
        assert np.max(np.abs(phi - ex[0])) < 10 * tol
        assert np.max(np.abs(grad - ex[1])) < 100 * tol
        # too few terms: the truncation shows (the bound is not vacuous here)
        phi2, _ = sog.long_range_taylor(p, x, q, max(1, Q // 4), t)
        assert np.max(np.abs(phi2 - ex[0])) > 100 * tol
