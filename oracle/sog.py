"""Step-by-step spectral SOG evaluation (the oracle).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Plain NumPy/SciPy, fp64,
no blocking or fusion: each function follows one passage of PAPER.md in the
paper's order and notation, on the plan's scalar parameters (oracle/plan.py).

    phi_i = Phi^N_i + Phi^mid_i + Phi^long_i - Phi^self_i
    F_i   = -q_i grad phi(r_i)
    U     = 1/2 sum_i q_i phi_i

Readings used: R6 stencil, R7 padding, R9 two-sided proxies,
R10 expm1 at kdot=0, R11 analytic gather gradient, R12 normalisations,
R14 coordinates.  Every function here is pinned by tests/test_oracle_*.py.
"""
from __future__ import annotations

import functools
import math

import numpy as np
import scipy.fft
import scipy.special
from numpy.polynomial import chebyshev as npcheb
from scipy.spatial import cKDTree

from .plan import Plan, cheb_T, cheb_nodes

_WORKERS = -1  # scipy.fft: all host cores


# ----------------------------------------------------------------------------- geometry
def canonicalize(xyz: np.ndarray, plan: Plan) -> np.ndarray:
    """R14: wrap x,y into [-L/2, L/2) (P:106-117 periodic in x,y); z must lie in the
    closed interval [-Lz/2, Lz/2] (free direction), else ValueError."""
    xyz = np.array(xyz, dtype=np.float64, copy=True)
    if not np.all(np.isfinite(xyz)):
        raise ValueError("non-finite position")
    for d, L in ((0, plan.Lx), (1, plan.Ly)):
        xyz[:, d] = xyz[:, d] - L * np.floor((xyz[:, d] + 0.5 * L) / L)
        xyz[:, d] = np.where(xyz[:, d] >= 0.5 * L, xyz[:, d] - L, xyz[:, d])
    if np.any(np.abs(xyz[:, 2]) > 0.5 * plan.Lz):
        raise ValueError("z outside [-Lz/2, Lz/2]")
    return xyz


def min_image(d: np.ndarray, L: float) -> np.ndarray:
    """Minimum-image displacement in a periodic direction (Assumption 1)."""
    return d - L * np.round(d / L)


# ----------------------------------------------------------------------------- near field
def near_kernel(plan: Plan, r: np.ndarray):
    """N(r) = 1/r - F(r), F(r) = sum_{l=0}^{M} w_l exp(-r^2/s_l^2), for r < r_c, else 0
    (Eqs. eq::SOGDEcomp, eq::SOGField); returns (N, dN/dr).  Exact sum."""
    w, s = plan.weights()
    r = np.asarray(r, dtype=np.float64)
    e = np.exp(-(r[..., None] / s) ** 2) * w
    F = e.sum(-1)
    dF = (e * (-2.0 * r[..., None] / s ** 2)).sum(-1)
    inside = r < plan.rc
    N = np.where(inside, 1.0 / r - F, 0.0)
    dN = np.where(inside, -1.0 / r ** 2 - dF, 0.0)
    return N, dN


def _near_pairs_accumulate(plan, xyz, q, ti, sj, out_phi, out_grad, out_rows):
    dx = min_image(xyz[ti, 0] - xyz[sj, 0], plan.Lx)
    dy = min_image(xyz[ti, 1] - xyz[sj, 1], plan.Ly)
    dz = xyz[ti, 2] - xyz[sj, 2]                       # z never wrapped (free)
    r = np.sqrt(dx * dx + dy * dy + dz * dz)
    keep = (r < plan.rc) & (r > 0.0)
    ti, sj, dx, dy, dz, r = ti[keep], sj[keep], dx[keep], dy[keep], dz[keep], r[keep]
    N, dN = near_kernel(plan, r)
    rows = out_rows[ti]
    np.add.at(out_phi, rows, q[sj] * N)
    g = q[sj] * dN / r
    np.add.at(out_grad, (rows, 0), g * dx)
    np.add.at(out_grad, (rows, 1), g * dy)
    np.add.at(out_grad, (rows, 2), g * dz)


def near_field(plan: Plan, xyz, q, targets=None, brute_force=None):
    """Phi^N_i = sum'_n sum_j q_j N(|r_ij + n L|) (Eq. eq::phiNDR) and its
    gradient; only r < r_c <= min(Lx,Ly)/2 contributes, i.e. the minimum image
    (P:264 cell list).  Candidate pairs come from a periodic k-d tree (library
    neighbour search) or, for brute_force=True, the O(N^2) double loop."""
    N = len(q)
    tgt = np.arange(N) if targets is None else np.asarray(targets)
    rows = np.full(N, -1, dtype=np.int64)
    rows[tgt] = np.arange(len(tgt))
    phi = np.zeros(len(tgt))
    grad = np.zeros((len(tgt), 3))
    if brute_force is None:
        brute_force = N * len(tgt) <= 4_000_000
    if brute_force:
        chunk = max(1, 2_000_000 // N)
        for c0 in range(0, len(tgt), chunk):
            t = tgt[c0:c0 + chunk]
            ti = np.repeat(t, N)
            sj = np.tile(np.arange(N), len(t))
            _near_pairs_accumulate(plan, xyz, q, ti, sj, phi, grad, rows)
        return phi, grad
    pos = np.empty_like(xyz)
    pos[:, 0] = np.mod(xyz[:, 0] + 0.5 * plan.Lx, plan.Lx)
    pos[:, 1] = np.mod(xyz[:, 1] + 0.5 * plan.Ly, plan.Ly)
    pos[:, 0] = np.where(pos[:, 0] >= plan.Lx, 0.0, pos[:, 0])
    pos[:, 1] = np.where(pos[:, 1] >= plan.Ly, 0.0, pos[:, 1])
    pos[:, 2] = xyz[:, 2] + 0.5 * plan.Lz
    box = [plan.Lx, plan.Ly, plan.Lz + 4.0 * plan.rc + 1.0]   # z box large: never wraps
    tree = cKDTree(pos, boxsize=box)
    rq = plan.rc * (1.0 + 1e-9)
    for c0 in range(0, len(tgt), 65536):
        t = tgt[c0:c0 + 65536]
        lists = tree.query_ball_point(pos[t], rq, workers=_WORKERS)
        cnt = np.fromiter((len(l) for l in lists), dtype=np.int64, count=len(t))
        sj = np.fromiter((j for l in lists for j in l), dtype=np.int64, count=int(cnt.sum()))
        ti = np.repeat(t, cnt)
        _near_pairs_accumulate(plan, xyz, q, ti, sj, phi, grad, rows)
    return phi, grad


def self_coefficient(plan: Plan) -> float:
    """Phi^self_i / q_i = sum_{l=0}^{M} w_l (Eq. eq::phiNDR)."""
    w, _ = plan.weights()
    return float(w.sum())


# ----------------------------------------------------------------------------- windows
def gaussian_window_hat(k, H: float, S: float):
    """W_hat_GS(k) = sqrt(pi/S) H exp(-k^2 H^2 / (4S)) (Eq. eq::GS), the
    untruncated closed form used for deconvolution (R6)."""
    return math.sqrt(math.pi / S) * H * np.exp(-(np.asarray(k) ** 2) * H * H / (4.0 * S))


def kb_window(d, H: float, beta: float):
    """Kaiser-Bessel window W_KB(x) = I0(beta sqrt(1 - (x/H)^2)) / I0(beta) for |x| <= H,
    0 otherwise (Remark rmk::PWindow; Kaiser 1980)."""
    d = np.asarray(d, dtype=np.float64)
    t = np.clip(1.0 - (d / H) ** 2, 0.0, None)
    return np.where(np.abs(d) <= H, scipy.special.i0(beta * np.sqrt(t)) / scipy.special.i0(beta), 0.0)


def kb_window_hat(k, H: float, beta: float):
    """Fourier transform of W_KB: 2H sinh(sqrt(beta^2 - (kH)^2)) / (I0(beta) sqrt(beta^2 - (kH)^2))
    (sin / sqrt form for kH > beta), used for deconvolution as the Gaussian's closed form is."""
    a = beta * beta - (np.asarray(k, dtype=np.float64) * H) ** 2
    r = np.sqrt(np.abs(a))
    rs = np.where(r == 0.0, 1.0, r)
    f = np.where(a > 0.0, np.sinh(r) / rs, np.where(r == 0.0, 1.0, np.sin(r) / rs))
    return 2.0 * H * f / scipy.special.i0(beta)


def es_window(d, H: float, beta: float):
    """"Exponential of semicircle" window exp(beta (sqrt(1 - (x/H)^2) - 1)) for |x| <= H, else 0
    (Remark rmk::PWindow; Barnett et al. 2019)."""
    d = np.asarray(d, dtype=np.float64)
    t = np.clip(1.0 - (d / H) ** 2, 0.0, None)
    return np.where(np.abs(d) <= H, np.exp(beta * (np.sqrt(t) - 1.0)), 0.0)


def es_window_hat(k, H: float, beta: float):
    """Fourier transform of the ES window (no closed form): with x = H sin(theta),
    H int_{-pi/2}^{pi/2} exp(beta (cos theta - 1)) cos(k H sin theta) cos theta dtheta, by adaptive
    quadrature (R6-ES)."""
    import warnings
    from scipy.integrate import IntegrationWarning, quad
    warnings.simplefilter("ignore", IntegrationWarning)    # round-off notices near 1e-16 relative
    ks = np.atleast_1d(np.asarray(k, dtype=np.float64))
    out = np.empty_like(ks)
    for i, kk in enumerate(ks):
        f = lambda th: math.exp(beta * (math.cos(th) - 1.0)) * math.cos(kk * H * math.sin(th)) * math.cos(th)
        out[i] = H * quad(f, -0.5 * math.pi, 0.5 * math.pi, epsabs=1e-17, epsrel=1e-13, limit=400)[0]
    return out.reshape(np.shape(k)) if np.ndim(k) else out[0]


POLY_WINDOWS = {"kb": kb_window, "es": es_window}


def window_half_width(window: str, P: int, h: float) -> float:
    """Support half-width H: (P-1)h/2 for the Gaussian (Eq. eq::GS); P h/2 for the
    polynomial windows KB / ES (R6-KB: every one of the P stencil points stays inside the support
    for all particle offsets, so each stencil point's weight is analytic in the offset)."""
    return (P * h if window in POLY_WINDOWS else (P - 1) * h) / 2.0


@functools.lru_cache(maxsize=64)
def kb_stencil_polys(P: int, beta: float, nu: int, window: str = "kb"):
    """R6-KB (the paper's polynomial windows, Remark rmk::PWindow P:477-480): for stencil
    point j = 0..P-1 and the particle's offset u = x/h + I/2 - g0 in [-1/2, 1/2), the weight
    W_KB((j - p - u) h) is replaced by its degree-nu interpolant at the nu+1 first-kind
    Chebyshev points of u in [-1/2, 1/2] (Chebyshev series in t = 2u).  h cancels (the window
    scales with H = P h / 2).  Returns the (P, nu+1) Chebyshev coefficients.

    The interpolation coefficients a_n = (2 - delta_n0)/(nu+1) sum_i f(t_i) T_n(t_i) are formed in
    40-digit arithmetic (mpmath) and rounded once: in double they carry ~1e-15 absolute noise,
    which the derivative series (the forces, R11) amplifies by ~nu^2 to ~1e-12 relative (the
    interpolant is the definition; its rounding noise is not)."""
    import mpmath as mp
    p = (P - 1) // 2
    n1 = nu + 1
    with mp.workdps(40):
        H = mp.mpf(P) / 2
        bb = mp.mpf(beta)
        i0b = mp.besseli(0, bb)

        def w(x):
            r = 1 - (x / H) ** 2
            if r < 0:
                return mp.mpf(0)
            return mp.besseli(0, bb * mp.sqrt(r)) / i0b if window == "kb" else mp.exp(bb * (mp.sqrt(r) - 1))

        ang = [(i + mp.mpf(1) / 2) * mp.pi / n1 for i in range(n1)]
        C = np.empty((P, n1))
        for j in range(P):
            f = [w((j - p) - mp.cos(a) / 2) for a in ang]
            for n in range(n1):
                acc = mp.fsum(f[i] * mp.cos(n * ang[i]) for i in range(n1))
                C[j, n] = float(acc * (1 if n == 0 else 2) / n1)
    C.setflags(write=False)
    return C


def window_hat(plan: Plan, k, H: float, long: bool = False):
    """Closed-form window transform for the deconvolution (R6 / R6-KB)."""
    shape = plan.Sl if long else plan.S
    if plan.window == "kb":
        return kb_window_hat(k, H, shape)
    if plan.window == "es":
        return es_window_hat(k, H, shape)
    return gaussian_window_hat(k, H, shape)


def stencil(x: np.ndarray, I: int, h: float, P: int, S: float, periodic: bool, window: str = "gs", nu: int = 0):
    """R6: the P (odd) consecutive grid points centred at the nearest grid point
    g0 = floor(x/h + I/2 + 1/2) of the grid x_g = (g - I/2) h; window
    W(x_g - x) = exp(-S ((x_g - x)/H)^2), H = (P-1)h/2 (Eq. eq::GS),
    evaluated at all P points; window == "kb": the polynomial Kaiser-Bessel weights of
    kb_stencil_polys.  Returns (flat index, W, dW/dx_particle)."""
    p = (P - 1) // 2
    H = window_half_width(window, P, h)
    g0 = np.floor(x / h + (I / 2.0 + 0.5)).astype(np.int64)
    g = g0[:, None] + np.arange(-p, p + 1)[None, :]
    if window in POLY_WINDOWS:
        u = x / h + I / 2.0 - g0                 # in [-1/2, 1/2)
        C = kb_stencil_polys(P, S, nu, window)
        W = np.stack([npcheb.chebval(2.0 * u, C[j]) for j in range(P)], axis=1)
        dW = np.stack([npcheb.chebval(2.0 * u, npcheb.chebder(C[j])) * 2.0 / h for j in range(P)], axis=1)
    else:
        d = (g - I / 2.0) * h - x[:, None]
        W = np.exp(-S * (d / H) ** 2)
        dW = 2.0 * S * d / (H * H) * W          # d/dx_i W(x_i - x_g)  (R11)
    if periodic:
        g = np.mod(g, I)
    elif np.any(g < 0) or np.any(g >= I):
        raise ValueError("stencil leaves the extended z grid (R7 violated)")
    return g, W, dW


# ----------------------------------------------------------------------------- mid range
def mid_multiplier(plan: Plan) -> np.ndarray:
    """Scaling factor of Eq. eq::widehat-tilde on the rfftn half spectrum:
    tau_hat^mid(k)/k^2 * 4 pi |W_hat|^-2 = pi^{3/2} sum_{l<=m} w_l s_l^3
    exp(-s_l^2 |k|^2 / 4) / (W_hat_x W_hat_y W_hat_z)^2   (R12),
    k_d = 2 pi n_d / L_d with L_z -> L_z^* (P:580).  |k|^2 = kx^2 + ky^2 + kz^2, so each term
    is the product of per-axis factors exp(-s^2 k_d^2 / 4) / W_hat_d^2; the sum over l is the
    (l)-contraction of the x-y factor table with the z factor table."""
    w, s = plan.weights()
    kx = 2.0 * np.pi * np.fft.fftfreq(plan.Ix, d=plan.hx)
    ky = 2.0 * np.pi * np.fft.fftfreq(plan.Iy, d=plan.hy)
    kz = 2.0 * np.pi * np.fft.rfftfreq(plan.Izs, d=plan.hz)
    Hx, Hy, Hz = (window_half_width(plan.window, plan.P, h) for h in (plan.hx, plan.hy, plan.hz))
    Wx, Wy, Wz = window_hat(plan, kx, Hx), window_hat(plan, ky, Hy), window_hat(plan, kz, Hz)
    L = plan.m + 1
    Fxy = np.empty((L, plan.Ix * plan.Iy))
    Fz = np.empty((L, len(kz)))
    for ell in range(L):
        fx = w[ell] * s[ell] ** 3 * np.exp(-s[ell] ** 2 * kx ** 2 / 4.0) / Wx ** 2
        fy = np.exp(-s[ell] ** 2 * ky ** 2 / 4.0) / Wy ** 2
        Fxy[ell] = (fx[:, None] * fy[None, :]).ravel()
        Fz[ell] = np.exp(-s[ell] ** 2 * kz ** 2 / 4.0) / Wz ** 2
    return (math.pi ** 1.5 * (Fxy.T @ Fz)).reshape(plan.Ix, plan.Iy, len(kz))


def mid_stencils(plan: Plan, xyz):
    sx = stencil(xyz[:, 0], plan.Ix, plan.hx, plan.P, plan.S, True, plan.window, plan.nu)
    sy = stencil(xyz[:, 1], plan.Iy, plan.hy, plan.P, plan.S, True, plan.window, plan.nu)
    sz = stencil(xyz[:, 2], plan.Izs, plan.hz, plan.P, plan.S, False, plan.window, plan.nu)
    return sx, sy, sz


def mid_spread(plan: Plan, xyz, q) -> np.ndarray:
    """Algorithm 1 step 1 (gridding, Eq. eq::gridding):
    S[g] = sum_j q_j W(x_g-x_j)_* W(y_g-y_j)_* W(z_g-z_j) on the I_x x I_y x I_z^* grid."""
    (gx, Wx, _), (gy, Wy, _), (gz, Wz, _) = mid_stencils(plan, xyz)
    G = np.zeros(plan.Ix * plan.Iy * plan.Izs)
    for a in range(plan.P):
        for b in range(plan.P):
            base = (gx[:, a] * plan.Iy + gy[:, b]) * plan.Izs
            idx = base[:, None] + gz
            val = (q * Wx[:, a] * Wy[:, b])[:, None] * Wz
            np.add.at(G, idx.ravel(), val.ravel())
    return G.reshape(plan.Ix, plan.Iy, plan.Izs)


def mid_spread_loops(plan: Plan, xyz, q) -> np.ndarray:
    """The same sum as mid_spread (Eq. eq::gridding) accumulated particle by particle in
    plain C loops (oracle/c/oracle_c.c: oracle_mid_spread), for full BASELINE sizes (N = 1e7) where
    np.add.at over 1.3e10 stencil points would take many minutes.  Pinned equal to mid_spread
    (tests/test_oracle_pins.py::test_mid_spread_loops_equals_add_at)."""
    from . import cext
    (gx, Wx, _), (gy, Wy, _), (gz, Wz, _) = mid_stencils(plan, xyz)
    G = np.zeros(plan.Ix * plan.Iy * plan.Izs)
    # visit particles in (x, y, z) stencil-start order (cache locality only: the sum is order-free)
    order = np.lexsort((gz[:, 0], gy[:, 0], gx[:, 0]))
    a = [np.ascontiguousarray(v[order]) for v in (gx, gy, gz, Wx, Wy, Wz, np.asarray(q, dtype=np.float64))]
    cext.lib().oracle_mid_spread(len(q), plan.P, plan.Ix, plan.Iy, plan.Izs, *[cext.ptr(v) for v in a], cext.ptr(G))
    return G.reshape(plan.Ix, plan.Iy, plan.Izs)


def mid_solve(plan: Plan, S: np.ndarray) -> np.ndarray:
    """Algorithm 1 steps 2-4: forward 3D FFT, scaling, backward 3D FFT."""
    Shat = scipy.fft.rfftn(S, workers=_WORKERS)
    Shat *= mid_multiplier(plan)
    return scipy.fft.irfftn(Shat, s=S.shape, workers=_WORKERS)


def mid_gather(plan: Plan, xyz, Psi: np.ndarray):
    """Algorithm 1 step 5 (gathering, Eq. eq::Phiconv discretised by the trapezoidal
    rule): phi_i = V_h sum_g W W W Psi[g]; gradient with W' (R11)."""
    (gx, Wx, dWx), (gy, Wy, dWy), (gz, Wz, dWz) = mid_stencils(plan, xyz)
    flat = Psi.ravel()
    n = len(xyz)
    phi = np.zeros(n)
    grad = np.zeros((n, 3))
    for a in range(plan.P):
        for b in range(plan.P):
            base = (gx[:, a] * plan.Iy + gy[:, b]) * plan.Izs
            vals = flat[base[:, None] + gz]
            t0 = (Wz * vals).sum(1)
            t1 = (dWz * vals).sum(1)
            phi += Wx[:, a] * Wy[:, b] * t0
            grad[:, 0] += dWx[:, a] * Wy[:, b] * t0
            grad[:, 1] += Wx[:, a] * dWy[:, b] * t0
            grad[:, 2] += Wx[:, a] * Wy[:, b] * t1
    Vh = plan.hx * plan.hy * plan.hz
    return Vh * phi, Vh * grad


def mid_range(plan: Plan, xyz, q, targets=None, loops=None):
    """Phi^mid (Algorithm 1) at the targets, with gradient.  loops=True spreads with
    mid_spread_loops (default above 2e5 particles), else with mid_spread."""
    tgt = slice(None) if targets is None else np.asarray(targets)
    n = len(q) if targets is None else len(tgt)
    if plan.m < 0:
        return np.zeros(n), np.zeros((n, 3))
    if loops is None:
        loops = len(q) > 200_000
    Psi = mid_solve(plan, (mid_spread_loops if loops else mid_spread)(plan, xyz, q))
    return mid_gather(plan, xyz[tgt], Psi)


# ----------------------------------------------------------------------------- long range
def long_kernel(plan: Plan) -> np.ndarray:
    """K_ab(kdot) on the rfft2 half plane, shape (Pc, Pc, Ilx, Ily//2+1):
    pi sum_{l=m+1}^{M} w_l s_l^2 exp(-s_l^2 |kdot|^2 / 4) E_l(z_a - z_b) / (W_hat_x W_hat_y)^2
    with E_l(d) = exp(-d^2/s_l^2), and expm1(-d^2/s_l^2) at kdot = 0 (R10).
    Derivation: Eq. eq::trun2 + two-sided Chebyshev proxies (R9) + the
    window sandwich of Eq. eq::phi2M / eq::overlineSscal."""
    w, s = plan.weights()
    za = 0.5 * plan.Lz * cheb_nodes(plan.Pc)
    d2 = (za[:, None] - za[None, :]) ** 2
    kx = 2.0 * np.pi * np.fft.fftfreq(plan.Ilx, d=plan.hlx)
    ky = 2.0 * np.pi * np.fft.rfftfreq(plan.Ily, d=plan.hly)
    k2 = kx[:, None] ** 2 + ky[None, :] ** 2
    K = np.zeros((plan.Pc, plan.Pc) + k2.shape)
    K0 = np.zeros((plan.Pc, plan.Pc))
    nonzero = k2 > 0.0
    for ell in range(plan.m + 1, plan.M + 1):
        E = np.exp(-d2 / s[ell] ** 2)
        spec = np.where(nonzero, w[ell] * s[ell] ** 2 * np.exp(-s[ell] ** 2 * k2 / 4.0), 0.0)
        K += E[:, :, None, None] * spec[None, None]
        K0 += w[ell] * s[ell] ** 2 * np.expm1(-d2 / s[ell] ** 2)
    K[:, :, 0, 0] = K0
    Hx = window_half_width(plan.window, plan.Pl, plan.hlx)
    Hy = window_half_width(plan.window, plan.Pl, plan.hly)
    What = window_hat(plan, kx, Hx, long=True)[:, None] * window_hat(plan, ky, Hy, long=True)[None, :]
    return math.pi * K / What[None, None] ** 2


def long_basis(plan: Plan, z: np.ndarray):
    """Lagrange basis L_a(z) at the Pc Chebyshev proxies and dL_a/dz (App. A.2)."""
    x = 2.0 * np.asarray(z) / plan.Lz
    V = cheb_T(cheb_nodes(plan.Pc), plan.Pc)
    Vinv = np.linalg.inv(V)
    T = cheb_T(x, plan.Pc)
    # T_n'(x) via T'_{n+1} = 2 T_n + 2 x T'_n - T'_{n-1}
    dT = np.zeros_like(T)
    if plan.Pc > 1:
        dT[..., 1] = 1.0
    for n in range(1, plan.Pc - 1):
        dT[..., n + 1] = 2.0 * T[..., n] + 2.0 * x * dT[..., n] - dT[..., n - 1]
    return T @ Vinv, (dT @ Vinv) * (2.0 / plan.Lz)


def long_stencils(plan: Plan, xyz):
    sx = stencil(xyz[:, 0], plan.Ilx, plan.hlx, plan.Pl, plan.Sl, True, plan.window, plan.nul)
    sy = stencil(xyz[:, 1], plan.Ily, plan.hly, plan.Pl, plan.Sl, True, plan.window, plan.nul)
    return sx, sy


def long_spread(plan: Plan, xyz, q) -> np.ndarray:
    """Anterpolation to the proxy layers (Alg. 2 step 1, two-sided form R9):
    S_b[g] = sum_j q_j L_b(z_j) W(x_g-x_j)_* W(y_g-y_j)_*  (P:529)."""
    (gx, Wx, _), (gy, Wy, _) = long_stencils(plan, xyz)
    Lb, _ = long_basis(plan, xyz[:, 2])
    G = np.zeros(plan.Pc * plan.Ilx * plan.Ily)
    layer = np.arange(plan.Pc) * (plan.Ilx * plan.Ily)
    for a in range(plan.Pl):
        for b in range(plan.Pl):
            idx = (gx[:, a] * plan.Ily + gy[:, b])[:, None] + layer[None, :]
            val = (q * Wx[:, a] * Wy[:, b])[:, None] * Lb
            np.add.at(G, idx.ravel(), val.ravel())
    return G.reshape(plan.Pc, plan.Ilx, plan.Ily)


def long_spread_dense(plan: Plan, xyz, q, chunk: int = 200_000) -> np.ndarray:
    """The same sum as long_spread for small long grids at full BASELINE sizes: each particle's
    window rows are written out densely over the Ilx (Ily) grid points (zeros off the stencil), and
    the sum over particles j of (q_j L_b(z_j) Wx_j(gx)) Wy_j(gy) is one matrix product per chunk
    of particles (a library GEMM as the j-contraction).  Pinned equal to long_spread
    (tests/test_oracle_pins.py::test_long_spread_dense_equals_add_at)."""
    (gx, Wx, _), (gy, Wy, _) = long_stencils(plan, xyz)
    Lb, _ = long_basis(plan, xyz[:, 2])
    q = np.asarray(q, dtype=np.float64)
    G = np.zeros((plan.Pc * plan.Ilx, plan.Ily))
    for c0 in range(0, len(q), chunk):
        sl = slice(c0, c0 + chunk)
        n = len(q[sl])
        rows = np.repeat(np.arange(n), plan.Pl)
        Dx = np.zeros((n, plan.Ilx))
        Dy = np.zeros((n, plan.Ily))
        np.add.at(Dx, (rows, gx[sl].ravel()), Wx[sl].ravel())
        np.add.at(Dy, (rows, gy[sl].ravel()), Wy[sl].ravel())
        T = (q[sl, None] * Lb[sl])[:, :, None] * Dx[:, None, :]          # (n, Pc, Ilx)
        G += T.reshape(n, -1).T @ Dy
    return G.reshape(plan.Pc, plan.Ilx, plan.Ily)


def long_solve(plan: Plan, S: np.ndarray) -> np.ndarray:
    """Alg. 2 steps 2-4: 2D FFT per layer, scaling by the wide
    Gaussians' spectra coupled across layers (K_ab), backward 2D FFT per layer."""
    Shat = scipy.fft.rfft2(S, axes=(1, 2), workers=_WORKERS)
    K = long_kernel(plan)
    Shat2 = np.einsum("abxy,bxy->axy", K, Shat)
    return scipy.fft.irfft2(Shat2, s=S.shape[1:], axes=(1, 2), workers=_WORKERS)


def long_gather(plan: Plan, xyz, Psi: np.ndarray):
    """Alg. 2 step 5 (Eq. eq::SOGLong): phi_i = h_x h_y sum_g W W sum_a L_a(z_i) Psi_a[g]."""
    (gx, Wx, dWx), (gy, Wy, dWy) = long_stencils(plan, xyz)
    La, dLa = long_basis(plan, xyz[:, 2])
    n = len(xyz)
    phi = np.zeros(n)
    grad = np.zeros((n, 3))
    flat = Psi.reshape(plan.Pc, -1)
    for a in range(plan.Pl):
        for b in range(plan.Pl):
            vals = flat[:, gx[:, a] * plan.Ily + gy[:, b]].T          # (n, Pc)
            t0 = (La * vals).sum(1)
            t1 = (dLa * vals).sum(1)
            phi += Wx[:, a] * Wy[:, b] * t0
            grad[:, 0] += dWx[:, a] * Wy[:, b] * t0
            grad[:, 1] += Wx[:, a] * dWy[:, b] * t0
            grad[:, 2] += Wx[:, a] * Wy[:, b] * t1
    A = plan.hlx * plan.hly
    return A * phi, A * grad


# ------------------------------------------- App. C: one-sided Taylor form of Alg. 2 steps 1-3
# Not on the GPU path (NEXT #3): kept as a checked reference for the measured
# comparison with the two-sided K_ab form (tests/test_oracle_pins.py::test_taylor_variant_*).
def taylor_bound(plan: Plan, Q: int) -> float:
    """Lemma lemma::Taylor (Eq. eq::Taylor2) for the variable App. C expands in
    (R23): the Lagrange remainder x^Q / Q! at x = (z_a - z_j)^2 / s^2 <= L_z^2 / s_{m+1}^2 = 1/eta^2
    (z_a - z_j spans [-L_z, L_z], twice the lemma's interval, so (2 eta)^{2Q} becomes eta^{2Q}),
    eta = s_{m+1} / L_z here."""
    _, s = plan.weights()
    eta = s[plan.m + 1] / plan.Lz
    return 1.0 / (math.factorial(Q) * eta ** (2 * Q))


def long_spread_taylor(plan: Plan, xyz, q, Q: int) -> np.ndarray:
    """App. C: S^p_grid([r, z_a]) = sum_j q_j W(r - r_j) ((z_a - z_j)/L_z)^{2p},
    p = 0..Q-1, on the long grid x the Pc Chebyshev proxies z_a; shape (Q, Pc, Ilx, Ily)."""
    (gx, Wx, _), (gy, Wy, _) = long_stencils(plan, xyz)
    za = 0.5 * plan.Lz * cheb_nodes(plan.Pc)
    d = (za[None, :] - xyz[:, 2][:, None]) / plan.Lz                       # (n, Pc)
    mom = np.stack([d ** (2 * p) for p in range(Q)], axis=1).reshape(len(q), -1)   # (n, Q Pc)
    G = np.zeros(Q * plan.Pc * plan.Ilx * plan.Ily)
    layer = np.arange(Q * plan.Pc) * (plan.Ilx * plan.Ily)
    for a in range(plan.Pl):
        for b in range(plan.Pl):
            idx = (gx[:, a] * plan.Ily + gy[:, b])[:, None] + layer[None, :]
            val = (q * Wx[:, a] * Wy[:, b])[:, None] * mom
            np.add.at(G, idx.ravel(), val.ravel())
    return G.reshape(Q, plan.Pc, plan.Ilx, plan.Ily)


def long_coeff_taylor(plan: Plan, Q: int) -> np.ndarray:
    """A_p(kdot) = (-1)^p / p! |W_hat(kdot)|^{-2} sum_{l>m} w_l L_z^{2p} / s_l^{2p-2}
    e^{-s_l^2 |kdot|^2 / 4}, with the factor pi of Eq. eq::trun2 as in long_kernel and, at kdot = 0,
    the p = 0 term dropped (R10: the constant of e^{-d^2/s^2} is the expm1 that long_kernel removes);
    shape (Q, Ilx, Ily//2+1)."""
    w, s = plan.weights()
    kx = 2.0 * np.pi * np.fft.fftfreq(plan.Ilx, d=plan.hlx)
    ky = 2.0 * np.pi * np.fft.rfftfreq(plan.Ily, d=plan.hly)
    k2 = kx[:, None] ** 2 + ky[None, :] ** 2
    A = np.zeros((Q,) + k2.shape)
    for p in range(Q):
        for ell in range(plan.m + 1, plan.M + 1):
            A[p] += w[ell] * s[ell] ** 2 * (plan.Lz / s[ell]) ** (2 * p) * np.exp(-s[ell] ** 2 * k2 / 4.0)
        A[p] *= (-1) ** p / math.factorial(p)
    A[0, 0, 0] = 0.0
    Hx = window_half_width(plan.window, plan.Pl, plan.hlx)
    Hy = window_half_width(plan.window, plan.Pl, plan.hly)
    What = window_hat(plan, kx, Hx, long=True)[:, None] * window_hat(plan, ky, Hy, long=True)[None, :]
    return math.pi * A / What[None] ** 2


def long_range_taylor(plan: Plan, xyz, q, Q: int, targets=None):
    """Phi^long by App. C: 2D FFT of every (p, z_a) layer, S_hat_scal(kdot, z_a) = sum_p A_p(kdot)
    S_hat^p(kdot, z_a), inverse 2D FFT per proxy layer, and the gather of Alg. 2 step 5
    (window in x, y, Chebyshev interpolation in z at the target: the moments are polynomials of
    degree 2(Q-1) in z_a, exact in the Pc-point interpolant when Pc >= 2Q - 1)."""
    tgt = slice(None) if targets is None else np.asarray(targets)
    G = long_spread_taylor(plan, xyz, q, Q)
    Ghat = scipy.fft.rfft2(G, axes=(2, 3), workers=_WORKERS)
    Psi_hat = np.einsum("pxy,paxy->axy", long_coeff_taylor(plan, Q), Ghat)
    Psi = scipy.fft.irfft2(Psi_hat, s=G.shape[2:], axes=(1, 2), workers=_WORKERS)
    return long_gather(plan, xyz[tgt], Psi)


# --------------------------------------------------- long range without FFT (Alg. 3, App. B)
def long_modes(plan: Plan):
    """R8-D mode set: kx = 2 pi n / Lx, n = -Kx..Kx; ky = 2 pi n / Ly, n = 0..Ky (half plane:
    the field is real, so the ky < 0 modes are the conjugates of ky > 0)."""
    kx = 2.0 * np.pi * np.arange(-plan.Kx, plan.Kx + 1) / plan.Lx
    ky = 2.0 * np.pi * np.arange(0, plan.Ky + 1) / plan.Ly
    return kx, ky


def long_kernel_direct(plan: Plan) -> np.ndarray:
    """K_ab(kdot) = (pi / (Lx Ly)) sum_{l>m} w_l s_l^2 exp(-s_l^2 |kdot|^2/4) E_l(z_a - z_b), shape
    (Pc, Pc, 2Kx+1, Ky+1): the 2D Fourier series of the x,y-periodised wide Gaussians (Eq.
    eq::gridnonfft) at the proxies (R9), R10 at kdot = 0; no window, no deconvolution."""
    w, s = plan.weights()
    za = 0.5 * plan.Lz * cheb_nodes(plan.Pc)
    d2 = (za[:, None] - za[None, :]) ** 2
    kx, ky = long_modes(plan)
    k2 = kx[:, None] ** 2 + ky[None, :] ** 2
    K = np.zeros((plan.Pc, plan.Pc) + k2.shape)
    K0 = np.zeros((plan.Pc, plan.Pc))
    nonzero = k2 > 0.0
    for ell in range(plan.m + 1, plan.M + 1):
        E = np.exp(-d2 / s[ell] ** 2)
        spec = np.where(nonzero, w[ell] * s[ell] ** 2 * np.exp(-s[ell] ** 2 * k2 / 4.0), 0.0)
        K += E[:, :, None, None] * spec[None, None]
        K0 += w[ell] * s[ell] ** 2 * np.expm1(-d2 / s[ell] ** 2)
    K[:, :, plan.Kx, 0] = K0
    return math.pi / (plan.Lx * plan.Ly) * K


def long_spread_direct(plan: Plan, xyz, q) -> np.ndarray:
    """Alg. 3 step 1 in the two-sided proxy form (R9): S_b(kdot) = sum_j q_j L_b(z_j)
    exp(-i kdot . r_j), a type-1 nonuniform DFT per proxy layer; shape (Pc, 2Kx+1, Ky+1)."""
    kx, ky = long_modes(plan)
    Lb, _ = long_basis(plan, xyz[:, 2])
    ex = np.exp(-1j * np.outer(xyz[:, 0], kx))                # (N, nkx)
    ey = np.exp(-1j * np.outer(xyz[:, 1], ky))                # (N, nky)
    return np.einsum("jb,jx,jy->bxy", q[:, None] * Lb, ex, ey)


def long_solve_direct(plan: Plan, S: np.ndarray) -> np.ndarray:
    """Alg. 3 step 2: the wide Gaussians' spectra coupled across the proxies."""
    return np.einsum("abxy,bxy->axy", long_kernel_direct(plan), S)


def long_gather_direct(plan: Plan, xyz, Psi: np.ndarray):
    """Alg. 3 step 3 (Eq. eq::3.13A): phi_i = sum_a L_a(z_i) sum_kdot Psi_a(kdot)
    exp(i kdot . r_i) over the full plane = Re of the half-plane sum with weight 1 (ky = 0) or 2."""
    kx, ky = long_modes(plan)
    La, dLa = long_basis(plan, xyz[:, 2])
    c = np.where(ky > 0, 2.0, 1.0)
    ex = np.exp(1j * np.outer(xyz[:, 0], kx))
    ey = np.exp(1j * np.outer(xyz[:, 1], ky)) * c[None, :]
    E = ex[:, :, None] * ey[:, None, :]                       # (N, nkx, nky)
    A = np.einsum("jxy,axy->ja", E, Psi)                      # sum over modes per layer
    Ax = np.einsum("jxy,axy->ja", E * (1j * kx)[None, :, None], Psi)
    Ay = np.einsum("jxy,axy->ja", E * (1j * ky)[None, None, :], Psi)
    phi = np.real((La * A).sum(1))
    grad = np.stack([np.real((La * Ax).sum(1)), np.real((La * Ay).sum(1)), np.real((dLa * A).sum(1))], axis=1)
    return phi, grad


def long_range(plan: Plan, xyz, q, targets=None):
    """Phi^long (Algorithm 2 with two-sided Chebyshev proxies, R9; or Algorithm 3 without FFT
    when plan.long_method == "direct") at the targets."""
    tgt = slice(None) if targets is None else np.asarray(targets)
    if plan.long_method == "direct":
        Psi = long_solve_direct(plan, long_spread_direct(plan, xyz, q))
        return long_gather_direct(plan, xyz[tgt], Psi)
    dense = len(q) > 200_000 and plan.Ilx * plan.Ily <= 4096
    Psi = long_solve(plan, (long_spread_dense if dense else long_spread)(plan, xyz, q))
    return long_gather(plan, xyz[tgt], Psi)


# ----------------------------------------------------------------------------- total
def evaluate(plan: Plan, xyz, q, targets=None, parts: bool = False):
    """phi_i = Phi^N + Phi^mid + Phi^long - q_i sum w_l and
    F_i = -q_i grad phi, at all particles or the given targets."""
    xyz = canonicalize(xyz, plan)
    q = np.asarray(q, dtype=np.float64)
    if abs(q.sum()) > 1e-12 * np.abs(q).sum():
        raise ValueError("system not charge neutral (P:119-121)")
    tq = q if targets is None else q[np.asarray(targets)]
    pn, gn = near_field(plan, xyz, q, targets)
    pm, gm = mid_range(plan, xyz, q, targets)
    pl, gl = long_range(plan, xyz, q, targets)
    phi = pn + pm + pl - tq * self_coefficient(plan)
    grad = gn + gm + gl
    force = -tq[:, None] * grad
    if parts:
        return phi, force, {"near": (pn, gn), "mid": (pm, gm), "long": (pl, gl)}
    return phi, force


def energy(q, phi) -> float:
    """U = 1/2 sum_i q_i phi_i."""
    return 0.5 * float(np.dot(q, phi))
