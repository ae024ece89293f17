"""Parameter selection for the spectral SOG solver (oracle side).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  The CUDA library has its
own, independent implementation of the same rules (paper_2412_04595_b200/csrc/
plan.cpp); tests/test_abi_plan.py::test_plan_rules_match_oracle compares the two.

The paper gives the ingredients (section 4.3) with
unit-prefactor O(.) estimates; the concrete rules are the readings R1-R9 of
DESIGN.md ("Readings of the paper").  Every constant below is named there.
"""
from __future__ import annotations

import dataclasses
import functools
import math

import numpy as np
from scipy.special import erfcinv

# Table 1: b, r0, omega, energy error, M_E, force error, M_F.
TABLE1 = (
    (2.0, 1.9892536839080267, 0.9944464927622323, 3.12e-2, 16, 9.93e-3, 11),
    (1.62976708826776469, 2.7520026668023417, 1.0078069793438068, 2.33e-3, 31, 6.21e-4, 16),
    (1.48783512395703226, 3.7554672283554990, 0.9919117057598183, 2.29e-4, 46, 7.98e-5, 26),
    (1.32070036405934420, 4.3914554711638349, 1.0018891411481198, 1.18e-6, 76, 5.76e-7, 41),
    (1.21812525709410644, 5.6355288151271085, 1.0009014615603334, 7.14e-10, 166, 5.14e-10, 71),
    (1.14878150173321925, 7.2956245490719404, 1.0000368348358225, 1.30e-15, 271, 1.98e-14, 116),
)

# ---- plan constants (R2, R4-R9); tuned on B200 / calibrated vs Ewald2D ----
RC_FACTOR = 3.25     # R2: r_c = RC_FACTOR * rho^(-1/3)  (GPU-tuned plan knob, R2)
ETA = 0.3            # R4: range-splitting factor
KAPPA = 1.15         # R5/R8: Nyquist safety, h <= pi s /(2 KAPPA sqrt(ln 1/tol))
WIN_C = 0.3          # R6: window error target eps_w = WIN_C * tol
PAD_C = 10.0         # R7: z padding  s_m * sqrt(ln(PAD_C/tol))
CHEB_C = 0.1         # R9: Chebyshev two-variable interpolation target CHEB_C * tol
CHEB_FLOOR = 5e-14   # R9: rounding floor of the interpolation test
FFT_COST = 30.0      # R6: cost of one FFT grid point in units of one stencil point (B200-measured model)
LONG_FFT_COST = 30.0
KB_BETA = 2.2        # R6-KB: Kaiser-Bessel shape beta = KB_BETA * P (R6-KB; cf. beta = 2.5 P)
KB_NU_EXTRA = 3      # R6-KB: polynomial degree nu = P + KB_NU_EXTRA of the Chebyshev-interpolated window
KB_RATE = (0.4, 0.92)  # R6-KB: window error ~ 10^(a - b P) at h = h_Nyquist (calibrated)
TOL_MIN = 2e-14      # Table 1 force floor 1.98e-14
TOL_MAX = 1e-1


def select_row(tol: float):
    """R1: the coarsest Table-1 row whose force error is <= tol."""
    if not (TOL_MIN <= tol <= TOL_MAX):
        raise ValueError(f"tol {tol} outside [{TOL_MIN}, {TOL_MAX}]")
    for row in TABLE1:
        if row[5] <= tol:
            return row
    raise ValueError("infeasible tolerance")


@functools.lru_cache(maxsize=32)
def c1_solve(b: float, tol: float):
    """NEXT #4: the C^1 continuity solve for a general b (Eq. eq::2.35z): with sigma = 1,
    r_0 and omega solve  r_0 F(r_0) - 1 = 0  and  r_0^2 F'(r_0) + 1 = 0,
    F(r) = omega w_0 e^{-r^2/s_0^2} + G(r),  G(r) = sum_{l>=1} w_l e^{-r^2/s_l^2},
    w_l = sqrt(2/pi) b^-l ln b, s_l = sqrt(2) b^l (the sum runs until w_l < 1e-55).
    Eliminating omega with the first equation leaves one equation in r,
        h(r) = 1 - r^2 + r^3 G(r) + r^2 G'(r) = 0,   omega = (1/r - G(r)) e^{r^2/2} / w_0(omega=1),
    whose roots are not unique.  The paper's rule: the smallest root r_0 whose last two
    eq::convrate terms are below tol -- here the larger of the energy and force forms,
    with s_{-1} = s_0 / b, w_{-1} = b w_0 from the weight formula (P:331 prints "s_{-1} = b s_0";
    DESIGN.md reading R22).  Roots are bracketed by sign changes of h on a 0.02 grid of r in [1, 20]
    and refined in 40-digit arithmetic (mpmath): for b -> 1 the residual of the system sits at the BSA
    error level (~1e-13 at b = 1.17) over whole intervals of r, so double precision cannot locate
    r_0, and omega = ... e^{r^2/2} amplifies rounding by e^{r_0^2/2}.  Returns (r0, omega) as floats.
    Pinned: Table 1's simple-root rows (b = 2, 1.4878...) come back to the printed digits, and every
    printed row satisfies h(r_0) ~ 0 (tests/test_oracle_pins.py::test_c1_solve_*)."""
    import mpmath as mp
    with mp.workdps(40):
        bb = mp.mpf(b)
        c = mp.sqrt(2 / mp.pi) * mp.log(bb)

        def G(r):
            g, dg, l = mp.mpf(0), mp.mpf(0), 1
            while True:
                s2 = 2 * bb ** (2 * l)
                w = c * bb ** (-l)
                e = w * mp.e ** (-r * r / s2)
                g += e
                dg += e * (-2 * r / s2)
                if w < mp.mpf(10) ** -55:
                    return g, dg
                l += 1

        def h(r):
            g, dg = G(r)
            return 1 - r * r + r ** 3 * g + r * r * dg

        def terms(r):
            g, _ = G(r)
            om = (1 / r - g) * mp.e ** (r * r / 2) / c
            s0, sm1, wm1 = mp.sqrt(2), mp.sqrt(2) / bb, c * bb
            te = abs(wm1 * mp.e ** (-r * r / sm1 ** 2)) + abs((om - 1) * c * mp.e ** (-r * r / s0 ** 2))
            tf = abs(wm1 / sm1 ** 2 * mp.e ** (-r * r / sm1 ** 2)) + abs((om - 1) * c / s0 ** 2 * mp.e ** (-r * r / s0 ** 2))
            return om, max(te, tf)

        # sign changes of h on the 0.02 grid, located with a float64 evaluation of the same sum
        # (|h| between roots is >= ~1e-14 for b >= 1.15, far above its rounding), then refined in
        # 40 digits
        rg = 1.0 + 0.02 * np.arange(951)
        ell = np.arange(1, int(130.0 / math.log(b)) + 2)
        s2 = 2.0 * b ** (2.0 * ell)
        e = (math.sqrt(2 / math.pi) * math.log(b) * b ** (-ell.astype(float)))[None, :] * np.exp(-rg[:, None] ** 2 / s2)
        hg = 1 - rg ** 2 + rg ** 3 * e.sum(1) + rg ** 2 * (e * (-2 * rg[:, None] / s2)).sum(1)
        for i in range(len(rg) - 1):
            if hg[i] * hg[i + 1] < 0:
                lo, hi = mp.mpf(rg[i]), mp.mpf(rg[i + 1])
                hlo = h(lo)
                if hlo * h(hi) > 0:
                    continue                        # a float64 artefact: no bracket in 40 digits
                for _ in range(64):                 # bisection to 0.02 * 2^-64 ~ 1e-21 (h is smooth)
                    mid = (lo + hi) / 2
                    hm = h(mid)
                    if hlo * hm <= 0:
                        hi = mid
                    else:
                        lo, hlo = mid, hm
                root = (lo + hi) / 2
                om, t = terms(root)
                if t <= tol:
                    return float(root), float(om)
    raise ValueError(f"no C^1 root with error terms <= {tol} for b = {b}")


def sog_nodes_weights(b: float, sigma: float, omega: float, M: int):
    """w_l = (pi/2)^(-1/2) b^(-l) sigma^(-1) log b, s_l = sqrt(2) b^l sigma;
    w_0 carries the extra factor omega."""
    ell = np.arange(M + 1, dtype=np.float64)
    w = (math.pi / 2.0) ** -0.5 * b ** (-ell) / sigma * math.log(b)
    w[0] *= omega
    s = math.sqrt(2.0) * b ** ell * sigma
    return w, s


def is_friendly(n: int) -> bool:
    for p in (2, 3, 5, 7):
        while n % p == 0:
            n //= p
    return n == 1


def friendly_even(n: int) -> int:
    """Smallest even integer >= n whose prime factors are in {2,3,5,7} (FFT sizes)."""
    n = max(int(n), 2)
    if n % 2:
        n += 1
    while not is_friendly(n):
        n += 2
    return n


def z_friendly_even(n: int) -> int:
    """Padded z size Izs (R7-Z): the smallest even 2^a 3^b or 2^a 5^b >= n (sizes the library's fused
    z pass has a radix set for), unless that exceeds 4096 (beyond the fused pass): then
    friendly_even(n).  Any Izs >= the R7 minimum is a valid padding (P:460-462 only needs the
    free direction padded by at least the Gaussian's reach)."""
    base = friendly_even(n)
    if base > 4096:
        return base
    m = base
    while True:
        r = m
        while r % 2 == 0:
            r //= 2
        r3, r5 = r, r
        while r3 % 3 == 0:
            r3 //= 3
        while r5 % 5 == 0:
            r5 //= 5
        if r3 == 1 or r5 == 1:
            return m
        m += 2


def window_h_alias(P: int, S: float, eps_w: float, s: float) -> float:
    """Largest mesh size h for which the aliasing term of Thm 4.2,
    exp(-pi^2 mu (P-1)^2 / (4 s^2 S)) with mu = s^2 - H^2/S, H=(P-1)h/2,
    stays <= eps_w.  Returns 0 if no h > 0 works (P too small for S)."""
    a = P - 1.0
    rhs = 1.0 - 4.0 * S * math.log(1.0 / eps_w) / (math.pi ** 2 * a * a)
    if rhs <= 0.0:
        return 0.0
    return 2.0 * s * math.sqrt(S) / a * math.sqrt(rhs)


def choose_window(s: float, eps_w: float, tol: float, cost_fn):
    """R6: Gaussian window W=exp(-S (x/H)^2).  S = erfcinv(eps_w)^2 so the
    erfc(sqrt S) term of Thms 4.2/4.3 is eps_w; the support P (odd) and mesh size
    h minimise cost_fn(P, h) subject to the aliasing bound and the Nyquist
    truncation h <= pi s / (2 KAPPA sqrt(ln 1/tol)) (Thm 4.1 with R5's exponent)."""
    S = float(erfcinv(eps_w)) ** 2
    h_nyq = math.pi * s / (2.0 * KAPPA * math.sqrt(math.log(1.0 / tol)))
    best = None
    for P in range(3, 61, 2):
        ha = window_h_alias(P, S, eps_w, s)
        if ha <= 0.0:
            continue
        h = min(h_nyq, ha)
        c = cost_fn(P, h)
        if best is None or c < best[0]:
            best = (c, P, h)
    if best is None:
        raise ValueError("no feasible window")
    return best[1], S, best[2]


ES_BETA = 2.3        # R6-ES: exponential-of-semicircle shape beta = ES_BETA * P (cf. beta = 2.5 P)
ES_NU_EXTRA = 3      # R6-ES: nu = P + 3 as KB (the paper needs 1-2 more for ES; not with H = P h/2)


def choose_window_kb(s: float, eps_w: float, tol: float, window: str = "kb"):
    """R6-KB: Kaiser-Bessel window (Remark rmk::PWindow), shape beta = KB_BETA P,
    support P = the smallest odd P >= 5 with 10^(a - b P) <= eps_w, mesh size at the Nyquist
    bound of R5 (the window does not constrain h).  Returns (P, beta, h, nu)."""
    a, b = KB_RATE
    P = 5
    while 10.0 ** (a - b * P) > eps_w:
        P += 2
    h = math.pi * s / (2.0 * KAPPA * math.sqrt(math.log(1.0 / tol)))
    if window == "es":
        return P, ES_BETA * P, h, P + ES_NU_EXTRA
    return P, KB_BETA * P, h, P + KB_NU_EXTRA


def cheb_nodes(P: int) -> np.ndarray:
    """First-kind Chebyshev nodes x_i = cos((i-1/2) pi / P), i=1..P."""
    i = np.arange(1, P + 1, dtype=np.float64)
    return np.cos((i - 0.5) * np.pi / P)


def cheb_T(x: np.ndarray, P: int) -> np.ndarray:
    """T_n(x), n=0..P-1, by the three-term recurrence; shape x.shape+(P,)."""
    x = np.asarray(x, dtype=np.float64)
    T = np.empty(x.shape + (P,), dtype=np.float64)
    T[..., 0] = 1.0
    if P > 1:
        T[..., 1] = x
    for n in range(1, P - 1):
        T[..., n + 1] = 2.0 * x * T[..., n] - T[..., n - 1]
    return T


def lagrange_matrix(x: np.ndarray, P: int) -> np.ndarray:
    """Values L_a(x) of the interpolation basis: Chebyshev interpolation a = V^{-1} f
     followed by evaluation E a, i.e. L(x) = T(x) V^{-1}."""
    V = cheb_T(cheb_nodes(P), P)            # V(i,j) = T_j(x_i)
    return cheb_T(x, P) @ np.linalg.inv(V)


def cheb_two_sided_error(P: int, Lz: float, s: float, ntest: int = 65) -> float:
    """Max error of the two-variable interpolant sum_ab L_a(z) g(z_a-z_b) L_b(z')
    of g(d)=exp(-d^2/s^2) on a test grid of [-Lz/2, Lz/2]^2 (R9; Thm 3.1)."""
    xt = np.linspace(-1.0, 1.0, ntest)
    za = 0.5 * Lz * cheb_nodes(P)
    G = np.exp(-((za[:, None] - za[None, :]) / s) ** 2)
    Lt = lagrange_matrix(xt, P)
    approx = Lt @ G @ Lt.T
    zt = 0.5 * Lz * xt
    exact = np.exp(-((zt[:, None] - zt[None, :]) / s) ** 2)
    return float(np.max(np.abs(approx - exact)))


def choose_cheb(Lz: float, s: float, eps: float) -> int:
    """R9: smallest P (>=2) with two-sided interpolation error <= eps."""
    for P in range(2, 65):
        if cheb_two_sided_error(P, Lz, s) <= eps:
            return P
    raise ValueError("Chebyshev order > 64 needed")


@dataclasses.dataclass
class Plan:
    N: int
    Lx: float
    Ly: float
    Lz: float
    tol: float
    b: float
    r0: float
    omega: float
    rc: float
    sigma: float
    M: int
    m: int
    # mid-range grid (R5-R7); unused when m < 0
    Ix: int = 0
    Iy: int = 0
    Iz: int = 0           # interior z count, h_z = Lz / Iz
    Izs: int = 0          # extended z grid count I_z^*
    P: int = 0            # window support (odd)
    S: float = 0.0        # window shape: S (Gaussian) or beta (Kaiser-Bessel)
    # long-range (R8-R9)
    Ilx: int = 0
    Ily: int = 0
    Pl: int = 0
    Sl: float = 0.0
    Pc: int = 0           # Chebyshev proxy layers
    window: str = "gs"    # "gs": Gaussian (Eq. eq::GS); "kb": Kaiser-Bessel, polynomial weights (R6-KB)
    long_method: str = "fft"   # "fft": Alg. 2 (window + 2D FFT); "direct": Alg. 3 (App. B), R8-D modes
    Kx: int = 0           # direct: Fourier modes kx = 2 pi n / Lx, |n| <= Kx (R8-D)
    Ky: int = 0
    nu: int = 0           # KB: degree of the Chebyshev-interpolated window polynomials (mid)
    nul: int = 0          # KB: same for the long-range window

    # derived quantities (recomputed, never stored separately)
    @property
    def hx(self) -> float:
        return self.Lx / self.Ix

    @property
    def hy(self) -> float:
        return self.Ly / self.Iy

    @property
    def hz(self) -> float:
        return self.Lz / self.Iz

    @property
    def Lzs(self) -> float:
        return self.hz * self.Izs

    @property
    def hlx(self) -> float:
        return self.Lx / self.Ilx

    @property
    def hly(self) -> float:
        return self.Ly / self.Ily

    def weights(self):
        return sog_nodes_weights(self.b, self.sigma, self.omega, self.M)

    def describe(self) -> dict:
        d = dataclasses.asdict(self)
        return d


# R20: eq::optimiz with B200-calibrated costs in seconds (c5 stage times, R20):
# near per pair, mid spread+gather per stencil point, mid FFT+scale per grid point, long
# spread+gather per (particle x Pl^2 x Pc), long FFT+scale per long grid point and layer
GPU_COST = {"pair": 1.35e-11, "stencil": 1.39e-12, "grid": 2.6e-11, "long": 4.33e-13, "lgrid": 3.6e-11}
OPT_RC = (2.75, 3.0, 3.25, 3.5, 3.75)
OPT_ETA = (0.2, 0.25, 0.3, 0.35, 0.4, 0.5)


def plan_cost(p: "Plan") -> float:
    """R20 predicted evaluation time (s) of a plan: the terms of eq::comp weighted by the
    measured B200 costs; near pairs from the cutoff sphere clipped to the box height."""
    c = GPU_COST
    rho = p.N / (p.Lx * p.Ly * p.Lz)
    vol = min(4.0 / 3.0 * math.pi * p.rc ** 3, math.pi * p.rc ** 2 * p.Lz)
    t = c["pair"] * p.N * rho * vol
    if p.m >= 0:
        t += c["stencil"] * p.N * p.P ** 3 + c["grid"] * p.Ix * p.Iy * p.Izs
    t += c["long"] * p.N * p.Pl ** 2 * p.Pc + c["lgrid"] * p.Ilx * p.Ily * p.Pc
    return t


def make_plan(N: int, Lx: float, Ly: float, Lz: float, tol: float, **over) -> Plan:
    """Rules R1-R9.  Keyword overrides replace any chosen value
    (rc_factor, eta, b-row via `row`, or any Plan field).  optimize=True: R20, the plan of least
    predicted time over r_c factors OPT_RC x range splits OPT_ETA (first minimum in that order)."""
    if over.pop("optimize", False):
        best, bc = None, None
        for f in OPT_RC:
            for e in OPT_ETA:
                q = make_plan(N, Lx, Ly, Lz, tol, rc_factor=f, eta=e, **over)
                if q.Pc > 32 or q.Pl > 25 or (q.m >= 0 and q.P > 25):
                    continue                       # outside the GPU path's compiled range
                c = plan_cost(q)
                if bc is None or c < bc:
                    best, bc = q, c
        return best
    if N < 1 or not all(math.isfinite(v) and v > 0 for v in (Lx, Ly, Lz)):
        raise ValueError("invalid N or box")
    b_general = over.pop("b", None)
    if b_general is not None:                               # NEXT #4: C^1 solve for this b
        if not (1.0 < b_general <= 2.0):
            raise ValueError("b must lie in (1, 2]")
        b = float(b_general)
        r0, omega = c1_solve(b, tol)
        over.pop("row", None)
    else:
        row = over.pop("row", None) or select_row(tol)
        b, r0, omega = row[0], row[1], row[2]
    rc_factor = over.pop("rc_factor", RC_FACTOR)
    window = over.pop("window", "gs")
    if window not in ("gs", "kb", "es"):
        raise ValueError("window must be 'gs', 'kb' or 'es'")
    long_method = over.pop("long_method", "fft")
    if long_method not in ("fft", "direct"):
        raise ValueError("long_method must be 'fft' or 'direct'")
    eta = over.pop("eta", ETA)
    rho = N / (Lx * Ly * Lz)
    rc = over.pop("rc", None)
    if rc is None:
        rc = min(rc_factor * rho ** (-1.0 / 3.0), 0.5 * min(Lx, Ly))
    if rc > 0.5 * min(Lx, Ly) * (1 + 1e-15):
        raise ValueError("r_c > min(Lx,Ly)/2")
    sigma = rc / r0
    s0 = math.sqrt(2.0) * sigma
    Lmax = max(Lx, Ly, Lz)
    M = over.pop("M", None)
    if M is None:                                            # R3
        M = max(0, math.ceil(math.log(Lmax / tol / s0) / math.log(b)))
        while s0 * b ** M < Lmax / tol:
            M += 1
        while M > 0 and s0 * b ** (M - 1) >= Lmax / tol:
            M -= 1
    m = over.pop("m", None)
    if m is None:                                            # R4
        m = -1
        for ell in range(M + 1):
            if s0 * b ** ell <= eta * Lz:
                m = ell
    m = min(m, M - 1)                                        # keep >= 1 long-range Gaussian
    p = Plan(N=N, Lx=Lx, Ly=Ly, Lz=Lz, tol=tol, b=b, r0=r0, omega=omega, rc=rc,
             sigma=sigma, M=M, m=m, window=window, long_method=long_method)
    eps_w = WIN_C * tol
    if m >= 0:
        sm = s0 * b ** m

        def cost_mid(P, h):
            pad = max(2.0 * ((P - 1) * h / 2.0 + h), sm * math.sqrt(math.log(PAD_C / tol)))
            return P ** 3 + FFT_COST * (Lx * Ly * (Lz + pad)) / (N * h ** 3)

        if window in ("kb", "es"):
            P, S, h, p.nu = choose_window_kb(s0, eps_w, tol, window)
        else:
            P, S, h = choose_window(s0, eps_w, tol, cost_mid)
        p.P, p.S = P, S
        p.Ix = friendly_even(math.ceil(Lx / h))
        p.Iy = friendly_even(math.ceil(Ly / h))
        p.Iz = max(1, math.ceil(Lz / h))
        Hz = (P - 1) * p.hz / 2.0
        pad = max(2.0 * (Hz + p.hz), sm * math.sqrt(math.log(PAD_C / tol)))   # R7
        p.Izs = z_friendly_even(math.ceil((Lz + pad) / p.hz))   # R7, R7-Z
    sl = s0 * b ** (m + 1)

    def cost_long(P, h):
        return P ** 2 + LONG_FFT_COST * (Lx * Ly) / (N * h ** 2)

    if window in ("kb", "es"):
        Pl, Sl, hl, p.nul = choose_window_kb(sl, eps_w, tol, window)   # R8 with R6-KB / R6-ES
    else:
        Pl, Sl, hl = choose_window(sl, eps_w, tol, cost_long)      # R8
    p.Pl, p.Sl = Pl, Sl
    p.Ilx = max(friendly_even(math.ceil(Lx / hl)), friendly_even(Pl))
    p.Ily = max(friendly_even(math.ceil(Ly / hl)), friendly_even(Pl))
    p.Pc = choose_cheb(Lz, sl, max(CHEB_C * tol, CHEB_FLOOR))        # R9
    if long_method == "direct":                                       # R8-D
        kcut = 2.0 * KAPPA * math.sqrt(math.log(1.0 / tol)) / sl
        p.Kx = math.ceil(kcut * Lx / (2.0 * math.pi))
        p.Ky = math.ceil(kcut * Ly / (2.0 * math.pi))
    for k, v in over.items():
        if not hasattr(p, k):
            raise KeyError(k)
        setattr(p, k, v)
    return p
