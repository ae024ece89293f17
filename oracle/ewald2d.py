"""Ewald2D reference for quasi-2D periodic Coulomb sums -- the oracle's own check.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  The paper's "true" solution
is Ewald2D (Parry 1975), cited without formula; this
is the textbook form.  With splitting parameter alpha and
A = Lx Ly, for target i (target-subsampled: cost O(N (images + modes)) each):

  real:       sum_j sum'_n q_j erfc(alpha |r_ij+n|)/|r_ij+n|
  kdot != 0:  (pi/A) sum_j q_j sum_k cos(k.rho_ij)/k [g(k,z_ij) + g(k,-z_ij)],
              g(k,z) = exp(kz) erfc(k/(2 alpha) + alpha z)
  kdot == 0:  -(2 pi/A) sum_j q_j [z_ij erf(alpha z_ij) + exp(-alpha^2 z_ij^2)/(alpha sqrt(pi))]
  self:       -2 alpha q_i / sqrt(pi)

and the analytic gradient of each term.  Pinned by alpha-independence and by
the alpha -> infinity quasi-2D limits (tests/test_oracle_pins.py::test_ewald2d_*).
"""
from __future__ import annotations

import math

import numpy as np
from scipy.special import erfc, erfcx, erf

_SQPI = math.sqrt(math.pi)


def _g(k, z, alpha):
    """g(k,z) = exp(kz) erfc(k/(2 alpha) + alpha z), evaluated stably."""
    x = k / (2.0 * alpha) + alpha * z
    pos = x >= 0
    out = np.empty(np.broadcast(k, z).shape)
    kk = np.broadcast_to(k, out.shape)
    zz = np.broadcast_to(z, out.shape)
    xx = np.broadcast_to(x, out.shape)
    out[pos] = erfcx(xx[pos]) * np.exp(-(kk[pos] / (2 * alpha)) ** 2 - (alpha * zz[pos]) ** 2)
    neg = ~pos
    out[neg] = np.exp(kk[neg] * zz[neg]) * erfc(xx[neg])
    return out


def ewald2d(xyz, q, L, targets=None, alpha=None, tol=1e-16):
    """Potential phi_i (self excluded) and gradient grad_i phi at the targets."""
    xyz = np.asarray(xyz, dtype=np.float64)
    q = np.asarray(q, dtype=np.float64)
    Lx, Ly, Lz = L
    A = Lx * Ly
    N = len(q)
    tgt = np.arange(N) if targets is None else np.asarray(targets)
    if alpha is None:
        alpha = 3.0 / min(Lx, Ly)
    rcut = math.sqrt(-math.log(tol)) / alpha + 0.0            # erfc(a r) ~ exp(-(a r)^2)
    kcut = 2.0 * alpha * math.sqrt(-math.log(tol))
    nx = int(math.ceil(rcut / Lx)) + 1
    ny = int(math.ceil(rcut / Ly)) + 1
    mx = int(math.ceil(kcut * Lx / (2 * math.pi)))
    my = int(math.ceil(kcut * Ly / (2 * math.pi)))
    # half-plane of kdot != 0 modes (pair k, -k): factor 2
    modes = []
    for a in range(0, mx + 1):
        for b in range(-my, my + 1):
            if a == 0 and b <= 0:
                continue
            kx, ky = 2 * math.pi * a / Lx, 2 * math.pi * b / Ly
            k = math.hypot(kx, ky)
            if k <= kcut:
                modes.append((kx, ky, k))
    modes = np.array(modes)
    phi = np.zeros(len(tgt))
    grad = np.zeros((len(tgt), 3))
    for it, i in enumerate(tgt):
        dx = xyz[i, 0] - xyz[:, 0]
        dy = xyz[i, 1] - xyz[:, 1]
        dz = xyz[i, 2] - xyz[:, 2]
        # real space
        for n1 in range(-nx, nx + 1):
            for n2 in range(-ny, ny + 1):
                X = dx + n1 * Lx
                Y = dy + n2 * Ly
                r = np.sqrt(X * X + Y * Y + dz * dz)
                mask = r < rcut
                if n1 == 0 and n2 == 0:
                    mask[i] = False
                if not mask.any():
                    continue
                rr = r[mask]
                qq = q[mask]
                er = erfc(alpha * rr)
                phi[it] += np.sum(qq * er / rr)
                dfr = -(er / rr ** 2 + 2 * alpha / _SQPI * np.exp(-(alpha * rr) ** 2) / rr)
                c = qq * dfr / rr
                grad[it, 0] += np.sum(c * X[mask])
                grad[it, 1] += np.sum(c * Y[mask])
                grad[it, 2] += np.sum(c * dz[mask])
        # kdot != 0 (each half-plane mode counted twice)
        if len(modes):
            kx = modes[:, 0:1]
            ky = modes[:, 1:2]
            k = modes[:, 2:3]
            ph = kx * dx[None, :] + ky * dy[None, :]
            gp = _g(k, dz[None, :], alpha)
            gm = _g(k, -dz[None, :], alpha)
            c = 2.0 * (math.pi / A) * q[None, :] / k
            cs = np.cos(ph)
            sn = np.sin(ph)
            phi[it] += np.sum(c * cs * (gp + gm))
            grad[it, 0] += np.sum(-c * kx * sn * (gp + gm))
            grad[it, 1] += np.sum(-c * ky * sn * (gp + gm))
            grad[it, 2] += np.sum(c * cs * k * (gp - gm))
        # kdot == 0
        phi[it] += -(2 * math.pi / A) * np.sum(q * (dz * erf(alpha * dz) + np.exp(-(alpha * dz) ** 2) / (alpha * _SQPI)))
        grad[it, 2] += -(2 * math.pi / A) * np.sum(q * erf(alpha * dz))
        # self
        phi[it] += -2.0 * alpha * q[i] / _SQPI
    return phi, grad


def ewald2d_targets(xyz, q, L, targets, tol=1e-12, alpha=None):
    """ewald2d() at sampled targets for large N (target-subsampled use): the same
    sums in plain C loops (oracle/c/oracle_c.c: oracle_ewald2d, one target per thread), with the
    real-space cutoff erfc(alpha r_cut) ~ tol and k_cut = 2 alpha sqrt(-ln tol).  alpha (a free
    splitting parameter: the result is alpha-independent) is chosen to minimise the loop count
    N (images + pairs + modes) per target.  Pinned equal to ewald2d at small N
    (tests/test_oracle_pins.py::test_ewald2d_c_loops_equal_numpy)."""
    from . import cext
    xyz = np.ascontiguousarray(xyz, dtype=np.float64)
    q = np.ascontiguousarray(q, dtype=np.float64)
    Lx, Ly, Lz = L
    N = len(q)
    rho = N / (Lx * Ly * Lz)
    s = math.sqrt(-math.log(tol))
    if alpha is None:
        best = None
        for a in np.geomspace(1e-3, 10.0, 400) / min(Lx, Ly) * 10:
            rc, kc = s / a, 2.0 * a * s
            shifts = (2 * (math.ceil(rc / Lx) + 1) + 1) * (2 * (math.ceil(rc / Ly) + 1) + 1)
            pairs = rho * min(4.0 / 3.0 * math.pi * rc ** 3, math.pi * rc * rc * Lz)
            modes = 0.5 * math.pi * (kc * Lx / (2 * math.pi)) * (kc * Ly / (2 * math.pi))
            cost = 1.5 * shifts * N + 25.0 * pairs + 80.0 * (modes + 1) * N
            if best is None or cost < best[0]:
                best = (cost, a)
        alpha = best[1]
    rcut = s / alpha
    kcut = 2.0 * alpha * s
    t = np.ascontiguousarray(np.asarray(targets, dtype=np.int64))
    phi = np.zeros(len(t))
    grad = np.zeros((len(t), 3))
    cext.lib().oracle_ewald2d(N, cext.ptr(xyz), cext.ptr(q), Lx, Ly, len(t), cext.ptr(t), alpha, rcut, kcut,
                              cext.ptr(phi), cext.ptr(grad))
    return phi, grad
