""""SOG-exact" component references: the mid- and long-range SOG sums evaluated
without grids, FFTs, windows or Chebyshev proxies.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Used to pin the spectral
components of oracle/sog.py ("exact result within the paper's error bound")
and to isolate the SOG decomposition error against Ewald2D.

  mid:  sum_j q_j sum_{n in Z^2} sum_{l<=m} w_l exp(-|r_ij + n L|^2 / s_l^2)      (Eq. eq::SOGdecomp)
        real-space image sum when s_l <= min(Lx,Ly)/3, else the Poisson dual
        (pi s^2/A) exp(-z^2/s^2) sum_kdot exp(-s^2 kdot^2/4) cos(kdot . rho)
  long: (pi/A) sum_j q_j sum_{l>m} w_l s_l^2 [exp(-z^2/s_l^2) sum_{kdot!=0} exp(-s_l^2 kdot^2/4) cos(kdot.rho)
        + expm1(-z^2/s_l^2)]                                                    (Eq. eq::trun2; R10)
Both include the j = i, n = 0 term, like the spectral solvers (the self term
removes it).  Gradients are analytic.
"""
from __future__ import annotations

import math

import numpy as np


def _modes(L, s, tol=1e-17):
    Lx, Ly = L
    kmax = 2.0 * math.sqrt(-math.log(tol)) / s
    mx = int(math.ceil(kmax * Lx / (2 * math.pi)))
    my = int(math.ceil(kmax * Ly / (2 * math.pi)))
    a, b = np.meshgrid(np.arange(-mx, mx + 1), np.arange(-my, my + 1), indexing="ij")
    kx = 2 * math.pi * a.ravel() / Lx
    ky = 2 * math.pi * b.ravel() / Ly
    return kx, ky


def gaussian_lattice_sum(xyz, q, L, s, targets, drop_constant=False):
    """sum_j q_j sum_{n in Z^2} exp(-|r_ij + nL|^2/s^2) and its gradient at targets.
    drop_constant=True returns the R10 form (kdot=0 mode uses expm1)."""
    Lx, Ly, _ = L
    A = Lx * Ly
    out = np.zeros(len(targets))
    grad = np.zeros((len(targets), 3))
    real = (s <= min(Lx, Ly) / 3.0) and not drop_constant
    if real:
        R = s * math.sqrt(-math.log(1e-18))
        nx = int(math.ceil(R / Lx)) + 1
        ny = int(math.ceil(R / Ly)) + 1
    else:
        kx, ky = _modes((Lx, Ly), s)
        k2 = kx ** 2 + ky ** 2
        spec = np.exp(-s * s * k2 / 4.0)
        nz = k2 > 0
    for it, i in enumerate(targets):
        dx = xyz[i, 0] - xyz[:, 0]
        dy = xyz[i, 1] - xyz[:, 1]
        dz = xyz[i, 2] - xyz[:, 2]
        if real:
            for n1 in range(-nx, nx + 1):
                for n2 in range(-ny, ny + 1):
                    X = dx + n1 * Lx
                    Y = dy + n2 * Ly
                    e = q * np.exp(-(X * X + Y * Y + dz * dz) / (s * s))
                    out[it] += e.sum()
                    c = -2.0 / (s * s) * e
                    grad[it] += (np.sum(c * X), np.sum(c * Y), np.sum(c * dz))
        else:
            ez = np.exp(-dz * dz / (s * s))
            ph = kx[nz, None] * dx[None, :] + ky[nz, None] * dy[None, :]
            cs = np.cos(ph) * spec[nz, None]
            sn = np.sin(ph) * spec[nz, None]
            qz = q * ez
            pre = math.pi * s * s / A
            out[it] += pre * np.sum(cs @ qz)
            grad[it, 0] += pre * np.sum(-(kx[nz, None] * sn) @ qz)
            grad[it, 1] += pre * np.sum(-(ky[nz, None] * sn) @ qz)
            grad[it, 2] += pre * np.sum((cs.sum(0)) * q * ez * (-2.0 * dz / (s * s)))
            # kdot = 0 mode
            if drop_constant:
                out[it] += pre * np.sum(q * np.expm1(-dz * dz / (s * s)))
            else:
                out[it] += pre * np.sum(qz)
            grad[it, 2] += pre * np.sum(q * ez * (-2.0 * dz / (s * s)))
    return out, grad


def mid_exact(plan, xyz, q, targets):
    w, s = plan.weights()
    phi = np.zeros(len(targets))
    grad = np.zeros((len(targets), 3))
    L = (plan.Lx, plan.Ly, plan.Lz)
    for ell in range(plan.m + 1):
        p, g = gaussian_lattice_sum(xyz, q, L, s[ell], targets)
        phi += w[ell] * p
        grad += w[ell] * g
    return phi, grad


def long_exact(plan, xyz, q, targets):
    w, s = plan.weights()
    phi = np.zeros(len(targets))
    grad = np.zeros((len(targets), 3))
    L = (plan.Lx, plan.Ly, plan.Lz)
    for ell in range(plan.m + 1, plan.M + 1):
        p, g = gaussian_lattice_sum(xyz, q, L, s[ell], targets, drop_constant=True)
        phi += w[ell] * p
        grad += w[ell] * g
    return phi, grad


def sog_exact(plan, xyz, q, targets):
    """Near (exact) + mid_exact + long_exact - self: isolates the decomposition error."""
    from . import sog
    pn, gn = sog.near_field(plan, xyz, q, targets)
    pm, gm = mid_exact(plan, xyz, q, targets)
    pl, gl = long_exact(plan, xyz, q, targets)
    tq = q[np.asarray(targets)]
    phi = pn + pm + pl - tq * sog.self_coefficient(plan)
    return phi, -tq[:, None] * (gn + gm + gl), {"near": (pn, gn), "mid": (pm, gm), "long": (pl, gl)}
