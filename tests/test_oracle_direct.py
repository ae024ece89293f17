"""Pins of the oracle's long range without FFT (Algorithm 3, App. B; SURVEY.md 8(f)
NEXT #1): direct type-1 / type-2 Fourier sums over the R8-D mode set with two-sided Chebyshev
proxies (R9).  Checked against the SOG-exact long sum, the FFT variant and Ewald2D.
"""
import math

import numpy as np
import pytest

from oracle import plan as P
from oracle import sog, sog_exact, ewald2d
from synth import config_system


@pytest.mark.parametrize("name", ["c1", "c4"])
@pytest.mark.parametrize("tol", [1e-4, 1e-6, 1e-8, 1e-10, 1e-12])
def test_direct_long_converges_to_exact(name, tol):
    """Alg. 3 -> the SOG-exact long sum (Eq. eq::gridnonfft) within the plan tolerance."""
    xyz, q, L = config_system(name, N=400)
    t = np.arange(12)
    p = P.make_plan(len(q), *L, tol, long_method="direct")
    x = sog.canonicalize(xyz, p)
    ex = sog_exact.long_exact(p, x, q, t)
    sp = sog.long_range(p, x, q, t)
    assert np.max(np.abs(sp[0] - ex[0])) < 10 * tol
    assert np.max(np.abs(sp[1] - ex[1])) < 100 * tol


def test_direct_matches_fft_variant():
    """Alg. 3 and Alg. 2 compute the same long-range field up to their truncations."""
    xyz, q, L = config_system("c1", N=500)
    t = np.arange(20)
    for tol in (1e-6, 1e-10):
        pd = P.make_plan(len(q), *L, tol, long_method="direct")
        pf = P.make_plan(len(q), *L, tol)
        x = sog.canonicalize(xyz, pd)
        a, b = sog.long_range(pd, x, q, t), sog.long_range(pf, x, q, t)
        assert np.max(np.abs(a[0] - b[0])) < 10 * tol
        assert np.max(np.abs(a[1] - b[1])) < 100 * tol


def test_direct_mode_rule_and_spectrum_tail():
    """R8-D: the first excluded mode's Gaussian factor exp(-s^2 k^2/4) of the narrowest long-range
    Gaussian is below tol, and dropping the outermost modes costs accuracy."""
    xyz, q, L = config_system("c1", N=300)
    t = np.arange(8)
    p = P.make_plan(len(q), *L, 1e-8, long_method="direct")
    sl = p.weights()[1][p.m + 1]
    kx = 2 * math.pi * (p.Kx + 1) / p.Lx
    assert math.exp(-sl ** 2 * kx ** 2 / 4) < 1e-8
    x = sog.canonicalize(xyz, p)
    ex = sog_exact.long_exact(p, x, q, t)[0]
    import dataclasses
    e_full = np.max(np.abs(sog.long_range(p, x, q, t)[0] - ex))
    e_cut = np.max(np.abs(sog.long_range(dataclasses.replace(p, Kx=p.Kx - 2, Ky=p.Ky - 2), x, q, t)[0] - ex))
    assert e_cut > 10 * e_full


def test_direct_tall_narrow_box_few_modes():
    """Two charges in a tall, narrow box (Lz = 10 Lx: only kdot = 0 and the first ring of modes
    survive R8-D): Alg. 3 still matches the SOG-exact image sum."""
    p = P.make_plan(2, 6.0, 6.0, 60.0, 1e-6, long_method="direct")
    xyz = np.array([[0.3, -0.7, 1.1], [-1.2, 0.4, -2.0]])
    q = np.array([1.0, -1.0])
    x = sog.canonicalize(xyz, p)
    ex = sog_exact.long_exact(p, x, q, np.arange(2))
    sp = sog.long_range(p, x, q, np.arange(2))
    assert np.max(np.abs(sp[0] - ex[0])) < 1e-5
    assert np.max(np.abs(sp[1] - ex[1])) < 1e-4


@pytest.mark.parametrize("name,N,tol", [("c1", 1000, 1e-6), ("c4", 3000, 1e-6), ("c2", 1500, 1e-8)])
def test_direct_total_vs_ewald2d(name, N, tol):
    """epsilon_r <= tol with Alg. 3 as the long-range solver."""
    xyz, q, L = config_system(name, N=N)
    t = np.arange(24)
    p = P.make_plan(len(q), *L, tol, long_method="direct")
    phi, F = sog.evaluate(p, xyz, q, targets=t)
    ref, g = ewald2d.ewald2d(xyz, q, L, targets=t)
    assert np.max(np.abs(phi - ref)) / np.max(np.abs(ref)) < tol
    Fref = -q[t, None] * g
    assert np.linalg.norm(F - Fref) / np.linalg.norm(Fref) < 10 * tol
