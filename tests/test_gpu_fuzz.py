"""Randomised parity sweep: seeded random boxes (aspect ratios from strongly confined to tall),
particle counts (ragged, not multiples of any tile), tolerances, windows and long-range methods,
each checked element-wise against the oracle at the fp64 bar (R13)."""
import numpy as np
import pytest

from oracle.plan import make_plan
from synth import uniform_system

from test_gpu_parity import check_total, need_gpu

pytestmark = pytest.mark.gpu

TOLS = (1e-4, 1e-6, 1e-8, 1e-10)


def case(seed):
    rng = np.random.default_rng(9000 + seed)
    N = int(rng.integers(300, 2500))
    rho = float(rng.uniform(0.3, 3.0))
    aspect = float(10.0 ** rng.uniform(-1.5, 1.0))         # Lz / Lx from 0.03 to 10
    lx = (N / rho / aspect) ** (1.0 / 3.0)
    L = (lx, lx * float(rng.uniform(0.8, 1.25)), lx * aspect)
    tol = TOLS[int(rng.integers(len(TOLS)))]
    window = ("gs", "kb", "es")[int(rng.integers(3))]
    xyz, q = uniform_system(N, L, 9100 + seed)
    return xyz, q, L, tol, window


@pytest.fixture(autouse=True)
def _gpu():
    need_gpu()


@pytest.mark.parametrize("seed", range(16))
def test_random_systems(seed):
    xyz, q, L, tol, window = case(seed)
    try:
        op = make_plan(len(q), *L, tol, window=window)
    except ValueError:
        pytest.skip("box outside the plan rules (r_c > min(Lx, Ly)/2)")
    if op.Pc > 32 or op.Pl > 25 or (op.m >= 0 and op.P > 25) or (window != "gs" and (op.Pl > 17 or op.P > 17)):
        pytest.skip("plan outside the compiled ranges")
    check_total(op, xyz, q)
    if op.Kx == 0:
        opd = make_plan(len(q), *L, tol, window=window, long_method="direct")
        if max(opd.Kx, opd.Ky) <= 6:
            check_total(opd, xyz, q)
