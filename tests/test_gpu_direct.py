"""GPU parity of the long range without FFT (Algorithm 3, App. B; SURVEY.md 8(f) NEXT #1,
DESIGN.md R8-D) against the oracle's Alg. 3 (tests/test_oracle_direct.py pins it), through the C-ABI.
"""
import numpy as np
import pytest
import torch

from oracle import sog as O
from oracle.plan import make_plan
from synth import config_system

from test_gpu_parity import TOL_FP32, TOL_FP64, check_total, gpu_plan, need_gpu, rel, run_gpu, to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _gpu():
    need_gpu()


def test_direct_c1_components_and_total():
    xyz, q, L = config_system("c1")
    op = make_plan(len(q), *L, 1e-6, long_method="direct")
    check_total(op, xyz, q)


@pytest.mark.parametrize("tol", [1e-4, 1e-8, 1e-12])
def test_direct_c2_tolerance_sweep_small(tol):
    xyz, q, L = config_system("c2", N=3000)
    check_total(make_plan(len(q), *L, tol, long_method="direct"), xyz, q)


@pytest.mark.parametrize("name", ["c4", "c5"])
def test_direct_shapes_small(name):
    xyz, q, L = config_system(name, N=5000)
    check_total(make_plan(len(q), *L, 1e-6, long_method="direct"), xyz, q)


def test_direct_with_kb_window():
    xyz, q, L = config_system("c5", N=5000)
    check_total(make_plan(len(q), *L, 1e-8, long_method="direct", window="kb"), xyz, q)


def test_direct_full_size_c4_sampled():
    """c4 (N=1e6, tall box) with Alg. 3: 100 sampled targets computed by the oracle."""
    xyz, q, L = config_system("c4")
    op = make_plan(len(q), *L, 1e-6, long_method="direct")
    t = np.random.default_rng(4).choice(len(q), 100, replace=False)
    phi_o, F_o = O.evaluate(op, xyz, q, targets=t)
    phi_g, F_g, _ = run_gpu(op, xyz, q)
    assert rel(phi_g[t], phi_o) <= TOL_FP64
    assert rel(F_g[t], F_o) <= TOL_FP64


def test_direct_fp32_mode():
    xyz, q, L = config_system("c4", N=4000)
    op = make_plan(len(q), *L, 1e-4, long_method="direct")
    pl = gpu_plan(op, precision="fp32")
    x, qq = to_dev(xyz, q)
    phi, F = pl.eval(x, qq)
    torch.cuda.synchronize()
    phi_o, F_o = O.evaluate(op, xyz, q)
    pl.close()
    assert rel(phi.cpu().numpy(), phi_o) <= TOL_FP32 and rel(F.cpu().numpy(), F_o) <= TOL_FP32


def test_direct_rejections():
    """Too many modes (a wide box) and the FFT-only debug stages are refused with an error."""
    from paper_2412_04595_b200 import Plan, SogError
    with pytest.raises(SogError):
        Plan(100000, (400.0, 400.0, 1.0), 1e-6, long_method="direct")
    xyz, q, L = config_system("c1")
    pl = gpu_plan(make_plan(len(q), *L, 1e-6, long_method="direct"))
    with pytest.raises(SogError):
        pl.debug_stage(3, *to_dev(xyz, q))
    pl.close()


def test_direct_library_rules_vs_ewald():
    from paper_2412_04595_b200 import Plan
    from oracle import ewald2d
    xyz, q, L = config_system("c1")
    pl = Plan(len(q), L, 1e-6, long_method="direct")
    phi, F = pl.eval(*to_dev(xyz, q))
    t = np.arange(0, 1000, 25)
    ref, g = ewald2d.ewald2d(xyz, q, L, targets=t)
    phi = phi.cpu().numpy()[t]
    assert np.max(np.abs(phi - ref)) / np.max(np.abs(ref)) < 1e-6
    assert rel(F.cpu().numpy()[t], -q[t, None] * g) < 1e-5
