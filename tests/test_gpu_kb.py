"""GPU parity of the Kaiser-Bessel window path (R6-KB) against
the oracle's KB path (tests/test_oracle_kb.py pins it), through the C-ABI, element by element.
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


def test_kb_c1_components_and_total():
    xyz, q, L = config_system("c1")
    op = make_plan(len(q), *L, 1e-6, window="kb")
    assert op.window == "kb" and op.P == 9
    check_total(op, xyz, q)


def test_kb_c1_stages():
    """Alg. 1 step 1 / step 4 and Alg. 2 step 1 / step 4 grids with the KB window."""
    xyz, q, L = config_system("c1")
    op = make_plan(len(q), *L, 1e-6, window="kb")
    x = O.canonicalize(xyz, op)
    pl = gpu_plan(op)
    xd, qd = to_dev(xyz, q)
    S_o = O.mid_spread(op, x, q)
    Psi_o = O.mid_solve(op, S_o)
    Sl_o = O.long_spread(op, x, q)
    Psil_o = O.long_solve(op, Sl_o)
    for stage, ref in ((1, S_o.transpose(2, 0, 1)), (2, Psi_o.transpose(2, 0, 1)), (3, Sl_o), (4, Psil_o)):
        g = pl.debug_stage(stage, xd, qd).cpu().numpy()
        assert g.shape == ref.shape
        assert rel(g, ref) <= TOL_FP64, (stage, rel(g, ref))
        assert np.max(np.abs(g - ref)) <= 1e-12 * np.max(np.abs(ref))


@pytest.mark.parametrize("tol", [1e-4, 1e-8, 1e-12])
def test_kb_c2_tolerance_sweep_small(tol):
    xyz, q, L = config_system("c2", N=3000)
    check_total(make_plan(len(q), *L, tol, window="kb"), xyz, q)


@pytest.mark.parametrize("name", ["c3", "c4", "c5"])
def test_kb_shapes_small(name):
    """Slab (c3: long grid beyond the small-grid kernels), tall box (c4), cube (c5)."""
    xyz, q, L = config_system(name, N=5000)
    check_total(make_plan(len(q), *L, 1e-6, window="kb"), xyz, q)


def test_kb_paper_shape_and_degree():
    """Explicit plan with the paper's Section 5.1 choices (beta = 2.5 P, nu = 10)."""
    xyz, q, L = config_system("c1")
    op = make_plan(len(q), *L, 1e-8, window="kb")
    import dataclasses
    op = dataclasses.replace(op, S=2.5 * op.P, nu=10, Sl=2.5 * op.Pl, nul=10)
    check_total(op, xyz, q)


def test_kb_full_size_c2_sampled():
    """c2 at N=1e5, tol 1e-6, KB: 200 sampled targets computed by the oracle one by one."""
    xyz, q, L = config_system("c2")
    op = make_plan(len(q), *L, 1e-6, window="kb")
    t = np.random.default_rng(0).choice(len(q), 200, replace=False)
    phi_o, F_o = O.evaluate(op, xyz, q, targets=t)
    phi_g, F_g, _ = run_gpu(op, xyz, q)
    assert rel(phi_g[t], phi_o) <= TOL_FP64
    assert rel(F_g[t], F_o) <= TOL_FP64


@pytest.mark.parametrize("name,N", [("c4", 4000), ("c1", 1000), ("c5", 20000)])
def test_kb_fp32_mode_vs_fp64_oracle(name, N):
    xyz, q, L = config_system(name, N=N)
    op = make_plan(len(q), *L, 1e-4, window="kb")
    pl = gpu_plan(op, precision="fp32")
    x, qq = to_dev(xyz, q)
    phi, F = pl.eval(x, qq)
    torch.cuda.synchronize()
    phi_o, F_o = O.evaluate(op, xyz, q)
    e_phi, e_F = rel(phi.cpu().numpy(), phi_o), rel(F.cpu().numpy(), F_o)
    pl.close()
    assert e_phi <= TOL_FP32 and e_F <= TOL_FP32, (e_phi, e_F)


def test_kb_library_rules_vs_ewald():
    """The library's own KB rules (Plan(window="kb")) at c1 reach tol vs Ewald2D."""
    from paper_2412_04595_b200 import Plan
    from oracle import ewald2d
    xyz, q, L = config_system("c1")
    pl = Plan(len(q), L, 1e-6, window="kb")
    phi, F = pl.eval(*to_dev(xyz, q))
    t = np.arange(0, 1000, 25)
    ref, g = ewald2d.ewald2d(xyz, q, L, targets=t)
    phi = phi.cpu().numpy()[t]
    assert np.max(np.abs(phi - ref)) / np.max(np.abs(ref)) < 1e-6
    assert rel(F.cpu().numpy()[t], -q[t, None] * g) < 1e-5


# ------------------------------------------------------------------ ES window (R6-ES), same kernels
def test_es_c1_components_and_total():
    xyz, q, L = config_system("c1")
    check_total(make_plan(len(q), *L, 1e-6, window="es"), xyz, q)


@pytest.mark.parametrize("tol", [1e-4, 1e-8, 1e-12])
def test_es_c2_tolerance_sweep_small(tol):
    xyz, q, L = config_system("c2", N=3000)
    check_total(make_plan(len(q), *L, tol, window="es"), xyz, q)


def test_es_c5_small_and_fp32():
    xyz, q, L = config_system("c5", N=5000)
    check_total(make_plan(len(q), *L, 1e-6, window="es"), xyz, q)
    xyz, q, L = config_system("c4", N=4000)
    op = make_plan(len(q), *L, 1e-4, window="es")
    pl = gpu_plan(op, precision="fp32")
    x, qq = to_dev(xyz, q)
    phi, F = pl.eval(x, qq)
    torch.cuda.synchronize()
    phi_o, F_o = O.evaluate(op, xyz, q)
    pl.close()
    assert rel(phi.cpu().numpy(), phi_o) <= TOL_FP32 and rel(F.cpu().numpy(), F_o) <= TOL_FP32
