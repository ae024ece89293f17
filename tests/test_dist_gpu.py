"""x-slab decomposition on one GPU: R virtual ranks in one process (loopback
exchange backend), same kernels and exchange steps as the NCCL path.  The assembled result
must equal the single-GPU evaluation (same plan) to rounding and the oracle within 1e-12."""
import dataclasses

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import sog as O
from oracle.plan import TABLE1, make_plan
from synth import config_system

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b))


def slab_plan(name, N, R, tol=1e-6, half=False, window="gs"):
    xyz, q, L = config_system(name, N=N)
    if half:   # every particle in the lower half of x: the upper ranks own nothing
        xyz = xyz.copy()
        xyz[:, 0] = -0.5 * L[0] + 0.5 * (xyz[:, 0] + 0.5 * L[0])
    op = make_plan(len(q), *L, tol, window=window)
    if op.m >= 0 and op.Ix % R:
        ix = op.Ix
        while ix % R or ix % 2:
            ix += 1
        op = dataclasses.replace(op, Ix=ix)
    params = dataclasses.asdict(op)
    params["row"] = [r[0] for r in TABLE1].index(op.b)
    return xyz, q, L, op, params


def run_slabs(xyz, q, L, op, params, R):
    from paper_2412_04595_b200 import DistPlan, Plan, slab_owner
    owner = slab_owner(xyz[:, 0], L[0], R)
    idx = [np.nonzero(owner == r)[0] for r in range(R)]
    nmax = max(1, max(len(i) for i in idx))
    dp = DistPlan(len(q), nmax, L, op.tol, R, loopback=True, params=params)
    xs = [torch.from_numpy(np.ascontiguousarray(xyz[i])).cuda() for i in idx]
    qs = [torch.from_numpy(np.ascontiguousarray(q[i])).cuda() for i in idx]
    phis, fs = dp.eval(xs, qs)
    torch.cuda.synchronize()
    phi = np.empty(len(q))
    F = np.empty((len(q), 3))
    for r in range(R):
        phi[idx[r]] = phis[r].cpu().numpy()
        F[idx[r]] = fs[r].cpu().numpy()
    pl = Plan(len(q), L, op.tol, params=params)
    p1, F1 = pl.eval(torch.from_numpy(xyz).cuda(), torch.from_numpy(q).cuda())
    torch.cuda.synchronize()
    d = dp.describe()
    dp.close()
    pl.close()
    return phi, F, p1.cpu().numpy(), F1.cpu().numpy(), d


@pytest.mark.parametrize("R", [2, 3, 4])
def test_loopback_cube_matches_single_and_oracle(R):
    xyz, q, L, op, params = slab_plan("c5", 20000, R)
    phi, F, p1, F1, d = run_slabs(xyz, q, L, op, params, R)
    assert d["ranks"] == R and d["slab_planes"] * R == d["Ix"]
    assert rel(phi, p1) <= 1e-13 and rel(F, F1) <= 1e-13, (rel(phi, p1), rel(F, F1))
    phi_o, F_o = O.evaluate(op, xyz, q)
    assert rel(phi, phi_o) <= 1e-12 and rel(F, F_o) <= 1e-12, (rel(phi, phi_o), rel(F, F_o))


def test_loopback_kb_window_three_ranks():
    """x-slab path with the Kaiser-Bessel window (R6-KB): equals the single-GPU plan and the oracle."""
    xyz, q, L, op, params = slab_plan("c5", 20000, 3, window="kb")
    phi, F, p1, F1, _ = run_slabs(xyz, q, L, op, params, 3)
    assert rel(phi, p1) <= 1e-13 and rel(F, F1) <= 1e-13, (rel(phi, p1), rel(F, F1))
    phi_o, F_o = O.evaluate(op, xyz, q)
    assert rel(phi, phi_o) <= 1e-12 and rel(F, F_o) <= 1e-12, (rel(phi, phi_o), rel(F, F_o))


def test_loopback_slab_box_two_ranks():
    """c3 shape (thin slab, wide in x,y): two ranks, long-range proxies exercised."""
    xyz, q, L, op, params = slab_plan("c3", 8000, 2)
    phi, F, p1, F1, _ = run_slabs(xyz, q, L, op, params, 2)
    assert rel(phi, p1) <= 1e-13 and rel(F, F1) <= 1e-13, (rel(phi, p1), rel(F, F1))


def test_loopback_empty_ranks():
    """Every particle in the lower half of x: ranks 2, 3 of 4 own nothing (halo only)."""
    xyz, q, L, op, params = slab_plan("c5", 12000, 4, half=True)
    phi, F, p1, F1, _ = run_slabs(xyz, q, L, op, params, 4)
    assert rel(phi, p1) <= 1e-13 and rel(F, F1) <= 1e-13, (rel(phi, p1), rel(F, F1))


def test_nccl_plumbing_selftest():
    """The library's run-time-bound NCCL calls (communicator, grouped send/recv, all-reduce) on one
    GPU: the multi-GPU x-slab path uses exactly these calls."""
    from paper_2412_04595_b200 import load_library
    import ctypes
    lib = load_library()
    lib.sog_nccl_selftest.restype = ctypes.c_int
    torch.cuda.init()
    rc = lib.sog_nccl_selftest()
    assert rc == 0, lib.sog_last_error().decode()


def test_particle_outside_its_slab_is_rejected():
    from paper_2412_04595_b200 import DistPlan, SogError
    xyz, q, L, op, params = slab_plan("c5", 4000, 2)
    dp = DistPlan(len(q), len(q), L, op.tol, 2, loopback=True, params=params)
    x = torch.from_numpy(xyz).cuda()
    qq = torch.from_numpy(q).cuda()
    empty_x = torch.empty(0, 3, dtype=torch.float64, device="cuda")
    empty_q = torch.empty(0, dtype=torch.float64, device="cuda")
    with pytest.raises(SogError):       # all particles handed to rank 0
        dp.eval([x, empty_x], [qq, empty_q])
    dp.close()


def test_clustered_halo_is_rejected_without_overflow():
    """Every own particle of rank 0 sits within the halo width of its right edge, with a capacity
    far above the halo capacity: the selects must not write past their buffers, every rank must
    return the same error, and the plan must still evaluate a valid input afterwards."""
    from paper_2412_04595_b200 import DistPlan, SogError, slab_owner
    xyz, q, L, op, params = slab_plan("c5", 6000, 2)
    R = 2
    owner = slab_owner(xyz[:, 0], L[0], R)
    idx = [np.nonzero(owner == r)[0] for r in range(R)]
    nmax = 4 * max(len(i) for i in idx)
    dp = DistPlan(len(q), nmax, L, op.tol, R, loopback=True, params=params)
    cap = dp.describe()["halo_capacity"]
    assert cap < nmax
    n = min(nmax, 3 * cap)                       # > cap particles in rank 0's right halo strip
    rng = np.random.default_rng(5)
    c = np.empty((n, 3))
    c[:, 0] = -1e-3 * rng.random(n) - 1e-9       # just left of the slab edge x = 0
    c[:, 1] = (rng.random(n) - 0.5) * L[1]
    c[:, 2] = (rng.random(n) - 0.5) * L[2]
    cq = np.where(np.arange(n) % 2 == 0, 1.0, -1.0)
    if n % 2:
        cq[-1] = 0.0
    xs = [torch.from_numpy(c).cuda(), torch.from_numpy(np.ascontiguousarray(xyz[idx[1]])).cuda()]
    qs = [torch.from_numpy(cq).cuda(), torch.from_numpy(np.ascontiguousarray(q[idx[1]])).cuda()]
    with pytest.raises(SogError) as e:
        dp.eval(xs, qs)
    assert "capacity" in str(e.value)
    torch.cuda.synchronize()                     # no fault
    xs = [torch.from_numpy(np.ascontiguousarray(xyz[i])).cuda() for i in idx]
    qs = [torch.from_numpy(np.ascontiguousarray(q[i])).cuda() for i in idx]
    phis, _ = dp.eval(xs, qs)
    assert all(torch.isfinite(p).all() for p in phis)
    dp.close()


def test_dist_validation_errors():
    """The x-slab path rejects invalid input as sog_eval does (non-finite, z range, non-neutral),
    with the status summed over ranks (a rank's own particles need not be neutral)."""
    from paper_2412_04595_b200 import DistPlan, SogError, slab_owner
    xyz, q, L, op, params = slab_plan("c5", 4000, 2)
    owner = slab_owner(xyz[:, 0], L[0], 2)
    idx = [np.nonzero(owner == r)[0] for r in range(2)]
    dp = DistPlan(len(q), max(len(i) for i in idx), L, op.tol, 2, loopback=True, params=params)

    def run(x, qq):
        return dp.eval([torch.from_numpy(np.ascontiguousarray(x[i])).cuda() for i in idx],
                       [torch.from_numpy(np.ascontiguousarray(qq[i])).cuda() for i in idx])

    run(xyz, q)
    for mod, code in (("z", -3), ("nan", -4), ("q", -2)):
        x, qq = xyz.copy(), q.copy()
        j = idx[1][3]
        if mod == "z":
            x[j, 2] = 0.51 * L[2]
        elif mod == "nan":
            x[j, 1] = np.nan
        else:
            qq[j] += 0.25
        with pytest.raises(SogError) as e:
            run(x, qq)
        assert e.value.code == code, (mod, e.value.code)
    phis, _ = run(xyz, q)
    assert all(torch.isfinite(p).all() for p in phis)
    dp.close()


def test_output_tensor_validation():
    """Caller-supplied outputs of the wrong dtype, shape or device are refused before any write."""
    from paper_2412_04595_b200 import Plan
    xyz, q, L = config_system("c1", N=500)
    op = make_plan(len(q), *L, 1e-6)
    pl = Plan(len(q), L, 1e-6)
    x, qq = torch.from_numpy(xyz).cuda(), torch.from_numpy(q).cuda()
    good_phi = torch.empty(len(q), dtype=torch.float64, device="cuda")
    good_F = torch.empty(len(q), 3, dtype=torch.float64, device="cuda")
    for phi, F in ((good_phi.float(), good_F), (good_phi[:-1], good_F), (good_phi, good_F[:-1]),
                   (good_phi, good_F.cpu()), (good_phi, good_F.t().contiguous().t())):
        with pytest.raises(ValueError):
            pl.eval(x, qq, phi, F)
    pl.eval(x, qq, good_phi, good_F)
    assert torch.isfinite(good_phi).all()
    pl.close()


def test_dist_phase_timings_and_own_targets():
    """SOG_TIMING on the x-slab path: per-phase device times of local rank 0 (the near field runs on
    the side stream with own targets only); results unchanged by the timing mode."""
    from paper_2412_04595_b200 import DistPlan, slab_owner
    xyz, q, L, op, params = slab_plan("c5", 20000, 2)
    owner = slab_owner(xyz[:, 0], L[0], 2)
    idx = [np.nonzero(owner == r)[0] for r in range(2)]
    dp = DistPlan(len(q), max(len(i) for i in idx), L, op.tol, 2, loopback=True, params=params)
    xs = [torch.from_numpy(np.ascontiguousarray(xyz[i])).cuda() for i in idx]
    qs = [torch.from_numpy(np.ascontiguousarray(q[i])).cuda() for i in idx]
    p0, _ = dp.eval(xs, qs)
    dp.set_flags(validate=True, timing=True)
    p1, _ = dp.eval(xs, qs)
    t = dp.timings()
    assert len(t) == 12 and t["near"] > 0 and t["a2a_fwd"] > 0 and t["long_allreduce"] >= 0
    assert all(torch.equal(a, b) for a, b in zip(p0, p1))
    dp.close()
