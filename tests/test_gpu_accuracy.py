"""Accuracy of the GPU path against Ewald2D at the full BASELINE sizes (the paper's metric).

epsilon_r = relative L-infinity potential error vs Ewald2D (R13) at sampled
targets must be <= tol, with the LIBRARY's own plan rules (Plan(N, L, tol): R1-R9) at every
BASELINE configuration: c2 at 1e-4 / 1e-8 / 1e-12, c3, c4 (fp64, and fp32 mode at 1e-4), c5; also
c5 with the Kaiser-Bessel window and with the direct (non-FFT) long range.  Forces: relative L2
at the same targets <= 10 tol (the SPEC's acceptance factor; the plan's b-row bounds the
force error by tol on the decomposition, R1).  Ewald2D at N up to 1e7 is the target-subsampled
form of oracle/ewald2d.py in plain C loops (pinned to the NumPy form)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import ewald2d
from synth import config_system

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


CASES = [("c2", 1e-4, {}), ("c2", 1e-8, {}), ("c2", 1e-12, {}), ("c3", 1e-6, {}), ("c4", 1e-6, {}),
         ("c4", 1e-4, {"precision": "fp32"}), ("c5", 1e-6, {}), ("c5", 1e-6, {"window": "kb"}),
         ("c5", 1e-6, {"long_method": "direct"})]


@pytest.mark.parametrize("name,tol,kw", CASES, ids=[f"{c[0]}-{c[1]:g}-{'-'.join(c[2].values()) or 'default'}" for c in CASES])
def test_full_size_accuracy_vs_ewald2d(name, tol, kw):
    from paper_2412_04595_b200 import Plan
    xyz, q, L = config_system(name)
    N = len(q)
    pl = Plan(N, L, tol, **kw)
    phi, F = pl.eval(torch.from_numpy(xyz).cuda(), torch.from_numpy(q).cuda())
    phi, F = phi.cpu().numpy(), F.cpu().numpy()
    pl.close()
    nt = 32 if N >= 10 ** 7 else 64
    t = np.random.default_rng(11).choice(N, nt, replace=False)
    ref, g = ewald2d.ewald2d_targets(xyz, q, L, t, tol=min(1e-11, 1e-4 * tol))
    Fref = -q[t, None] * g
    eps_r = np.max(np.abs(phi[t] - ref)) / np.max(np.abs(ref))
    eF = np.linalg.norm(F[t] - Fref) / np.linalg.norm(Fref)
    print(f"{name} tol={tol:g} {kw}: eps_r={eps_r:.3e} force rel L2={eF:.3e}")
    assert eps_r <= tol, eps_r
    assert eF <= 10 * tol, eF
