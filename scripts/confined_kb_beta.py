"""NEXT #3 (strongly confined regime): the paper's confined-regime long window (KB, nu = 8,
beta = 7.5 P) against this code's R6-KB rule (beta = 2.2 P, nu = P + 3), measured with the
oracle on the setting of the paper's Fig. thin (Lx = Ly = 100, N = 1000 random
monovalent charges, eta = 0.294 so that no mid-range solver is needed, gamma = Lx/Lz = 100 and 500).

For each long window support Pl the long-range potential by Algorithm 2 (window + 2D FFT per proxy
layer) is compared with Algorithm 3 (direct Fourier sums, no window, R8-D) at the same Chebyshev
proxies, so the difference is the window / grid error alone (Fig. thin (a)).  Test infrastructure:
calls only oracle/ and synth/.  Output: one line per (gamma, Pl, rule), relative L2 error of phi.

    python scripts/confined_kb_beta.py > profiles/r02_confined_kb_beta.txt
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from oracle import sog as O  # noqa: E402
from oracle.plan import make_plan  # noqa: E402


def system(N, L, Lz, seed):
    rng = np.random.default_rng(seed)
    xyz = np.column_stack([rng.uniform(-L / 2, L / 2, N), rng.uniform(-L / 2, L / 2, N),
                           rng.uniform(-Lz / 2, Lz / 2, N)])
    q = np.where(np.arange(N) % 2 == 0, 1.0, -1.0)
    return xyz, q


def main():
    N, L, tol = 1000, 100.0, 1e-10
    print("# gamma Pl rule beta nu rel_L2(phi_long, Alg.2 vs Alg.3) |  plan: Ilx Pc m")
    for gamma in (100.0, 500.0):
        Lz = L / gamma
        xyz, q = system(N, L, Lz, 7)
        base = make_plan(N, L, L, Lz, tol, window="kb", eta=0.294)
        assert base.m < 0, "eta = 0.294: all Gaussians long-range (no mid solver), as in P:1044"
        ref_plan = make_plan(N, L, L, Lz, tol, window="kb", eta=0.294, long_method="direct")
        xyz_c = O.canonicalize(xyz, ref_plan)
        phi_ref, _ = O.long_range(ref_plan, xyz_c, q)
        for Pl in (5, 7, 9, 11, 13):
            for rule, beta, nu in (("R6-KB", 2.2 * Pl, Pl + 3), ("paper-confined", 7.5 * Pl, 8),
                                   ("beta7.5P,nu=P+3", 7.5 * Pl, Pl + 3), ("beta2.2P,nu=8", 2.2 * Pl, 8)):
                p = make_plan(N, L, L, Lz, tol, window="kb", eta=0.294, Pl=Pl, Sl=beta, nul=nu,
                              Pc=ref_plan.Pc)
                phi, _ = O.long_range(p, O.canonicalize(xyz, p), q)
                err = np.linalg.norm(phi - phi_ref) / np.linalg.norm(phi_ref)
                print(f"{gamma:6.0f} {Pl:3d} {rule:15s} {beta:6.1f} {nu:3d} {err:.3e} | {p.Ilx} {p.Pc} {p.m}",
                      flush=True)


if __name__ == "__main__":
    main()
