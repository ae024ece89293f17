"""Stage-by-stage GPU vs oracle comparison for one plan (diagnostics; not a test).
usage: python scripts/diag_stages.py CONFIG N TOL WINDOW"""
import dataclasses
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from oracle import sog as O  # noqa: E402
from oracle.plan import TABLE1, make_plan  # noqa: E402
from synth import config_system  # noqa: E402
from paper_2412_04595_b200 import Plan  # noqa: E402


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def run(op, xyz, q, label):
    d = dataclasses.asdict(op)
    d["row"] = [r[0] for r in TABLE1].index(op.b)
    pl = Plan(op.N, (op.Lx, op.Ly, op.Lz), op.tol, params=d)
    x = O.canonicalize(xyz, op)
    xd, qd = torch.from_numpy(xyz).cuda(), torch.from_numpy(q).cuda()
    out = [label, f"P={op.P} Pl={op.Pl} Pc={op.Pc} m={op.m}"]
    if op.m >= 0:
        S = O.mid_spread(op, x, q)
        Psi = O.mid_solve(op, S)
        g1 = pl.debug_stage(1, xd, qd).cpu().numpy()
        g2 = pl.debug_stage(2, xd, qd).cpu().numpy()
        out.append(f"S {rel(g1, S.transpose(2, 0, 1)):.2e} Psi {rel(g2, Psi.transpose(2, 0, 1)):.2e}")
    Sl = O.long_spread(op, x, q)
    Pl = O.long_solve(op, Sl)
    g3 = pl.debug_stage(3, xd, qd).cpu().numpy()
    g4 = pl.debug_stage(4, xd, qd).cpu().numpy()
    out.append(f"Sl {rel(g3, Sl):.2e} Psil {rel(g4, Pl):.2e}")
    comp = pl.components(xd, qd).cpu().numpy()
    _, _, parts = O.evaluate(op, xyz, q, parts=True)
    for c, k in enumerate(("near", "mid", "long")):
        po, go = parts[k]
        if np.linalg.norm(po) > 0:
            out.append(f"{k} phi {rel(comp[c][:, 0], po):.2e} grad {rel(comp[c][:, 1:], go):.2e}")
    print(" | ".join(out), flush=True)
    pl.close()


if __name__ == "__main__":
    cfg, N, tol = sys.argv[1], int(sys.argv[2]), float(sys.argv[3])
    for w in sys.argv[4].split(","):
        xyz, q, L = config_system(cfg, N=N)
        run(make_plan(len(q), *L, tol, window=w), xyz, q, f"{cfg} N={N} tol={tol:g} {w}")
