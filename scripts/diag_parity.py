"""Diagnostic: per-component and per-stage GPU vs oracle errors on a small case."""
import dataclasses, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import sog as O
from oracle.plan import make_plan, TABLE1
from paper_2412_04595_b200 import Plan
from synth import config_system

def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
N = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
xyz, q, L = config_system(name, N=N)
op = make_plan(len(q), *L, 1e-6)
d = dataclasses.asdict(op); d["row"] = [r[0] for r in TABLE1].index(op.b)
pl = Plan(len(q), L, 1e-6, params=d)
print("plan", op)
print("lib describe", pl.describe())
xd, qd = torch.from_numpy(xyz).cuda(), torch.from_numpy(q).cuda()
x = O.canonicalize(xyz, op)
phi_o, F_o, parts = O.evaluate(op, xyz, q, parts=True)
comp = pl.components(xd, qd).cpu().numpy()
for c, nm in enumerate(("near", "mid", "long")):
    po, go = parts[nm]
    print(nm, "phi rel %.3e grad rel %.3e  |o| %.3e |g| %.3e" % (rel(comp[c][:, 0], po), rel(comp[c][:, 1:], go),
          np.abs(po).max(), np.abs(comp[c][:, 0]).max()))
S_o = O.mid_spread(op, x, q); Psi_o = O.mid_solve(op, S_o)
Sl_o = O.long_spread(op, x, q); Psil_o = O.long_solve(op, Sl_o)
for st, ref in ((1, S_o.transpose(2, 0, 1)), (2, Psi_o.transpose(2, 0, 1)), (3, Sl_o), (4, Psil_o)):
    g = pl.debug_stage(st, xd, qd).cpu().numpy()
    print("stage", st, "rel %.3e  |ref| %.3e |g| %.3e" % (rel(g, ref), np.abs(ref).max(), np.abs(g).max()))
phi, F = pl.eval(xd, qd)
print("total phi rel %.3e F rel %.3e" % (rel(phi.cpu().numpy(), phi_o), rel(F.cpu().numpy(), F_o)))
