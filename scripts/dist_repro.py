"""Small x-slab loopback reproduction (for compute-sanitizer runs)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
from test_dist_gpu import slab_plan, run_slabs, rel
R = int(sys.argv[1]) if len(sys.argv) > 1 else 2
N = int(sys.argv[2]) if len(sys.argv) > 2 else 4000
xyz, q, L, op, params = slab_plan("c5", N, R)
phi, F, p1, F1, d = run_slabs(xyz, q, L, op, params, R)
print(d)
print("rel phi", rel(phi, p1), "rel F", rel(F, F1))
