"""CPU oracle for the spectral SOG quasi-2D electrostatics hot path.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s `cpu_baseline` / `--impl reference` legs may import or run
anything under `oracle/`.  The product path (`paper_2412_04595_b200`) never
does, and shares no code, tables or constants with it.

Modules
  plan       -- parameter selection rules R1-R9, Table 1, the window
                rules R6-KB / R6-ES, the direct long-range modes R8-D, the R20 optimiser.
  sog        -- the step-by-step spectral SOG evaluation (near, mid, long by Alg. 2 or Alg. 3,
                self) with Gaussian, Kaiser-Bessel or ES windows.
  ewald2d    -- textbook Ewald2D (Parry 1975) reference, the oracle's own check.
  sog_exact  -- "SOG-exact" component references (image sums / Poisson dual).

Parity status: every function is pinned by a `-m "not gpu"` test in
tests/test_oracle_*.py except where its docstring says "parity unpinned".
"""
