"""CPU-only checks of the C-ABI library: it loads, exports every symbol include/sog.h
declares, and its host-side plan rules (sog_plan_choose) agree with the oracle's."""
import ctypes
import dataclasses
import os
import re

import pytest

from paper_2412_04595_b200 import sog as B
from oracle.plan import make_plan
from synth import CONFIGS

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "sog.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sog_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = B.load_library()
    names = header_functions()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(B.EXPORTS)


def test_nm_exports_are_c_symbols():
    out = os.popen(f"nm -D --defined-only {B.lib_path()}").read()
    for n in header_functions():
        assert re.search(rf"\bT {n}$", out, flags=re.M), n


CASES = [(c.name, c.N, c.L, t) for c in CONFIGS.values()
         for t in ((1e-4, 1e-6, 1e-8, 1e-12) if c.name == "c2" else (c.tol,))]
CASES += [("tiny", 2, (20.0, 20.0, 20.0), 1e-6), ("confined", 5000, (60.0, 60.0, 0.5), 1e-6),
          ("tall", 3000, (6.0, 7.0, 90.0), 1e-4), ("dense", 100000, (10.0, 10.0, 10.0), 1e-8)]


@pytest.mark.parametrize("window,long_method", [("gs", "fft"), ("kb", "fft"), ("es", "fft"), ("gs", "direct")])
@pytest.mark.parametrize("name,N,L,tol", CASES)
def test_plan_rules_match_oracle(name, N, L, tol, window, long_method):
    ora = dataclasses.asdict(make_plan(N, *L, tol, window=window, long_method=long_method))
    if long_method == "direct" and max(ora["Kx"], ora["Ky"]) > 63:
        with pytest.raises(B.SogError):       # too many modes for the direct sums (library bound)
            B.choose_params(N, L, tol, window=window, long_method=long_method)
        return
    lib_p = B.choose_params(N, L, tol, window=window, long_method=long_method)
    for k, v in ora.items():
        if k == "window":
            assert lib_p[k] == B.WINDOWS[v]
        elif k == "long_method":
            assert lib_p[k] == B.LONG_METHODS[v]
        elif isinstance(v, int):
            assert lib_p[k] == v, (k, lib_p[k], v)
        else:
            assert abs(lib_p[k] - v) <= 1e-13 * abs(v), (k, lib_p[k], v)


@pytest.mark.parametrize("name,N,L,tol", CASES)
def test_optimised_plan_matches_oracle(name, N, L, tol):
    """R20 (eq::optimiz with B200 costs): library and oracle pick the same plan."""
    lib_p = B.choose_params(N, L, tol, optimize=True)
    ora = dataclasses.asdict(make_plan(N, *L, tol, optimize=True))
    for k, v in ora.items():
        if k in ("window", "long_method"):
            continue
        if isinstance(v, int):
            assert lib_p[k] == v, (k, lib_p[k], v)
        else:
            assert abs(lib_p[k] - v) <= 1e-13 * abs(v), (k, lib_p[k], v)


def test_plan_choose_errors():
    lib = B.load_library()
    o = B.Opts()
    assert lib.sog_plan_choose(100, 10.0, 10.0, 10.0, 1e-15, ctypes.byref(o), None, 0) == -5
    assert lib.sog_plan_choose(0, 10.0, 10.0, 10.0, 1e-6, ctypes.byref(o), None, 0) == -1
    assert lib.sog_plan_choose(100, -1.0, 10.0, 10.0, 1e-6, ctypes.byref(o), None, 0) == -1
    assert b"tol" in lib.sog_last_error() or b"box" in lib.sog_last_error()
    # explicit parameters are validated: r_c beyond min(Lx,Ly)/2 is rejected
    p = dataclasses.asdict(make_plan(1000, 10.0, 10.0, 10.0, 1e-6))
    o.explicit_params = 1
    for k in B.PLAN_FIELDS:
        if k == "row":
            continue
        setattr(o, k, type(getattr(o, k))(p[k]))
    o.row = 3
    assert lib.sog_plan_choose(1000, 10.0, 10.0, 10.0, 1e-6, ctypes.byref(o), None, 0) > 0
    o.rc = 6.0
    assert lib.sog_plan_choose(1000, 10.0, 10.0, 10.0, 1e-6, ctypes.byref(o), None, 0) == -1
    o.rc = p["rc"]
    o.Izs = 10
    assert lib.sog_plan_choose(1000, 10.0, 10.0, 10.0, 1e-6, ctypes.byref(o), None, 0) == -1


def test_table1_row_selection():
    for tol, row in ((1e-2, 0), (1e-3, 1), (1e-4, 2), (1e-6, 3), (1e-8, 4), (1e-12, 5), (2e-14, 5)):
        assert B.choose_params(1000, (10.0, 10.0, 10.0), tol)["row"] == row


@pytest.mark.parametrize("b,tol", [(1.17, 1e-12), (1.25, 1e-8), (1.4, 1e-5)])
def test_general_b_c1_solve_matches_oracle(b, tol):
    """NEXT #4: the library's binary128 C^1 solve (plan.cpp c1_solve) and the oracle's 40-digit one
    (oracle/plan.py c1_solve) pick the same root; the plans agree field by field."""
    from paper_2412_04595_b200 import choose_params
    from oracle.plan import make_plan
    d = choose_params(2000, (12.0, 12.0, 12.0), tol, b=b)
    op = make_plan(2000, 12.0, 12.0, 12.0, tol, b=b)
    assert d["row"] == -1 and d["b"] == b
    assert abs(d["r0"] - op.r0) <= 1e-14 * op.r0 and abs(d["omega"] - op.omega) <= 1e-14
    for k in ("M", "m", "Ix", "Iy", "Izs", "P", "Pc", "Ilx"):
        assert d[k] == getattr(op, k), k


def test_sog_lib_override_stays_in_tree(monkeypatch, tmp_path):
    """SOG_LIB (A/B of in-tree builds) may name a build under the package's lib/ only."""
    lib_dir = os.path.dirname(B.lib_path())
    monkeypatch.setenv("SOG_LIB", "libsog_variant.so")
    assert B.lib_path() == os.path.join(os.path.realpath(lib_dir), "libsog_variant.so")
    monkeypatch.setenv("SOG_LIB", str(tmp_path / "libsog.so"))
    with pytest.raises(ImportError):
        B.lib_path()
    monkeypatch.delenv("SOG_LIB")
    assert B.lib_path() == os.path.join(lib_dir, "libsog.so")
