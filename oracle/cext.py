"""ctypes loader for oracle/c/oracle_c.c (plain C loops for full-size oracle runs).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  build() compiles it with gcc (-O2, OpenMP);
`ensure_built()` does the same on first use when the library is missing or stale.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "c", "oracle_c.c")
LIB = os.path.join(HERE, "lib", "liboracle_c.so")
_lib = None


def ensure_built(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        os.makedirs(os.path.dirname(LIB), exist_ok=True)
        # -O2 without -ffast-math: IEEE arithmetic in the order written
        subprocess.run(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", SRC, "-o", LIB + ".tmp", "-lm"], check=True)
        os.replace(LIB + ".tmp", LIB)
    return LIB


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(ensure_built())
        P = ctypes.c_void_p
        i64, d = ctypes.c_int64, ctypes.c_double
        L.oracle_mid_spread.argtypes = [i64, ctypes.c_int, i64, i64, i64, P, P, P, P, P, P, P, P]
        L.oracle_mid_spread.restype = None
        L.oracle_ewald2d.argtypes = [i64, P, P, d, d, i64, P, d, d, d, P, P]
        L.oracle_ewald2d.restype = None
        _lib = L
    return _lib


def ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)
