"""Builds (gcc) and loads oracle.c -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py)."""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(_HERE, "oracle.c")
SO = os.path.join(_HERE, "liboracle.so")
# No fast-math, no FMA contraction: every product is rounded before it is added (reading R14).
CFLAGS = ["-O2", "-fno-fast-math", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared", "-std=c11"]

_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(SO) or os.path.getmtime(SO) < os.path.getmtime(SRC):
        tmp = SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, SRC, "-o", tmp])
        os.replace(tmp, SO)
    return SO


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(SO)
        P = ctypes.POINTER
        i64p, f64p, u8p = P(ctypes.c_int64), P(ctypes.c_double), P(ctypes.c_uint8)
        L.orc_contract_naive.argtypes = [ctypes.c_int, i64p, i64p, i64p, i64p, ctypes.c_int, i64p, i64p,
                                         i64p, f64p, f64p, f64p, u8p, ctypes.c_double, ctypes.c_double]
        L.orc_contract_naive.restype = None
        L.orc_contract_gathered.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, f64p, f64p, f64p]
        L.orc_contract_gathered.restype = None
        L.orc_dot.argtypes = [ctypes.c_int64, f64p, f64p]
        L.orc_dot.restype = ctypes.c_double
        L.orc_dots.argtypes = [ctypes.c_int64, ctypes.c_int64, f64p, f64p, f64p]
        L.orc_dots.restype = None
        L.orc_matvec.argtypes = [ctypes.c_int64, ctypes.c_int64, f64p, f64p, f64p]
        L.orc_matvec.restype = None
        L.orc_contract3_naive.argtypes = [ctypes.c_int, i64p, i64p, i64p, i64p, i64p, ctypes.c_int, i64p, i64p,
                                          i64p, i64p, f64p, f64p, f64p, f64p, u8p, ctypes.c_double,
                                          ctypes.c_double]
        L.orc_contract3_naive.restype = None
        _lib = L
    return _lib


def ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(ctypes.POINTER(ctype))


def i64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64))


def f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))
