"""TEST INFRASTRUCTURE ONLY — ctypes loader of oracle/build/liboracle.so (the C
restatement of the reference kernels) plus the bounded CPU-baseline runner
used by bench.py. Not importable from the product package."""
from __future__ import annotations

import ctypes
import os
import subprocess
import time

import numpy as np

from . import cutbench_oracle as orc

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "build", "liboracle.so")
_lib = None


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        lib = ctypes.CDLL(LIB)
        vp, i64, i32, f64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
        lib.or_run_gates.argtypes = [vp, i32, vp, vp, vp, vp, i64, i64, i32]
        lib.or_axpy_outer.argtypes = [vp, i64, i64, vp, vp, i64, f64, f64, i32]
        lib.or_outer_into.argtypes = [vp, vp, i64, vp, i64, i32]
        lib.or_zero.argtypes = [vp, i64, i32]
        lib.or_max_threads.restype = i32
        _lib = lib
    return _lib


def simulate(q, kinds, qa, qb, params=None, threads=1):
    lib = load()
    amps = orc.zero_state(q)
    k = np.ascontiguousarray(kinds, np.uint8)
    a = np.ascontiguousarray(qa, np.int64)
    b = np.ascontiguousarray(qb, np.int64)
    p = np.ascontiguousarray(params if params is not None else np.zeros((len(k), 3)), np.float64)
    lib.or_run_gates(amps.ctypes.data, q, k.ctypes.data, a.ctypes.data, b.ctypes.data, p.ctypes.data,
                     0, len(k), threads)
    return amps


def merge_rows(seg_states, table, coeffs, rows, threads=1):
    """Reference merge (merging.py:156-186) restricted to output rows [r0, r1)
    of the final (hi x seg0) fold, n = 2 only. Returns (acc, seconds)."""
    lib = load()
    if len(seg_states) != 2:
        raise ValueError("bounded C merge sample supports n = 2")
    lo_states, hi_states = seg_states
    width = len(lo_states[0])
    r0, r1 = rows
    t0 = time.perf_counter()
    acc = np.empty((r1 - r0) * width, dtype=np.complex128)
    lib.or_zero(acc.ctypes.data, acc.size, threads)
    for m in range(table.shape[1]):
        hi = np.ascontiguousarray(hi_states[table[1, m]])
        lo = np.ascontiguousarray(lo_states[table[0, m]])
        c = complex(coeffs[m])
        lib.or_axpy_outer(acc.ctypes.data, r0, r1, hi.ctypes.data, lo.ctypes.data, width, c.real, c.imag,
                          threads)
    return acc, time.perf_counter() - t0


def max_threads() -> int:
    return int(load().or_max_threads())
