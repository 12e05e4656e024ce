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
    of the final (segments n-1..1) x segment-0 fold, with the reference's
    structure: zero-filled accumulator (merging.py:117), then per term m one
    read-modify-write axpy pass acc += alpha_m * hi_m (x) psi_0 (merging.py:
    86-94); for n >= 3 hi_m is the Kronecker product of segments n-1..1
    (the reference's _outer_into fold, merging.py:140-150), built per term.
    Returns (acc, seconds)."""
    lib = load()
    n = len(seg_states)
    lo_states = seg_states[0]
    width = len(lo_states[0])
    r0, r1 = rows
    t0 = time.perf_counter()
    acc = np.empty((r1 - r0) * width, dtype=np.complex128)
    lib.or_zero(acc.ctypes.data, acc.size, threads)
    for m in range(table.shape[1]):
        if n == 2:
            hi = np.ascontiguousarray(seg_states[1][table[1, m]])
            h0, h1 = r0, r1
        else:
            cur = seg_states[n - 1][table[n - 1, m]]
            for i in range(n - 2, 0, -1):
                cur = np.multiply.outer(cur, seg_states[i][table[i, m]]).ravel()
            hi = np.ascontiguousarray(cur[r0:r1])
            h0, h1 = 0, r1 - r0
        lo = np.ascontiguousarray(lo_states[table[0, m]])
        c = complex(coeffs[m])
        # or_axpy_outer writes acc rows [h0, h1) relative to row h0 of hi
        lib.or_axpy_outer(acc.ctypes.data, h0, h1, hi.ctypes.data, lo.ctypes.data, width, c.real, c.imag,
                          threads)
    return acc, time.perf_counter() - t0


def max_threads() -> int:
    return int(load().or_max_threads())
