"""ctypes binding of libcutsim.so (the sm_100a C-ABI declared in include/cutsim.h).

There is no CPU fallback: if the library or a CUDA device is missing, every
compute entry point raises ``NativeUnavailableError``.
"""
from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from .errors import (
    BudgetExceededError,
    CapacityError,
    CutbenchError,
    DeviceError,
    NativeUnavailableError,
    UnsupportedTopologyError,
    ValidationError,
)

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libcutsim.so")

CS_C128 = 0
CS_C64 = 1

_ERRORS = {
    1: ValidationError,
    2: CapacityError,
    3: DeviceError,
    4: DeviceError,
    5: CutbenchError,
    6: NativeUnavailableError,
    7: UnsupportedTopologyError,
    8: BudgetExceededError,
}

_i32, _i64, _u64, _vp, _dp = (ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_void_p,
                              ctypes.POINTER(ctypes.c_double))

# name -> (restype, argtypes); exactly the functions include/cutsim.h declares
SIGNATURES = {
    "cs_version": (ctypes.c_int, []),
    "cs_last_error": (ctypes.c_char_p, []),
    "cs_device_count": (ctypes.c_int, [_vp]),
    "cs_set_option": (ctypes.c_int, [ctypes.c_char_p, _i64]),
    "cs_get_option": (_i64, [ctypes.c_char_p]),
    "cs_launch_count": (_i64, []),
    "cs_jit_wait": (ctypes.c_int, [ctypes.c_double]),
    "cs_init_basis": (ctypes.c_int, [_vp, _i32, _i64, _i64, _i32, _vp]),
    "cs_copy_to_host": (ctypes.c_int, [_vp, _vp, _i64, _vp]),
    "cs_sim_families": (ctypes.c_int, [_i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _vp]),
    "cs_sim_batch": (ctypes.c_int, [_i32, _vp, _vp, _vp, _vp, _vp, _i64, _vp, _i64, _i64, _u64, _i32,
                                    _i32, _vp]),
    "cs_sim_batch_until": (ctypes.c_int, [_i32, _vp, _vp, _vp, _vp, _vp, _i64, _vp, _i64, _i64, _u64, _i32,
                                          _i32, _vp, ctypes.c_double]),
    "cs_sweep_plan_json": (ctypes.c_int, [_i32, _vp, _vp, _vp, _vp, _vp, _i64, _i32, _i32, _vp, _i64,
                                          _vp]),
    "cs_jit_selftest": (ctypes.c_int, [_i32, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i32, _vp]),
    "cs_merge_terms": (ctypes.c_int, [_i32, _i32, _vp, _vp, _vp, _vp, _i64, _vp, _i64, _i64, _i64,
                                      _vp, _i64, _i32, _i32, _vp]),
    "cs_merge_chain_plan": (ctypes.c_int, [_i32, _vp, _vp, _vp, _i32, _vp, _vp, _i32, _i32, _vp, _vp,
                                           _vp]),
    "cs_merge_chain": (ctypes.c_int, [_i32, _vp, _vp, _vp, _vp, _i32, _vp, _vp, _i32, _i64, _i64, _vp,
                                      _vp, _i64, _i32, _vp]),
    "cs_cut_workspace": (ctypes.c_int, [_i32, _vp, _vp, _vp, _vp, _i64, _i32, _vp, _i32, _i32, _vp, _vp,
                                        _vp]),
    "cs_cut_run": (ctypes.c_int, [_i32, _vp, _vp, _vp, _vp, _i64, _i32, _vp, _i32, _i64, _i64, _vp, _vp,
                                  _i64, _i32, _vp, _vp, _vp]),
    "cs_cut_shard_plan": (ctypes.c_int, [_i32, _vp, _vp, _vp, _vp, _i64, _i32, _vp, _i32, _i32, _i32, _vp]),
    "cs_cut_run_sharded": (ctypes.c_int, [_i32, _vp, _vp, _vp, _vp, _i64, _i32, _vp, _vp, _i32, _i32, _i64, _i64,
                                          _vp, _vp, _i64, _i32, _vp, _vp, _vp]),
    "cs_cut_host_workspace": (ctypes.c_int, [_i32, _vp, _vp, _vp, _vp, _i64, _i32, _vp, _i32, _i32, _vp]),
    "cs_cut_run_to_host": (ctypes.c_int, [_i32, _vp, _vp, _vp, _vp, _i64, _i32, _vp, _i32, _vp, _vp, _i64, _i32,
                                          _vp, _vp]),
    "cs_cut_describe_json": (ctypes.c_int, [_i32, _vp, _vp, _vp, _vp, _i64, _i32, _vp, _vp, _i64, _vp]),
    "cs_cut_tables": (ctypes.c_int, [_i32, _vp, _vp, _vp, _vp, _i64, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                     _vp, _vp, _i64, _i64, _vp]),
    "cs_maxabsdiff": (ctypes.c_int, [_vp, _vp, _i64, _i32, _vp, _vp]),
    "cs_maxabs": (ctypes.c_int, [_vp, _i64, _i32, _vp, _vp]),
    "cs_inner": (ctypes.c_int, [_vp, _vp, _i64, _i32, _vp, _vp]),
    "cs_gather": (ctypes.c_int, [_vp, _vp, _i64, _vp, _i32, _vp]),
    "cs_nccl_load": (ctypes.c_int, [ctypes.c_char_p]),
    "cs_nccl_unique_id": (ctypes.c_int, [_vp]),
    "cs_nccl_comm_init": (ctypes.c_int, [_i32, _i32, _vp, _i32, _vp]),
    "cs_nccl_comm_destroy": (ctypes.c_int, [_vp]),
    "cs_allgather_states": (ctypes.c_int, [_vp, _vp, _i64, _vp, _vp]),
    "cs_sendrecv": (ctypes.c_int, [_vp, _vp, _vp, _i64, _i32, _vp]),
}

_lock = threading.Lock()
_lib = None
_load_error = None


def load() -> ctypes.CDLL:
    """Load (once) and type the library; raise NativeUnavailableError if absent."""
    global _lib, _load_error
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise NativeUnavailableError(
                f"{LIB_PATH} is not built; run __graft_entry__.build() (nvcc, sm_100a). "
                "This package has no CPU fallback."
            )
        try:
            lib = ctypes.CDLL(LIB_PATH)
        except OSError as exc:
            _load_error = exc
            raise NativeUnavailableError(f"cannot load {LIB_PATH}: {exc}") from exc
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def last_error() -> str:
    msg = load().cs_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str) -> None:
    if rc != 0:
        exc = _ERRORS.get(int(rc), CutbenchError)
        raise exc(f"{what}: {last_error()}")


def ptr(arr) -> int:
    """Address of a numpy array (must stay alive across the call) or None."""
    if arr is None:
        return None
    if arr.flags.writeable and arr.size:
        return ctypes.addressof(ctypes.c_char.from_buffer(arr))  # 3x cheaper than .ctypes.data
    return arr.ctypes.data


def c_i32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int32)


def c_i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


def c_f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def set_option(key: str, value: int) -> None:
    check(load().cs_set_option(key.encode(), int(value)), f"cs_set_option({key})")


def get_option(key: str) -> int:
    return int(load().cs_get_option(key.encode()))


def launch_count() -> int:
    return int(load().cs_launch_count())


def jit_wait(timeout_s: float = -1.0) -> None:
    """Block until the background kernel compiler (jit = 3) is idle."""
    check(load().cs_jit_wait(float(timeout_s)), "cs_jit_wait")


def sweep_plan_json(nq, table, slots=None, tile_bits=0, dtype=CS_C128) -> str:
    """Host-only: the sweep schedule of a gate table (no GPU needed)."""
    lib = load()
    k = np.ascontiguousarray(table.kinds, dtype=np.uint8)
    qa, qb, prm = c_i64(table.qa), c_i64(table.qb), c_f64(table.params)
    sl = c_i32(slots) if slots is not None else None
    need = np.zeros(1, dtype=np.int64)
    check(lib.cs_sweep_plan_json(nq, ptr(k), ptr(qa), ptr(qb), ptr(prm), ptr(sl), len(k), tile_bits,
                                 dtype, None, 0, ptr(need)), "cs_sweep_plan_json")
    buf = ctypes.create_string_buffer(int(need[0]))
    check(lib.cs_sweep_plan_json(nq, ptr(k), ptr(qa), ptr(qb), ptr(prm), ptr(sl), len(k), tile_bits,
                                 dtype, buf, int(need[0]), ptr(need)), "cs_sweep_plan_json")
    return buf.value.decode()


def jit_selftest(nq, table, slots=None, n_states=1, dtype=CS_C128) -> int:
    """Host-only: compile the NVRTC-specialised sweep kernels; CUBIN bytes."""
    lib = load()
    k = np.ascontiguousarray(table.kinds, dtype=np.uint8)
    qa, qb, prm = c_i64(table.qa), c_i64(table.qb), c_f64(table.params)
    sl = c_i32(slots) if slots is not None else None
    out = np.zeros(1, np.int64)
    check(lib.cs_jit_selftest(nq, ptr(k), ptr(qa), ptr(qb), ptr(prm), ptr(sl), len(k), n_states, dtype,
                              ptr(out)), "cs_jit_selftest")
    return int(out[0])


def chain_plan(n, seg_nq, seg_ncuts, seg_cut_ids, c_total, cut_boundary, term_coef,
               force_bond=-1, dtype=CS_C128):
    """Host-only: (workspace_bytes, bond, q_low) of the chain-contracted merge."""
    lib = load()
    a_nq, a_nc, a_ids = c_i32(seg_nq), c_i32(seg_ncuts), c_i32(seg_cut_ids if len(seg_cut_ids) else [0])
    a_b = c_i32(cut_boundary if len(cut_boundary) else [0])
    a_t = c_f64(term_coef)
    ws = np.zeros(1, np.int64)
    bond = np.zeros(1, np.int32)
    qlow = np.zeros(1, np.int32)
    check(lib.cs_merge_chain_plan(n, ptr(a_nq), ptr(a_nc), ptr(a_ids), c_total, ptr(a_b), ptr(a_t),
                                  force_bond, dtype, ptr(ws), ptr(bond), ptr(qlow)),
          "cs_merge_chain_plan")
    return int(ws[0]), int(bond[0]), int(qlow[0])


def _table_args(table):
    k = np.ascontiguousarray(table.kinds, dtype=np.uint8)
    return k, c_i64(table.qa), c_i64(table.qb), c_f64(table.params)


def cut_workspace(nq, table, sizes, force_bond=-1, dtype=CS_C128):
    """Host-only: (workspace_bytes, q_low, c_total) of cs_cut_run."""
    k, qa, qb, prm = _table_args(table)
    sz = c_i32(sizes)
    ws = np.zeros(1, np.int64)
    ql = np.zeros(1, np.int32)
    ct = np.zeros(1, np.int32)
    check(load().cs_cut_workspace(nq, ptr(k), ptr(qa), ptr(qb), ptr(prm), len(k), len(sz), ptr(sz), force_bond,
                                  dtype, ptr(ws), ptr(ql), ptr(ct)), "cs_cut_workspace")
    return int(ws[0]), int(ql[0]), int(ct[0])


def cut_shard_plan(nq, table, sizes, world, rank, dtype=CS_C128) -> dict:
    """Host-only: the sharded pipeline's layout for `rank` of `world`
    (cs_cut_shard_plan): workspace bytes, q_low, the rank's default output
    range and its chunk [var_begin, var_end) of the flattened variant list."""
    k, qa, qb, prm = _table_args(table)
    sz = c_i32(sizes)
    info = np.zeros(8, np.int64)
    check(load().cs_cut_shard_plan(nq, ptr(k), ptr(qa), ptr(qb), ptr(prm), len(k), len(sz), ptr(sz), world, rank,
                                   dtype, ptr(info)), "cs_cut_shard_plan")
    keys = ("workspace_bytes", "q_low", "out_begin", "out_end", "var_begin", "var_end", "per", "total")
    return {k_: int(v) for k_, v in zip(keys, info)}


def cut_tables(nq, table, sizes):
    """Host-only C++ plan + decompose as flat numpy tables:
    (cuts [c,4], seg_counts [n,2], kinds, qa, qb, params [G,3], slots, cut_ids)."""
    k, qa, qb, prm = _table_args(table)
    sz = c_i32(sizes)
    n = len(sz)
    n2 = int(np.count_nonzero(k >= 5))  # CX = 5, CZ = 6, U3 = 7 (a bound is enough)
    gcap = len(k) + 4 * n2 + 1
    ccap = n2 + 1
    cuts = np.empty((ccap, 4), np.int64)
    counts = np.empty((n, 2), np.int32)
    ok = np.empty(gcap, np.uint8)
    oa = np.empty(gcap, np.int64)
    ob = np.empty(gcap, np.int64)
    op = np.empty((gcap, 3), np.float64)
    osl = np.empty(gcap, np.int32)
    oc = np.empty(2 * ccap, np.int32)
    need = np.zeros(2, np.int64)
    check(load().cs_cut_tables(nq, ptr(k), ptr(qa), ptr(qb), ptr(prm), len(k), n, ptr(sz), ptr(cuts), ptr(counts),
                               ptr(ok), ptr(oa), ptr(ob), ptr(op), ptr(osl), ptr(oc), gcap, ccap, ptr(need)),
          "cs_cut_tables")
    g, c = int(need[0]), int(need[1])
    return cuts[:c], counts, ok[:g], oa[:g], ob[:g], op[:g], osl[:g], oc[:int(counts[:, 1].sum())]


def cut_describe(nq, table, sizes) -> dict:
    """Host-only: the C++ preprocess (cuts and per-segment templates)."""
    import json

    lib = load()
    k, qa, qb, prm = _table_args(table)
    sz = c_i32(sizes)
    need = np.zeros(1, np.int64)
    check(lib.cs_cut_describe_json(nq, ptr(k), ptr(qa), ptr(qb), ptr(prm), len(k), len(sz), ptr(sz), None, 0,
                                   ptr(need)), "cs_cut_describe_json")
    buf = ctypes.create_string_buffer(int(need[0]))
    check(lib.cs_cut_describe_json(nq, ptr(k), ptr(qa), ptr(qb), ptr(prm), len(k), len(sz), ptr(sz), buf,
                                   int(need[0]), ptr(need)), "cs_cut_describe_json")
    return json.loads(buf.value.decode())
