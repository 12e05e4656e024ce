"""The cut pipeline end to end: preprocess -> batched subcircuit simulation ->
merge, with per-stage timing (the stage boundaries of the reference harness,
`/root/reference/pkg/src/cutbench/harness.py:125-151`: t_pre = plan_cut +
decompose, t_sub = all subcircuit simulations, t_merge = merge_input_from +
merge).

``run_cut`` is what a user calls instead of the reference's per-variant loop
`[[simulate(c) for c in fam.circuits] for fam in subs.segments]`: every variant
family is one batched sweep sequence on the device, and the merge is the chain
kernel writing the state (or this GPU's shard of it) once.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _device, _native
from .circuits import Circuit
from .cutting import decompose, plan_cut
from .engine import DEFAULT_MAX_QUBITS, StateVec, check_capacity, simulate_family
from .merging import ChainSpec, ShardedState, merge_chain_device


@dataclass
class StageTimes:
    """Seconds per stage. pre is host time; sub/merge are CUDA-event times."""

    pre: float = 0.0
    sub: float = 0.0
    merge: float = 0.0

    @property
    def cut(self) -> float:
        return self.pre + self.sub + self.merge


@dataclass
class Prepared:
    """Host-side preprocess result (t_pre)."""

    circuit: Circuit
    n: int
    subs: object
    chain: ChainSpec


def preprocess(circuit: Circuit, n: int) -> Prepared:
    plan = plan_cut(circuit, n)
    subs = decompose(circuit, plan)
    return Prepared(circuit, n, subs, ChainSpec.from_plan(plan))


def simulate_segments(prep: Prepared, *, dtype=np.complex128, max_qubits=DEFAULT_MAX_QUBITS):
    """Device batches [2^{c_i}, 2^{q_i}] of every segment's variants (t_sub)."""
    return simulate_families(prep.subs.segments, dtype=dtype, max_qubits=max_qubits)


def simulate_families(fams, *, dtype=np.complex128, max_qubits=DEFAULT_MAX_QUBITS):
    """Device batches [2^{c_i}, 2^{q_i}] of the given segment families.

    Segments are independent, so each family runs on its own side stream
    (forked from and joined back into the current stream): the short,
    latency-bound sweep chains of different segments overlap on the GPU."""
    if len(fams) == 1:
        return [simulate_family(fams[0], dtype=dtype, max_qubits=max_qubits)]
    fast = _simulate_families_native(fams, dtype, max_qubits)
    if fast is not None:
        return fast
    t = _device.torch()
    main = t.cuda.current_stream()
    fork = t.cuda.Event()
    fork.record(main)
    outs, joins = [], []
    for j, fam in enumerate(fams):
        s = _side_stream(j)
        s.wait_event(fork)
        with t.cuda.stream(s):
            outs.append(simulate_family(fam, dtype=dtype, max_qubits=max_qubits))
            ev = t.cuda.Event()
            ev.record(s)
        joins.append(ev)
    for ev, o in zip(joins, outs):
        main.wait_event(ev)
        o.record_stream(main)
    return outs


def _simulate_families_native(fams, dtype, max_qubits):
    """All families of one C++-planned decomposition in ONE native call
    (cs_sim_families: schedules, side streams and joins inside libcutsim),
    reading the templates straight from the planner's concatenated tables.
    None when the families are not such a set (or a template was replaced)."""
    src0 = getattr(fams[0], "_src", None)
    if src0 is None:
        return None
    nt = src0[0]
    g = 0
    for f in fams:
        src = getattr(f, "_src", None)
        if src is None or src[0] is not nt or src[1] != g or f.slots is not src[5]:
            return None
        t_ = f.template
        cols = src[4]
        if t_ is not src[3] or t_.kinds is not cols[0] or t_.qa is not cols[1] or t_.qb is not cols[2] \
                or t_.params is not cols[3]:
            return None  # the template (or a column of it) was replaced: not the planner's tables any more
        g += src[2]
    for f in fams:
        check_capacity(f.num_qubits, max_qubits)
    _device.require_cuda()
    t = _device.torch()
    tdt = _device.torch_dtype(dtype)
    outs = [t.empty((f.num_variants, 1 << f.num_qubits), dtype=tdt, device="cuda") for f in fams]
    # the per-family counts and the planner tables' addresses are fixed for a
    # decomposition: built once per family set (the API path pays ~1 us per
    # pointer conversion), kept with the tables they point into
    key = tuple(map(id, fams))
    args = _FAMILY_ARGS.get(key)
    if args is None or args[0] is not nt:
        _cuts, _counts, k, a, b, p, sl, _cid = nt
        nq = np.array([f.num_qubits for f in fams], np.int32)
        gcount = np.array([f._src[2] for f in fams], np.int64)
        ns = np.array([f.num_variants for f in fams], np.int64)
        ptr = _native.ptr
        args = (nt, nq, gcount, ns, tuple(fams),
                (ptr(nq), ptr(gcount), ptr(k), ptr(a), ptr(b), ptr(p), ptr(sl)), ptr(ns))
        if len(_FAMILY_ARGS) >= 64:
            _FAMILY_ARGS.clear()
        _FAMILY_ARGS[key] = args
    ptrs = (ctypes.c_uint64 * len(outs))(*[o.data_ptr() for o in outs])
    _native.check(_native.load().cs_sim_families(len(fams), *args[5], ptrs, args[6], _device.code_of(dtype),
                                                 _device.stream_ptr()), "cs_sim_families")
    return outs


# decomposition (family tuple) -> (tables, arrays, families kept alive, pointers)
_FAMILY_ARGS: dict = {}


_SIDE_STREAMS: dict = {}


def _side_stream(j: int):
    t = _device.torch()
    key = (t.cuda.current_device(), j % 4)
    if key not in _SIDE_STREAMS:
        _SIDE_STREAMS[key] = t.cuda.Stream()
    return _SIDE_STREAMS[key]


_WORKSPACE: dict = {}


def cut_workspace_tensor(nbytes: int):
    """The per-device workspace of cs_cut_run (grown on demand, reused). It is
    shared by every run_cut call on the device without an explicit
    ``workspace=``, which is safe for calls ordered on one stream; callers
    running cut pipelines concurrently on several streams pass their own."""
    t = _device.torch()
    dev = t.cuda.current_device()
    ws = _WORKSPACE.get(dev)
    if ws is None or ws.numel() < nbytes:
        ws = t.empty(max(nbytes, 1), dtype=t.uint8, device="cuda")
        _WORKSPACE[dev] = ws
    return ws


def run_cut(circuit: Circuit, n: int, *, dtype=np.complex128, max_qubits: int = DEFAULT_MAX_QUBITS,
            out=None, out_range=None, timers: StageTimes | None = None, workspace=None, sizes=None,
            force_bond: int = -1, events=None):
    """Cut-simulate ``circuit`` into n equal segments (or ``sizes``) and return
    the merged state (a device StateVec, or a ShardedState when ``out_range``
    selects a shard). One native call (cs_cut_run): C++ preprocess, batched
    variant sweeps on side streams, chain merge written once into ``out``.
    ``timers`` synchronises and fills pre/sub/merge; ``events`` (three
    torch.cuda.Event with timing) are recorded around the two device stages
    without synchronising. Reference: harness.py:125-145 (cut leg)."""
    from . import _native
    from .errors import ValidationError

    q = circuit.num_qubits
    check_capacity(q, max_qubits)
    if sizes is None:
        if n < 2:
            raise ValidationError(f"segment count must be >= 2, got {n}")
        if q % n:
            raise ValidationError(f"q must be divisible by n: q={q}, n={n}")
        sizes = (q // n,) * n
    t = _device.require_cuda()
    code = _device.code_of(dtype)
    ws_bytes, qlow, _c = _native.cut_workspace(q, circuit.table, sizes, force_bond, code)
    if workspace is None:
        workspace = cut_workspace_tensor(ws_bytes)
    begin, end = (0, 1 << q) if out_range is None else tuple(out_range)
    if not (0 <= begin <= end <= (1 << q)):
        raise ValidationError(f"output range [{begin}, {end}) outside [0, 2^{q})")
    if out is None:
        _device.check_free((end - begin) * np.dtype(dtype).itemsize, "state")
        out = _device.empty_shape((end - begin,), dtype)
    else:
        _device.check_out(out, end - begin, dtype)
    if workspace is not None and (workspace.device.type != "cuda" or not workspace.is_contiguous()
                                  or workspace.numel() * workspace.element_size() < ws_bytes):
        raise ValidationError(f"workspace must be a contiguous CUDA buffer of >= {ws_bytes} bytes")
    k, qa, qb, prm = _native._table_args(circuit.table)
    sz = _native.c_i32(sizes)
    stage = np.zeros(3) if timers is not None else None
    evp = None
    if events is not None:
        for ev in events:
            if not ev.cuda_event:  # torch creates the cudaEvent_t on first record
                ev.record()
        evp = (ctypes.c_void_p * 3)(*(ev.cuda_event for ev in events))
    _native.check(
        _native.load().cs_cut_run(q, _native.ptr(k), _native.ptr(qa), _native.ptr(qb), _native.ptr(prm), len(k),
                                  len(sz), _native.ptr(sz), force_bond, begin, end, out.data_ptr(),
                                  workspace.data_ptr(), workspace.numel() * workspace.element_size(), code, _device.stream_ptr(),
                                  evp, _native.ptr(stage)),
        "cs_cut_run",
    )
    if timers is not None:
        timers.pre, timers.sub, timers.merge = (float(v) / 1e3 for v in stage)
    if (begin, end) != (0, 1 << q):
        return ShardedState(q, begin, end, out)
    return StateVec(q, device=out)


def run_cut_sharded_native(circuit: Circuit, n: int, *, rank: int = 0, world: int = 1, comm=None,
                           dtype=np.complex128, out=None, out_range=None, workspace=None,
                           timers: dict | None = None, events=None, max_qubits: int = 34):
    """One rank's share of the multi-GPU cut pipeline in ONE native call
    (cs_cut_run_sharded): C++ preprocess, this rank's chunk of the variant
    list simulated in place, one in-place NCCL all-gather (``comm``, a
    comm.NcclComm; None = simulate every variant here, no exchange), then the
    chain merge of this rank's output rows (default: parallel.shard_range).
    Returns a ShardedState (or a StateVec when the range is the whole state).
    ``timers`` (a dict) receives pre/sub/exchange/merge seconds (synchronises);
    ``events`` = four timing torch.cuda.Events recorded around the stages.
    Each rank computes rows [begin, end) of reference merging.py:156-186."""
    from . import _native
    from .errors import ValidationError

    q = circuit.num_qubits
    check_capacity(q, max_qubits)
    if n < 2 or q % n:
        raise ValidationError(f"q must be divisible by n >= 2: q={q}, n={n}")
    t = _device.require_cuda()
    code = _device.code_of(dtype)
    sizes = (q // n,) * n
    lay = _native.cut_shard_plan(q, circuit.table, sizes, world, rank, code)
    begin, end = (lay["out_begin"], lay["out_end"]) if out_range is None else tuple(out_range)
    if not (0 <= begin <= end <= (1 << q)):
        raise ValidationError(f"output range [{begin}, {end}) outside [0, 2^{q})")
    if out is None:
        _device.check_free((end - begin) * np.dtype(dtype).itemsize, "state shard")
        out = _device.empty_shape((end - begin,), dtype)
    else:
        _device.check_out(out, end - begin, dtype)
    if workspace is None:
        workspace = t.empty(max(lay["workspace_bytes"], 1), dtype=t.uint8, device="cuda")
    elif workspace.numel() * workspace.element_size() < lay["workspace_bytes"] or not workspace.is_contiguous():
        raise ValidationError(f"workspace must be a contiguous CUDA buffer of >= {lay['workspace_bytes']} bytes")
    k, qa, qb, prm = _native._table_args(circuit.table)
    sz = _native.c_i32(sizes)
    stage = np.zeros(4) if timers is not None else None
    evp = None
    if events is not None:
        for ev in events:
            if not ev.cuda_event:  # torch creates the cudaEvent_t on first record
                ev.record()
        evp = (ctypes.c_void_p * 4)(*(ev.cuda_event for ev in events))
    handle = comm.handle if comm is not None else None
    _native.check(
        _native.load().cs_cut_run_sharded(q, _native.ptr(k), _native.ptr(qa), _native.ptr(qb), _native.ptr(prm),
                                          len(k), len(sz), _native.ptr(sz), handle, world, rank, begin, end,
                                          out.data_ptr(), workspace.data_ptr(),
                                          workspace.numel() * workspace.element_size(), code,
                                          _device.stream_ptr(), evp, _native.ptr(stage)),
        "cs_cut_run_sharded",
    )
    if timers is not None:
        for key, v in zip(("pre", "sub", "exchange", "merge"), stage):
            timers[key] = float(v) / 1e3
    if (begin, end) != (0, 1 << q):
        return ShardedState(q, begin, end, out)
    return StateVec(q, device=out)


def shard_workspace_bytes(circuit: Circuit, n: int, world: int, dtype=np.complex128) -> int:
    from . import _native

    q = circuit.num_qubits
    return _native.cut_shard_plan(q, circuit.table, (q // n,) * n, world, 0, _device.code_of(dtype))[
        "workspace_bytes"]


def cut_simulate(circuit: Circuit, n: int, **kw) -> StateVec:
    return run_cut(circuit, n, **kw)


def run_cut_to_host(circuit: Circuit, n: int, host_out, *, dtype=np.complex128, chunks: int = 8,
                    workspace=None, timers: StageTimes | None = None, max_qubits: int = DEFAULT_MAX_QUBITS,
                    sizes=None):
    """Cut-simulate and deliver the full state into ``host_out`` (a host
    tensor or array of 2^q amplitudes, ideally pinned): the reference API's
    contract of returning host memory. One native call (cs_cut_run_to_host):
    the merge runs in ``chunks`` row ranges into two device staging buffers
    and each chunk's device->host copy overlaps the next chunk's merge
    (PCIe-bound); returns when ``host_out`` is complete."""
    from . import _native
    from .errors import ValidationError

    q = circuit.num_qubits
    check_capacity(q, max_qubits)
    _device.require_cuda()
    if sizes is None:
        if n < 2 or q % n:
            raise ValidationError(f"q must be divisible by n >= 2: q={q}, n={n}")
        sizes = (q // n,) * n
    if isinstance(host_out, np.ndarray):
        if host_out.size != 1 << q or host_out.dtype != np.dtype(dtype) or not host_out.flags.c_contiguous:
            raise ValidationError("host_out must be a contiguous array of 2^q amplitudes of the dtype")
        host_ptr = host_out.ctypes.data
    else:
        _device.check_out(host_out, 1 << q, dtype, "host_out", device="cpu")
        host_ptr = host_out.data_ptr()
    k, qa, qb, prm = _native._table_args(circuit.table)
    sz = _native.c_i32(sizes)
    code = _device.code_of(dtype)
    need = np.zeros(1, np.int64)
    _native.check(_native.load().cs_cut_host_workspace(q, _native.ptr(k), _native.ptr(qa), _native.ptr(qb),
                                                       _native.ptr(prm), len(k), len(sz), _native.ptr(sz), chunks,
                                                       code, _native.ptr(need)), "cs_cut_host_workspace")
    if workspace is None or workspace.numel() * workspace.element_size() < int(need[0]):
        workspace = cut_workspace_tensor(int(need[0]))
    stage = np.zeros(3) if timers is not None else None
    _native.check(_native.load().cs_cut_run_to_host(q, _native.ptr(k), _native.ptr(qa), _native.ptr(qb),
                                                    _native.ptr(prm), len(k), len(sz), _native.ptr(sz), chunks,
                                                    host_ptr, workspace.data_ptr(), workspace.numel() * workspace.element_size(), code,
                                                    _device.stream_ptr(), _native.ptr(stage)),
                  "cs_cut_run_to_host")
    if timers is not None:
        timers.pre, timers.sub, timers.merge = (float(v) / 1e3 for v in stage)
    return host_out


def host_workspace_bytes(circuit: Circuit, n: int, *, chunks: int = 8, dtype=np.complex128) -> int:
    """Device workspace run_cut_to_host needs (variant states, merge
    intermediates and two staging buffers of 2^q / chunks amplitudes)."""
    from . import _native

    q = circuit.num_qubits
    k, qa, qb, prm = _native._table_args(circuit.table)
    sz = _native.c_i32((q // n,) * n)
    need = np.zeros(1, np.int64)
    _native.check(_native.load().cs_cut_host_workspace(q, _native.ptr(k), _native.ptr(qa), _native.ptr(qb),
                                                       _native.ptr(prm), len(k), len(sz), _native.ptr(sz), chunks,
                                                       _device.code_of(dtype), _native.ptr(need)),
                  "cs_cut_host_workspace")
    return int(need[0])


