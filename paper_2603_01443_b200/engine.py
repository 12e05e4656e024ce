"""Dense state-vector simulation on the B200 (drop-in for cutbench.engine).

Same contract as `/root/reference/pkg/src/cutbench/engine.py`:
  * complex128 amplitudes, qubit j = bit j (qubit 0 = LSB) (`engine.py:1-11`);
  * ``simulate(circuit, *, max_qubits=30, deadline=None) -> StateVec`` applies
    every gate in order to |0...0> (`engine.py:158-168`); ``apply_gate``
    mutates in place (`engine.py:171-181`); ``tensor(a, b)`` puts ``a`` on the
    low qubits (`engine.py:184-189`); dump/load use little-endian (re, im)
    float64 pairs (`engine.py:192-202`);
  * the qubit guard raises ``CapacityError`` before any allocation
    (`engine.py:54-59`); an expired cooperative deadline raises
    ``BudgetExceededError`` between launches (`engine.py:142-155`).

How it differs: the work runs in the sm_100a sweep kernel (libcutsim
``cs_sim_batch``) — gates are lowered to fused 2x2/diagonal ops, tiled into
shared-memory sweeps, and a whole cut-variant family runs in one batch.
``StateVec`` keeps its amplitudes on the GPU; ``.amps`` copies them to a host
numpy array on first access (and writes back into the same array object on
later accesses, so in-place semantics match the reference).
"""
from __future__ import annotations

import time

import numpy as np

from . import _device, _native
from .circuits import Circuit, Gate, GateTable
from .errors import BudgetExceededError, CapacityError, ValidationError

DEFAULT_MAX_QUBITS = 30


class StateVec:
    """Length-2^num_qubits amplitude vector, resident on host or device.

    Exactly one copy is authoritative at a time: ``amps`` hands out the host
    array (synchronising it from the device when needed); device operations
    take the device tensor (uploading the host array when it is newer).
    """

    __slots__ = ("num_qubits", "_host", "_dev", "_owner", "dtype", "_keep", "_row_of")

    def __init__(self, num_qubits: int, amps=None, *, device=None, dtype=None, row_of=None):
        self.num_qubits = int(num_qubits)
        self._keep = None
        self._row_of = row_of  # (family batch, row) when device is that batch's row
        n = 1 << self.num_qubits
        if device is not None:
            if amps is not None:
                raise ValidationError("pass either host amps or a device tensor")
            if tuple(device.shape) != (n,):
                raise ValidationError(
                    f"state vector for {num_qubits} qubit(s) must have length {n}, "
                    f"got {tuple(device.shape)}"
                )
            self._dev = device
            self._host = None
            self._owner = "device"
            self.dtype = np.complex64 if str(device.dtype) == "torch.complex64" else np.complex128
        else:
            arr = np.asarray(amps)
            if arr.shape != (n,):
                raise ValidationError(
                    f"state vector for {num_qubits} qubit(s) must have length {n}, got {arr.shape}"
                )
            self._host = arr
            self._dev = None
            self._owner = "host"
            self.dtype = np.complex64 if arr.dtype == np.complex64 else np.complex128

    @classmethod
    def batch_row(cls, num_qubits: int, batch, row: int, dtype) -> "StateVec":
        """Row ``row`` of a device family batch [2^c, 2^num_qubits] (trusted
        shape: built by the library itself). The row tensor is materialised on
        first use, so handing out a family's states costs no torch calls."""
        sv = cls.__new__(cls)
        sv.num_qubits = num_qubits
        sv._keep = None
        sv._row_of = (batch, row)
        sv._dev = None
        sv._host = None
        sv._owner = "device"
        sv.dtype = dtype
        return sv

    def _devt(self):
        d = self._dev
        if d is None and self._row_of is not None:
            b, v = self._row_of
            d = self._dev = b[v]
        return d

    # -- host view ---------------------------------------------------------
    @property
    def amps(self) -> np.ndarray:
        if self._owner == "device":
            if self._host is None or self._host.dtype != self.dtype:
                self._host = np.empty(1 << self.num_qubits, dtype=self.dtype)
            _device.to_host(self._devt(), out=self._host)
            self._owner = "host"
        return self._host

    @amps.setter
    def amps(self, value):
        arr = np.asarray(value)
        if arr.shape != (1 << self.num_qubits,):
            raise ValidationError("amplitude array has the wrong length")
        self._host = arr
        self._owner = "host"

    # -- device view ---------------------------------------------------------
    def device_tensor(self, *, for_write: bool = False):
        """The device tensor (uploads the host copy if it is newer). When
        ``for_write`` the caller mutates it, so the host copy becomes stale."""
        if self._owner == "host":
            src = self._host
            if src.dtype not in (np.complex128, np.complex64):
                src = src.astype(np.complex128)
            t = _device.torch()
            dev = self._devt()
            if dev is None or str(dev.dtype) != str(_device.torch_dtype(src.dtype)):
                self._dev = _device.from_host(src)
            else:
                dev.copy_(t.from_numpy(np.ascontiguousarray(src)))
            self.dtype = src.dtype.type
            if for_write:
                self._owner = "device"
        elif for_write:
            self._owner = "device"
        return self._devt()

    def _sync_handed_out(self) -> None:
        """The reference's apply_gate mutates ``amps`` in place
        (engine.py:171-181): if a host array exists (the state was built from
        one, or ``amps`` was read), copy the device result back INTO that same
        array so references a caller holds see the new amplitudes. Both copies
        are then current ("both")."""
        if self._host is not None and self._host.dtype == self.dtype and self._host.flags.writeable \
                and self._host.flags.c_contiguous:
            _device.to_host(self._devt(), out=self._host)
            self._owner = "both"

    def on_device_only(self) -> bool:
        """The device tensor is the current copy (no newer host amplitudes)."""
        return self._owner in ("device", "both")

    @property
    def on_device(self) -> bool:
        return self._owner in ("device", "both")

    def norm(self) -> float:
        if self._owner in ("device", "both"):
            re, _ = inner(self, self)
            return float(np.sqrt(max(re, 0.0)))
        return float(np.linalg.norm(self._host))

    @classmethod
    def zero_state(cls, num_qubits: int) -> "StateVec":
        amps = np.zeros(1 << num_qubits, dtype=np.complex128)
        amps[0] = 1.0
        return cls(num_qubits, amps)

    def __repr__(self) -> str:
        return f"StateVec(num_qubits={self.num_qubits}, on={self._owner}, dtype={np.dtype(self.dtype).name})"


def check_capacity(num_qubits: int, max_qubits: int = DEFAULT_MAX_QUBITS) -> None:
    if num_qubits > max_qubits:
        raise CapacityError(
            f"{num_qubits} qubits exceeds the memory guard of {max_qubits} qubits "
            f"(2^{num_qubits} amplitudes)"
        )


def _expired(deadline) -> bool:
    return deadline is not None and time.monotonic() > deadline


def run_table(states, nq: int, table: GateTable, *, slots=None, variant_base: int = 0,
              init_zero: bool = False, dtype=np.complex128, stream=None, deadline=None) -> None:
    """Launch the sweep kernel on a device batch [n_states, 2^nq] (in place).
    deadline (time.monotonic() seconds): checked after every sweep launch in
    the library (cs_sim_batch_until), BudgetExceededError once passed."""
    lib = _native.load()
    k = np.ascontiguousarray(table.kinds, dtype=np.uint8)
    qa = _native.c_i64(table.qa)
    qb = _native.c_i64(table.qb)
    prm = _native.c_f64(table.params)
    sl = _native.c_i32(slots) if slots is not None else None
    n_states = states.shape[0] if states.dim() == 2 else 1
    stride = states.stride(0) if states.dim() == 2 else (1 << nq)
    if deadline is not None and nq >= 1:
        _native.check(
            lib.cs_sim_batch_until(nq, _native.ptr(k), _native.ptr(qa), _native.ptr(qb), _native.ptr(prm),
                                   _native.ptr(sl), len(k), states.data_ptr(), n_states, stride,
                                   int(variant_base), 1 if init_zero else 0, _device.code_of(dtype),
                                   _device.stream_ptr(stream), float(deadline)),
            "cs_sim_batch_until",
        )
        return
    _native.check(
        lib.cs_sim_batch(nq, _native.ptr(k), _native.ptr(qa), _native.ptr(qb), _native.ptr(prm),
                         _native.ptr(sl), len(k), states.data_ptr(), n_states, stride,
                         int(variant_base), 1 if init_zero else 0, _device.code_of(dtype),
                         _device.stream_ptr(stream)),
        "cs_sim_batch",
    )


def simulate_table(nq: int, table: GateTable, *, n_states: int = 1, slots=None,
                   deadline=None, dtype=np.complex128, out=None, stream=None, variant_base: int = 0):
    """Simulate a (template) table for a batch of variant states; returns the
    device tensor [n_states, 2^nq]. With a deadline the library synchronises
    and checks it after every sweep launch (BudgetExceededError)."""
    _device.require_cuda()
    if _expired(deadline):
        raise BudgetExceededError(f"simulation exceeded its deadline after 0/{len(table)} gates")
    states = out if out is not None else _device.empty(n_states, nq, dtype)
    # with a deadline the library checks it after every sweep launch (the
    # fused program is unchanged; granularity = one sweep)
    run_table(states, nq, table, slots=slots, init_zero=True, dtype=dtype, stream=stream,
              variant_base=variant_base, deadline=deadline)
    return states


def simulate(circuit: Circuit, *, max_qubits: int = DEFAULT_MAX_QUBITS, deadline: float | None = None,
             dtype=np.complex128) -> StateVec:
    """Apply every gate in order to |0...0> on the GPU and return the state.

    A variant circuit of decompose() (reference cutting.py:237-247) is served
    from one batched simulation of its whole segment family
    (SegmentFamily.claim_state): the reference's per-variant loop costs one
    launch sequence per family instead of one per variant."""
    check_capacity(circuit.num_qubits, max_qubits)
    origin = getattr(circuit, "_origin", None)
    if origin is not None and deadline is None:
        fam, b = origin
        batch, row = fam.claim_state(b, dtype, lambda: simulate_family(fam, dtype=dtype, max_qubits=max_qubits))
        return StateVec.batch_row(circuit.num_qubits, batch, row, np.dtype(dtype).type)
    states = simulate_table(circuit.num_qubits, circuit.table, deadline=deadline, dtype=dtype)
    return StateVec(circuit.num_qubits, device=states[0])


def simulate_family(family, *, deadline=None, dtype=np.complex128, max_qubits: int = DEFAULT_MAX_QUBITS):
    """All 2^{c_i} variants of one SegmentFamily in one batched launch
    sequence. Returns the device batch [2^{c_i}, 2^{q_i}]."""
    check_capacity(family.num_qubits, max_qubits)
    return simulate_table(family.num_qubits, family.template, n_states=family.num_variants,
                          slots=family.slots, deadline=deadline, dtype=dtype)


def apply_gate(state: StateVec, gate: Gate) -> StateVec:
    """Apply one gate in place and return the same state."""
    for q in gate.qubits:
        if q >= state.num_qubits:
            raise ValidationError(
                f"gate {gate.kind.value}{gate.qubits} out of range for {state.num_qubits} qubit(s)"
            )
    _device.require_cuda()
    tiny = Circuit(state.num_qubits, (gate,))
    dev = state.device_tensor(for_write=True)
    run_table(dev.view(1, -1), state.num_qubits, tiny.table, init_zero=False, dtype=state.dtype)
    state._sync_handed_out()
    return state


def apply_circuit(state: StateVec, circuit: Circuit) -> StateVec:
    """Apply a whole circuit in place (one sweep schedule)."""
    if circuit.num_qubits != state.num_qubits:
        raise ValidationError("circuit and state qubit counts differ")
    _device.require_cuda()
    dev = state.device_tensor(for_write=True)
    run_table(dev.view(1, -1), state.num_qubits, circuit.table, init_zero=False, dtype=state.dtype)
    state._sync_handed_out()
    return state


def tensor(a: StateVec, b: StateVec, *, max_qubits: int = DEFAULT_MAX_QUBITS) -> StateVec:
    """Product state with ``a`` on the low-index qubits and ``b`` on the high ones
    (the K = 1 case of the merge kernel)."""
    total = a.num_qubits + b.num_qubits
    check_capacity(total, max_qubits)
    _device.require_cuda()
    dt = np.complex64 if (a.dtype == np.complex64 and b.dtype == np.complex64) else np.complex128
    da = a.device_tensor()
    db = b.device_tensor()
    if np.dtype(a.dtype) != np.dtype(dt):
        da = da.to(_device.torch_dtype(dt))
    if np.dtype(b.dtype) != np.dtype(dt):
        db = db.to(_device.torch_dtype(dt))
    out = _device.empty(1, total, dt)[0]
    zero = np.zeros(1, np.int32)
    coef = np.array([1.0, 0.0])
    lib = _native.load()
    _native.check(
        lib.cs_merge_terms(1, 1, _native.ptr(zero), _native.ptr(zero), _native.ptr(coef),
                           db.data_ptr(), 1 << b.num_qubits, da.data_ptr(), 1 << a.num_qubits,
                           0, 1 << b.num_qubits, out.data_ptr(), 1 << total, 0, _device.code_of(dt),
                           _device.stream_ptr()),
        "cs_merge_terms(tensor)",
    )
    return StateVec(total, device=out)


def inner(a: StateVec, b: StateVec) -> tuple[float, float]:
    """<a|b> on the device (deterministic two-pass reduction)."""
    if a.num_qubits != b.num_qubits:
        raise ValidationError("inner product of states with different qubit counts")
    da, db = a.device_tensor(), b.device_tensor()
    if da.dtype != db.dtype:
        raise ValidationError("inner product of states with different dtypes")
    res = np.zeros(2)
    _native.check(_native.load().cs_inner(da.data_ptr(), db.data_ptr(), da.numel(),
                                          _device.code_of(a.dtype), _native.ptr(res),
                                          _device.stream_ptr()), "cs_inner")
    return float(res[0]), float(res[1])


def max_abs_diff(a: StateVec, b: StateVec) -> float:
    """max_i |a_i - b_i| on the device."""
    if a.num_qubits != b.num_qubits:
        raise ValidationError("comparing states with different qubit counts")
    da, db = a.device_tensor(), b.device_tensor()
    if da.dtype != db.dtype:
        raise ValidationError("comparing states with different dtypes")
    res = np.zeros(1)
    _native.check(_native.load().cs_maxabsdiff(da.data_ptr(), db.data_ptr(), da.numel(),
                                               _device.code_of(a.dtype), _native.ptr(res),
                                               _device.stream_ptr()), "cs_maxabsdiff")
    return float(res[0])


def gather(state: StateVec, idx) -> np.ndarray:
    """Selected amplitudes state[idx] (device gather, host result)."""
    t = _device.torch()
    dev = state.device_tensor()
    ix = t.as_tensor(np.ascontiguousarray(idx, dtype=np.int64), device="cuda")
    n = 1 << state.num_qubits
    if ix.numel() and (int(ix.min()) < 0 or int(ix.max()) >= n):
        raise ValidationError("gather index out of range")
    out = t.empty(ix.numel(), dtype=dev.dtype, device="cuda")
    _native.check(_native.load().cs_gather(dev.data_ptr(), ix.data_ptr(), ix.numel(), out.data_ptr(),
                                           _device.code_of(state.dtype), _device.stream_ptr()),
                  "cs_gather")
    return out.cpu().numpy()


def dump_amplitudes(state: StateVec, path) -> None:
    """Binary dump: little-endian float64 (re, im) pairs in index order."""
    data = np.ascontiguousarray(state.amps, dtype="<c16")
    with open(path, "wb") as fh:
        fh.write(data.tobytes())


def load_amplitudes(path, num_qubits: int) -> StateVec:
    with open(path, "rb") as fh:
        amps = np.frombuffer(fh.read(), dtype="<c16").astype(np.complex128)
    return StateVec(num_qubits, amps)


__all__ = [
    "DEFAULT_MAX_QUBITS",
    "StateVec",
    "apply_circuit",
    "apply_gate",
    "check_capacity",
    "dump_amplitudes",
    "gather",
    "inner",
    "load_amplitudes",
    "max_abs_diff",
    "simulate",
    "simulate_family",
    "simulate_table",
    "tensor",
]



def dump_shard(shard, prefix, *, rank: int, world: int) -> str:
    """Per-rank amplitude dump of a sharded state: the reference's format
    (little-endian float64 (re, im) pairs, engine.py:192-196) for amplitudes
    [begin, end), plus a JSON manifest written by rank 0. `shard` is a
    ShardedState or a (num_qubits, begin, end, tensor-or-array) tuple."""
    import json

    if hasattr(shard, "device"):
        q, begin, end, data = shard.num_qubits, shard.begin, shard.end, shard.device
    else:
        q, begin, end, data = shard
    arr = data.cpu().numpy() if hasattr(data, "cpu") else np.asarray(data)
    if arr.shape != (end - begin,):
        raise ValidationError("shard length does not match its range")
    path = f"{prefix}.rank{rank}-of-{world}.bin"
    with open(path, "wb") as fh:
        fh.write(np.ascontiguousarray(arr, dtype="<c16").tobytes())
    if rank == 0:
        with open(f"{prefix}.manifest.json", "w") as fh:
            json.dump({"num_qubits": q, "world": world, "format": "<c16 (re, im) pairs, index order",
                       "shards": [f"{prefix}.rank{r}-of-{world}.bin" for r in range(world)]}, fh)
    return path


def load_shards(prefix) -> StateVec:
    """Reassemble a full host StateVec from dump_shard files."""
    import json

    with open(f"{prefix}.manifest.json") as fh:
        man = json.load(fh)
    parts = []
    for path in man["shards"]:
        with open(path, "rb") as fh:
            parts.append(np.frombuffer(fh.read(), dtype="<c16"))
    return StateVec(man["num_qubits"], np.concatenate(parts).astype(np.complex128))
