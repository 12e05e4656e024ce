"""Distributed uncut simulator for states that do not fit one GPU (q >= 33 on
8 x B200) — the full-state cross-check of the
sharded cut pipeline.

Layout: world = 2^g ranks; the top g index bits select the rank, so rank r
holds amplitudes [r * 2^nloc, (r + 1) * 2^nloc), nloc = q - g. The simulator
tracks a permutation pi (logical qubit -> physical index bit). Gates run on
the local shard with the sm_100a sweep kernel after translation:
  * diagonal gates and controls on a global bit are resolved per rank (the
    bit is constant on the shard): dropped, reduced to a local gate, or a
    scalar phase (X P X P on a local qubit, fused to diag(p, p));
  * a dense gate (H, X, U3, CX target) on a global bit first swaps that bit
    with the top local bit: rank r and its partner r ^ 2^j exchange one
    contiguous half shard over NCCL (one send + one recv per rank) — the only
    collective;
  * at the end pi is restored (global swaps, then local SWAPs as 3 CX).
The result on rank r is exactly rows [r * 2^nloc, (r + 1) * 2^nloc) of
`simulate(circuit)` (reference engine.py:158-168).

`run_local(table, shard)` and `exchange(send_half, recv_buf, partner)`
default to the GPU kernel and NCCL point-to-point; the CPU tests inject a
numpy oracle and gloo.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .circuits import (
    KIND_CX,
    KIND_CZ,
    KIND_H,
    KIND_S,
    KIND_SDG,
    KIND_T,
    KIND_U3,
    KIND_X,
    Circuit,
    GateTable,
)
from .errors import ValidationError

DENSE = (KIND_H, KIND_X, KIND_U3)
PHASE1 = (KIND_T, KIND_S, KIND_SDG)


@dataclass
class Swap:
    local_bit: int   # physical local position (always the top local bit)
    global_bit: int  # physical global position (>= nloc)


@dataclass
class Segment:
    gates: list       # [(kind, a, b, params)] on LOGICAL qubits
    perm: list        # logical -> physical at the start of the segment


def plan(circuit: Circuit, world: int):
    """Rank-independent schedule: alternating gate segments and swaps, plus
    the final restoration (as swaps and local SWAP = 3 CX segments)."""
    if world < 1 or world & (world - 1):
        raise ValidationError(f"world size must be a power of two, got {world}")
    q = circuit.num_qubits
    g = world.bit_length() - 1
    nloc = q - g
    if nloc < 1:
        raise ValidationError(f"{q} qubits cannot be spread over {world} ranks")
    perm = list(range(q))
    steps = []
    cur: list = []

    def flush():
        nonlocal cur
        if cur:
            steps.append(Segment(cur, list(perm)))
            cur = []

    top = nloc - 1

    def phys_swap(p1, p2):
        flush()
        steps.append(Swap(p1, p2))
        l1, l2 = perm.index(p1), perm.index(p2)
        perm[l1], perm[l2] = p2, p1

    def swap_in(logical):
        phys_swap(top, perm[logical])

    k, qa, qb, prm = circuit.kinds, circuit.qa, circuit.qb, circuit.params
    for i in range(circuit.gate_count):
        kind, a, b = int(k[i]), int(qa[i]), int(qb[i])
        target = a if kind in DENSE else (b if kind == KIND_CX else None)
        if target is not None and perm[target] >= nloc:
            swap_in(target)
        cur.append((kind, a, b, tuple(prm[i])))
    # restore pi: global positions first (a logical qubit parked at another
    # global position is brought to the top local bit first)
    for gpos in range(nloc, q):
        p = perm[gpos]
        if p == gpos:
            continue
        if p >= nloc:
            phys_swap(top, p)
        elif p != top:
            _local_swap(cur, perm, p, top)
        phys_swap(top, gpos)
    for pos in range(nloc):
        if perm[pos] != pos:
            _local_swap(cur, perm, perm[pos], pos)
    flush()
    assert perm == list(range(q))
    return steps, nloc


def _local_swap(cur, perm, pa, pb):
    """Append SWAP of physical local bits pa, pb (as 3 CX on the logical
    qubits currently there) and update pi."""
    la, lb = perm.index(pa), perm.index(pb)
    cur += [(KIND_CX, la, lb, (0.0, 0.0, 0.0)), (KIND_CX, lb, la, (0.0, 0.0, 0.0)),
            (KIND_CX, la, lb, (0.0, 0.0, 0.0))]
    perm[la], perm[lb] = pb, pa


def _scalar(p_kind):
    """Gates multiplying the shard by the phase of p_kind: X P X P on qubit 0."""
    return [(KIND_X, 0, -1), (p_kind, 0, -1), (KIND_X, 0, -1), (p_kind, 0, -1)]


def local_table(seg: Segment, rank: int, nloc: int) -> GateTable:
    """Translate a segment to this rank's local gate table (physical local bits)."""
    perm = list(seg.perm)
    kinds, qa, qb, prm = [], [], [], []

    def emit(kind, a, b=-1, p=(0.0, 0.0, 0.0)):
        kinds.append(kind)
        qa.append(a)
        qb.append(b)
        prm.append(p)

    def gbit(pos):
        return (rank >> (pos - nloc)) & 1

    for kind, a, b, p in seg.gates:
        pa = perm[a]
        pb = perm[b] if kind in (KIND_CX, KIND_CZ) else -1
        if kind in DENSE:
            emit(kind, pa, -1, p)
        elif kind in PHASE1:
            if pa < nloc:
                emit(kind, pa)
            elif gbit(pa):
                for g in _scalar(kind):
                    emit(*g)
        elif kind == KIND_CZ:
            la, lb = pa < nloc, pb < nloc
            if la and lb:
                emit(KIND_CZ, pa, pb)
            elif la or lb:
                loc, glob = (pa, pb) if la else (pb, pa)
                if gbit(glob):
                    emit(KIND_S, loc)
                    emit(KIND_S, loc)
            elif gbit(pa) and gbit(pb):
                for g in _scalar(KIND_S) + _scalar(KIND_S):
                    emit(*g)
        elif kind == KIND_CX:
            if pb >= nloc:
                raise AssertionError("CX target must be local after scheduling")
            if pa < nloc:
                emit(KIND_CX, pa, pb)
            elif gbit(pa):
                emit(KIND_X, pb)
        else:
            raise ValidationError(f"unknown gate kind {kind}")
    n = len(kinds)
    return GateTable(np.array(kinds, np.uint8), np.array(qa, np.int64), np.array(qb, np.int64),
                     np.array(prm, np.float64).reshape(n, 3))


def simulate_distributed(circuit: Circuit, *, rank: int, world: int, group=None, dtype=np.complex128,
                         run_local=None, exchange=None, init=None, comm=None):
    """This rank's shard of the uncut state (device tensor by default). The
    half-shard swaps go through `comm` (comm.NcclComm: libcutsim's grouped
    ncclSend/ncclRecv) when given, else torch.distributed P2P on `group`."""
    import torch

    steps, nloc = plan(circuit, world)
    half = 1 << (nloc - 1)
    if run_local is None:
        from . import _device
        from .engine import run_table

        from . import _native

        shard = _device.empty(1, nloc, dtype)[0]
        pending_init = [rank == 0]  # rank 0's |0..0> not written yet
        if rank != 0:
            shard.zero_()

        def run_local(table, sh):
            # rank 0's first local segment starts from |0..0> inside the
            # library (zero-start tiles); afterwards the shard holds the state
            run_table(sh.view(1, -1), nloc, table, dtype=dtype, init_zero=pending_init[0])
            pending_init[0] = False

        def ensure_init():
            if pending_init[0]:
                _native.check(_native.load().cs_init_basis(shard.data_ptr(), nloc, 1, 0, _device.code_of(dtype),
                                                           _device.stream_ptr()), "cs_init_basis")
                pending_init[0] = False
    else:
        shard = init(nloc) if init is not None else None

        def ensure_init():
            pass
    if exchange is None and comm is not None:
        exchange = comm.sendrecv
    if exchange is None:
        import torch.distributed as dist

        def exchange(send, recv, partner):
            ops = [dist.P2POp(dist.isend, send, partner, group), dist.P2POp(dist.irecv, recv, partner, group)]
            for req in dist.batch_isend_irecv(ops):
                req.wait()
    buf = None
    # ranks whose shard can be non-zero: from |0..0> only rank 0, and a swap
    # on global bit j spreads it to the partner. Every rank tracks the same
    # set; an all-zero shard stays zero under its local gates (skipped) and
    # two all-zero partners skip their exchange.
    nonzero = {0}
    for st in steps:
        if isinstance(st, Segment):
            table = local_table(st, rank, nloc)
            if len(table) and rank in nonzero:
                run_local(table, shard)
        else:
            b = (rank >> (st.global_bit - nloc)) & 1
            partner = rank ^ (1 << (st.global_bit - nloc))
            bit = 1 << (st.global_bit - nloc)
            was = set(nonzero)
            nonzero |= {r ^ bit for r in was}
            if rank not in was and partner not in was:
                continue
            # keep local bit == b, exchange the half with local bit != b
            part = shard[half:] if b == 0 else shard[:half]
            if buf is None:
                buf = torch.empty_like(part)
            ensure_init()
            exchange(torch.view_as_real(part.contiguous()), torch.view_as_real(buf), partner)
            part.copy_(buf)
    ensure_init()
    return shard


def simulate_emulated(circuit: Circuit, world: int, *, dtype=np.complex128):
    """All ranks of `simulate_distributed` in lockstep on ONE device: the same
    schedule and per-rank gate tables, with the NCCL exchange replaced by a
    device copy between the partner shards. Validates the distributed path on
    a single GPU; returns the full state as one device tensor."""
    from . import _device, _native
    from .engine import run_table

    steps, nloc = plan(circuit, world)
    half = 1 << (nloc - 1)
    full = _device.empty(world, nloc, dtype)
    full.zero_()
    _native.check(_native.load().cs_init_basis(full.data_ptr(), nloc, 1, 0, _device.code_of(dtype),
                                               _device.stream_ptr()), "cs_init_basis")
    nonzero = {0}  # as in simulate_distributed
    for st in steps:
        if isinstance(st, Segment):
            for r in range(world):
                table = local_table(st, r, nloc)
                if len(table) and r in nonzero:
                    run_table(full[r].view(1, -1), nloc, table, dtype=dtype)
        else:
            j = st.global_bit - nloc
            nonzero |= {r ^ (1 << j) for r in set(nonzero)}
            for r in range(world):
                if (r >> j) & 1:
                    continue
                partner = r | (1 << j)
                # rank r (bit 0) sends its upper half, the partner (bit 1) its lower half
                tmp = full[r, half:].clone()
                full[r, half:].copy_(full[partner, :half])
                full[partner, :half].copy_(tmp)
    return full.view(-1)
