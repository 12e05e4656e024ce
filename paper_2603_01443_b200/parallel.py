"""Multi-GPU cut pipeline: output sharded on the high-order amplitude bits,
subcircuit variants split across ranks, and ONE exchange — an all-gather of
the (small) subcircuit state vectors over NCCL/NVLink. The 2^q output never
moves.

One process per GPU (torch.distributed, backend "nccl" on B200s; the same
code runs under "gloo" on CPU for the host-logic tests, with the compute
steps injected).

Reference: the reference is single-process (no collectives anywhere,
SURVEY.md §2); the sharded merge computes exactly the rows [begin, end) of
merging.py:156-186's result on each rank.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ValidationError


@dataclass(frozen=True)
class Slice:
    segment: int
    v0: int
    v1: int


def shard_range(num_qubits: int, world: int, rank: int, unit_bits: int) -> tuple[int, int]:
    """Amplitudes [begin, end) owned by `rank`: contiguous, high bits first,
    aligned to 2^unit_bits (the row length of the final product)."""
    if world < 1 or not (0 <= rank < world):
        raise ValidationError(f"bad rank {rank} of world {world}")
    rows = 1 << (num_qubits - unit_bits)
    if world > rows:
        raise ValidationError(f"{world} ranks but only {rows} output rows")
    r0 = rows * rank // world
    r1 = rows * (rank + 1) // world
    return r0 << unit_bits, r1 << unit_bits


def variant_slices(counts: list[int], world: int, rank: int) -> list[Slice]:
    """Split the flattened list of all segments' variants (segment-major) into
    `world` near-equal contiguous chunks; return rank's chunk as per-segment
    slices."""
    total = int(sum(counts))
    per = -(-total // world)
    g0, g1 = min(total, rank * per), min(total, (rank + 1) * per)
    out = []
    base = 0
    for seg, c in enumerate(counts):
        a, b = max(g0, base), min(g1, base + c)
        if a < b:
            out.append(Slice(seg, a - base, b - base))
        base += c
    return out


def gather_states(local: dict, counts: list[int], lengths: list[int], world: int, rank: int,
                  all_gather, make_buffer):
    """Assemble every segment's full variant batch on every rank.

    local: {segment: tensor [v1 - v0, len]} for this rank's slices.
    all_gather(list_out, tensor): the collective (dist.all_gather).
    make_buffer(n_floats): a zeroed float64 tensor on the right device.
    Returns a list of [count_j, len_j] complex tensors (views of one buffer).
    """
    total = int(sum(counts))
    per = -(-total // world)
    offs = np.concatenate([[0], np.cumsum([c * n for c, n in zip(counts, lengths)])]).astype(np.int64)
    # every rank sends a fixed-size chunk: its `per` states padded to max length
    max_len = max(lengths)
    mine = make_buffer(per * max_len * 2)
    for sl in variant_slices(counts, world, rank):
        t = local[sl.segment]
        flat_index0 = sum(counts[:sl.segment]) + sl.v0 - rank * per
        n = lengths[sl.segment]
        real = _as_real(t).reshape(sl.v1 - sl.v0, n * 2)
        for i in range(sl.v1 - sl.v0):
            mine[(flat_index0 + i) * max_len * 2:(flat_index0 + i) * max_len * 2 + n * 2] = real[i]
    # the receive buffers are consecutive views of one allocation (what a
    # single all-gather writes; dist.all_gather takes them as a list)
    parts = list(make_buffer(world * per * max_len * 2).split(per * max_len * 2))
    all_gather(parts, mine)
    full = make_buffer(int(offs[-1]) * 2)
    g = 0
    for seg, (c, n) in enumerate(zip(counts, lengths)):
        for v in range(c):
            r, k = divmod(g, per)
            src = parts[r][k * max_len * 2:k * max_len * 2 + n * 2]
            dst0 = (int(offs[seg]) + v * n) * 2
            full[dst0:dst0 + n * 2] = src
            g += 1
    out = []
    for seg, (c, n) in enumerate(zip(counts, lengths)):
        chunk = full[int(offs[seg]) * 2:int(offs[seg + 1]) * 2]
        out.append(_as_complex(chunk).reshape(c, n))
    return out


def _as_real(t):
    import torch

    return torch.view_as_real(t.contiguous()).reshape(-1)


def _as_complex(t):
    import torch

    return torch.view_as_complex(t.reshape(-1, 2))


def run_cut_sharded(circuit, n: int, *, rank: int, world: int, dtype=np.complex128, out=None,
                    group=None, simulate_slice=None, merge_shard=None, all_gather=None, merge_events=None,
                    comm=None):
    """Cut pipeline on `world` ranks; returns (ShardedState-like tensor, (begin, end)).

    With no injected functions and a `comm` (a comm.NcclComm; or world 1)
    the whole rank step is ONE native call (pipeline.run_cut_sharded_native
    -> cs_cut_run_sharded). Otherwise the host-orchestrated form runs:
    simulate_slice(family, v0, v1) -> tensor [v1-v0, 2^q_i] and
    merge_shard(chain, batches, (begin, end)) -> tensor default to the sm_100a
    kernels; the CPU tests inject oracle-backed versions, and the all-gather
    is torch.distributed's collective on `group`."""
    import torch
    import torch.distributed as dist

    from .pipeline import preprocess, run_cut_sharded_native

    if np.dtype(dtype) != np.complex128:
        raise ValidationError("the sharded path exchanges complex128 states")
    q = circuit.num_qubits
    native = (simulate_slice is None and merge_shard is None and all_gather is None
              and (comm is not None or world == 1) and q % n == 0)
    if native:
        # the device path: ONE native call per rank (cs_cut_run_sharded) — C++
        # preprocess, this rank's variant chunk simulated in place, the
        # in-place NCCL all-gather, the chain merge of this rank's rows
        timers = {} if merge_events is not None else None
        evs = None
        if merge_events is not None:
            evs = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        res = run_cut_sharded_native(circuit, n, rank=rank, world=world, comm=comm, dtype=dtype, out=out,
                                     events=evs)
        if merge_events is not None:
            merge_events["start"], merge_events["end"] = evs[2], evs[3]
            merge_events["events"] = evs
        from .merging import ShardedState

        if isinstance(res, ShardedState):
            return res.device, (res.begin, res.end)
        return res.device_tensor(), (0, 1 << q)
    prep = preprocess(circuit, n)
    fams = prep.subs.segments
    counts = [f.num_variants for f in fams]
    lengths = [1 << f.num_qubits for f in fams]
    if simulate_slice is None:
        from .engine import simulate_table

        def simulate_slice(fam, v0, v1):
            return simulate_table(fam.num_qubits, fam.template, n_states=v1 - v0, slots=fam.slots,
                                  dtype=dtype, variant_base=v0)
    local = {}
    for sl in variant_slices(counts, world, rank):
        local[sl.segment] = simulate_slice(fams[sl.segment], sl.v0, sl.v1)
    if local:
        device = next(iter(local.values())).device
    else:
        device = "cuda" if dist.get_backend(group) == "nccl" else "cpu"

    def make_buffer(nf):
        return torch.zeros(nf, dtype=torch.float64, device=device)

    if all_gather is None and comm is not None:
        all_gather = comm.gather_parts
    if all_gather is None:
        def all_gather(parts, mine):
            dist.all_gather(parts, mine, group=group)
    batches = gather_states(local, counts, lengths, world, rank, all_gather, make_buffer)
    chain = prep.chain
    _, _, qlow = chain.plan()
    begin, end = shard_range(circuit.num_qubits, world, rank, qlow)
    if merge_shard is None:
        from .merging import merge_chain_device

        if merge_events is not None:
            merge_events["start"] = torch.cuda.Event(enable_timing=True)
            merge_events["end"] = torch.cuda.Event(enable_timing=True)
            merge_events["start"].record()
        res = merge_chain_device(chain, [b.contiguous() for b in batches], dtype=dtype, out=out,
                                 out_range=(begin, end))
        if merge_events is not None:
            merge_events["end"].record()
    else:
        res = merge_shard(chain, batches, (begin, end))
    return res, (begin, end)

