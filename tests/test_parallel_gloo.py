"""Multi-rank host logic of the sharded cut pipeline, on CPU with gloo
(world_size 2 and 3): variant split, all-gather reassembly, output shard
ranges. The compute steps are injected with oracle-backed functions (this is
a test of the exchange/sharding logic, not of the kernels)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import cutbench_oracle as orc
from paper_2603_01443_b200 import generators as G
from paper_2603_01443_b200.parallel import run_cut_sharded, shard_range, variant_slices


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def oracle_simulate_slice(fam, v0, v1):
    out = []
    for v in range(v0, v1):
        t = fam.variant_table(v)
        out.append(orc.simulate(fam.num_qubits, t.kinds, t.qa, t.qb, t.params))
    return torch.from_numpy(np.stack(out))


def oracle_merge_shard(chain, batches, rng):
    # rebuild the reference merge table from the chain structure, merge fully, slice
    n = chain.n
    m = np.arange(1 << chain.c_total)
    table = np.zeros((n, m.size), np.int64)
    pos = 0
    for seg in range(n):
        for lb in range(chain.seg_ncuts[seg]):
            j = chain.seg_cut_ids[pos]
            pos += 1
            table[seg] |= ((m >> j) & 1) << lb
    states = [list(b.numpy()) for b in batches]
    full = orc.merge(states, table, orc.coefficients(chain.c_total))
    return torch.from_numpy(full[rng[0]:rng[1]].copy())


def _worker(rank, world, port, spec_args, n, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        circ = G.build_brickwall(G.BrickwallSpec(*spec_args))
        res, rng = run_cut_sharded(circ, n, rank=rank, world=world,
                                   simulate_slice=oracle_simulate_slice,
                                   merge_shard=oracle_merge_shard)
        result_q.put((rank, rng, res.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,spec_args,n", [
    (2, (10, 4, 2, 2, 0), 2),
    (2, (9, 4, 3, 4, 1), 3),
    (3, (8, 4, 4, 4, 2), 4),
])
def test_sharded_pipeline_matches_oracle(world, spec_args, n):
    ctx = mp.get_context("spawn")
    q_out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, spec_args, n, q_out)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q_out.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    results.sort()
    q = spec_args[0]
    full = np.concatenate([r[2] for r in results])
    assert [r[1] for r in results][0][0] == 0 and results[-1][1][1] == 1 << q
    k, a, b, p = orc.brickwall(*spec_args)
    ref, _, _, _ = orc.cut_pipeline(q, k, a, b, p, n)
    assert np.abs(full - ref).max() < 1e-12
    assert np.abs(full - orc.simulate(q, k, a, b, p)).max() < 1e-10


def test_shard_ranges_partition_the_state():
    for world in (1, 2, 3, 4, 8):
        spans = [shard_range(30, world, r, 15) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == 1 << 30
        for (a0, a1), (b0, _b1) in zip(spans, spans[1:]):
            assert a1 == b0 and (a1 - a0) % (1 << 15) == 0


def test_variant_slices_cover_each_variant_once():
    for counts in ([4, 4], [4, 16, 4], [4, 8, 4, 2]):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                for sl in variant_slices(counts, world, r):
                    seen += [(sl.segment, v) for v in range(sl.v0, sl.v1)]
            assert sorted(seen) == [(s, v) for s, c in enumerate(counts) for v in range(c)]


def test_sharded_dump_round_trip(tmp_path):
    from paper_2603_01443_b200.engine import dump_shard, load_shards

    full = (np.arange(16) + 1j * np.arange(16)[::-1]).astype(np.complex128)
    prefix = str(tmp_path / "state")
    for r in range(4):
        dump_shard((4, 4 * r, 4 * r + 4, full[4 * r:4 * r + 4]), prefix, rank=r, world=4)
    back = load_shards(prefix)
    assert back.num_qubits == 4 and np.array_equal(back.amps, full)
    raw = open(f"{prefix}.rank1-of-4.bin", "rb").read()
    assert np.array_equal(np.frombuffer(raw, "<f8"), np.stack([full[4:8].real, full[4:8].imag], 1).ravel())


def _native_layout_worker(rank, world, port, spec_args, n, result_q):
    """One rank of the cs_cut_run_sharded data flow with gloo standing in for
    NCCL: the layout (workspace chunks, the rank's variant chunk, its output
    rows) comes from the library's own host-only cs_cut_shard_plan; the rank
    fills ITS chunk of the flat variant array in place (oracle-simulated
    states, segment-major), one all-gather of equal chunks completes the
    array, and the segment batches are read straight out of it (no
    reassembly) for the merge of the rank's rows."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2603_01443_b200 import _native
        from paper_2603_01443_b200.cutting import decompose, plan_cut
        from paper_2603_01443_b200.merging import ChainSpec

        circ = G.build_brickwall(G.BrickwallSpec(*spec_args))
        q = circ.num_qubits
        lay = _native.cut_shard_plan(q, circ.table, [q // n] * n, world, rank)
        plan = plan_cut(circ, n)
        fams = decompose(circ, plan).segments
        counts = [f.num_variants for f in fams]
        L = 1 << (q // n)
        per, total = lay["per"], lay["total"]
        assert total == sum(counts) and per == -(-total // world)
        flat = torch.zeros(world * per, L, dtype=torch.complex128)
        first = np.concatenate([[0], np.cumsum(counts)])
        for g in range(lay["var_begin"], lay["var_end"]):  # this rank's chunk only
            seg = int(np.searchsorted(first, g, side="right") - 1)
            t = fams[seg].variant_table(g - int(first[seg]))
            flat[g] = torch.from_numpy(orc.simulate(q // n, t.kinds, t.qa, t.qb, t.params))
        mine = flat[rank * per:(rank + 1) * per].clone()
        dist.all_gather(list(flat.split(per)), mine)
        batches = [flat[int(first[s]):int(first[s + 1])] for s in range(n)]
        rng = (lay["out_begin"], lay["out_end"])
        res = oracle_merge_shard(ChainSpec.from_plan(plan), batches, rng)
        result_q.put((rank, rng, res.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,spec_args,n", [
    (2, (10, 4, 2, 2, 0), 2),
    (2, (12, 4, 4, 4, 1), 4),
    (3, (9, 4, 3, 4, 2), 3),
])
def test_native_shard_layout_matches_oracle(world, spec_args, n):
    ctx = mp.get_context("spawn")
    q_out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_native_layout_worker, args=(r, world, port, spec_args, n, q_out))
             for r in range(world)]
    for p in procs:
        p.start()
    results = sorted(q_out.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    q = spec_args[0]
    full = np.concatenate([r[2] for r in results])
    spans = [r[1] for r in results]
    assert spans[0][0] == 0 and spans[-1][1] == 1 << q
    assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    k, a, b, p = orc.brickwall(*spec_args)
    assert np.abs(full - orc.simulate(q, k, a, b, p)).max() < 1e-10
