"""Distributed uncut simulator (q > one GPU): schedule, per-rank gate
resolution and half-shard exchanges, on CPU with gloo at world 2 and 4 (the
local compute is the numpy oracle, injected; the exchange is the real
torch.distributed point-to-point path)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import cutbench_oracle as orc
from paper_2603_01443_b200 import circuits as C
from paper_2603_01443_b200 import generators as G
from paper_2603_01443_b200.distributed import Segment, Swap, plan, simulate_distributed


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _circuit(kind, args):
    if kind == "brickwall":
        return G.build_brickwall(G.BrickwallSpec(*args))
    return C.build_staircase(C.BenchmarkSpec(*args))


def _worker(rank, world, port, kind, args, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        circ = _circuit(kind, args)
        nloc = circ.num_qubits - (world.bit_length() - 1)

        def init(n):
            t = torch.zeros(1 << n, dtype=torch.complex128)
            if rank == 0:
                t[0] = 1
            return t

        def run_local(table, shard):
            a = shard.numpy()
            orc.run_gates(a, table.kinds, table.qa, table.qb, table.params)

        def exchange(send, recv, partner):
            ops = [dist.P2POp(dist.isend, send.clone(), partner), dist.P2POp(dist.irecv, recv, partner)]
            for r in dist.batch_isend_irecv(ops):
                r.wait()

        shard = simulate_distributed(circ, rank=rank, world=world, run_local=run_local, exchange=exchange,
                                     init=init)
        out_q.put((rank, shard.numpy().copy(), nloc))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,kind,args", [
    (2, "brickwall", (6, 4, 2, 2, 0)),
    (4, "brickwall", (8, 5, 2, 2, 1)),
    (4, "staircase", (8, 2, 2)),
    (2, "staircase", (5, 5, 1)),
])
def test_distributed_matches_oracle(world, kind, args):
    ctx = mp.get_context("spawn")
    q_out = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, args, q_out)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q_out.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = np.concatenate([r[1] for r in res])
    circ = _circuit(kind, args)
    ref = orc.simulate(circ.num_qubits, circ.kinds, circ.qa, circ.qb, circ.params)
    assert np.abs(full - ref).max() < 1e-12


def test_plan_restores_permutation_and_counts_swaps():
    circ = G.build_brickwall(G.BASELINE_CONFIGS["cfg5_q34_n2_c2"])
    steps, nloc = plan(circ, 8)
    assert nloc == 31
    swaps = [s for s in steps if isinstance(s, Swap)]
    segs = [s for s in steps if isinstance(s, Segment)]
    assert all(s.local_bit == 30 and s.global_bit >= 31 for s in swaps)
    assert sum(len(s.gates) for s in segs) >= circ.gate_count
    assert 10 <= len(swaps) <= 80  # a few swaps per U3 layer on the 3 global qubits
