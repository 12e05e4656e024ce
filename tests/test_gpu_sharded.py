"""The sharded (multi-GPU) cut pipeline's one native call per rank,
cs_cut_run_sharded (pipeline.run_cut_sharded_native), on one GPU.

* comm = None: the rank simulates every variant itself (no exchange) and
  writes its rows — any (rank, world) share can be computed and checked on one
  GPU without ranks waiting on each other;
* a world-1 NCCL communicator: the in-place all-gather runs;
* one GPU's share of the 8-GPU q=34 job (BASELINE cfg5) and of the 4-GPU
  q=32 n=4 job, sampled against the CPU oracle.
Each rank's rows are rows [begin, end) of reference merging.py:156-186.
"""
import numpy as np
import pytest

from oracle import cutbench_oracle as orc

pytestmark = pytest.mark.gpu

TOL = 1e-10


@pytest.fixture(scope="module")
def cb():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_01443_b200 as pkg

    return pkg


def oracle_samples(circ, n, idx):
    q = circ.num_qubits
    sizes = [q // n] * n
    k, qa, qb, p = circ.kinds, circ.qa, circ.qb, circ.params
    bgs, counts, _ = orc.plan(k, qa, qb, sizes)
    states = [[orc.simulate(sizes[s], *v) for v in orc.segment_variants(k, qa, qb, p, sizes, bgs, s)]
              for s in range(n)]
    return orc.sample_amplitudes(states, orc.merge_table(n, bgs, sum(counts)), orc.coefficients(sum(counts)),
                                 sizes, idx)


@pytest.mark.parametrize("q,d,n,c,seed", [(18, 5, 3, 4, 2), (20, 6, 2, 4, 1), (16, 5, 4, 4, 3), (14, 4, 2, 2, 0)])
@pytest.mark.parametrize("world", [2, 3, 8])
def test_every_rank_share_equals_the_full_state_rows(cb, q, d, n, c, seed, world):
    from paper_2603_01443_b200.pipeline import run_cut_sharded_native

    circ = cb.build_brickwall(cb.BrickwallSpec(q, d, n, c, seed))
    full = cb.run_cut(circ, n).amps
    ends = []
    for rank in range(world):
        sh = run_cut_sharded_native(circ, n, rank=rank, world=world)
        ends.append((sh.begin, sh.end))
        assert np.abs(sh.amps - full[sh.begin:sh.end]).max() < 1e-14
    assert ends[0][0] == 0 and ends[-1][1] == 1 << q
    assert all(a[1] == b[0] for a, b in zip(ends, ends[1:]))
    ref = orc.simulate(q, circ.kinds, circ.qa, circ.qb, circ.params)
    assert np.abs(full - ref).max() < TOL


def test_nccl_world1_exchange_and_stage_times(cb):
    import torch

    from paper_2603_01443_b200.comm import NcclComm
    from paper_2603_01443_b200.pipeline import run_cut_sharded_native

    comm = NcclComm.create(0, 1)
    try:
        circ = cb.build_brickwall(cb.BrickwallSpec(20, 6, 2, 2, 5))
        timers = {}
        sv = run_cut_sharded_native(circ, 2, rank=0, world=1, comm=comm, timers=timers)
        assert np.array_equal(sv.amps, cb.run_cut(circ, 2).amps)
        assert set(timers) == {"pre", "sub", "exchange", "merge"} and all(v >= 0 for v in timers.values())
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        run_cut_sharded_native(circ, 2, rank=0, world=1, comm=comm, events=evs)
        torch.cuda.synchronize()
        assert evs[2].elapsed_time(evs[3]) > 0
    finally:
        comm.destroy()


def test_unequal_sizes_and_bad_ranges_are_rejected(cb):
    from paper_2603_01443_b200.errors import ValidationError
    from paper_2603_01443_b200.pipeline import run_cut_sharded_native

    circ = cb.build_brickwall(cb.BrickwallSpec(12, 4, 2, 2, 0))
    with pytest.raises(ValidationError):
        run_cut_sharded_native(circ, 5)
    with pytest.raises(ValidationError):
        run_cut_sharded_native(circ, 2, rank=2, world=2)
    with pytest.raises(ValidationError):
        run_cut_sharded_native(circ, 2, out_range=(3, 100))


@pytest.mark.parametrize("name,n,world,ranks", [("cfg5_q34_n2_c2", 2, 8, (0, 5)), ("cfg5_q32_n4_c4", 4, 4, (3,)),
                                                ("cfg5_q32_n2_c4", 2, 8, (7,))])
def test_one_gpu_share_of_the_sharded_baseline_jobs(cb, name, n, world, ranks):
    """BASELINE cfg5: one rank's share through the same native call the
    multi-GPU bench runs (32 GiB for q=34 at 8 GPUs), sampled against the
    oracle's sum_m alpha_m prod_i psi_i^{r_i(m)}[x_i]."""
    import torch

    from paper_2603_01443_b200 import _native
    from paper_2603_01443_b200.pipeline import run_cut_sharded_native

    spec = cb.BASELINE_CONFIGS[name]
    circ = cb.build_brickwall(spec)
    old = _native.get_option("jit")
    _native.set_option("jit", 2)
    try:
        for rank in ranks:
            sh = run_cut_sharded_native(circ, n, rank=rank, world=world)
            idx = np.random.default_rng(rank + spec.q).integers(sh.begin, sh.end, size=4096)
            got = sh.device[torch.as_tensor(idx - sh.begin, device="cuda")].cpu().numpy()
            assert np.abs(got - oracle_samples(circ, n, idx)).max() < TOL
            del sh
            torch.cuda.empty_cache()
    finally:
        _native.set_option("jit", old)
