"""GPU parity: the sm_100a path (through the drop-in Python API over the
C-ABI) against the reference's golden outputs and the CPU oracle.

Tolerances (BASELINE.json north_star): complex128 max|d amp| <= 1e-10 and
1 - fidelity <= 1e-12; complex64 <= 1e-5. Hand values and per-gate checks
use the reference's own 1e-12 (tests/test_engine.py of the reference).
"""
import struct
import time

import numpy as np
import pytest

from conftest import golden_cases
from oracle import cutbench_oracle as orc

pytestmark = pytest.mark.gpu

TOL = 1e-10
FID_TOL = 1e-12
TOL_C64 = 1e-5


@pytest.fixture(scope="module")
def cb():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_01443_b200 as pkg

    return pkg


def fidelity(a, b):
    a = np.asarray(a, np.complex128)
    b = np.asarray(b, np.complex128)
    return abs(np.vdot(a, b)) ** 2 / (np.vdot(a, a).real * np.vdot(b, b).real)


def circuit_from(cb, golden, key):
    q = int(golden[f"{key}/q"])
    return cb.Circuit.from_table(q, cb.GateTable(golden[f"{key}/kinds"], golden[f"{key}/qa"],
                                                 golden[f"{key}/qb"]))


# -- reference KATs (tests/test_engine.py of the reference) --------------------
def test_known_answers(cb):
    from paper_2603_01443_b200.circuits import cx, cz, h, s, x

    assert np.allclose(cb.simulate(cb.Circuit(1, [h(0)])).amps, [2 ** -0.5, 2 ** -0.5], atol=1e-15)
    assert np.allclose(cb.simulate(cb.Circuit(2, [h(0), h(1), cz(0, 1)])).amps,
                       np.array([1, 1, 1, -1]) / 2, atol=1e-15)
    e = np.zeros(8)
    e[0] = 1
    assert np.array_equal(cb.simulate(cb.Circuit(3, [])).amps, e)
    for j in range(5):
        got = cb.simulate(cb.Circuit(5, [x(j)])).amps
        want = np.zeros(32)
        want[1 << j] = 1
        assert np.array_equal(got, want)
    sv = cb.StateVec(1, np.array([0, 1], dtype=complex))
    cb.apply_gate(sv, s(0))
    assert np.allclose(sv.amps, [0, 1j])
    sv = cb.StateVec(2, np.full(4, 0.5, dtype=complex))
    cb.apply_gate(sv, cz(0, 1))
    assert np.allclose(sv.amps, [0.5, 0.5, 0.5, -0.5])
    a = cb.StateVec(1, np.array([1, 0], dtype=complex))
    b = cb.StateVec(1, np.array([0, 1], dtype=complex))
    assert np.allclose(cb.tensor(a, b).amps, [0, 0, 1, 0])
    sv = cb.simulate(cb.Circuit(2, [h(0), cx(0, 1)]))
    assert sv.norm() == pytest.approx(1.0, abs=1e-14)


def test_dump_bytes(cb, tmp_path):
    from paper_2603_01443_b200.circuits import cx, h

    sv = cb.simulate(cb.Circuit(2, [h(0), cx(0, 1)]))
    path = tmp_path / "state.bin"
    cb.dump_amplitudes(sv, path)
    vals = struct.unpack("<8d", path.read_bytes())
    rt = np.sqrt(0.5)
    assert np.allclose(vals, [rt, 0, 0, 0, 0, 0, rt, 0], atol=1e-12)
    back = cb.load_amplitudes(path, 2)
    assert np.array_equal(back.amps, sv.amps)


def test_every_gate_on_random_state_vs_dense_oracle(cb, rng):
    from paper_2603_01443_b200.circuits import cx, cz, h, s, sdg, t, u3, x

    gates = [h(1), x(0), t(2), s(1), sdg(0), cx(0, 2), cx(2, 0), cz(1, 2), u3(1, 0.3, 1.1, -0.7)]
    for g in gates:
        amps = rng.normal(size=8) + 1j * rng.normal(size=8)
        amps /= np.linalg.norm(amps)
        sv = cb.StateVec(3, amps.copy())
        cb.apply_gate(sv, g)
        c = cb.Circuit(3, [g])
        k, qa, qb, p = c.kinds, c.qa, c.qb, c.params
        ref = amps.copy()
        orc.run_gates(ref, k, qa, qb, p)
        assert np.abs(sv.amps - ref).max() < 1e-12


def test_in_place_semantics_and_guards(cb):
    from paper_2603_01443_b200.circuits import x

    host = np.array([1, 0], dtype=complex)
    sv = cb.StateVec(1, host)
    cb.apply_gate(sv, x(0))
    assert sv.amps is host and np.allclose(host, [0, 1])
    with pytest.raises(cb.ValidationError):
        cb.apply_gate(sv, x(1))
    with pytest.raises(cb.CapacityError):
        cb.simulate(cb.Circuit(31, []), max_qubits=30)
    with pytest.raises(cb.CapacityError):
        cb.simulate(cb.Circuit(64, []))
    with pytest.raises(cb.BudgetExceededError):
        cb.simulate(cb.build_staircase(cb.BenchmarkSpec(8, 2, 2)), deadline=time.monotonic() - 1)
    sv = cb.simulate(cb.build_staircase(cb.BenchmarkSpec(4, 2, 1)), deadline=time.monotonic() + 60)
    assert abs(sv.norm() - 1) < 1e-10


# -- reference golden outputs ---------------------------------------------------
@pytest.mark.parametrize("key", golden_cases())
def test_uncut_matches_reference(cb, golden, key):
    circ = circuit_from(cb, golden, key)
    got = cb.simulate(circ).amps
    assert np.abs(got - golden[f"{key}/uncut"]).max() < 1e-12


@pytest.mark.parametrize("key", golden_cases())
def test_cut_pipeline_matches_reference(cb, golden, key):
    circ = circuit_from(cb, golden, key)
    n = int(golden[f"{key}/n"])
    plan = cb.plan_cut(circ, n)
    subs = cb.decompose(circ, plan)
    # the reference harness's per-variant loop, through the drop-in API
    states = [[cb.simulate(c) for c in fam.circuits] for fam in subs.segments]
    for fam, sts in zip(subs.segments, states):
        ref = golden[f"{key}/seg{fam.segment}/states"]
        for v, sv in enumerate(sts):
            assert np.abs(sv.amps - ref[v]).max() < 1e-12
    merged = cb.merge(cb.merge_input_from(subs, states))
    assert np.abs(merged.amps - golden[f"{key}/merged"]).max() < 1e-12
    # batched family path + chain merge
    out = cb.run_cut(circ, n)
    assert np.abs(out.amps - golden[f"{key}/merged"]).max() < 1e-12
    assert np.abs(out.amps - golden[f"{key}/uncut"]).max() < TOL


def test_generic_merge_permuted_table(cb, golden):
    # reference tests/test_merging.py:51-76 (blocked path and permutation soundness)
    for key in ("stair_q4_n2_b13", "stair_q6_n2_b3", "stair_q8_n4_b2"):
        circ = circuit_from(cb, golden, key)
        n = int(golden[f"{key}/n"])
        subs = cb.decompose(circ, cb.plan_cut(circ, n))
        states = [[cb.simulate(c) for c in fam.circuits] for fam in subs.segments]
        base = cb.merge(cb.merge_input_from(subs, states))
        perm = np.random.default_rng(11).permutation(len(subs.coeffs))
        shuffled = cb.MergeInput(states, subs.coeffs[perm], subs.merge_table[:, perm], circ.num_qubits)
        assert shuffled.chain is None
        again = cb.merge(shuffled)
        assert np.abs(base.amps - again.amps).max() < 1e-12
        assert np.abs(again.amps - golden[f"{key}/uncut"]).max() < TOL


def test_merge_streaming_matches_merge(cb, golden):
    key = "stair_q6_n3_b2"
    circ = circuit_from(cb, golden, key)
    subs = cb.decompose(circ, cb.plan_cut(circ, 3))
    states = [[cb.simulate(c) for c in fam.circuits] for fam in subs.segments]
    a = cb.merge(cb.merge_input_from(subs, states))
    fams = [f.circuits for f in subs.segments]
    b = cb.merge_streaming(lambda s, i: cb.simulate(fams[s][i]), subs.coeffs, subs.merge_table, 6)
    assert np.abs(a.amps - b.amps).max() < 1e-12
    with pytest.raises(cb.ValidationError):
        cb.merge_streaming(lambda s, i: cb.simulate(fams[s][i]), subs.coeffs, subs.merge_table, 7)


def test_merge_validation_errors(cb):
    from paper_2603_01443_b200.circuits import h

    circ = cb.Circuit(4, [h(0)])
    subs = cb.decompose(circ, cb.plan_cut(circ, 2))
    states = [[cb.simulate(c) for c in f.circuits] for f in subs.segments]
    with pytest.raises(cb.CapacityError):
        cb.merge(cb.merge_input_from(subs, states), max_qubits=3)
    with pytest.raises(cb.ValidationError):
        cb.MergeInput(states, subs.coeffs, subs.merge_table, num_qubits=5)


# -- BASELINE U3 family vs the oracle ---------------------------------------------
@pytest.mark.parametrize("q,d,n,c,seed", [(12, 4, 2, 1, 0), (20, 10, 2, 2, 0), (12, 5, 3, 4, 1),
                                          (16, 6, 4, 4, 2), (18, 5, 3, 2, 3), (16, 8, 2, 6, 4)])
def test_u3_cut_pipeline_vs_oracle(cb, q, d, n, c, seed):
    circ = cb.build_brickwall(cb.BrickwallSpec(q, d, n, c, seed))
    k, qa, qb, p = circ.kinds, circ.qa, circ.qb, circ.params
    ref_uncut = orc.simulate(q, k, qa, qb, p)
    cut = cb.run_cut(circ, n).amps
    assert np.abs(cut - ref_uncut).max() < TOL
    assert 1 - fidelity(cut, ref_uncut) < FID_TOL
    uncut = cb.simulate(circ).amps
    assert np.abs(uncut - ref_uncut).max() < TOL
    if q <= 12:
        ref_cut, _, _, _ = orc.cut_pipeline(q, k, qa, qb, p, n)
        assert np.abs(cut - ref_cut).max() < TOL


@pytest.mark.parametrize("tile_bits", [4, 7, 10, 12])
def test_multi_sweep_uncut_vs_oracle(cb, tile_bits):
    from paper_2603_01443_b200 import _native

    old = _native.get_option("tile_bits")
    try:
        _native.set_option("tile_bits", tile_bits)
        for q, d, seed in [(14, 6, 0), (18, 4, 1)]:
            circ = cb.build_brickwall(cb.BrickwallSpec(q, d, 2, 3, seed))
            ref = orc.simulate(q, circ.kinds, circ.qa, circ.qb, circ.params)
            assert np.abs(cb.simulate(circ).amps - ref).max() < TOL
    finally:
        _native.set_option("tile_bits", old)


def test_staircase_multi_sweep_and_cx(cb):
    # CX with control/target on either side of the tile boundary
    circ = cb.build_staircase(cb.BenchmarkSpec(q=16, n=2, blocks=2))
    ref = orc.simulate(16, circ.kinds, circ.qa, circ.qb)
    assert np.abs(cb.simulate(circ).amps - ref).max() < TOL
    cut = cb.run_cut(circ, 2).amps
    assert np.abs(cut - ref).max() < TOL


def test_complex64_mode(cb):
    circ = cb.build_brickwall(cb.BrickwallSpec(16, 6, 2, 2, 0))
    ref = orc.simulate(16, circ.kinds, circ.qa, circ.qb, circ.params)
    got = cb.run_cut(circ, 2, dtype=np.complex64).amps
    assert got.dtype == np.complex64
    assert np.abs(got - ref).max() < TOL_C64
    got_uncut = cb.simulate(circ, dtype=np.complex64).amps
    assert np.abs(got_uncut - ref).max() < TOL_C64


def test_sharded_output_ranges_concatenate(cb):
    circ = cb.build_brickwall(cb.BrickwallSpec(16, 5, 4, 4, 3))
    full = cb.run_cut(circ, 4).amps
    world = 4
    parts = []
    for r in range(world):
        lo, hi = r * (1 << 16) // world, (r + 1) * (1 << 16) // world
        shard = cb.run_cut(circ, 4, out_range=(lo, hi))
        parts.append(shard.amps)
    assert np.array_equal(np.concatenate(parts), full)


def test_forced_bonds_agree(cb):
    from paper_2603_01443_b200.merging import merge_chain_device
    from paper_2603_01443_b200.pipeline import preprocess, simulate_segments

    circ = cb.build_brickwall(cb.BrickwallSpec(16, 5, 4, 4, 7))
    prep = preprocess(circ, 4)
    batches = simulate_segments(prep)
    outs = [merge_chain_device(prep.chain, batches, force_bond=k).cpu().numpy() for k in range(3)]
    ref = orc.simulate(16, circ.kinds, circ.qa, circ.qb, circ.params)
    for o in outs:
        assert np.abs(o - ref).max() < TOL


# -- full size -----------------------------------------------------------------
def test_q30_cfg4a_cut_vs_gpu_uncut_and_sampled_oracle(cb):
    from paper_2603_01443_b200 import engine

    spec = cb.BASELINE_CONFIGS["cfg4a"]
    circ = cb.build_brickwall(spec)
    cut = cb.run_cut(circ, 2)
    uncut = cb.simulate(circ)
    diff = engine.max_abs_diff(cut, uncut)
    assert diff < TOL
    re, im = engine.inner(uncut, cut)
    n1 = engine.inner(cut, cut)[0]
    n2 = engine.inner(uncut, uncut)[0]
    assert 1 - (re * re + im * im) / (n1 * n2) < FID_TOL
    # sampled amplitudes against the CPU oracle's subcircuit states
    k, qa, qb, p = circ.kinds, circ.qa, circ.qb, circ.params
    sizes = [15, 15]
    bgs, counts, _ = orc.plan(k, qa, qb, sizes)
    states = []
    for seg in range(2):
        vs = orc.segment_variants(k, qa, qb, p, sizes, bgs, seg)
        states.append([orc.simulate(15, *v) for v in vs])
    tab = orc.merge_table(2, bgs, sum(counts))
    co = orc.coefficients(sum(counts))
    idx = np.random.default_rng(5).integers(0, 1 << 30, size=4096)
    want = orc.sample_amplitudes(states, tab, co, sizes, idx)
    got = engine.gather(cut, idx)
    assert np.abs(got - want).max() < TOL
    del cut, uncut


@pytest.mark.parametrize("c_total", [4, 6])
def test_q30_int8_tensor_core_merge_cut_vs_uncut(cb, c_total):
    """q=30 (15|15) with K = 2^c_total = 16 / 64 cut terms: the merge runs on
    the int8 tcgen05 kernel (ozaki.cu); the full 16 GiB state against the
    GPU uncut simulator and sampled amplitudes against the CPU oracle's
    subcircuit states."""
    from paper_2603_01443_b200 import _native, engine

    assert _native.get_option("merge_ozaki") == 1
    spec = cb.BrickwallSpec(30, 10, 2, c_total, 0)
    circ = cb.build_brickwall(spec)
    n0 = _native.launch_count()
    cut = cb.run_cut(circ, 2)
    assert _native.launch_count() - n0 >= 3  # prep_lo, prep_hi, the tcgen05 kernel
    uncut = cb.simulate(circ)
    assert engine.max_abs_diff(cut, uncut) < TOL
    re, im = engine.inner(uncut, cut)
    n1 = engine.inner(cut, cut)[0]
    n2 = engine.inner(uncut, uncut)[0]
    assert 1 - (re * re + im * im) / (n1 * n2) < FID_TOL
    k, qa, qb, p = circ.kinds, circ.qa, circ.qb, circ.params
    sizes = [15, 15]
    bgs, counts, _ = orc.plan(k, qa, qb, sizes)
    states = []
    for seg in range(2):
        vs = orc.segment_variants(k, qa, qb, p, sizes, bgs, seg)
        states.append([orc.simulate(15, *v) for v in vs])
    tab = orc.merge_table(2, bgs, sum(counts))
    co = orc.coefficients(sum(counts))
    idx = np.random.default_rng(7).integers(0, 1 << 30, size=2048)
    want = orc.sample_amplitudes(states, tab, co, sizes, idx)
    assert np.abs(engine.gather(cut, idx) - want).max() < TOL
    del cut, uncut


def test_q32_cfg5_c4_int8_merge_cut_vs_uncut(cb):
    """BASELINE cfg5 at full size on one GPU: q=32 (16|16), c_total=4 (K=16,
    int8 tcgen05 merge) — the 64 GiB cut state against the 64 GiB uncut
    state from the GPU simulator (needs ~130 GB of free device memory)."""
    import torch

    from paper_2603_01443_b200 import engine

    torch.cuda.empty_cache()
    free, _total = torch.cuda.mem_get_info()
    if free < 140 * 2**30:
        pytest.skip(f"needs ~140 GB free device memory, {free / 2**30:.0f} GiB free")
    circ = cb.build_brickwall(cb.BASELINE_CONFIGS["cfg5_q32_n2_c4"])
    cut = cb.run_cut(circ, 2, max_qubits=32)
    uncut = cb.simulate(circ, max_qubits=32)
    assert engine.max_abs_diff(cut, uncut) < TOL
    re, im = engine.inner(uncut, cut)
    n1 = engine.inner(cut, cut)[0]
    n2 = engine.inner(uncut, uncut)[0]
    assert 1 - (re * re + im * im) / (n1 * n2) < FID_TOL
    del cut, uncut
    torch.cuda.empty_cache()


def test_q30_cfg4b_three_way(cb):
    from paper_2603_01443_b200 import engine

    circ = cb.build_brickwall(cb.BASELINE_CONFIGS["cfg4b"])
    cut = cb.run_cut(circ, 3)
    uncut = cb.simulate(circ)
    assert engine.max_abs_diff(cut, uncut) < TOL
    del cut, uncut


def test_q34_shard_sampled_vs_oracle(cb):
    """One GPU's share of the 8-GPU q=34 job (rows [0, 2^17/8)) against the
    oracle's sampled amplitudes sum_m alpha_m prod_i psi_i[x_i]."""
    import torch

    from paper_2603_01443_b200.merging import merge_chain_device
    from paper_2603_01443_b200.parallel import shard_range
    from paper_2603_01443_b200.pipeline import preprocess, simulate_segments

    spec = cb.BASELINE_CONFIGS["cfg5_q34_n2_c2"]
    circ = cb.build_brickwall(spec)
    prep = preprocess(circ, 2)
    for rank in (0, 5):
        begin, end = shard_range(34, 8, rank, 17)
        out = merge_chain_device(prep.chain, simulate_segments(prep), out_range=(begin, end))
        k, qa, qb, p = circ.kinds, circ.qa, circ.qb, circ.params
        sizes = [17, 17]
        bgs, counts, _ = orc.plan(k, qa, qb, sizes)
        states = [[orc.simulate(17, *v) for v in orc.segment_variants(k, qa, qb, p, sizes, bgs, s)]
                  for s in range(2)]
        idx = np.random.default_rng(rank).integers(begin, end, size=2048)
        want = orc.sample_amplitudes(states, orc.merge_table(2, bgs, sum(counts)),
                                     orc.coefficients(sum(counts)), sizes, idx)
        got = out[torch.as_tensor(idx - begin, device="cuda")].cpu().numpy()
        assert np.abs(got - want).max() < TOL
        del out
        torch.cuda.empty_cache()


@pytest.mark.parametrize("world,q,d", [(2, 14, 6), (8, 16, 5), (4, 20, 4)])
def test_distributed_uncut_emulated_on_one_gpu(cb, world, q, d):
    """The q >= 33 distributed simulator's schedule and per-rank gate tables,
    all ranks in lockstep on one GPU (exchange = device copy)."""
    from paper_2603_01443_b200.distributed import simulate_emulated

    circ = cb.build_brickwall(cb.BrickwallSpec(q, d, 2, 2, world))
    got = simulate_emulated(circ, world).cpu().numpy()
    ref = orc.simulate(q, circ.kinds, circ.qa, circ.qb, circ.params)
    assert np.abs(got - ref).max() < TOL


def test_distributed_uncut_world1_default_path(cb):
    """simulate_distributed's own device path at one rank (rank 0 starts from
    |0..0> inside the library: zero-start tiles) equals simulate()."""
    from paper_2603_01443_b200.distributed import simulate_distributed

    circ = cb.build_brickwall(cb.BrickwallSpec(22, 6, 2, 2, 3))
    got = simulate_distributed(circ, rank=0, world=1).cpu().numpy()
    ref = cb.simulate(circ).amps
    assert np.abs(got - ref).max() < 1e-12


def test_run_cut_to_host_matches_device_state(cb):
    """The e2e path of bench.py (cs_cut_run_to_host: chunked merge overlapped
    with D2H into host memory) for pinned tensors, numpy arrays, ragged chunk
    counts, n = 3 and complex64."""
    import torch

    from paper_2603_01443_b200.pipeline import StageTimes, run_cut_to_host

    circ = cb.build_brickwall(cb.BrickwallSpec(20, 6, 2, 2, 3))
    dev = cb.run_cut(circ, 2).amps
    for chunks in (1, 3, 8, 64):
        host = torch.empty(1 << 20, dtype=torch.complex128, pin_memory=True)
        run_cut_to_host(circ, 2, host, chunks=chunks)
        assert np.array_equal(host.numpy(), dev), chunks
    arr = np.empty(1 << 20, np.complex128)
    t = StageTimes()
    run_cut_to_host(circ, 2, arr, timers=t)
    assert np.array_equal(arr, dev) and t.sub > 0 and t.merge > 0
    c3 = cb.build_brickwall(cb.BrickwallSpec(18, 5, 3, 4, 1))
    arr3 = np.empty(1 << 18, np.complex128)
    run_cut_to_host(c3, 3, arr3, chunks=5)
    assert np.array_equal(arr3, cb.run_cut(c3, 3).amps)
    a64 = np.empty(1 << 20, np.complex64)
    run_cut_to_host(circ, 2, a64, dtype=np.complex64)
    assert np.abs(a64 - dev).max() < 1e-5
    with pytest.raises(cb.ValidationError):
        run_cut_to_host(circ, 2, np.empty(10, np.complex128))


def test_sharded_pipeline_over_nccl_world1(cb):
    """run_cut_sharded through a real NCCL process group (world size 1 on one
    GPU: the all-gather path runs, no rank waits on another)."""
    import os
    import socket

    import torch
    import torch.distributed as dist

    from paper_2603_01443_b200.parallel import run_cut_sharded

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        circ = cb.build_brickwall(cb.BrickwallSpec(18, 5, 3, 4, 2))
        res, (b, e) = run_cut_sharded(circ, 3, rank=0, world=1)
        assert (b, e) == (0, 1 << 18)
        assert np.abs(res.cpu().numpy() - cb.run_cut(circ, 3).amps).max() < 1e-14
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("q,d,sizes,c,seed", [(12, 4, (6, 6), 1, 0), (15, 5, (5, 5, 5), 4, 1),
                                               (16, 5, (4, 4, 4, 4), 4, 3), (14, 6, (7, 7), 3, 4)])
def test_one_call_pipeline_equals_stepwise(cb, q, d, sizes, c, seed):
    """cs_cut_run (C++ preprocess + batched sweeps + chain merge in one call)
    is bit-identical to the step-by-step Python path and within TOL of the oracle."""
    from paper_2603_01443_b200.merging import merge_chain_device
    from paper_2603_01443_b200.pipeline import preprocess, simulate_segments

    n = len(sizes)
    circ = cb.build_brickwall(cb.BrickwallSpec(q, d, n, c, seed))
    one = cb.run_cut(circ, n).amps
    prep = preprocess(circ, n)
    step = merge_chain_device(prep.chain, simulate_segments(prep)).cpu().numpy()
    assert np.array_equal(one, step)
    ref = orc.simulate(q, circ.kinds, circ.qa, circ.qb, circ.params)
    assert np.abs(one - ref).max() < TOL


def test_one_call_pipeline_unequal_sizes_bonds_events(cb):
    import torch

    from paper_2603_01443_b200.errors import UnsupportedTopologyError, ValidationError

    circ = cb.build_staircase(cb.BenchmarkSpec(q=12, n=3, blocks=3))
    ref = orc.simulate(12, circ.kinds, circ.qa, circ.qb, circ.params)
    for sizes in [(3, 4, 5), (6, 6), (2, 5, 5)]:
        got = cb.run_cut(circ, len(sizes), sizes=sizes).amps
        assert np.abs(got - ref).max() < TOL
    circ = cb.build_brickwall(cb.BrickwallSpec(16, 5, 4, 4, 7))
    ref = orc.simulate(16, circ.kinds, circ.qa, circ.qb, circ.params)
    for k in range(3):
        assert np.abs(cb.run_cut(circ, 4, force_bond=k).amps - ref).max() < TOL
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    times = cb.StageTimes()
    got = cb.run_cut(circ, 4, events=evs, timers=times).amps
    assert np.abs(got - ref).max() < TOL
    assert evs[0].elapsed_time(evs[1]) > 0 and evs[1].elapsed_time(evs[2]) > 0
    assert times.pre > 0 and times.sub > 0 and times.merge > 0
    with pytest.raises(ValidationError):
        cb.run_cut(circ, 3)
    with pytest.raises(UnsupportedTopologyError):
        from paper_2603_01443_b200 import circuits as C

        cb.run_cut(C.Circuit(3, [C.h(0), C.cx(0, 2)]), 3)
    with pytest.raises(ValidationError):
        cb.run_cut(circ, 4, workspace=torch.empty(16, dtype=torch.uint8, device="cuda"),
                   out=torch.empty(1 << 16, dtype=torch.complex128, device="cuda"))


def test_native_nccl_comm_world1(cb):
    """libcutsim's NCCL binding on one GPU: all-gather, self send/recv, and the
    sharded pipeline routed through it."""
    import torch

    from paper_2603_01443_b200.comm import NcclComm
    from paper_2603_01443_b200.parallel import run_cut_sharded

    comm = NcclComm.create(0, 1)
    try:
        send = torch.arange(1000, dtype=torch.float64, device="cuda")
        recv = torch.empty_like(send)
        comm.all_gather(recv, send)
        torch.cuda.synchronize()
        assert torch.equal(recv, send)
        back = torch.empty_like(send)
        comm.sendrecv(send * 2, back, 0)
        torch.cuda.synchronize()
        assert torch.equal(back, send * 2)
        circ = cb.build_brickwall(cb.BrickwallSpec(16, 5, 2, 2, 4))
        res, (b, e) = run_cut_sharded(circ, 2, rank=0, world=1, comm=comm)
        assert (b, e) == (0, 1 << 16)
        assert np.array_equal(res.cpu().numpy(), cb.run_cut(circ, 2).amps)
    finally:
        comm.destroy()


def test_deadline_checked_per_sweep_without_splitting_the_program(cb):
    """simulate(deadline=...) runs the same fused program as without one
    (cs_sim_batch_until checks the budget after every sweep launch): results
    identical, and a budget that expires mid-run raises BudgetExceededError
    (the reference's cooperative timeout, engine.py:142-155)."""
    circ = cb.build_brickwall(cb.BrickwallSpec(24, 10, 2, 2, 1))
    free = cb.simulate(circ).amps
    timed = cb.simulate(circ, deadline=time.monotonic() + 60).amps
    assert np.array_equal(free, timed)
    big = cb.build_brickwall(cb.BrickwallSpec(28, 10, 2, 2, 1))
    cb.simulate(big, max_qubits=28)  # build (and compile) the program first
    with pytest.raises(cb.BudgetExceededError):
        cb.simulate(big, max_qubits=28, deadline=time.monotonic() + 1e-4)
