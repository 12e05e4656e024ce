"""Edge cases of the cut path on the GPU against the oracle: empty circuits,
no cuts (K = 1), one-qubit segments (n = q), the smallest q, thousands of
merge terms (launch chunking), repeated cuts at one position, complex64 with
n = 3, CX cuts with the target on either side, and the one-call pipeline on
all of them."""
import numpy as np
import pytest

from oracle import cutbench_oracle as orc

pytestmark = pytest.mark.gpu

TOL = 1e-10
TOL_C64 = 1e-5


@pytest.fixture(scope="module")
def cb():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_01443_b200 as pkg

    return pkg


def ref_state(c):
    return orc.simulate(c.num_qubits, c.kinds, c.qa, c.qb, c.params)


def both_paths(cb, circ, n, **kw):
    """run_cut (one native call) and the step-by-step drop-in API."""
    one = cb.run_cut(circ, n, **kw).amps
    subs = cb.decompose(circ, cb.plan_cut(circ, n))
    states = [[cb.simulate(c) for c in fam.circuits] for fam in subs.segments]
    step = cb.merge(cb.merge_input_from(subs, states)).amps
    return one, step


def test_empty_circuit(cb):
    from paper_2603_01443_b200.circuits import Circuit

    circ = Circuit(6, [])
    one, step = both_paths(cb, circ, 2)
    want = np.zeros(64, complex)
    want[0] = 1
    assert np.array_equal(one, want) and np.array_equal(step, want)
    assert np.array_equal(cb.simulate(circ).amps, want)


def test_no_cuts(cb):
    from paper_2603_01443_b200.circuits import Circuit, cz, h, t

    circ = Circuit(8, [h(i) for i in range(8)] + [cz(0, 1), t(3), cz(5, 6), h(7)])
    plan = cb.plan_cut(circ, 2)
    assert plan.c_total == 0
    one, step = both_paths(cb, circ, 2)
    ref = ref_state(circ)
    assert np.abs(one - ref).max() < TOL and np.abs(step - ref).max() < TOL


@pytest.mark.parametrize("q", [2, 3, 6])
def test_one_qubit_segments(cb, q):
    circ = cb.build_staircase(cb.BenchmarkSpec(q=q, n=q, blocks=2))
    one, step = both_paths(cb, circ, q)
    ref = ref_state(circ)
    assert np.abs(one - ref).max() < TOL and np.abs(step - ref).max() < TOL


def test_thousands_of_terms(cb):
    # c_total = 11 cuts on one boundary: K = 2048 terms (> one launch's table)
    circ = cb.build_brickwall(cb.BrickwallSpec(12, 4, 2, 11, 5))
    assert cb.plan_cut(circ, 2).c_total == 11
    one, step = both_paths(cb, circ, 2)
    ref = ref_state(circ)
    assert np.abs(one - ref).max() < TOL and np.abs(step - ref).max() < TOL


def test_repeated_cuts_same_layer(cb):
    # c > d forces several cuts into one layer at the same position
    circ = cb.build_brickwall(cb.BrickwallSpec(10, 2, 2, 5, 1))
    pos = [bg.position for bg in cb.plan_cut(circ, 2).boundary_gates]
    assert len(pos) == 5
    one, _ = both_paths(cb, circ, 2)
    assert np.abs(one - ref_state(circ)).max() < TOL


def test_complex64_three_segments(cb):
    circ = cb.build_brickwall(cb.BrickwallSpec(15, 6, 3, 4, 2))
    got = cb.run_cut(circ, 3, dtype=np.complex64).amps
    assert got.dtype == np.complex64
    assert np.abs(got - ref_state(circ)).max() < TOL_C64


def test_cx_cuts_both_orientations(cb):
    from paper_2603_01443_b200.circuits import Circuit, cx, h, t

    gates = [h(i) for i in range(8)] + [cx(3, 4), t(4), cx(4, 3), t(3), cx(3, 4), h(2), cx(4, 3)]
    circ = Circuit(8, gates)
    assert cb.plan_cut(circ, 2).c_total == 4
    one, step = both_paths(cb, circ, 2)
    ref = ref_state(circ)
    assert np.abs(one - ref).max() < TOL and np.abs(step - ref).max() < TOL


def test_unequal_sizes_one_call(cb):
    circ = cb.build_staircase(cb.BenchmarkSpec(q=10, n=2, blocks=3))
    ref = ref_state(circ)
    for sizes in [(1, 9), (9, 1), (3, 7), (2, 3, 5), (1, 1, 1, 7)]:
        got = cb.run_cut(circ, len(sizes), sizes=sizes).amps
        assert np.abs(got - ref).max() < TOL, sizes


@pytest.mark.parametrize("seed", range(12))
@pytest.mark.parametrize("jit", [0, 2])
def test_random_circuits_cut_equals_oracle(cb, seed, jit):
    """Random circuits over the full gate set (incl. U3, CX either way,
    repeated and back-to-back cuts) with random segment sizes: the one-call
    pipeline and the uncut simulator against the oracle, interpreter and
    NVRTC kernels."""
    from paper_2603_01443_b200 import _native
    from paper_2603_01443_b200.errors import UnsupportedTopologyError
    from test_host_cutting import _random_circuit

    rng = np.random.default_rng(1000 + seed)
    q = int(rng.integers(4, 11))
    circ = _random_circuit(rng, q, int(rng.integers(10, 70)))
    n = int(rng.integers(2, min(q, 4) + 1))
    cuts = np.sort(rng.choice(np.arange(1, q), size=n - 1, replace=False))
    sizes = tuple(int(v) for v in np.diff(np.concatenate([[0], cuts, [q]])))
    old = _native.get_option("jit")
    _native.set_option("jit", jit)
    try:
        ref = ref_state(circ)
        assert np.abs(cb.simulate(circ).amps - ref).max() < TOL
        try:
            got = cb.run_cut(circ, n, sizes=sizes).amps
        except UnsupportedTopologyError:
            return
        assert np.abs(got - ref).max() < TOL
    finally:
        _native.set_option("jit", old)


@pytest.mark.parametrize("jit", [0, 2])
def test_long_gate_tables_split_across_launches(cb, jit):
    """6800 gates on 12 qubits: register programs split into many launches
    (kMaxRegOps per launch, NVRTC cost guard) — interpreter and NVRTC."""
    from paper_2603_01443_b200 import _native

    circ = cb.build_brickwall(cb.BrickwallSpec(12, 400, 2, 3, 9))
    assert circ.gate_count > 6000
    old = _native.get_option("jit")
    _native.set_option("jit", jit)
    try:
        ref = ref_state(circ)
        assert np.abs(cb.simulate(circ).amps - ref).max() < TOL
        assert np.abs(cb.run_cut(circ, 2).amps - ref).max() < TOL
    finally:
        _native.set_option("jit", old)


def test_thousands_of_variants(cb):
    """c_total = 12 at n = 2: 4096 variants per segment in one batched launch
    sequence, a 4096-term merge."""
    circ = cb.build_brickwall(cb.BrickwallSpec(16, 6, 2, 12, 2))
    plan = cb.plan_cut(circ, 2)
    assert plan.c_total == 12 and cb.count_subcircuits(plan) == 2 * 4096
    got = cb.run_cut(circ, 2).amps
    assert np.abs(got - ref_state(circ)).max() < TOL


@pytest.mark.parametrize("q,d,n,c,seed", [(15, 5, 3, 10, 1), (15, 4, 5, 8, 3), (16, 3, 8, 7, 5)])
def test_many_segments_and_interior_cuts(cb, q, d, n, c, seed):
    """Chain contraction with wide interior bonds (10 cuts over n=3) and long
    chains (n = 5, 8 two-qubit segments), full state and a middle shard."""
    circ = cb.build_brickwall(cb.BrickwallSpec(q, d, n, c, seed))
    ref = ref_state(circ)
    full = cb.run_cut(circ, n).amps
    assert np.abs(full - ref).max() < TOL
    from paper_2603_01443_b200 import _native

    qlow = _native.cut_workspace(q, circ.table, [q // n] * n)[1]  # shard unit: the chosen bond's low side
    unit = 1 << qlow
    lo, hi = unit, min(1 << q, 3 * unit)
    shard = cb.run_cut(circ, n, out_range=(lo, hi))
    assert np.array_equal(shard.amps, full[lo:hi])


def test_reference_variant_loop_runs_one_batch_per_family(cb):
    """The reference's loop `[[simulate(c) for c in fam.circuits] ...]`
    (harness.py:136-139) costs one batched launch sequence per segment
    family; each call still returns a fresh, independent state equal to the
    variant circuit simulated on its own, and merge() reads the batch in
    place."""
    from paper_2603_01443_b200 import _native
    from paper_2603_01443_b200.circuits import h

    circ = cb.build_brickwall(cb.BrickwallSpec(14, 5, 2, 4, 3))
    subs = cb.decompose(circ, cb.plan_cut(circ, 2))
    fam = subs.segments[0]
    n0 = _native.launch_count()
    first = cb.simulate(fam.circuits[0])
    per_batch = _native.launch_count() - n0
    states = [[first] + [cb.simulate(c) for c in fam.circuits[1:]]]
    assert _native.launch_count() - n0 == per_batch  # the other variants came from the same batch
    states.append([cb.simulate(c) for c in subs.segments[1].circuits])
    for f, sts in zip(subs.segments, states):
        for b, sv in enumerate(sts):
            alone = cb.simulate(cb.Circuit.from_table(f.num_qubits, f.variant_table(b)))
            # one batched program vs a single-state one (other tiling): equal to rounding
            assert np.abs(sv.amps - alone.amps).max() < 1e-14
    merged = cb.merge(cb.merge_input_from(subs, states)).amps
    assert np.abs(merged - ref_state(circ)).max() < TOL
    again = cb.simulate(fam.circuits[1])  # a second request: a new pass, a fresh state
    cb.apply_gate(again, h(0))
    assert np.array_equal(states[0][1].amps, cb.simulate(fam.circuits[1]).amps)
