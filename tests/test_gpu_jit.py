"""NVRTC-specialised sweep kernels (cs_set_option("jit", 2)) against the
oracle: uncut multi-sweep circuits, cut-variant batches with slots,
controlled gates, complex64. The host-only NVRTC compile runs on CPU too."""
import numpy as np
import pytest

from oracle import cutbench_oracle as orc
from paper_2603_01443_b200 import _native
from paper_2603_01443_b200 import circuits as C
from paper_2603_01443_b200 import generators as G
from paper_2603_01443_b200.pipeline import preprocess


def test_nvrtc_compiles_generated_kernels_on_cpu():
    circ = G.build_brickwall(G.BrickwallSpec(14, 3, 2, 2, 0))
    prep = preprocess(circ, 2)
    fam = prep.subs.segments[0]
    assert _native.jit_selftest(fam.num_qubits, fam.template, fam.slots, n_states=fam.num_variants) > 1000
    stair = C.build_staircase(C.BenchmarkSpec(q=14, n=2, blocks=2))
    assert _native.jit_selftest(14, stair.table, n_states=1) > 1000


@pytest.mark.parametrize("dtype", [_native.CS_C128, _native.CS_C64])
def test_nvrtc_compiles_param_mode_kernels_on_cpu(dtype):
    """Param mode (jit_struct): the coefficients become kernel parameters;
    the generated sources still compile to sm_100a CUBINs."""
    old = (_native.get_option("jit"), _native.get_option("jit_struct"))
    _native.set_option("jit", 2)
    _native.set_option("jit_struct", 2)
    try:
        circ = G.build_brickwall(G.BrickwallSpec(14, 3, 2, 2, 0))
        fam = preprocess(circ, 2).subs.segments[1]
        assert _native.jit_selftest(fam.num_qubits, fam.template, fam.slots, n_states=fam.num_variants,
                                    dtype=dtype) > 1000
        assert _native.jit_selftest(14, circ.table, n_states=1, dtype=dtype) > 1000
    finally:
        _native.set_option("jit", old[0])
        _native.set_option("jit_struct", old[1])


@pytest.fixture
def jit_on():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    old = _native.get_option("jit")
    _native.set_option("jit", 2)
    yield
    _native.set_option("jit", old)


@pytest.mark.gpu
@pytest.mark.parametrize("q,d,n,c,seed", [(14, 5, 2, 3, 0), (18, 4, 2, 2, 1), (12, 4, 3, 4, 2)])
def test_jit_cut_and_uncut_match_oracle(jit_on, q, d, n, c, seed):
    import paper_2603_01443_b200 as cb

    circ = cb.build_brickwall(cb.BrickwallSpec(q, d, n, c, seed))
    ref = orc.simulate(q, circ.kinds, circ.qa, circ.qb, circ.params)
    assert np.abs(cb.simulate(circ).amps - ref).max() < 1e-10
    assert np.abs(cb.run_cut(circ, n).amps - ref).max() < 1e-10


@pytest.mark.gpu
def test_jit_controlled_gates_and_complex64(jit_on):
    import paper_2603_01443_b200 as cb

    circ = cb.build_staircase(cb.BenchmarkSpec(q=16, n=2, blocks=2))
    ref = orc.simulate(16, circ.kinds, circ.qa, circ.qb)
    assert np.abs(cb.simulate(circ).amps - ref).max() < 1e-10
    got = cb.simulate(circ, dtype=np.complex64).amps
    assert np.abs(got - ref).max() < 1e-5


@pytest.mark.gpu
@pytest.mark.parametrize("key", ["stair_q8_n4_b2", "stair_q6_n2_b3", "shadow_q9_d4_n3_c4_s3", "stair_q12_n3_b1",
                                 "padded_q6_n2_b1_p1"])
def test_jit_normalised_kernels_match_reference_golden(jit_on, golden, key):
    """The default specialised lowering (normalised 2x2s with deferred
    diagonals) on the reference's own golden uncut and merged states."""
    import paper_2603_01443_b200 as cb

    assert _native.get_option("dense_norm") == 2
    q, n = int(golden[f"{key}/q"]), int(golden[f"{key}/n"])
    circ = cb.Circuit.from_table(q, cb.GateTable(golden[f"{key}/kinds"], golden[f"{key}/qa"],
                                                 golden[f"{key}/qb"]))
    assert np.abs(cb.simulate(circ).amps - golden[f"{key}/uncut"]).max() < 1e-12
    assert np.abs(cb.run_cut(circ, n).amps - golden[f"{key}/merged"]).max() < 1e-12


@pytest.mark.gpu
def test_jit_q22_multisweep_u3(jit_on):
    import paper_2603_01443_b200 as cb

    circ = cb.build_brickwall(cb.BrickwallSpec(22, 8, 2, 3, 7))
    ref = orc.simulate(22, circ.kinds, circ.qa, circ.qb, circ.params)
    got = cb.simulate(circ).amps
    assert np.abs(got - ref).max() < 1e-10
    assert abs(np.vdot(got, got).real - 1) < 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("persistent,minb", [(1, 1), (0, 1), (0, 2)])
def test_jit_streaming_kernel_forms(jit_on, persistent, minb):
    """The opt-in persistent prefetching form and both launch-bound settings
    of the many-tile (streaming) kernels against the oracle."""
    import paper_2603_01443_b200 as cb

    old = _native.get_option("jit_persistent"), _native.get_option("jit_minb")
    _native.set_option("jit_persistent", persistent)
    _native.set_option("jit_minb", minb)
    try:
        circ = cb.build_brickwall(cb.BrickwallSpec(22, 4, 2, 2, 3))
        ref = orc.simulate(22, circ.kinds, circ.qa, circ.qb, circ.params)
        assert np.abs(cb.simulate(circ).amps - ref).max() < 1e-10
        stair = cb.build_staircase(cb.BenchmarkSpec(q=22, n=2, blocks=1))
        ref = orc.simulate(22, stair.kinds, stair.qa, stair.qb)
        assert np.abs(cb.simulate(stair).amps - ref).max() < 1e-10
    finally:
        _native.set_option("jit_persistent", old[0])
        _native.set_option("jit_minb", old[1])


@pytest.mark.gpu
def test_jit_deep_circuit_complex64_stays_finite(jit_on):
    """A 300-layer circuit through the normalised NVRTC kernels in complex64:
    without the growth budget the executed amplitudes would pass 2^128."""
    import paper_2603_01443_b200 as cb

    circ = cb.build_brickwall(cb.BrickwallSpec(12, 300, 2, 2, 4))
    ref = orc.simulate(12, circ.kinds, circ.qa, circ.qb, circ.params)
    got = cb.simulate(circ, dtype=np.complex64).amps
    assert np.isfinite(got).all() and np.abs(got - ref).max() < 1e-4
    assert np.abs(cb.simulate(circ).amps - ref).max() < 1e-10


@pytest.mark.gpu
def test_jit_apply_circuit_on_arbitrary_state(jit_on):
    """engine.apply_circuit (init = 0) on a random state through the normalised
    NVRTC kernels: the deferred diagonals and global scalar must land on any
    input state, not only |0...0>."""
    import paper_2603_01443_b200 as cb
    from paper_2603_01443_b200 import engine

    rng = np.random.default_rng(17)
    for q, d in ((10, 6), (16, 4)):
        circ = cb.build_brickwall(cb.BrickwallSpec(q, d, 2, 2, 5))
        amps = rng.normal(size=1 << q) + 1j * rng.normal(size=1 << q)
        amps /= np.linalg.norm(amps)
        sv = cb.StateVec(q, amps.copy())
        for _ in range(2):  # second pass: compiled program reused on a new state
            sv = cb.StateVec(q, amps.copy())
            engine.apply_circuit(sv, circ)
        ref = amps.copy()
        orc.run_gates(ref, circ.kinds, circ.qa, circ.qb, circ.params)
        assert np.abs(sv.amps - ref).max() < 1e-10


def _angles_perturbed(circ, seed):
    """The same gate structure with new U3 angles."""
    rng = np.random.default_rng(seed)
    p = circ.params.copy()
    u3 = circ.kinds == C.KIND_U3
    p[u3] = rng.uniform(0, np.pi, size=(int(u3.sum()), 3))
    return C.Circuit.from_table(circ.num_qubits, C.GateTable(circ.kinds, circ.qa, circ.qb, p))


@pytest.mark.gpu
@pytest.mark.parametrize("dtype,tol", [(np.complex128, 1e-10), (np.complex64, 1e-5)])
def test_param_mode_kernels_match_oracle(jit_on, dtype, tol):
    """jit_struct = 2: every program (uncut multi-sweep and variant batches)
    on structure-keyed kernels with the coefficients as kernel parameters."""
    import paper_2603_01443_b200 as cb

    old = _native.get_option("jit_struct")
    _native.set_option("jit_struct", 2)
    try:
        for spec in (cb.BrickwallSpec(16, 5, 2, 3, 4), cb.BrickwallSpec(12, 4, 3, 4, 5)):
            circ = cb.build_brickwall(spec)
            ref = orc.simulate(spec.q, circ.kinds, circ.qa, circ.qb, circ.params)
            assert np.abs(cb.simulate(circ, dtype=dtype).amps - ref).max() < tol
            assert np.abs(cb.run_cut(circ, spec.n, dtype=dtype).amps - ref).max() < tol
        stair = cb.build_staircase(cb.BenchmarkSpec(q=12, n=2, blocks=2))
        ref = orc.simulate(12, stair.kinds, stair.qa, stair.qb)
        assert np.abs(cb.simulate(stair, dtype=dtype).amps - ref).max() < tol
    finally:
        _native.set_option("jit_struct", old)


@pytest.mark.gpu
def test_structure_keyed_modules_are_reused_across_angles(jit_on):
    """A circuit with the same structure but new angles compiles no new
    kernel for its variant batches (param mode) and is still exact."""
    import paper_2603_01443_b200 as cb

    base = cb.build_brickwall(cb.BrickwallSpec(20, 6, 2, 2, 9))
    cb.run_cut(base, 2)
    for seed in (1, 2):
        circ = _angles_perturbed(base, seed)
        n0 = _native.get_option("jit_units_compiled")
        r0 = _native.get_option("jit_units_reused")
        got = cb.run_cut(circ, 2).amps
        assert _native.get_option("jit_units_compiled") == n0
        assert _native.get_option("jit_units_reused") > r0
        ref = orc.simulate(20, circ.kinds, circ.qa, circ.qb, circ.params)
        assert np.abs(got - ref).max() < 1e-10


@pytest.mark.gpu
def test_tiered_jit_runs_interpreter_then_compiled_kernels():
    """jit = 3: the first call of a new program runs the interpreter kernel
    while the module compiles in the background; after cs_jit_wait the same
    call runs the compiled kernels; all results exact."""
    import torch

    import paper_2603_01443_b200 as cb

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    old = _native.get_option("jit")
    _native.set_option("jit", 3)
    try:
        circ = cb.build_brickwall(cb.BrickwallSpec(18, 7, 2, 2, 31))
        ref = orc.simulate(18, circ.kinds, circ.qa, circ.qb, circ.params)
        n0 = _native.get_option("jit_units_compiled")
        first = cb.run_cut(circ, 2).amps
        _native.jit_wait(120)
        assert _native.get_option("jit_units_compiled") > n0
        second = cb.run_cut(circ, 2).amps
        assert np.abs(first - ref).max() < 1e-10 and np.abs(second - ref).max() < 1e-10
        u_first = cb.simulate(circ).amps
        _native.jit_wait(120)
        assert np.abs(cb.simulate(circ).amps - u_first).max() < 1e-12
    finally:
        _native.set_option("jit", old)


@pytest.mark.gpu
@pytest.mark.parametrize("qs,c,dtype,tol,cmax", [(12, 2, np.complex128, 1e-10, 16), (15, 2, np.complex128, 1e-10, 16),
                                                  (15, 4, np.complex128, 1e-10, 16), (16, 2, np.complex64, 1e-5, 16),
                                                  (13, 3, np.complex64, 1e-5, 16), (14, 6, np.complex128, 1e-10, 8)])
def test_cluster_resident_variant_batches(jit_on, qs, c, dtype, tol, cmax):
    """Variant batches of 12..16-qubit segments run as ONE cluster-resident
    kernel (each state in the shared memory of a CTA cluster, sweeps as
    phases separated by cluster barriers): one launch per family, equal to
    the per-launch kernels and the oracle."""
    import paper_2603_01443_b200 as cb
    from paper_2603_01443_b200.engine import simulate_family

    old = _native.get_option("cluster_max")
    _native.set_option("cluster_max", cmax)
    try:
        circ = cb.build_brickwall(cb.BrickwallSpec(2 * qs, 6, 2, c, qs))
        prep = preprocess(circ, 2)
        for fam in prep.subs.segments:
            simulate_family(fam, dtype=dtype)  # compile
            n0 = _native.launch_count()
            got = simulate_family(fam, dtype=dtype).cpu().numpy()
            assert _native.launch_count() - n0 == 1
            _native.set_option("cluster", 0)
            try:
                per_launch = simulate_family(fam, dtype=dtype).cpu().numpy()
            finally:
                _native.set_option("cluster", 1)
            for v in range(fam.num_variants):
                t = fam.variant_table(v)
                ref = orc.simulate(qs, t.kinds, t.qa, t.qb, t.params)
                assert np.abs(got[v] - ref).max() < tol
            assert np.abs(got - per_launch).max() < tol
        from paper_2603_01443_b200 import engine

        cut = cb.run_cut(circ, 2, dtype=dtype, max_qubits=32)
        assert engine.max_abs_diff(cut, cb.simulate(circ, dtype=dtype, max_qubits=32)) < tol
    finally:
        _native.set_option("cluster_max", old)


@pytest.mark.gpu
def test_cluster_resident_uncut_small_states(jit_on):
    """A single 12..15-qubit simulate() from |0..0> also runs cluster-resident
    (2^11-amplitude chunks: up to 16 CTAs per cluster)."""
    import paper_2603_01443_b200 as cb

    for q in (12, 14, 15):
        circ = cb.build_brickwall(cb.BrickwallSpec(q, 8, 3 if q % 2 else 2, 2, q))
        cb.simulate(circ)
        n0 = _native.launch_count()
        got = cb.simulate(circ).amps
        assert _native.launch_count() - n0 == 1
        assert np.abs(got - orc.simulate(q, circ.kinds, circ.qa, circ.qb, circ.params)).max() < 1e-10


@pytest.mark.gpu
def test_process_exits_cleanly_while_the_background_compiler_runs():
    """jit = 3 queues NVRTC compiles on a background thread; a process that
    exits while one is in flight used to crash inside nvrtcCompileProgram
    (NVRTC's destructors ran before the library's exit drain). Each child
    enqueues compiles of never-seen circuits and exits at once."""
    import subprocess
    import sys
    import os

    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys; sys.path.insert(0, %r)\n"
            "import paper_2603_01443_b200 as cb\n"
            "from paper_2603_01443_b200 import _native\n"
            "_native.set_option('jit', 3)\n"
            "for s in range(3):\n"
            "    cb.run_cut(cb.build_brickwall(cb.BrickwallSpec(16, 6, 2, 2, 900 + 7 * s + int(sys.argv[1]))), 2)\n"
            "print('done')\n") % root
    for run in range(3):
        r = subprocess.run([sys.executable, "-c", code, str(run)], capture_output=True, text=True, timeout=300)
        assert r.returncode == 0 and "done" in r.stdout, (r.returncode, r.stderr[-2000:])


@pytest.mark.gpu
@pytest.mark.parametrize("q,n,c", [(12, 3, 4), (16, 4, 5), (14, 2, 3)])
def test_sim_families_one_call_matches_per_family(jit_on, q, n, c):
    """cs_sim_families (every family of a decomposition in one native call,
    read from the planner's tables, families on forked streams) equals one
    simulate_family call per family; a family whose template was replaced
    takes the per-family path."""
    import torch

    from paper_2603_01443_b200.cutting import GateTable
    from paper_2603_01443_b200.engine import simulate_family
    from paper_2603_01443_b200.pipeline import _simulate_families_native, simulate_families

    circ = G.build_brickwall(G.BrickwallSpec(q, 5, n, c, 3))
    fams = preprocess(circ, n).subs.segments
    one = _simulate_families_native(fams, np.complex128, 30)
    assert one is not None and len(one) == n
    each = [simulate_family(f) for f in fams]
    torch.cuda.synchronize()
    for a, b in zip(one, each):
        assert a.shape == b.shape and torch.equal(a, b)
    t = fams[1].template
    fams[1].template = GateTable(t.kinds.copy(), t.qa, t.qb, t.params)
    assert _simulate_families_native(fams, np.complex128, 30) is None
    again = simulate_families(fams)
    torch.cuda.synchronize()
    for a, b in zip(again, each):
        assert torch.equal(a, b)
