"""Host-side preprocess (plan_cut / decompose / generators) against the
reference's golden tables and the oracle — CPU only, bit-exact (integer work)."""
import numpy as np
import pytest

from conftest import golden_cases, golden_tables
from oracle import cutbench_oracle as orc
from paper_2603_01443_b200 import circuits as C
from paper_2603_01443_b200 import cutting as K
from paper_2603_01443_b200 import generators as G
from paper_2603_01443_b200.errors import UnsupportedTopologyError, ValidationError


@pytest.fixture(params=["native", "numpy"])
def planner(request, monkeypatch):
    """Both planners behind plan_cut/decompose: libcutsim's C++ tables and
    the numpy restatement (used when the library cannot be loaded)."""
    if request.param == "numpy":
        monkeypatch.setattr(K, "_native_tables", lambda circuit, sizes: None)
    else:
        import os

        from paper_2603_01443_b200 import _native

        if not os.path.exists(_native.LIB_PATH):
            pytest.skip("libcutsim.so not built")
    return request.param


def _circuit(golden, key):
    q = int(golden[f"{key}/q"]) if f"{key}/q" in golden else None
    tab = C.GateTable(golden[f"{key}/kinds"], golden[f"{key}/qa"], golden[f"{key}/qb"])
    return C.Circuit.from_table(q, tab)


def _check_tables(golden, key, circ, n):
    plan = K.plan_cut(circ, n)
    subs = K.decompose(circ, plan)
    assert [bg.position for bg in plan.boundary_gates] == list(golden[f"{key}/positions"])
    assert [bg.boundary for bg in plan.boundary_gates] == list(golden[f"{key}/boundaries"])
    assert list(plan.c_i) == list(golden[f"{key}/c_i"])
    assert list(plan.c_per_boundary) == list(golden[f"{key}/c_per_boundary"])
    assert np.array_equal(subs.merge_table, golden[f"{key}/merge_table"])
    assert np.array_equal(subs.coeffs, golden[f"{key}/coeffs"])
    for fam in subs.segments:
        s = fam.segment
        assert np.array_equal(fam.template.kinds, golden[f"{key}/seg{s}/kinds"])
        assert np.array_equal(fam.template.qa, golden[f"{key}/seg{s}/qa"])
        assert np.array_equal(fam.template.qb, golden[f"{key}/seg{s}/qb"])
        assert np.array_equal(fam.patch_offsets, golden[f"{key}/seg{s}/patch"])
        assert np.array_equal(np.flatnonzero(fam.slots >= 0), np.sort(fam.patch_offsets))
    return plan, subs


@pytest.mark.parametrize("key", golden_cases())
def test_plan_and_decompose_match_reference(golden, key, planner):
    circ = _circuit(golden, key)
    _check_tables(golden, key, circ, int(golden[f"{key}/n"]))


@pytest.mark.parametrize("key", golden_tables())
def test_full_size_tables_match_reference(golden, key, planner):
    q, d, n, c, seed = (int(v) for v in golden[f"{key}/spec"])
    circ = G.build_brickwall(G.BrickwallSpec(q, d, n, c, seed, one_qubit="clifford_t"))
    assert circ.gate_count == int(golden[f"{key}/G"])
    _check_tables(golden, key, circ, n)
    # the U3 circuit has the identical structure (same positions, same tables)
    u3c = G.build_brickwall(G.BrickwallSpec(q, d, n, c, seed))
    plan = K.plan_cut(u3c, n)
    assert [bg.position for bg in plan.boundary_gates] == list(golden[f"{key}/positions"])


@pytest.mark.parametrize("q,d,n,c,seed", [(12, 4, 2, 1, 0), (30, 10, 3, 4, 0), (32, 10, 4, 4, 0),
                                          (24, 20, 2, 6, 2), (8, 3, 4, 2, 9)])
@pytest.mark.parametrize("shadow", [False, True])
def test_generator_matches_oracle_restatement(q, d, n, c, seed, shadow):
    circ = G.build_brickwall(G.BrickwallSpec(q, d, n, c, seed,
                                             one_qubit="clifford_t" if shadow else "u3"))
    k, a, b, p = orc.brickwall(q, d, n, c, seed, shadow=shadow)
    assert np.array_equal(circ.kinds, k)
    assert np.array_equal(circ.qa, a)
    assert np.array_equal(circ.qb, b)
    assert np.array_equal(circ.params, p)


def test_variant_tables_equal_oracle_variants(planner):
    k, a, b, p = orc.brickwall(9, 4, 3, 4, 1)
    circ = C.Circuit.from_table(9, C.GateTable(k, a, b, p))
    plan = K.plan_cut(circ, 3)
    subs = K.decompose(circ, plan)
    bgs, _, _ = orc.plan(k, a, b, [3, 3, 3])
    for fam in subs.segments:
        ref = orc.segment_variants(k, a, b, p, [3, 3, 3], bgs, fam.segment)
        assert len(ref) == fam.num_variants
        for v, (rk, ra, rb, rp) in enumerate(ref):
            sub = fam.circuits[v]
            assert np.array_equal(sub.kinds, rk)
            assert np.array_equal(sub.qa, ra)
            assert np.array_equal(sub.qb, rb)
            assert np.array_equal(sub.params, rp)


def test_cut_distribution():
    assert G.cut_distribution(4, 2) == [1, 1, 0]
    assert G.cut_distribution(4, 4) == [2, 1, 1]
    assert G.cut_distribution(3, 4) == [2, 2]
    assert G.cut_distribution(2, 6) == [6]


def test_reference_error_contract(planner):
    # tests/test_cutting.py:58-66, 75-83 of the reference
    circ = C.build_staircase(C.BenchmarkSpec(q=6, n=2, blocks=1))
    with pytest.raises(ValidationError):
        K.plan_cut(circ, 4)
    with pytest.raises(UnsupportedTopologyError):
        K.plan_cut(C.Circuit(3, [C.h(0), C.cx(0, 2)]), 3)
    with pytest.raises(ValidationError):
        K.plan_cut_sizes(circ, (2, 2))
    with pytest.raises(ValidationError):
        K.plan_cut_sizes(circ, (6,))
    plan = K.plan_cut_sizes(C.build_staircase(C.BenchmarkSpec(q=6, n=2, blocks=2)), (1, 5))
    assert plan.c_total == 2


def test_coefficients_exact():
    # reference tests/test_cutting.py:102-122
    co = K.coefficients_of(2)
    assert co[3] == 0.5j
    for c in (1, 2, 5, 8, 12):
        assert np.allclose(np.abs(K.coefficients_of(c)), 2.0 ** (-c / 2), rtol=1e-12)


def test_json_shape_and_lazy_circuits(planner):
    circ = C.build_staircase(C.BenchmarkSpec(q=4, n=2, blocks=1))
    subs = K.decompose(circ, K.plan_cut(circ, 2))
    data = subs.to_json_dict()
    assert data["merge_table"] == [[0, 1], [0, 1]]
    assert data["coeffs"] == [[0.5, -0.5], [0.5, 0.5]]
    rebuilt = C.Circuit.from_json_dict(data["segments"][0]["subcircuits"][0])
    assert rebuilt == subs.segments[0].circuits[0]
    fresh = C.Circuit(2, subs.segments[1].circuits[1].gates)
    assert np.array_equal(fresh.kinds, subs.segments[1].circuits[1].kinds)


def test_u3_gate_and_json_round_trip():
    c = C.Circuit(2, [C.u3(0, 0.1, 0.2, 0.3), C.cz(0, 1), C.h(1)])
    assert c.kinds.tolist() == [C.KIND_U3, C.KIND_CZ, C.KIND_H]
    assert np.allclose(c.params[0], [0.1, 0.2, 0.3])
    again = C.Circuit.from_json(c.to_json())
    assert again == c
    with pytest.raises(ValidationError):
        C.Gate(C.GateKind.U3, (0,))
    with pytest.raises(ValidationError):
        C.Circuit(2, [C.h(2)])


def test_staircase_and_padded_generators_match_oracle():
    for q, blocks in [(2, 1), (6, 3), (9, 2)]:
        circ = C.build_staircase(C.BenchmarkSpec(q=q, n=q if q < 3 else 3, blocks=blocks))
        k, a, b, _ = orc.staircase(q, blocks)
        assert np.array_equal(circ.kinds, k) and np.array_equal(circ.qa, a)
        assert np.array_equal(circ.qb, b)
    c = C.build_depth_padded(C.BenchmarkSpec(q=6, n=2, blocks=1, depth_pad_exponent=2))
    assert c.gate_count == C.build_staircase(C.BenchmarkSpec(q=6, n=2, blocks=1)).gate_count + 200
    assert C.compute_depth(C.Circuit(2, [C.h(0), C.cx(0, 1), C.h(1)])) == 3


@pytest.mark.parametrize("key", golden_cases())
def test_native_preprocess_matches_python_and_reference(golden, key, monkeypatch):
    """cs_cut_run's C++ preprocess == the numpy planner (pinned to the reference)."""
    import os

    monkeypatch.setattr(K, "_native_tables", lambda circuit, sizes: None)
    from paper_2603_01443_b200 import _native

    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("libcutsim.so not built")
    circ = _circuit(golden, key)
    n = int(golden[f"{key}/n"])
    q = circ.num_qubits
    d = _native.cut_describe(q, circ.table, [q // n] * n)
    plan = K.plan_cut(circ, n)
    subs = K.decompose(circ, plan)
    assert [c[0] for c in d["cuts"]] == list(golden[f"{key}/positions"])
    assert [c[1] for c in d["cuts"]] == list(golden[f"{key}/boundaries"])
    for fam, seg in zip(subs.segments, d["segments"]):
        assert np.array_equal(np.array(seg["kinds"], np.uint8), fam.template.kinds)
        assert np.array_equal(np.array(seg["qa"]), fam.template.qa)
        assert np.array_equal(np.array(seg["qb"]), fam.template.qb)
        assert np.array_equal(np.array(seg["slots"]), fam.slots)
        assert tuple(seg["cut_ids"]) == fam.cut_ids


@pytest.mark.parametrize("name", list(G.BASELINE_CONFIGS))
def test_native_preprocess_full_size_u3(name, monkeypatch):
    import os

    monkeypatch.setattr(K, "_native_tables", lambda circuit, sizes: None)
    from paper_2603_01443_b200 import _native

    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("libcutsim.so not built")
    spec = G.BASELINE_CONFIGS[name]
    circ = G.build_brickwall(spec)
    d = _native.cut_describe(spec.q, circ.table, [spec.q // spec.n] * spec.n)
    subs = K.decompose(circ, K.plan_cut(circ, spec.n))
    for fam, seg in zip(subs.segments, d["segments"]):
        assert np.array_equal(np.array(seg["kinds"], np.uint8), fam.template.kinds)
        assert np.array_equal(np.array(seg["params"]).reshape(-1, 3), fam.template.params)
        assert np.array_equal(np.array(seg["slots"]), fam.slots)
    with pytest.raises(UnsupportedTopologyError):
        _native.cut_describe(3, C.Circuit(3, [C.h(0), C.cx(0, 2)]).table, [1, 1, 1])


def test_native_preprocess_validation_matches_python(monkeypatch):
    """cs_cut_run's planner rejects what plan_cut_sizes rejects
    (reference cutting.py:70-136 error contract)."""
    import os

    monkeypatch.setattr(K, "_native_tables", lambda circuit, sizes: None)
    from paper_2603_01443_b200 import _native

    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("libcutsim.so not built")
    circ = G.build_brickwall(G.BrickwallSpec(8, 3, 2, 2, 0))
    for sizes in ([8], [4, 5], [4, 4, 0], [0, 8], [-1, 9]):
        with pytest.raises(ValidationError):
            K.plan_cut_sizes(circ, tuple(sizes))
        with pytest.raises(ValidationError):
            _native.cut_describe(8, circ.table, sizes)
    d = _native.cut_describe(8, circ.table, [2, 2, 2, 2])
    plan = K.plan_cut_sizes(circ, (2, 2, 2, 2))
    assert [c[0] for c in d["cuts"]] == [bg.position for bg in plan.boundary_gates]
    assert [c[1] for c in d["cuts"]] == [bg.boundary for bg in plan.boundary_gates]


def _random_circuit(rng, q, g):
    """Random gate table over the reference gate set + U3; two-qubit gates
    only between qubits at distance <= 2 (so small segments can be crossed
    by non-adjacent spans, exercising the topology error too)."""
    kinds, qa, qb, prm = [], [], [], []
    for _ in range(g):
        k = int(rng.integers(0, 8))
        a = int(rng.integers(0, q))
        b = -1
        if k in (5, 6):
            b = a + int(rng.choice([-2, -1, 1, 2]))
            if not 0 <= b < q:
                b = a - 1 if a > 0 else a + 1
        kinds.append(k)
        qa.append(a)
        qb.append(b)
        prm.append(rng.uniform(0, 6.3, 3) if k == 7 else np.zeros(3))
    return C.Circuit.from_table(q, C.GateTable(np.array(kinds, np.uint8), np.array(qa), np.array(qb),
                                               np.array(prm)))


@pytest.mark.parametrize("seed", range(40))
def test_native_and_numpy_planners_agree_on_random_circuits(seed, monkeypatch):
    import os

    from paper_2603_01443_b200 import _native

    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("libcutsim.so not built")
    rng = np.random.default_rng(seed)
    q = int(rng.integers(2, 12))
    circ = _random_circuit(rng, q, int(rng.integers(0, 60)))
    n = int(rng.integers(2, q + 1))
    cuts = np.sort(rng.choice(np.arange(1, q), size=n - 1, replace=False))
    sizes = tuple(int(v) for v in np.diff(np.concatenate([[0], cuts, [q]])))
    results = []
    for native in (True, False):
        if not native:
            monkeypatch.setattr(K, "_native_tables", lambda circuit, sizes: None)
        try:
            plan = K.plan_cut_sizes(circ, sizes)
            subs = K.decompose(circ, plan)
            results.append(("ok", plan, subs))
        except UnsupportedTopologyError:
            results.append(("topology", None, None))
    assert results[0][0] == results[1][0]
    if results[0][0] == "ok":
        (_, p1, s1), (_, p2, s2) = results
        assert p1 == p2
        assert np.array_equal(s1.merge_table, s2.merge_table) and np.array_equal(s1.coeffs, s2.coeffs)
        for f1, f2 in zip(s1.segments, s2.segments):
            for col in ("kinds", "qa", "qb", "params"):
                assert np.array_equal(getattr(f1.template, col), getattr(f2.template, col)), col
            assert np.array_equal(f1.slots, f2.slots) and np.array_equal(f1.patch_offsets, f2.patch_offsets)
            assert f1.cut_ids == f2.cut_ids
