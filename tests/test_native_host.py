"""CPU checks of the native library's host side (no kernels are launched):
the C-ABI loads and exports every symbol include/cutsim.h declares; the gate
lowering, fusion and sweep scheduling (executed here by a numpy interpreter of
the exported schedule) reproduce the oracle; the chain-merge planner picks
the documented bonds and validates its input."""
import json
import os
import re

import numpy as np
import pytest

from conftest import ROOT
from oracle import cutbench_oracle as orc
from paper_2603_01443_b200 import _native
from paper_2603_01443_b200 import circuits as C
from paper_2603_01443_b200 import cutting as K
from paper_2603_01443_b200 import generators as G
from paper_2603_01443_b200.errors import NativeUnavailableError, ValidationError

HEADER = os.path.join(ROOT, "include", "cutsim.h")

pytestmark = pytest.mark.skipif(not os.path.exists(_native.LIB_PATH),
                                reason="libcutsim.so not built (run __graft_entry__.build())")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(cs_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    lib = _native.load()
    decl = declared_symbols()
    assert len(decl) >= 14
    for name in decl:
        assert hasattr(lib, name), name
    assert set(decl) == set(_native.SIGNATURES), "ctypes table and header disagree"
    assert lib.cs_version() >= 10000


def test_options_round_trip_and_errors():
    old = _native.get_option("tile_bits")
    _native.set_option("tile_bits", 10)
    assert _native.get_option("tile_bits") == 10
    _native.set_option("tile_bits", old)
    with pytest.raises(ValidationError):
        _native.set_option("tile_bits", 40)
    with pytest.raises(ValidationError):
        _native.set_option("no_such_option", 1)
    assert "unknown option" in _native.last_error()


def execute_schedule(plan, nq, variant=0, garbage=False):
    """Interpret the exported sweep schedule on a full numpy state. Before
    every sweep, check the zero-start tile bound the kernels rely on: every
    non-zero amplitude lies in a tile t < 2^z (tile-id bit j <-> qubit oq[j]).
    garbage=True models the kernels without the zeroing pass: memory starts
    as NaN, the first sweep's launched tile starts from |0..0>, and every
    later sweep reads an amplitude of its launched tiles as 0 when its
    tile-local index has a bit of the sweep's zero_local_mask ("zl") set —
    the result must still be finite and exact."""
    amps = orc.zero_state(nq)
    idx = np.arange(1 << nq, dtype=np.int64)
    if garbage:
        amps[:] = np.nan
    for k, sw in enumerate(plan["sweeps"]):
        high = 0
        for q in sw["oq"][sw["z"]:]:
            high |= 1 << q
        L, hq = sw["L"], sw["hq"]
        glob = list(range(L)) + list(hq)
        if garbage:
            launched = (idx & high) == 0
            if k == 0:
                amps[launched] = 0
                amps[0] = 1
            else:
                zq = 0
                for p, q in enumerate(glob):
                    if (sw["zl"] >> p) & 1:
                        zq |= 1 << q
                amps[launched & ((idx & zq) != 0)] = 0
        else:
            assert not np.any((idx[np.abs(amps) > 0] & high) != 0), "amplitude outside the zero-start tiles"
        ents = sw["entries"]
        i = 0
        while i < len(ents):
            e = ents[i]
            src = e
            step = 1
            if e["slot"] >= 0:
                src = ents[i + ((variant >> e["slot"]) & 1)]
                step = 2
            mask = e["omask"]
            for p in range(32):
                if (e["lmask"] >> p) & 1:
                    mask |= 1 << glob[p]
            m = np.array(src["m"]).reshape(4, 2)
            m = m[:, 0] + 1j * m[:, 1]
            sel = (idx & mask) == mask
            if e["type"] == 1:
                amps[sel] *= m[0]
            else:
                t = glob[e["target"]]
                zero = sel & (((idx >> t) & 1) == 0)
                i0 = idx[zero]
                i1 = i0 | (1 << t)
                a, b = amps[i0].copy(), amps[i1].copy()
                amps[i0] = m[0] * a + m[1] * b
                amps[i1] = m[2] * a + m[3] * b
            i += step
    return amps


@pytest.fixture(params=[(1, 0, 0), (2, 0, 0), (1, 1, 0), (2, 1, 0), (1, 1, 1)],
                ids=["fuse-complex", "fuse-split-u3", "normalised", "split-normalised", "normalised-diag-pivot"])
def fuse_mode(request):
    """The lowerings: fused complex 2x2s (interpreter default), split U3 =
    phase . Ry . phase with commuted phases, normalised 2x2s with the
    deferred diagonals (the specialised-kernel default), and the param-mode
    form normalised by the structural (diagonal) pivot (jit_struct)."""
    keys = ("fuse", "dense_norm", "jit", "jit_struct")
    old = [_native.get_option(k) for k in keys]
    _native.set_option("fuse", request.param[0])
    _native.set_option("dense_norm", request.param[1])
    if request.param[2]:
        _native.set_option("jit", 2)
        _native.set_option("jit_struct", 2)
    yield request.param
    for k, v in zip(keys, old):
        _native.set_option(k, v)


@pytest.mark.parametrize("tile_bits", [4, 6, 12])
@pytest.mark.parametrize("q,d,n,c,seed", [(9, 4, 3, 4, 1), (10, 5, 2, 3, 0), (14, 3, 2, 2, 2)])
def test_schedule_reproduces_oracle_uncut(q, d, n, c, seed, tile_bits, fuse_mode):
    circ = G.build_brickwall(G.BrickwallSpec(q, d, n, c, seed))
    plan = json.loads(_native.sweep_plan_json(q, circ.table, tile_bits=tile_bits))
    T = plan["sweeps"][0]["T"]
    assert T == min(q, tile_bits)  # an explicit tile size applies to small states too
    got = execute_schedule(plan, q)
    ref = orc.simulate(q, circ.kinds, circ.qa, circ.qb, circ.params)
    assert np.abs(got - ref).max() < 1e-12


def test_cost_aware_zero_start_schedule_reproduces_oracle():
    """From 2^22 amplitudes up the planner prices tile sets by the tiles they
    launch (sweep_windows 3, zero-start tiles): the schedule of a q=22
    brick-wall — many sweeps, most of them over a few tiles — executed here
    (with the zero-start bound asserted before every sweep) equals the oracle;
    its early sweeps launch a fraction of the tiles."""
    q = 22
    circ = G.build_brickwall(G.BrickwallSpec(q, 4, 2, 2, 5))
    plan3 = json.loads(_native.sweep_plan_json(q, circ.table))
    old = _native.get_option("sweep_windows")
    _native.set_option("sweep_windows", 1)
    try:
        plan1 = json.loads(_native.sweep_plan_json(q, circ.table))
    finally:
        _native.set_option("sweep_windows", old)

    assert plan3["sweeps"][0]["z"] == 0 and any(sw["z"] < q - sw["T"] for sw in plan3["sweeps"][1:])
    assert plan3 != plan1
    got = execute_schedule(plan3, q)
    ref = orc.simulate(q, circ.kinds, circ.qa, circ.qb, circ.params)
    assert np.abs(got - ref).max() < 1e-12


@pytest.mark.parametrize("q,d,n,c,seed,tile_bits", [(22, 4, 2, 2, 5, 0), (16, 5, 2, 3, 1, 8), (15, 6, 3, 4, 2, 6),
                                                    (14, 3, 2, 2, 0, 4)])
def test_zero_start_without_zeroing_reproduces_oracle(q, d, n, c, seed, tile_bits):
    """The register-tile kernels skip the zeroing pass when the sweeps hold
    every qubit: each sweep loads as 0 the amplitudes whose tile-local index
    has a bit of its zero_local_mask (a qubit no earlier sweep held) and never
    reads a tile outside 2^z. Executed here on NaN-initialised memory, the
    schedule still gives the oracle's state, and the masks are what the
    support implies."""
    circ = G.build_brickwall(G.BrickwallSpec(q, d, n, c, seed))
    plan = json.loads(_native.sweep_plan_json(q, circ.table, tile_bits=tile_bits))
    held = 0
    for sw in plan["sweeps"]:
        glob = list(range(sw["L"])) + list(sw["hq"])
        assert sw["zl"] == sum(1 << p for p, g in enumerate(glob) if not (held >> g) & 1)
        for g in glob:
            held |= 1 << g
    assert held == (1 << q) - 1
    assert any(sw["zl"] for sw in plan["sweeps"][1:])
    got = execute_schedule(plan, q, garbage=True)
    assert np.all(np.isfinite(got))
    ref = orc.simulate(q, circ.kinds, circ.qa, circ.qb, circ.params)
    assert np.abs(got - ref).max() < 1e-12


@pytest.mark.parametrize("key", ["stair_q8_n4_b2", "stair_q6_n2_b3", "shadow_q9_d4_n3_c4_s3",
                                 "padded_q6_n2_b1_p1"])
def test_schedule_of_variant_templates_matches_reference_states(golden, key, fuse_mode):
    q, n = int(golden[f"{key}/q"]), int(golden[f"{key}/n"])
    circ = C.Circuit.from_table(q, C.GateTable(golden[f"{key}/kinds"], golden[f"{key}/qa"],
                                               golden[f"{key}/qb"]))
    subs = K.decompose(circ, K.plan_cut(circ, n))
    for fam in subs.segments:
        for tb in (2, 3, 0):
            plan = json.loads(_native.sweep_plan_json(fam.num_qubits, fam.template, fam.slots,
                                                      tile_bits=tb))
            ref = golden[f"{key}/seg{fam.segment}/states"]
            for v in range(fam.num_variants):
                got = execute_schedule(plan, fam.num_qubits, v)
                assert np.abs(got - ref[v]).max() < 1e-12


def test_depth_padded_fusion_collapses_pad():
    circ = C.build_depth_padded(C.BenchmarkSpec(q=6, n=2, blocks=1, depth_pad_exponent=3))
    plan = json.loads(_native.sweep_plan_json(6, circ.table))
    n_entries = sum(len(s["entries"]) for s in plan["sweeps"])
    assert circ.gate_count > 2000 and n_entries < 60
    got = execute_schedule(plan, 6)
    ref = orc.simulate(6, circ.kinds, circ.qa, circ.qb)
    assert np.abs(got - ref).max() < 1e-10


def test_split_u3_lowering_counts():
    """fuse=2 on cfg4a: one real rotation per U3 and one merged phase per
    qubit per layer (plus the trailing ones); CZs untouched."""
    circ = G.build_brickwall(G.BASELINE_CONFIGS["cfg4a"])
    old = _native.get_option("fuse")
    try:
        _native.set_option("fuse", 2)
        plan = json.loads(_native.sweep_plan_json(30, circ.table))
    finally:
        _native.set_option("fuse", old)
    ents = [e for s in plan["sweeps"] for e in s["entries"]]
    dense = [e for e in ents if e["type"] == 0]
    assert len(dense) == 300 and all(e["m"][1::2] == [0, 0, 0, 0] for e in dense)  # real
    n_cz = int((circ.kinds == C.KIND_CZ).sum())
    assert len(ents) - len(dense) == n_cz + 300 + 30


def test_normalised_dense_ops_have_unit_pivots():
    circ = G.build_brickwall(G.BASELINE_CONFIGS["cfg4a"])
    old = _native.get_option("dense_norm")
    try:
        _native.set_option("dense_norm", 1)
        plan = json.loads(_native.sweep_plan_json(30, circ.table))
    finally:
        _native.set_option("dense_norm", old)
    dense = [e for s in plan["sweeps"] for e in s["entries"] if e["type"] == 0]
    unit = 0
    for e in dense:
        m = np.array(e["m"]).reshape(2, 2, 2)  # row, col, (re, im)
        for r in range(2):
            ones = [c for c in range(2) if tuple(m[r, c]) == (1.0, 0.0)]
            if ones:
                other = m[r, 1 - ones[0]]
                assert np.hypot(*other) <= 1 + 1e-12
                unit += 1
    # every row of every dense op but the last (which carries the global scalar)
    assert unit >= 2 * len(dense) - 2


def test_diagonal_pivot_keeps_the_structure_of_new_angles():
    """Param mode (jit_struct) normalises every row by its diagonal entry, so
    which coefficients are exactly 1 does not depend on the angles: two
    circuits of one structure (new U3 angles) lower to the same pattern."""
    circ = G.build_brickwall(G.BrickwallSpec(14, 6, 2, 2, 3))
    rng = np.random.default_rng(1)
    p2 = circ.params.copy()
    u3 = circ.kinds == C.KIND_U3
    p2[u3] = rng.uniform(0.3, 2.8, size=(int(u3.sum()), 3))
    circ2 = C.Circuit.from_table(14, C.GateTable(circ.kinds, circ.qa, circ.qb, p2))
    keys = ("dense_norm", "jit", "jit_struct")
    old = [_native.get_option(k) for k in keys]
    try:
        _native.set_option("dense_norm", 1)
        _native.set_option("jit", 2)
        _native.set_option("jit_struct", 2)

        def pattern(c):
            plan = json.loads(_native.sweep_plan_json(14, c.table))
            return [(e["type"], tuple(tuple(np.array(e["m"]) == 1.0)), tuple(tuple(np.array(e["m"]) == 0.0)))
                    for s in plan["sweeps"] for e in s["entries"]], plan

        a, plan = pattern(circ)
        b, _ = pattern(circ2)
        assert a == b
        got = execute_schedule(plan, 14)
        assert np.abs(got - orc.simulate(14, circ.kinds, circ.qa, circ.qb, circ.params)).max() < 1e-12
    finally:
        for k, v in zip(keys, old):
            _native.set_option(k, v)


def test_uncut_q30_schedule_is_compact():
    circ = G.build_brickwall(G.BASELINE_CONFIGS["cfg4a"])
    plan = json.loads(_native.sweep_plan_json(30, circ.table))
    sweeps = plan["sweeps"]
    ops = sum(len(s["entries"]) for s in sweeps)
    # edge qubits skip the odd-layer CZ, so their U3 pairs fuse
    assert ops < circ.gate_count
    assert len(sweeps) <= 40


def test_lowering_rejects_bad_tables():
    bad = C.GateTable(np.array([9], np.uint8), np.array([0]), np.array([-1]))
    with pytest.raises(ValidationError):
        _native.sweep_plan_json(2, bad)
    out_of_range = C.GateTable(np.array([0], np.uint8), np.array([5]), np.array([-1]))
    with pytest.raises(ValidationError):
        _native.sweep_plan_json(2, out_of_range)
    slot_on_h = C.GateTable(np.array([0], np.uint8), np.array([0]), np.array([-1]))
    with pytest.raises(ValidationError):
        _native.sweep_plan_json(2, slot_on_h, np.array([0], np.int32))


def _chain(spec):
    circ = G.build_brickwall(spec)
    from paper_2603_01443_b200.merging import ChainSpec

    return ChainSpec.from_plan(K.plan_cut(circ, spec.n))


@pytest.mark.parametrize("name,bond,qlow,ws", [
    ("cfg4a", 0, 15, 0),
    ("cfg5_q34_n2_c2", 0, 17, 0),
    ("cfg5_q32_n4_c4", 1, 16, 2 * 2 * (1 << 16) * 16),   # middle bond: rank 2
])
def test_chain_plan_bonds(name, bond, qlow, ws):
    ch = _chain(G.BASELINE_CONFIGS[name])
    got_ws, got_bond, got_qlow = ch.plan()
    assert (got_bond, got_qlow) == (bond, qlow)
    assert got_ws == ws


def test_chain_plan_cfg4b_rank4_and_small_workspace():
    ch = _chain(G.BASELINE_CONFIGS["cfg4b"])
    ws, bond, qlow = ch.plan()
    assert bond in (0, 1)
    assert ws == 4 * (1 << 20) * 16  # one 2^20-amplitude intermediate per bond value


def test_chain_plan_validation():
    with pytest.raises(ValidationError):
        _native.chain_plan(2, [3, 3], [1, 2], [0, 0, 1], 1, [0], [0.5, -0.5, 0.5, 0.5])
    with pytest.raises(ValidationError):
        _native.chain_plan(1, [3], [0], [], 0, [], [0.5, -0.5, 0.5, 0.5])


def test_compute_entry_points_fail_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2603_01443_b200 import engine

    with pytest.raises(NativeUnavailableError):
        engine.simulate(C.Circuit(2, [C.h(0)]))


def test_family_fast_path_needs_the_planner_tables_and_fails_loudly_without_gpu():
    """pipeline.simulate_families runs a C++-planned decomposition's families
    in one native call only while every template column is still the
    planner's own array (identity, not equality); without a GPU that path
    raises instead of falling back."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2603_01443_b200 import generators as G
    from paper_2603_01443_b200.cutting import decompose, plan_cut
    from paper_2603_01443_b200.pipeline import _simulate_families_native

    circ = G.build_brickwall(G.BrickwallSpec(12, 4, 2, 2, 0))
    fams = decompose(circ, plan_cut(circ, 2)).segments
    with pytest.raises(NativeUnavailableError):
        _simulate_families_native(fams, np.complex128, 30)
    fams[1].template.qa = fams[1].template.qa.copy()  # same values, not the planner's array
    assert _simulate_families_native(fams, np.complex128, 30) is None
    fams2 = decompose(circ, plan_cut(circ, 2)).segments
    assert _simulate_families_native(fams2[1:], np.complex128, 30) is None  # not from the first row


def execute_reg_programs(plan, nq, variant=0):
    """Interpret the register-tile programs (rsweep kernel input) on a full
    numpy state: tile bit b is qubit b (< L) or hq[b - L]; register bit k is
    tile bit rpos[k]; thread-index bit m is the m-th non-register tile bit."""
    amps = orc.zero_state(nq)
    idx = np.arange(1 << nq, dtype=np.int64)
    for sw in plan["sweeps"]:
        T, L, RB = sw["T"], sw["L"], sw["RB"]
        glob = list(range(L)) + list(sw["hq"])
        rpos = [T - RB + k for k in range(RB)]
        ops = sw["ops"]
        i = 0
        while i < len(ops):
            op = ops[i]
            if op["kind"] == 2:
                rpos = op["rpos"][:RB]
                i += 1
                continue
            src, step = op, 1
            if op["slot"] >= 0:
                src = ops[i + ((variant >> op["slot"]) & 1)]
                step = 2
            tbits = [b for b in range(T) if b not in rpos]
            mask = op["omask"]
            for m in range(32):
                if (op["tmask"] >> m) & 1:
                    mask |= 1 << glob[tbits[m]]
            for k in range(RB):
                if (op["rmask"] >> k) & 1:
                    mask |= 1 << glob[rpos[k]]
            mm = np.array(src["m"]).reshape(4, 2)
            mm = mm[:, 0] + 1j * mm[:, 1]
            sel = (idx & mask) == mask
            if op["kind"] == 1:
                amps[sel] *= mm[0]
            else:
                t = glob[rpos[op["k"]]]
                zero = sel & (((idx >> t) & 1) == 0)
                i0 = idx[zero]
                i1 = i0 | (1 << t)
                a, b = amps[i0].copy(), amps[i1].copy()
                amps[i0] = mm[0] * a + mm[1] * b
                amps[i1] = mm[2] * a + mm[3] * b
            i += step
        assert rpos == [T - RB + k for k in range(RB)], "program must end in the canonical mapping"
    return amps


def _reg_plan(nq, table, slots=None, tile_bits=0):
    _native.set_option("plan_json", 1)
    try:
        return json.loads(_native.sweep_plan_json(nq, table, slots, tile_bits=tile_bits))
    finally:
        _native.set_option("plan_json", 0)


@pytest.mark.parametrize("tile_bits", [4, 6, 9, 12])
@pytest.mark.parametrize("q,d,n,c,seed", [(9, 4, 3, 4, 1), (14, 3, 2, 2, 2), (16, 3, 4, 3, 5)])
def test_register_programs_reproduce_oracle(q, d, n, c, seed, tile_bits, fuse_mode):
    circ = G.build_brickwall(G.BrickwallSpec(q, d, n, c, seed))
    plan = _reg_plan(q, circ.table, tile_bits=tile_bits)
    got = execute_reg_programs(plan, q)
    ref = orc.simulate(q, circ.kinds, circ.qa, circ.qb, circ.params)
    assert np.abs(got - ref).max() < 1e-12


@pytest.mark.parametrize("key", ["stair_q8_n4_b2", "stair_q6_n2_b3", "shadow_q9_d4_n3_c4_s3",
                                 "stair_q12_n3_b1"])
def test_register_programs_of_variant_templates(golden, key, fuse_mode):
    q, n = int(golden[f"{key}/q"]), int(golden[f"{key}/n"])
    circ = C.Circuit.from_table(q, C.GateTable(golden[f"{key}/kinds"], golden[f"{key}/qa"],
                                               golden[f"{key}/qb"]))
    subs = K.decompose(circ, K.plan_cut(circ, n))
    for fam in subs.segments:
        for tb in (2, 3, 0):
            plan = _reg_plan(fam.num_qubits, fam.template, fam.slots, tile_bits=tb)
            ref = golden[f"{key}/seg{fam.segment}/states"]
            for v in range(fam.num_variants):
                got = execute_reg_programs(plan, fam.num_qubits, v)
                assert np.abs(got - ref[v]).max() < 1e-12


@pytest.mark.parametrize("dtype,bound", [(_native.CS_C128, 200.5), (_native.CS_C64, 20.5)])
def test_normalised_lowering_bounds_amplitude_growth(dtype, bound):
    """Each normalised 2x2 inflates the executed state by up to 1/2 bit; the
    planner re-applies the pending scale before the budget (2^200 for c128,
    2^20 for c64) is exceeded, so deep circuits cannot overflow. Checked by
    executing the exported schedule of a 600-layer circuit step by step."""
    circ = G.build_brickwall(G.BrickwallSpec(8, 600, 2, 2, 0))
    old = _native.get_option("dense_norm")
    try:
        _native.set_option("dense_norm", 1)
        plan = json.loads(_native.sweep_plan_json(8, circ.table, dtype=dtype))
    finally:
        _native.set_option("dense_norm", old)
    amps = orc.zero_state(8)
    idx = np.arange(256)
    peak = 0.0
    for sw in plan["sweeps"]:
        glob = list(range(sw["L"])) + list(sw["hq"])
        for e in sw["entries"]:
            mask = e["omask"]
            for p in range(32):
                if (e["lmask"] >> p) & 1:
                    mask |= 1 << glob[p]
            m = np.array(e["m"]).reshape(4, 2)
            m = m[:, 0] + 1j * m[:, 1]
            sel = (idx & mask) == mask
            if e["type"] == 1:
                amps[sel] *= m[0]
            else:
                t = glob[e["target"]]
                i0 = idx[sel & (((idx >> t) & 1) == 0)]
                i1 = i0 | (1 << t)
                a, b = amps[i0].copy(), amps[i1].copy()
                amps[i0] = m[0] * a + m[1] * b
                amps[i1] = m[2] * a + m[3] * b
            peak = max(peak, float(np.abs(amps).max()))
    assert np.log2(peak) <= bound
    ref = orc.simulate(8, circ.kinds, circ.qa, circ.qb, circ.params)
    assert np.abs(amps - ref).max() < 1e-12
