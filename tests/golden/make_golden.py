"""Generate the golden fixtures by running the REAL reference (`cutbench`).

Run in the build container only (the reference tree does not exist on the
GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden.py

Writes tests/golden/reference_golden.npz. Contents (all produced by the
reference's own functions, `cutbench.engine.simulate`, `cutting.plan_cut`,
`cutting.decompose`, `merging.merge`):

  * staircase family (reference-native, parity tier A) and depth-padded;
  * "shadow" brick-wall circuits: the BASELINE U3 family with every U3 slot
    holding a reference gate (H/X/T/S by floor(4u)), built from the oracle's
    generator so the fixture is independent of the product;
  * cut tables of the full-size BASELINE configs computed by the reference on
    their shadows (positions, c_i, per-segment templates and patch offsets,
    merge table, coefficients) — the U3 circuits have the same structure.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

import cutbench as cb  # noqa: E402  (the reference, via PYTHONPATH)
from cutbench.circuits import Gate, GateKind  # noqa: E402

from oracle import cutbench_oracle as orc  # noqa: E402

KIND_NAMES = {0: GateKind.H, 1: GateKind.X, 2: GateKind.T, 3: GateKind.S, 4: GateKind.Sdg,
              5: GateKind.CX, 6: GateKind.CZ}


def ref_circuit(q, kinds, qa, qb):
    gates = []
    for k, a, b in zip(kinds, qa, qb):
        kind = KIND_NAMES[int(k)]
        qs = (int(a), int(b)) if kind.arity == 2 else (int(a),)
        gates.append(Gate(kind, qs))
    return cb.Circuit(q, gates)


def dump_cut(out, key, circ, n, with_states):
    plan = cb.plan_cut(circ, n)
    subs = cb.decompose(circ, plan)
    out[f"{key}/positions"] = np.array([bg.position for bg in plan.boundary_gates], np.int64)
    out[f"{key}/boundaries"] = np.array([bg.boundary for bg in plan.boundary_gates], np.int64)
    out[f"{key}/c_i"] = np.array(plan.c_i, np.int64)
    out[f"{key}/c_per_boundary"] = np.array(plan.c_per_boundary, np.int64)
    out[f"{key}/merge_table"] = subs.merge_table
    out[f"{key}/coeffs"] = subs.coeffs
    for fam in subs.segments:
        base = fam.circuits[0]
        out[f"{key}/seg{fam.segment}/kinds"] = base.kinds
        out[f"{key}/seg{fam.segment}/qa"] = base.qa
        out[f"{key}/seg{fam.segment}/qb"] = base.qb
        # patch offsets = where variant 2^k differs from variant 0
        patches = []
        for k in range(plan.c_i[fam.segment]):
            diff = np.flatnonzero(fam.circuits[1 << k].kinds != base.kinds)
            assert diff.size == 1
            patches.append(int(diff[0]))
        out[f"{key}/seg{fam.segment}/patch"] = np.array(patches, np.int64)
        if with_states:
            out[f"{key}/seg{fam.segment}/states"] = np.stack(
                [cb.simulate(c).amps for c in fam.circuits])
    if with_states:
        states = [[cb.simulate(c) for c in fam.circuits] for fam in subs.segments]
        out[f"{key}/merged"] = cb.merge(cb.merge_input_from(subs, states)).amps


def main():
    out = {}
    cases = []
    # staircase family: (q, n, blocks) from the reference's own tests
    for q, n, blocks in [(2, 2, 1), (4, 2, 2), (6, 3, 2), (8, 4, 2), (8, 2, 3), (12, 3, 1),
                         (6, 2, 3), (4, 2, 13), (10, 2, 4)]:
        key = f"stair_q{q}_n{n}_b{blocks}"
        circ = cb.build_staircase(cb.BenchmarkSpec(q=q, n=n, blocks=blocks))
        out[f"{key}/kinds"], out[f"{key}/qa"], out[f"{key}/qb"] = circ.kinds, circ.qa, circ.qb
        out[f"{key}/q"] = np.int64(q)
        out[f"{key}/n"] = np.int64(n)
        out[f"{key}/uncut"] = cb.simulate(circ).amps
        dump_cut(out, key, circ, n, with_states=True)
        cases.append(key)
    key = "padded_q6_n2_b1_p1"
    circ = cb.build_depth_padded(cb.BenchmarkSpec(q=6, n=2, blocks=1, depth_pad_exponent=1))
    out[f"{key}/kinds"], out[f"{key}/qa"], out[f"{key}/qb"] = circ.kinds, circ.qa, circ.qb
    out[f"{key}/q"] = np.int64(6)
    out[f"{key}/n"] = np.int64(2)
    out[f"{key}/uncut"] = cb.simulate(circ).amps
    dump_cut(out, key, circ, 2, with_states=True)
    cases.append(key)

    # shadow brick-wall circuits (small: full states)
    for q, d, n, c, seed in [(12, 4, 2, 1, 0), (8, 6, 2, 3, 1), (8, 5, 4, 4, 2),
                             (9, 4, 3, 4, 3), (12, 4, 3, 2, 4), (10, 10, 2, 2, 0),
                             (12, 3, 2, 6, 5)]:
        key = f"shadow_q{q}_d{d}_n{n}_c{c}_s{seed}"
        k, a, b, _ = orc.brickwall(q, d, n, c, seed, shadow=True)
        circ = ref_circuit(q, k, a, b)
        out[f"{key}/kinds"], out[f"{key}/qa"], out[f"{key}/qb"] = circ.kinds, circ.qa, circ.qb
        out[f"{key}/q"] = np.int64(q)
        out[f"{key}/n"] = np.int64(n)
        out[f"{key}/uncut"] = cb.simulate(circ).amps
        dump_cut(out, key, circ, n, with_states=True)
        cases.append(key)

    # full-size BASELINE configs: cut tables only (reference on the shadow)
    big = []
    for name, (q, d, n, c, seed) in {
        "cfg1": (12, 4, 2, 1, 0), "cfg2": (20, 10, 2, 2, 0), "cfg3_d10_c6": (24, 10, 2, 6, 0),
        "cfg4a": (30, 10, 2, 2, 0), "cfg4b": (30, 10, 3, 4, 0), "cfg5_q32_n4_c4": (32, 10, 4, 4, 0),
        "cfg5_q32_n2_c4": (32, 10, 2, 4, 0), "cfg5_q34_n2_c2": (34, 10, 2, 2, 0),
    }.items():
        key = f"table_{name}"
        k, a, b, _ = orc.brickwall(q, d, n, c, seed, shadow=True)
        circ = ref_circuit(q, k, a, b)
        out[f"{key}/spec"] = np.array([q, d, n, c, seed], np.int64)
        out[f"{key}/G"] = np.int64(circ.gate_count)
        dump_cut(out, key, circ, n, with_states=False)
        big.append(key)

    out["cases"] = np.array(cases)
    out["tables"] = np.array(big)
    path = os.path.join(HERE, "reference_golden.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {len(cases)} state cases, {len(big)} table cases, "
          f"{os.path.getsize(path) / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
