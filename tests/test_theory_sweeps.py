"""Host side of the threshold study (cost model, boundary fit, crossovers,
reports, CLI `threshold`) against golden vectors produced by the reference
(tests/golden/make_golden_theory.py) — CPU only."""
import io
import json
import os
from contextlib import redirect_stdout

import numpy as np
import pytest

from paper_2603_01443_b200 import boundary_fit, cli, sweeps, theory
from paper_2603_01443_b200.errors import DegenerateFitError, ValidationError
from paper_2603_01443_b200.harness import TimingBreakdown

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_theory.json")))


def test_threshold_line_and_uniform():
    for n, want in GOLD["threshold_line"].items():
        assert theory.threshold_line(int(n)) == pytest.approx(want, rel=1e-15)
    for case in GOLD["threshold_uniform"]:
        r = theory.threshold_uniform(*case["args"])
        assert r.c_total_max == pytest.approx(case["c_total_max"], rel=1e-15)
        assert (r.slope, r.satisfied) == (pytest.approx(case["slope"]), case["satisfied"])
    with pytest.raises(ValidationError):
        theory.threshold_uniform(25, 2)
    with pytest.raises(ValidationError):
        theory.threshold_line(1)


def test_cost_scalings_and_regimes():
    for case in GOLD["n_sub"]:
        assert theory.n_sub_uniform(*case["args"]) == case["value"]
    for case in GOLD["regime"]:
        q, n, c, d, ds = case["args"]
        rr = theory.regime_ratios(theory.CostParams(q=q, n=n, c=c, depth=d, seg_depth=ds))
        assert rr.regime == case["regime"]
        for k in ("r_pre_sub", "r_pre_merge", "r_sub_merge"):
            assert getattr(rr, k) == pytest.approx(case[k], rel=1e-13)
    for case in GOLD["predict"]:
        q, n, c, d, ds, ns = case["args"]
        p = theory.CostParams(q=q, n=n, c=c, depth=d, seg_depth=ds)
        assert theory.predict_costs(p, ns) == pytest.approx(case["value"], rel=1e-15)
    for case in GOLD["nonuniform"]:
        q, n, c, d, ds, ns = case["args"]
        p = theory.CostParams(q=q, n=n, c=c, depth=d, seg_depth=ds)
        assert theory.threshold_nonuniform(p, ns) == case["value"]
    for args, err in GOLD["errors"].items():
        if args == "one_class":
            continue
        with pytest.raises(ValidationError):
            theory.CostParams(**json.loads(args))
        assert err == "ValidationError"


@pytest.mark.parametrize("i", range(4))
def test_boundary_fit_matches_reference(i):
    case = GOLD["fits"][i]
    f = boundary_fit.fit_weighted_line(np.array(case["points"]), np.array(case["deltas"]), tuple(case["init"]),
                                       iterations=case["iterations"])
    assert f.slope == pytest.approx(case["slope"], rel=1e-9, abs=1e-12)
    assert f.intercept == pytest.approx(case["intercept"], rel=1e-9, abs=1e-12)
    assert np.allclose(f.w, case["w"], rtol=1e-9, atol=1e-12)
    assert f.weighted_accuracy == pytest.approx(case["weighted_accuracy"], rel=1e-12)
    assert f.margin_violations == case["margin_violations"]
    assert np.allclose(f.weights, case["weights"], rtol=1e-14)
    assert np.array_equal(f.predict(f.points), np.where(f.decision_values(f.points) >= 0, 1, -1))


def test_boundary_fit_errors():
    with pytest.raises(DegenerateFitError):
        boundary_fit.fit_weighted_line(np.array([[2.0, 1.0], [4.0, 1.0]]), np.array([-1.0, -2.0]), (0.5, 0.0))
    with pytest.raises(DegenerateFitError):
        boundary_fit.fit_weighted_line(np.array([[2.0, 1.0]]), np.array([np.nan]), (0.5, 0.0))
    with pytest.raises(ValidationError):
        boundary_fit.fit_weighted_line(np.zeros((3, 3)), np.zeros(3), (0.5, 0.0))
    with pytest.raises(ValidationError):
        boundary_fit.fit_weighted_line(np.zeros((3, 2)), np.zeros(2), (0.5, 0.0))


def _row(q, c, delta, n=2, pre=1e-3, sub=2e-3, merge=1e-3, status="ok"):
    t_orig = 1.0
    return TimingBreakdown(q, n, c, 10, 100, pre, sub, merge, (1 + delta) * t_orig, t_orig, delta, 1, status)


def test_fit_boundary_and_reports_from_sweep():
    case = GOLD["fits"][0]
    rows = [_row(int(q), int(c), d) for (q, c), d in zip(case["points"], case["deltas"])]
    rows.append(_row(30, 3, float("nan"), status="timeout-orig"))
    sw = sweeps.SweepResult(points=rows, metadata={"n": 2})
    f = sweeps.fit_boundary(sw)
    assert f.slope == pytest.approx(case["slope"], rel=1e-9)
    assert sweeps.fit_boundary(rows).intercept == pytest.approx(case["intercept"], rel=1e-9)
    rep = sweeps.boundary_fit_report(f, tag="t")
    assert rep["kind"] == "boundary-fit" and rep["machine_tag"] == "t" and len(rep["points"]) == len(rows) - 1
    csv = sweeps.sweep_report(sw).splitlines()
    assert csv[0].split(",")[:5] == ["q", "n", "c_total", "D", "G"] and len(csv) == len(rows) + 1
    with pytest.raises(ValidationError):
        sweeps.SweepResult(points=[rows[0], rows[0]], metadata={})


def test_detect_crossovers_matches_reference():
    case = GOLD["crossovers"][0]
    rows = [_row(q, 6, 0.0, pre=pre, sub=sub, merge=mer, status=st) for q, pre, sub, mer, st in case["rows"]]
    c = sweeps.detect_crossovers(rows)
    assert (c.q_pre_cross, c.q_sub_cross) == (case["q_pre_cross"], case["q_sub_cross"])
    with pytest.raises(ValidationError):
        sweeps.detect_crossovers(rows + [_row(18, 4, 0.0)])
    rep = sweeps.crossover_report(c, rows)
    assert rep["kind"] == "crossovers" and len(rep["series"]) == len(rows)


def test_cli_threshold_matches_reference():
    for case in GOLD["cli_threshold"]:
        buf = io.StringIO()
        with redirect_stdout(buf):
            rc = cli.main(case["argv"])
        assert rc == case["rc"]
        got = json.loads(buf.getvalue())
        want = case["json"]
        assert got.keys() == want.keys()
        for k, v in want.items():
            assert got[k] == (pytest.approx(v, rel=1e-15) if isinstance(v, float) else v)


def test_cli_ranges_and_grid_validation():
    assert cli.parse_range("8") == [8]
    assert cli.parse_range("2:8:2") == [2, 4, 6, 8]
    assert cli.parse_range("3:5") == [3, 4, 5]
    for bad in ("a", "1:2:0", "1:2:3:4"):
        with pytest.raises(ValidationError):
            cli.parse_range(bad)
    with pytest.raises(ValidationError):
        cli.parse_int_list("1,x")
    # grid validation happens before any device work
    with pytest.raises(ValidationError):
        sweeps.sweep_heatmap([6], [3], n=3)
    with pytest.raises(ValidationError):
        sweeps.sweep_heatmap(n=5)
    with pytest.raises(ValidationError):
        sweeps.sweep_heatmap([6], [2], family="ladder")
    with pytest.raises(ValidationError):
        sweeps.split_sweep(7, [1])
    with pytest.raises(ValidationError):
        sweeps.scan_feasible([0], 0.0)
    assert cli.main(["sweep", "--q", "6", "--c", "3", "--n", "3"]) == cli.EXIT_VALIDATION


def test_install_as_cutbench_aliases_reference_modules():
    import sys

    import paper_2603_01443_b200 as pkg

    name = "cutbench_alias_test"
    pkg.install_as_cutbench(name)
    try:
        import importlib

        cbm = importlib.import_module(name)
        assert cbm.__dropin_of__ is pkg and cbm.simulate is pkg.simulate
        h = importlib.import_module(f"{name}.harness")
        assert h.sweep_heatmap is sweeps.sweep_heatmap and h.measure is pkg.measure
        assert importlib.import_module(f"{name}.costmodel").threshold_uniform is theory.threshold_uniform
        assert importlib.import_module(f"{name}.svmfit").fit_weighted_line is boundary_fit.fit_weighted_line
        assert importlib.import_module(f"{name}.cutting").plan_cut is pkg.plan_cut
        # every name the reference package exports (cutbench/__init__.py:68-125)
        for attr in ("BenchmarkSpec", "BoundaryFit", "BoundaryGate", "BudgetExceededError", "CapacityError",
                     "Circuit", "CostParams", "Crossovers", "CutPlan", "CutbenchError", "DEFAULT_MAX_QUBITS",
                     "DegenerateFitError", "FeasibilityScan", "Gate", "GateKind", "MergeInput", "RegimeRatios",
                     "StateVec", "SubcircuitSet", "SweepResult", "ThresholdReport", "TimingBreakdown",
                     "UnsupportedTopologyError", "ValidationError", "apply_gate", "breakdown_series",
                     "build_benchmark", "build_depth_padded", "build_staircase", "compute_depth",
                     "count_subcircuits", "decompose", "detect_crossovers", "dump_amplitudes", "fit_boundary",
                     "fit_weighted_line", "measure", "merge", "merge_input_from", "merge_streaming",
                     "n_sub_uniform", "plan_cut", "plan_cut_sizes", "predict_costs", "regime_ratios",
                     "scan_feasible", "simulate", "split_sweep", "sweep_heatmap", "tensor", "threshold_line",
                     "threshold_nonuniform", "threshold_uniform"):
            assert hasattr(cbm, attr), attr
        with pytest.raises(RuntimeError):
            sys.modules["cutbench_alias_other"] = object()
            pkg.install_as_cutbench("cutbench_alias_other")
    finally:
        for k in [k for k in sys.modules if k.startswith(name) or k.startswith("cutbench_alias_other")]:
            del sys.modules[k]
