"""The threshold-study drivers on the GPU (small grids): stage-sum identity,
row schema, crossovers, feasibility scan, split sweep, CLI round trip."""
import io
import json
import math
from contextlib import redirect_stdout

import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sw():
    from paper_2603_01443_b200 import sweeps

    return sweeps


def test_sweep_heatmap_staircase(sw):
    res = sw.sweep_heatmap([4, 6, 8], [1, 2], n=2, repetitions=2, tag="box")
    assert [(p.q, p.c_total) for p in res.points] == [(q, c) for q in (4, 6, 8) for c in (1, 2)]
    for p in res.points:
        assert p.status == "ok" and p.reps == 2
        assert p.t_cut == pytest.approx(p.t_pre + p.t_sub + p.t_merge)
        assert p.delta == pytest.approx((p.t_cut - p.t_orig) / p.t_orig)
    assert res.metadata["machine_tag"] == "box" and res.metadata["family"] == "staircase"
    csv = sw.format_csv(res.points).splitlines()
    assert len(csv) == 7


def test_sweep_heatmap_brickwall_seeds_and_fit(sw):
    from paper_2603_01443_b200.errors import DegenerateFitError

    res = sw.sweep_heatmap([12, 14], [1, 4, 8], n=2, repetitions=1, family="brickwall", depth=5, seeds=(0, 1))
    assert res.metadata["seeds"] == [0, 1] and all(p.reps == 2 for p in res.points)
    try:
        fit = sw.fit_boundary(res)
        assert math.isfinite(fit.slope)
    except DegenerateFitError:
        pass  # all points on one side at these tiny sizes is a legitimate outcome


def test_breakdown_feasible_split(sw):
    rows = sw.breakdown_series([4, 6, 8], n=2, c_total=2, repetitions=1)
    cross = sw.detect_crossovers(rows)
    rep = sw.crossover_report(cross, rows)
    assert [r["q"] for r in rep["series"]] == [4, 6, 8]
    scans = sw.scan_feasible([None], 5.0, n=2, c_total=2, q_start=4, q_stop=10)
    assert scans[0].q_max_cut == 10 and scans[0].q_max_orig == 10 and len(scans[0].rows) == 4
    res = sw.split_sweep(6, [1, 2], repetitions=1)
    assert {p.split for p in res.points} == set(range(1, 6)) and set(res.best_split) == {1, 2}
    assert all(p.ratio == pytest.approx(p.t_cut / p.t_orig) for p in res.points)


def test_cli_sweep_json(sw, tmp_path):
    from paper_2603_01443_b200 import cli

    out = tmp_path / "sweep.json"
    fit = tmp_path / "fit.json"
    rc = cli.main(["sweep", "--q", "4:8:2", "--c", "1:2", "--reps", "1", "--format", "json", "--out", str(out),
                   "--fit", str(fit)])
    assert rc in (cli.EXIT_OK, cli.EXIT_DEGENERATE_FIT)
    data = json.loads(out.read_text())
    assert data["kind"] == "sweep" and len(data["points"]) == 6
    buf = io.StringIO()
    with redirect_stdout(buf):
        assert cli.main(["breakdown", "--q", "4:6:2", "--c", "2", "--reps", "1", "--report", "-"]) == 0
    assert "q_pre_cross" in buf.getvalue()


def test_reference_style_code_through_alias():
    """Code written against the reference (`import cutbench ...`) runs on the
    GPU path after install_as_cutbench(): the harness's cut pipeline
    (harness.py:125-145) and measure()."""
    import sys

    import numpy as np

    import paper_2603_01443_b200 as pkg
    from oracle import cutbench_oracle as orc

    pkg.install_as_cutbench("cutbench_gpu_alias")
    try:
        import importlib

        cutbench = importlib.import_module("cutbench_gpu_alias")
        harness = importlib.import_module("cutbench_gpu_alias.harness")
        spec = cutbench.BenchmarkSpec(q=10, n=2, blocks=3)
        circuit = cutbench.build_benchmark(spec)
        plan = cutbench.plan_cut(circuit, spec.n)
        subs = cutbench.decompose(circuit, plan)
        states = [[cutbench.simulate(c) for c in fam.circuits] for fam in subs.segments]
        merged = cutbench.merge(cutbench.merge_input_from(subs, states))
        ref = orc.simulate(10, circuit.kinds, circuit.qa, circuit.qb)
        assert np.abs(merged.amps - ref).max() < 1e-10
        row = harness.measure(spec, 2)
        assert row.status == "ok" and row.t_cut == pytest.approx(row.t_pre + row.t_sub + row.t_merge)
    finally:
        for k in [k for k in sys.modules if k.startswith("cutbench_gpu_alias")]:
            del sys.modules[k]


def test_measure_native_cut_path(sw):
    from paper_2603_01443_b200 import harness
    from paper_2603_01443_b200.generators import BrickwallSpec

    row = harness.measure(BrickwallSpec(16, 5, 2, 3, 1), 2, cut_path="native")
    assert row.status == "ok" and row.t_pre > 0 and row.t_sub > 0 and row.t_merge > 0
    assert row.t_cut == pytest.approx(row.t_pre + row.t_sub + row.t_merge)
    res = sw.sweep_heatmap([12], [1, 2], n=2, repetitions=1, family="brickwall", depth=4, cut_path="native")
    assert res.metadata["cut_path"] == "native" and len(res.points) == 2
