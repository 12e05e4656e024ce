"""CLI shim and harness mirror. CPU: argument handling, preprocess, exit
codes; GPU: cutrun --verify and measure()'s timing contract
(reference tests/test_harness.py:42-72, tests/test_cli.py:69-92)."""
import json
import math

import pytest

from paper_2603_01443_b200 import cli
from paper_2603_01443_b200.circuits import BenchmarkSpec
from paper_2603_01443_b200.generators import BrickwallSpec


def test_preprocess_json(tmp_path, capsys):
    """Reference cli.py:136-143: the SubcircuitSet JSON goes to --out (or
    stdout); --summary adds a plan line on stderr."""
    path = tmp_path / "subs.json"
    rc = cli.main(["preprocess", "--q", "6", "--n", "3", "--blocks", "2", "--out", str(path), "--summary"])
    assert rc == cli.EXIT_OK
    data = json.loads(path.read_text())
    assert data["c_total"] == 4 and len(data["segments"]) == 3
    assert "N_sub=24" in capsys.readouterr().err
    rc = cli.main(["preprocess", "--q", "6", "--n", "3", "--blocks", "2", "--machine-tag", "x", "--reps", "1"])
    assert rc == cli.EXIT_OK
    assert json.loads(capsys.readouterr().out) == data


def test_validation_exit_code(capsys):
    assert cli.main(["preprocess", "--q", "7", "--n", "2"]) == cli.EXIT_VALIDATION


def test_brickwall_preprocess(capsys):
    rc = cli.main(["preprocess", "--family", "brickwall", "--q", "12", "--n", "2", "--d", "4", "--c", "1"])
    assert rc == 0
    assert json.loads(capsys.readouterr().out)["c_total"] == 1


def test_capacity_exit_code_before_any_device_work():
    assert cli.main(["simulate", "--q", "32", "--n", "2", "--guard", "30"]) == cli.EXIT_CAPACITY


@pytest.mark.gpu
def test_cutrun_verify(capsys):
    rc = cli.main(["cutrun", "--family", "brickwall", "--q", "16", "--n", "2", "--d", "6", "--c", "3",
                   "--verify"])
    assert rc == 0
    out = capsys.readouterr().out
    err = float(out.split("reconstruction_linf_error=")[1].split()[0])
    assert err < 1e-10


@pytest.mark.gpu
def test_cutrun_streaming_verify(capsys):
    """Reference cli.py:97-108: --streaming merges through merge_streaming."""
    rc = cli.main(["cutrun", "--q", "8", "--n", "2", "--blocks", "2", "--streaming", "--verify",
                   "--machine-tag", "t"])
    assert rc == 0
    out = capsys.readouterr().out
    assert float(out.split("reconstruction_linf_error=")[1].split()[0]) < 1e-10


@pytest.mark.gpu
def test_measure_contract():
    from paper_2603_01443_b200 import harness

    tb = harness.measure(BenchmarkSpec(q=8, n=2, blocks=2), repetitions=2)
    for v in (tb.t_pre, tb.t_sub, tb.t_merge, tb.t_orig):
        assert math.isfinite(v) and v > 0
    assert tb.t_cut == tb.t_pre + tb.t_sub + tb.t_merge
    assert tb.status == "ok" and len(tb.samples["orig"]) == 2
    tb = harness.measure(BrickwallSpec(q=12, d=4, n=2, c_total=1), repetitions=1, pipelines=("orig",))
    assert math.isnan(tb.t_pre) and math.isfinite(tb.t_orig)
    tb = harness.measure(BenchmarkSpec(q=10, n=2, blocks=3), repetitions=1, budget=1e-9)
    assert tb.status == "timeout-cut+orig" and math.isnan(tb.delta)
    csv = harness.format_csv([tb])
    assert csv.splitlines()[0].split(",") == list(harness.CSV_COLUMNS)
