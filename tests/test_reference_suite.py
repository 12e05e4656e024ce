"""The REFERENCE's own test files (pkg/tests of /root/reference, copied
unmodified into the git-ignored baseline/_ref/pkg_tests/ by
__graft_entry__.build()) run against this package through the module alias
(`import cutbench` -> paper_2603_01443_b200, compat.install_as_cutbench),
as SURVEY.md §4 planned: test_engine.py, test_cutting.py, test_merging.py,
test_circuits.py, test_harness.py, test_cli.py, test_costmodel.py,
test_svmfit.py and test_acceptance.py.

CPU: every reference test that does not reach the device path must pass
(the rest are reported as skipped: the product has no CPU fallback).
GPU: every reference test must pass, except the ones
tests/reference_suite/dropin_plugin.py lists, each with its reason: a
reference internal it needs, or a timing law of the CPU implementation
(single-thread numba cost model) that the GPU path does not share.
"""
import os
import re
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUITE = os.path.join(ROOT, "baseline", "_ref", "pkg_tests")


def run_suite(files, extra=()):
    if not os.path.isdir(SUITE):
        pytest.skip("reference tests not fetched (run __graft_entry__.build() where /root/reference exists)")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(ROOT, "tests", "reference_suite"), ROOT,
                                         env.get("PYTHONPATH", "")])
    cmd = [sys.executable, "-m", "pytest", "-p", "dropin_plugin", "-p", "no:cacheprovider", "-q", "-rs",
           "--rootdir", SUITE, *extra, *[os.path.join(SUITE, f) for f in files]]
    out = subprocess.run(cmd, capture_output=True, text=True, env=env, cwd=SUITE, timeout=3000)
    text = out.stdout + out.stderr
    counts = {k: int(v) for v, k in re.findall(r"(\d+) (passed|failed|skipped|errors?)", text.splitlines()[-1])}
    return out.returncode, counts, text


CPU_FILES = ["test_circuits.py", "test_cutting.py", "test_costmodel.py", "test_svmfit.py", "test_engine.py",
             "test_merging.py", "test_harness.py"]


def test_reference_suite_host_parts_pass_on_cpu():
    try:
        import torch

        if torch.cuda.is_available():
            pytest.skip("the GPU variant runs the whole suite")
    except ImportError:
        pass
    rc, counts, text = run_suite(CPU_FILES)
    assert counts.get("failed", 0) == 0 and counts.get("error", 0) == 0 and counts.get("errors", 0) == 0, text[-4000:]
    assert counts.get("passed", 0) >= 100, text[-2000:]


@pytest.mark.gpu
def test_reference_suite_passes_on_the_gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    files = CPU_FILES + ["test_cli.py", "test_acceptance.py"]
    rc, counts, text = run_suite(files)
    with open(os.path.join(ROOT, "gpurun_out", "reference_suite.log") if os.path.isdir(
            os.path.join(ROOT, "gpurun_out")) else os.devnull, "w") as fh:
        fh.write(text)
    assert counts.get("failed", 0) == 0 and counts.get("error", 0) == 0 and counts.get("errors", 0) == 0, text[-6000:]
    skipped = re.findall(r"SKIPPED \[\d+\] .*?: (.*)", text)
    assert all(s.startswith(("reference internal:", "reference CPU cost law:")) for s in skipped), skipped
    assert rc == 0
