"""The raw ctypes binding shown in INTEGRATION.md §2 (what a maintainer would
add to the reference) runs as written against libcutsim.so and agrees with
the oracle."""
import os
import re

import numpy as np
import pytest

from oracle import cutbench_oracle as orc

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _snippets():
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    sec = text[text.index("## 2."):text.index("## 3.")]
    code = "\n".join(re.findall(r"```python\n(.*?)```", sec, re.S))
    return code.replace("/path/to/paper_2603_01443_b200/libcutsim.so",
                        os.path.join(ROOT, "paper_2603_01443_b200", "libcutsim.so"))


def test_integration_snippets_run():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_01443_b200 as cb

    ns = {}
    exec(compile(_snippets(), "INTEGRATION.md", "exec"), ns)
    circ = cb.build_staircase(cb.BenchmarkSpec(q=12, n=2, blocks=3))
    ref = orc.simulate(12, circ.kinds, circ.qa, circ.qb)
    assert np.abs(ns["simulate_device"](circ).cpu().numpy() - ref).max() < 1e-10
    out, stage = ns["cut_run_device"](circ, 2)
    assert np.abs(out.cpu().numpy() - ref).max() < 1e-10 and stage.min() >= 0
    subs = cb.decompose(circ, cb.plan_cut(circ, 2))
    states = [[ns["simulate_device"](c) for c in fam.circuits] for fam in subs.segments]
    merged = ns["merge2_device"](states[0], states[1], subs.merge_table, subs.coeffs)
    assert np.abs(merged.cpu().numpy() - ref).max() < 1e-10
