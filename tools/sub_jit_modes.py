"""Subcircuit (variant-batch) stage of cs_cut_run under the interpreter and
the NVRTC kernels, per segment size:  python tools/sub_jit_modes.py"""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2603_01443_b200 as cb  # noqa: E402
from paper_2603_01443_b200 import _native  # noqa: E402

for q in (16, 20, 24, 26, 28, 30):
    circ = cb.build_brickwall(cb.BrickwallSpec(q, 10, 2, 2, 0))
    row = []
    for jit in (0, 2):
        _native.set_option("jit", jit)
        t = cb.StageTimes()
        for _ in range(3):
            cb.run_cut(circ, 2, timers=t)
        subs = []
        for _ in range(10):
            cb.run_cut(circ, 2, timers=t)
            subs.append(t.sub)
        row.append(np.median(subs) * 1e6)
    print(f"q={q} (segments of {q // 2}): sub interpreter {row[0]:.1f} us, nvrtc {row[1]:.1f} us", flush=True)
