"""Wall-time breakdown of the drop-in API cut path (harness._cut_once, batched)
into its Python / native pieces at small q (median of N passes, device synced
around every piece).   python tools/api_stage_breakdown.py [q] [c] [d]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_01443_b200 as cb  # noqa: E402
from paper_2603_01443_b200 import _native, harness  # noqa: E402
from paper_2603_01443_b200.cutting import decompose, plan_cut  # noqa: E402
from paper_2603_01443_b200.engine import StateVec  # noqa: E402
from paper_2603_01443_b200.merging import merge, merge_input_from  # noqa: E402
from paper_2603_01443_b200.pipeline import simulate_families  # noqa: E402

q = int(sys.argv[1]) if len(sys.argv) > 1 else 24
c = int(sys.argv[2]) if len(sys.argv) > 2 else 4
d = int(sys.argv[3]) if len(sys.argv) > 3 else 10
_native.set_option("jit", 2)
circ = cb.build_brickwall(cb.BrickwallSpec(q, d, 2, c, 0))
N = 50
rec = {}


def t(name, fn, sync=True):
    if sync:
        torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn()
    if sync:
        torch.cuda.synchronize()
    rec.setdefault(name, []).append(time.perf_counter() - t0)
    return r


for i in range(N + 5):
    plan = t("plan_cut", lambda: plan_cut(circ, 2))
    subs = t("decompose", lambda: decompose(circ, plan))
    batches = t("simulate_families(launch)", lambda: simulate_families(subs.segments), sync=False)
    t("  sync after sub", lambda: None)
    states = t("StateVec rows", lambda: [[StateVec.batch_row(f.num_qubits, b, v, np.complex128) for v in range(f.num_variants)]
                                         for f, b in zip(subs.segments, batches)], sync=False)
    mi = t("merge_input_from", lambda: merge_input_from(subs, states), sync=False)
    out = t("merge(launch)", lambda: merge(mi), sync=False)
    t("  sync after merge", lambda: None)
    if i == 4:
        rec.clear()
for k, v in rec.items():
    print(f"{k:28s} {np.median(v) * 1e6:8.1f} us")
for f in (harness._cut_once, harness._cut_once_native):
    tt = [f(circ, 2, max_qubits=30, deadline=None)[:3] for _ in range(30)]
    print(f.__name__, "pre/sub/merge us:", [round(1e6 * float(np.median([x[i] for x in tt])), 1) for i in range(3)])
