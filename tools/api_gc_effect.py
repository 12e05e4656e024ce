"""The drop-in API cut path (harness._cut_once) with and without gc.collect()
between passes (the reference's measure() protocol collects after every
pipeline run): median stage times.   python tools/api_gc_effect.py [q] [c] [d]"""
import gc
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2603_01443_b200 as cb  # noqa: E402
from paper_2603_01443_b200 import _native, harness  # noqa: E402

q = int(sys.argv[1]) if len(sys.argv) > 1 else 24
c = int(sys.argv[2]) if len(sys.argv) > 2 else 4
d = int(sys.argv[3]) if len(sys.argv) > 3 else 10
_native.set_option("jit", 2)
circ = cb.build_brickwall(cb.BrickwallSpec(q, d, 2, c, 0))
for f in (harness._cut_once, harness._cut_once_native):
    for collect in (False, True):
        for _ in range(3):
            f(circ, 2, max_qubits=30, deadline=None)
        t = []
        for _ in range(30):
            r = f(circ, 2, max_qubits=30, deadline=None)
            t.append(r[:3])
            del r
            if collect:
                gc.collect()
        med = [round(1e6 * float(np.median([x[i] for x in t])), 1) for i in range(3)]
        print(f"{f.__name__:18s} gc={collect!s:5s} pre/sub/merge us {med}  sum {sum(med):.0f}", flush=True)
