"""Host-side cost of the drop-in API cut path (harness._cut_once, the
reference's call sequence) vs the one-call pipeline at small q: stage times
and a cProfile of repeated passes.
    python tools/api_path_profile.py [q] [c] [d]"""
import cProfile
import os
import pstats
import sys
import time

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
    for _ in range(3):
        f(circ, 2, max_qubits=30, deadline=None)
    t = [f(circ, 2, max_qubits=30, deadline=None)[:3] for _ in range(20)]
    print(f.__name__, "pre/sub/merge ms:", [round(1e3 * float(np.median([x[i] for x in t])), 3) for i in range(3)])
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    harness._cut_once(circ, 2, max_qubits=30, deadline=None)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
