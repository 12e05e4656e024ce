"""Host-side cost of the drop-in API cut path (harness._cut_once) at small q:
cProfile of repeated passes (q=24, d=10, c=2).  python tools/api_path_profile.py"""
import cProfile
import pstats
import sys

sys.path.insert(0, ".")
import paper_2603_01443_b200 as cb  # noqa: E402
from paper_2603_01443_b200 import _native, harness  # noqa: E402

_native.set_option("jit", 2)
circ = cb.build_brickwall(cb.BrickwallSpec(24, 10, 2, 2, 0))
for _ in range(3):
    harness._cut_once(circ, 2, max_qubits=30, deadline=None)
import time  # noqa: E402

t = []
for _ in range(20):
    r = harness._cut_once(circ, 2, max_qubits=30, deadline=None)
    t.append(r[:3])
import numpy as np  # noqa: E402

print("pre/sub/merge ms:", [round(1e3 * float(np.median([x[i] for x in t])), 3) for i in range(3)])
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    harness._cut_once(circ, 2, max_qubits=30, deadline=None)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
