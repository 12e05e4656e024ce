"""cProfile of the drop-in cut pipeline (harness._cut_once) at small q, where
host overhead dominates:  python tools/profile_host_cut.py [q] [c]"""
import cProfile
import pstats
import sys

sys.path.insert(0, ".")
import paper_2603_01443_b200 as cb  # noqa: E402
from paper_2603_01443_b200 import _native, harness  # noqa: E402

q, c = (int(v) for v in sys.argv[1:3]) if len(sys.argv) > 2 else (20, 2)
_native.set_option("jit", 2)
circ = cb.build_brickwall(cb.BrickwallSpec(q, 10, 2, c, 0))
for _ in range(5):
    harness._cut_once(circ, 2, max_qubits=30, deadline=None)
    harness._orig_once(circ, max_qubits=30, deadline=None)
acc = [0.0, 0.0, 0.0]
for _ in range(50):
    t = harness._cut_once(circ, 2, max_qubits=30, deadline=None)
    for i in range(3):
        acc[i] += t[i] / 50
print("stage means (ms):", [round(a * 1e3, 3) for a in acc])
pr = cProfile.Profile()
pr.enable()
for _ in range(50):
    harness._cut_once(circ, 2, max_qubits=30, deadline=None)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
