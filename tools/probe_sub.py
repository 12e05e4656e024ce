"""Probe host vs device time of the subcircuit stage (diagnostic)."""
import cProfile
import pstats
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2603_01443_b200 as cb  # noqa: E402
from paper_2603_01443_b200.pipeline import preprocess, simulate_segments  # noqa: E402

circ = cb.build_brickwall(cb.BASELINE_CONFIGS["cfg4a"])
prep = preprocess(circ, 2)
for _ in range(3):
    simulate_segments(prep)
torch.cuda.synchronize()
N = 20
t0 = time.perf_counter()
for _ in range(N):
    simulate_segments(prep)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host issue {1e3*(t1-t0)/N:.3f} ms/iter, total incl drain {1e3*(t2-t0)/N:.3f} ms/iter")
pr = cProfile.Profile()
pr.enable()
for _ in range(N):
    simulate_segments(prep)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
