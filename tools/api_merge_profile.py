"""cProfile of the drop-in merge call (merge_input_from + merge) at small q.
    python tools/api_merge_profile.py [q] [c] [d]"""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_01443_b200 as cb  # noqa: E402
from paper_2603_01443_b200 import _native  # noqa: E402
from paper_2603_01443_b200.cutting import decompose, plan_cut  # noqa: E402
from paper_2603_01443_b200.engine import StateVec  # noqa: E402
from paper_2603_01443_b200.merging import merge, merge_input_from  # noqa: E402
from paper_2603_01443_b200.pipeline import simulate_families  # noqa: E402

q = int(sys.argv[1]) if len(sys.argv) > 1 else 24
c = int(sys.argv[2]) if len(sys.argv) > 2 else 4
d = int(sys.argv[3]) if len(sys.argv) > 3 else 10
_native.set_option("jit", 2)
circ = cb.build_brickwall(cb.BrickwallSpec(q, d, 2, c, 0))
subs = decompose(circ, plan_cut(circ, 2))
batches = simulate_families(subs.segments)
states = [[StateVec.batch_row(f.num_qubits, b, v, np.complex128) for v in range(f.num_variants)]
          for f, b in zip(subs.segments, batches)]
for _ in range(20):
    merge(merge_input_from(subs, states))
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    merge(merge_input_from(subs, states))
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(30)
import time  # noqa: E402

from paper_2603_01443_b200.merging import ChainSpec, merge_chain_device  # noqa: E402

chain = ChainSpec.from_plan(subs.plan)
out = torch.empty(1 << q, dtype=torch.complex128, device="cuda")
for _ in range(20):
    merge_chain_device(chain, batches, out=out)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(200):
    merge_chain_device(chain, batches, out=out)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"merge_chain_device host {1e6 * (t1 - t0) / 200:.1f} us/call, incl. device drain {1e6 * (t2 - t0) / 200:.1f} us/call")
lib = _native.load()
t0 = time.perf_counter()
for _ in range(200):
    lib.cs_version()
print(f"ctypes call {1e6 * (time.perf_counter() - t0) / 200:.2f} us")
