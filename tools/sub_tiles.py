"""Variant-batch stage vs forced tile size (NVRTC kernels):
python tools/sub_tiles.py Q T1,T2,..."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2603_01443_b200 as cb  # noqa: E402
from paper_2603_01443_b200 import _native  # noqa: E402

q = int(sys.argv[1])
_native.set_option("jit", 2)
circ = cb.build_brickwall(cb.BrickwallSpec(q, 10, 2, 2, 0))
for tb in [int(v) for v in sys.argv[2].split(",")]:
    _native.set_option("tile_bits", tb)
    t = cb.StageTimes()
    for _ in range(3):
        cb.run_cut(circ, 2, timers=t)
    subs = []
    for _ in range(10):
        cb.run_cut(circ, 2, timers=t)
        subs.append(t.sub)
    print(f"q={q} tile_bits={tb}: sub {np.median(subs) * 1e6:.1f} us", flush=True)
