"""Uncut simulator with and without the zero-start tile bound (option
zero_start_tiles): time per simulate at q (default 30) and max |diff|.
    python tools/uncut_zero_start.py [q]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2603_01443_b200 as cb  # noqa: E402
from paper_2603_01443_b200 import _native, engine  # noqa: E402

q = int(sys.argv[1]) if len(sys.argv) > 1 else 30
_native.set_option("jit", 2)
circ = cb.build_brickwall(cb.BrickwallSpec(q, 10, 2, 2, 0))
res = {}
for z in (0, 1):
    _native.set_option("zero_start_tiles", z)
    for _ in range(2):
        st = engine.simulate(circ, max_qubits=34)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        st = engine.simulate(circ, max_qubits=34)
    e1.record()
    e1.synchronize()
    res[z] = (e0.elapsed_time(e1) / 3, st.device_tensor().clone() if q <= 30 else None)
    print(f"q={q} zero_start_tiles={z}: {res[z][0]:.2f} ms", flush=True)
    del st
if q <= 30:
    print("max|diff|", (res[0][1] - res[1][1]).abs().max().item())
