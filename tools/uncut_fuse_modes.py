"""Uncut simulator, NVRTC-specialised, under the two lowerings (fuse=1: fused
complex 2x2s; fuse=2: U3 split into phase . Ry . phase with commuted
phases): time and agreement.  python tools/uncut_fuse_modes.py [cfg]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2603_01443_b200 as cb  # noqa: E402
from paper_2603_01443_b200 import _native, engine  # noqa: E402

_native.set_option("jit", 2)
name = sys.argv[1] if len(sys.argv) > 1 else "cfg4a"
circ = cb.build_brickwall(cb.BASELINE_CONFIGS[name])
states = {}
for fuse in (1, 2):
    _native.set_option("fuse", fuse)
    sv = cb.simulate(circ, max_qubits=circ.num_qubits)  # build + compile
    del sv
    torch.cuda.synchronize()
    times = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        sv = cb.simulate(circ, max_qubits=circ.num_qubits)
        e1.record()
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
        if len(times) < 3:
            del sv
    states[fuse] = sv
    print(f"{name} fuse={fuse}: {np.median(times):.1f} ms  ({[round(t, 1) for t in times]})", flush=True)
    if circ.num_qubits > 30:
        break
if len(states) == 2:
    print("max|diff| =", engine.max_abs_diff(states[1], states[2]))
