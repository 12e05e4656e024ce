"""Uncut simulator (NVRTC kernels) vs tile size:  python tools/uncut_tiles.py T [cfg]"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2603_01443_b200 as cb  # noqa: E402
from paper_2603_01443_b200 import _native  # noqa: E402

_native.set_option("jit", 2)
_native.set_option("tile_bits", int(sys.argv[1]))
name = sys.argv[2] if len(sys.argv) > 2 else "cfg4a"
circ = cb.build_brickwall(cb.BASELINE_CONFIGS[name])
nsw = len(json.loads(_native.sweep_plan_json(circ.num_qubits, circ.table))["sweeps"])
sv = cb.simulate(circ, max_qubits=circ.num_qubits)
del sv
times = []
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sv = cb.simulate(circ, max_qubits=circ.num_qubits)
    e1.record()
    e1.synchronize()
    times.append(e0.elapsed_time(e1))
    del sv
print(f"{name} tile_bits={sys.argv[1]} sweeps={nsw}: {np.median(times):.1f} ms", flush=True)
