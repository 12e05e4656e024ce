"""Uncut simulator (NVRTC kernels) with a given __launch_bounds__ min-blocks
for the generated kernels:  python tools/uncut_minb.py MINB [cfg] [REG_BITS]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2603_01443_b200 as cb  # noqa: E402
from paper_2603_01443_b200 import _native  # noqa: E402

_native.set_option("jit", 2)
_native.set_option("jit_minb", int(sys.argv[1]))
if len(sys.argv) > 3:
    _native.set_option("reg_bits", int(sys.argv[3]))
if len(sys.argv) > 4:
    _native.set_option("jit_persistent", int(sys.argv[4]))
if len(sys.argv) > 5:
    _native.set_option("reg_reorder", int(sys.argv[5]))
if len(sys.argv) > 6:
    _native.set_option("sweep_windows", int(sys.argv[6]))
name = sys.argv[2] if len(sys.argv) > 2 else "cfg4a"
circ = cb.build_brickwall(cb.BASELINE_CONFIGS[name])
sv = cb.simulate(circ, max_qubits=circ.num_qubits)
ref = sv.device_tensor()[:1 << 20].clone()
del sv
times = []
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sv = cb.simulate(circ, max_qubits=circ.num_qubits)
    e1.record()
    e1.synchronize()
    times.append(e0.elapsed_time(e1))
    assert torch.equal(sv.device_tensor()[:1 << 20], ref)
    del sv
print(f"{name} jit_minb={sys.argv[1]} reg_bits={_native.get_option('reg_bits')} "
      f"persistent={_native.get_option('jit_persistent')} reorder={_native.get_option('reg_reorder')} windows={_native.get_option('sweep_windows')}: {np.median(times):.1f} ms {[round(t, 1) for t in times]}", flush=True)
