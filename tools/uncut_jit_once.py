"""Uncut simulator with NVRTC-specialised kernels (ncu target)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2603_01443_b200 as cb  # noqa: E402
from paper_2603_01443_b200 import _native  # noqa: E402

_native.set_option("jit", 2)
circ = cb.build_brickwall(cb.BASELINE_CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg4a"])
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 1):
    sv = cb.simulate(circ, max_qubits=circ.num_qubits)
torch.cuda.synchronize()
print("ok")
