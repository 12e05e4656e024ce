"""One warm uncut simulate of a BASELINE workload (for ncu launch lists):
python tools/uncut_one.py [workload] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2603_01443_b200 as cb  # noqa: E402
from paper_2603_01443_b200 import _native  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4a"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
spec = cb.BASELINE_CONFIGS[name]
circ = cb.build_brickwall(spec)
_native.set_option("jit", 3)
sv = cb.simulate(circ, max_qubits=spec.q)
del sv
_native.jit_wait(600)
for _ in range(reps):
    sv = cb.simulate(circ, max_qubits=spec.q)
    torch.cuda.synchronize()
    del sv
print("ok")
