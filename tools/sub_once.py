"""Run the subcircuit stage of one config a few times (ncu target):
python tools/sub_once.py [cfg] [reps] [jit]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2603_01443_b200 as cb  # noqa: E402
from paper_2603_01443_b200.pipeline import preprocess, simulate_segments  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4a"
if len(sys.argv) > 3:
    from paper_2603_01443_b200 import _native

    _native.set_option("jit", int(sys.argv[3]))
spec = cb.BASELINE_CONFIGS[name]
prep = preprocess(cb.build_brickwall(spec), spec.n)
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 3):
    simulate_segments(prep)
torch.cuda.synchronize()
print("ok")
