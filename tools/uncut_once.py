"""Run the uncut simulator on one BASELINE config (ncu target)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2603_01443_b200 as cb  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4a"
circ = cb.build_brickwall(cb.BASELINE_CONFIGS[name])
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 1):
    sv = cb.simulate(circ, max_qubits=circ.num_qubits)
torch.cuda.synchronize()
print("ok", sv)
