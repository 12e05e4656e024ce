"""Per-launch view of one cfg4a cut step (for ncu's launch list): one warm-up
step (NVRTC compile, jit = 2), then `--steps` measured steps. Run under
  ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 12 \
      --csv --log-file launches.csv python tools/sub_stage_launches.py
The variant stage is every launch before the merge kernel."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2603_01443_b200 as cb  # noqa: E402
from paper_2603_01443_b200 import _native  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--workload", default="cfg4a")
args = ap.parse_args()
_native.set_option("jit", 2)
spec = cb.BASELINE_CONFIGS[args.workload]
circ = cb.build_brickwall(spec)
out = torch.empty(1 << spec.q, dtype=torch.complex128, device="cuda")
n0 = _native.launch_count()
cb.run_cut(circ, spec.n, out=out, max_qubits=spec.q)
torch.cuda.synchronize()
print("launches per step:", _native.launch_count() - n0)
evs = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
for _ in range(args.steps):
    cb.run_cut(circ, spec.n, out=out, events=evs, max_qubits=spec.q)
    torch.cuda.synchronize()
    print(f"sub {evs[0].elapsed_time(evs[1]) * 1e3:.1f} us  merge {evs[1].elapsed_time(evs[2]) * 1e3:.1f} us")
