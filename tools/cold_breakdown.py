"""Where a never-seen circuit's extra time goes (bench cold leg): run_cut on
new seeds with stage timers (pre = C++ plan + schedules + module lookup;
sub / merge = device events) next to a warm circuit.
    python tools/cold_breakdown.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2603_01443_b200 as cb  # noqa: E402
from paper_2603_01443_b200 import _native  # noqa: E402

_native.set_option("jit", 3)
spec = cb.BASELINE_CONFIGS["cfg4a"]
q = spec.q
out = torch.empty(1 << q, dtype=torch.complex128, device="cuda")
warm = cb.build_brickwall(spec)
for _ in range(3):
    cb.run_cut(warm, 2, out=out, max_qubits=q)
torch.cuda.synchronize()
_native.jit_wait(600)
for label, seeds in (("warm", [0] * 5), ("cold", range(1000, 1005))):
    for sd in seeds:
        circ = warm if label == "warm" else cb.build_brickwall(cb.BrickwallSpec(q, spec.d, 2, spec.c_total, sd))
        t = cb.StageTimes()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        cb.run_cut(circ, 2, out=out, max_qubits=q, timers=t)
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) * 1e3
        print(f"{label} seed {sd}: wall {wall:.3f} ms  pre {t.pre * 1e3:.3f}  sub {t.sub * 1e3:.3f}  merge {t.merge * 1e3:.3f}",
              flush=True)
