"""Cold circuits (a seed the library has not seen every step, bench.py's
cold leg) with option OPTION = A vs B, interleaved: host wall time of a
synchronised run_cut and its variant stage (stage events).
    python tools/cold_ab.py OPTION A B [workload] [steps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_01443_b200 as cb  # noqa: E402
from paper_2603_01443_b200 import _native  # noqa: E402
from paper_2603_01443_b200.generators import BrickwallSpec  # noqa: E402

opt, va, vb = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
name = sys.argv[4] if len(sys.argv) > 4 else "cfg4a"
steps = int(sys.argv[5]) if len(sys.argv) > 5 else 8
_native.set_option("jit", 3)
spec = cb.BASELINE_CONFIGS[name]
out = torch.empty(1 << spec.q, dtype=torch.complex128, device="cuda")
warm = cb.build_brickwall(spec)
for _ in range(3):
    cb.run_cut(warm, spec.n, out=out, max_qubits=spec.q)
torch.cuda.synchronize()
_native.jit_wait(600)
wall = {va: [], vb: []}
sub = {va: [], vb: []}
seed = 5000
for i in range(steps):
    for g in ((va, vb) if i % 2 == 0 else (vb, va)):
        _native.set_option(opt, g)
        c = cb.build_brickwall(BrickwallSpec(spec.q, spec.d, spec.n, spec.c_total, seed))
        seed += 1
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        cb.run_cut(c, spec.n, out=out, max_qubits=spec.q, events=ev)
        torch.cuda.synchronize()
        wall[g].append(time.perf_counter() - t0)
        sub[g].append(ev[0].elapsed_time(ev[1]))
        _native.jit_wait(600)
for g in (va, vb):
    print(f"{name} cold {opt}={g}: {1e3 * np.median(wall[g]):.3f} ms per step "
          f"(variant stage {1e3 * np.median(sub[g]):.0f} us)", flush=True)
