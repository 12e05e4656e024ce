"""Does recording stage events per step change the step time? Interleaved
blocks of 10 cfg4a steps with and without per-step events.
    python tools/step_events_ab.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_01443_b200 as cb  # noqa: E402
from paper_2603_01443_b200 import _native  # noqa: E402

_native.set_option("jit", 3)
spec = cb.BASELINE_CONFIGS["cfg4a"]
circ = cb.build_brickwall(spec)
q = spec.q
ws_bytes, _, _ = _native.cut_workspace(q, circ.table, [q // 2] * 2)
out = torch.empty(1 << q, dtype=torch.complex128, device="cuda")
ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
for _ in range(3):
    cb.run_cut(circ, 2, out=out, workspace=ws, max_qubits=q)
torch.cuda.synchronize()
_native.jit_wait(600)
evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(10)]
res = {True: [], False: []}
for rnd in range(6):
    for with_ev in (True, False) if rnd % 2 == 0 else (False, True):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for i in range(10):
            cb.run_cut(circ, 2, out=out, workspace=ws, events=evs[i] if with_ev else None, max_qubits=q)
        b.record()
        torch.cuda.synchronize()
        res[with_ev].append(a.elapsed_time(b) / 10 * 1e3)
for k, v in res.items():
    print(f"events={k}: per step us {[round(x, 1) for x in v]} median {np.median(v):.1f}")
