import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2603_01443_b200 as cb
from paper_2603_01443_b200 import _native
_native.set_option("jit", 3)
spec = cb.BASELINE_CONFIGS["cfg4a"]; circ = cb.build_brickwall(spec); q = spec.q
ws_bytes, _, _ = _native.cut_workspace(q, circ.table, [q // 2] * 2)
out = torch.empty(1 << q, dtype=torch.complex128, device="cuda")
ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
for _ in range(3): cb.run_cut(circ, 2, out=out, workspace=ws, max_qubits=q)
torch.cuda.synchronize(); _native.jit_wait(600); cb.run_cut(circ, 2, out=out, workspace=ws, max_qubits=q); torch.cuda.synchronize()
evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(20)]
import time
s0 = torch.cuda.Event(enable_timing=True); s0.record()
h = []
for i in range(20):
    t0 = time.perf_counter()
    cb.run_cut(circ, 2, out=out, workspace=ws, events=evs[i], max_qubits=q)
    h.append((time.perf_counter() - t0) * 1e6)
s1 = torch.cuda.Event(enable_timing=True); s1.record(); torch.cuda.synchronize()
print("host us per call", [round(x) for x in h])
print("per step", s0.elapsed_time(s1) / 20 * 1e3, "us")
gaps = [evs[i][2].elapsed_time(evs[i + 1][0]) * 1e3 for i in range(19)]
print("gap ev2->next ev0 us", [round(g, 1) for g in gaps])
print("sub", [round(e[0].elapsed_time(e[1]) * 1e3, 1) for e in evs])
print("first ev0 after start", s0.elapsed_time(evs[0][0]) * 1e3)
# the same loop without per-step events
torch.cuda.synchronize()
s0 = torch.cuda.Event(enable_timing=True); s0.record()
for i in range(20):
    cb.run_cut(circ, 2, out=out, workspace=ws, max_qubits=q)
s1 = torch.cuda.Event(enable_timing=True); s1.record(); torch.cuda.synchronize()
print("per step without events", s0.elapsed_time(s1) / 20 * 1e3, "us")
