"""Uncut simulator under the tile-set policies (option sweep_windows: 1 most
absorbed dense ops per sweep, 2 with a one-sweep look-ahead, 3 cost-aware for
zero-start tiles): sweeps, full-sweep equivalents, time and max |diff| vs 1.
    python tools/uncut_windows.py [q,q,..] [d]"""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2603_01443_b200 as cb  # noqa: E402
from paper_2603_01443_b200 import _native, engine  # noqa: E402

qs = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [30]
d = int(sys.argv[2]) if len(sys.argv) > 2 else 10
_native.set_option("jit", 2)
for q in qs:
    circ = cb.build_brickwall(cb.BrickwallSpec(q, d, 2, 2, 0))
    ref = None
    for win in (1, 3):
        _native.set_option("sweep_windows", win)
        _native.set_option("dense_norm", 1)
        plan = json.loads(_native.sweep_plan_json(q, circ.table))
        _native.set_option("dense_norm", 2)
        eq = sum(2.0 ** (sw["z"] - (q - sw["T"])) for sw in plan["sweeps"])
        for _ in range(2):
            st = engine.simulate(circ, max_qubits=34)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            st = engine.simulate(circ, max_qubits=34)
        e1.record()
        e1.synchronize()
        t = st.device_tensor()
        if q <= 30:
            if ref is None:
                ref = t.clone()
                diff = 0.0
            else:
                diff = (t - ref).abs().max().item()
        else:
            diff = float("nan")
        del st, t
        print(f"q={q} d={d} windows={win}: {len(plan['sweeps'])} sweeps, {eq:.2f} full-sweep equivalents, "
              f"{e0.elapsed_time(e1) / 3:.2f} ms, max|diff| {diff:.2e}", flush=True)
    del ref
    torch.cuda.empty_cache()
_native.set_option("sweep_windows", 1)
