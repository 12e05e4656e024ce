"""Uncut simulator vs the tile's contiguous low qubits L (option low_bits)
with zero-start tiles: sweeps, full-sweep equivalents, time.
    python tools/uncut_low_bits.py [q,q,..] [L,L,..] [windows,..]"""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2603_01443_b200 as cb  # noqa: E402
from paper_2603_01443_b200 import _native, engine  # noqa: E402

qs = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [30]
Ls = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [5, 4, 3, 2]
wins = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [1, 2]
_native.set_option("jit", 2)
for q, L, win in [(q, L, w) for q in qs for L in Ls for w in wins]:
    circ = cb.build_brickwall(cb.BrickwallSpec(q, 10, 2, 2, 0))
    if True:
        _native.set_option("low_bits", L)
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
        del st
        print(f"q={q} L={L} windows={win}: {len(plan['sweeps'])} sweeps, {eq:.2f} full-sweep equivalents, "
              f"{e0.elapsed_time(e1) / 3:.2f} ms", flush=True)
_native.set_option("low_bits", 5)
_native.set_option("sweep_windows", 1)
