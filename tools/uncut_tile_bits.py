import json, sys, torch
sys.path.insert(0, '.')
import paper_2603_01443_b200 as cb
from paper_2603_01443_b200 import _native, engine
_native.set_option("jit", 2)
for q, d in ((30, 10), (30, 20), (32, 10)):
    circ = cb.build_brickwall(cb.BrickwallSpec(q, d, 2, 2, 0))
    for T in (11, 12, 13):
        _native.set_option("tile_bits", T)
        _native.set_option("dense_norm", 1)
        plan = json.loads(_native.sweep_plan_json(q, circ.table))
        _native.set_option("dense_norm", 2)
        eq = sum(2.0 ** (sw["z"] - (q - sw["T"])) for sw in plan["sweeps"])
        for _ in range(2): st = engine.simulate(circ, max_qubits=34)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3): st = engine.simulate(circ, max_qubits=34)
        e1.record(); e1.synchronize(); del st
        print(f"q={q} d={d} T={T}: {len(plan['sweeps'])} sweeps {eq:.2f} eq {e0.elapsed_time(e1)/3:.2f} ms", flush=True)
    _native.set_option("tile_bits", 0)
