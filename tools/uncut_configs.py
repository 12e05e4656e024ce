import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import paper_2603_01443_b200 as cb
from paper_2603_01443_b200 import _native
for name in ["cfg5_q32_n2_c4", "cfg5_q32_n2_c2", "cfg4a"]:
    spec = cb.BASELINE_CONFIGS[name]
    circ = cb.build_brickwall(spec)
    for jit in (2, 3):
        _native.set_option("jit", jit)
        sv = cb.simulate(circ, max_qubits=spec.q); del sv
        _native.jit_wait(600)
        ts = []
        for _ in range(3):
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); sv = cb.simulate(circ, max_qubits=spec.q); b.record(); b.synchronize(); ts.append(a.elapsed_time(b)); del sv
        print(name, "jit", jit, [round(t, 1) for t in ts], "ms", flush=True)
