"""Variant stage replayed from a captured CUDA graph (option stage_graphs) vs
launched directly: cfg4a / cfg5 steps in interleaved blocks, per-step time
and the steady-state variant stage, results identical.
    python tools/stage_graphs_ab.py [workload...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_01443_b200 as cb  # noqa: E402
from paper_2603_01443_b200 import _native  # noqa: E402

_native.set_option("jit", 3)
for name in sys.argv[1:] or ["cfg4a", "cfg4b", "cfg5_q32_n4_c4"]:
    spec = cb.BASELINE_CONFIGS[name]
    circ = cb.build_brickwall(spec)
    q = spec.q
    ws_bytes, _, _ = _native.cut_workspace(q, circ.table, [q // spec.n] * spec.n)
    out = torch.empty(1 << q, dtype=torch.complex128, device="cuda")
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        cb.run_cut(circ, spec.n, out=out, workspace=ws, max_qubits=q)
    torch.cuda.synchronize()
    _native.jit_wait(600)
    res = {0: [], 1: []}
    sub = {0: [], 1: []}
    probe = {}
    for rnd in range(4):
        for g in ((0, 1) if rnd % 2 == 0 else (1, 0)):
            _native.set_option("stage_graphs", g)
            cb.run_cut(circ, spec.n, out=out, workspace=ws, max_qubits=q)  # (captures on first use)
            torch.cuda.synchronize()
            evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(8)]
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for i in range(8):
                cb.run_cut(circ, spec.n, out=out, workspace=ws, events=evs[i], max_qubits=q)
            b.record()
            torch.cuda.synchronize()
            res[g].append(a.elapsed_time(b) / 8 * 1e3)
            sub[g].extend(e[0].elapsed_time(e[1]) * 1e3 for e in evs)
            probe[g] = out[:: (1 << q) // 4096].clone()
    same = torch.equal(probe[0], probe[1])
    print(f"{name}: direct {np.median(res[0]):.1f} us/step (sub {np.median(sub[0]):.1f}) | "
          f"graph {np.median(res[1]):.1f} us/step (sub {np.median(sub[1]):.1f}) | identical {same}", flush=True)
    _native.set_option("stage_graphs", 1)
    del out, ws
    torch.cuda.empty_cache()
