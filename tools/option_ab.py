"""Interleaved A/B of one library option over the cut pipeline's steady state
(device-resident run_cut steps in blocks of 8): per-step time, the variant
stage (stage events), and max|delta| between the two settings' outputs.
    python tools/option_ab.py OPTION A B [workload...]
e.g. python tools/option_ab.py cluster_loop 0 1 cfg4a cfg4b"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_01443_b200 as cb  # noqa: E402
from paper_2603_01443_b200 import _native  # noqa: E402

opt, va, vb = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
_native.set_option("jit", 3)
old = _native.get_option(opt)
for name in sys.argv[4:] or ["cfg4a", "cfg4b", "cfg5_q32_n2_c2"]:
    spec = cb.BASELINE_CONFIGS[name]
    circ = cb.build_brickwall(spec)
    q = spec.q
    out = torch.empty(1 << q, dtype=torch.complex128, device="cuda")
    res = {va: [], vb: []}
    sub = {va: [], vb: []}
    probe = {}
    for rnd in range(4):
        for g in ((va, vb) if rnd % 2 == 0 else (vb, va)):
            _native.set_option(opt, g)
            for _ in range(3):
                cb.run_cut(circ, spec.n, out=out, max_qubits=q)
            torch.cuda.synchronize()
            _native.jit_wait(600)
            evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(8)]
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for i in range(8):
                cb.run_cut(circ, spec.n, out=out, events=evs[i], max_qubits=q)
            b.record()
            torch.cuda.synchronize()
            res[g].append(a.elapsed_time(b) / 8 * 1e3)
            sub[g].extend(e[0].elapsed_time(e[1]) * 1e3 for e in evs)
            probe[g] = out[:: (1 << q) // 65536].clone()
    d = (probe[va] - probe[vb]).abs().max().item()
    print(f"{name}: {opt}={va} {np.median(res[va]):.1f} us/step (sub {np.median(sub[va]):.1f}) | "
          f"{opt}={vb} {np.median(res[vb]):.1f} us/step (sub {np.median(sub[vb]):.1f}) | max|d| {d:.2e}",
          flush=True)
    _native.set_option(opt, old)
    del out
    torch.cuda.empty_cache()
