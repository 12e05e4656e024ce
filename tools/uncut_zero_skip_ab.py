"""Interleaved A/B of the zero_skip option on the uncut simulator (a start
from |0..0> with zero-start tiles: 1 = skip loads of still-zero amplitudes and
the zeroing pass, 0 = zero the state once and load every launched tile):
device time per simulate and max|delta| between the two outputs.
    python tools/uncut_zero_skip_ab.py [workload ...]   (default cfg4a cfg5_q32_n2_c2)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_01443_b200 as cb  # noqa: E402
from paper_2603_01443_b200 import _native  # noqa: E402

for jit in (3, 0):
    _native.set_option("jit", jit)
    for name in sys.argv[1:] or ["cfg4a", "cfg5_q32_n2_c2"]:
        spec = cb.BASELINE_CONFIGS[name]
        circ = cb.build_brickwall(spec)
        q = spec.q
        if jit == 0 and q > 30:
            continue
        t = {0: [], 1: []}
        for rnd in range(6):
            for g in ((0, 1) if rnd % 2 == 0 else (1, 0)):
                _native.set_option("zero_skip", g)
                sv = cb.simulate(circ, max_qubits=q)
                del sv
                _native.jit_wait(600)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                a.record()
                sv = cb.simulate(circ, max_qubits=q)
                b.record()
                b.synchronize()
                t[g].append(a.elapsed_time(b))
                del sv
        # full-state comparison on one pair
        _native.set_option("zero_skip", 0)
        s0 = cb.simulate(circ, max_qubits=q).device_tensor().clone()
        _native.set_option("zero_skip", 1)
        s1 = cb.simulate(circ, max_qubits=q).device_tensor()
        d = max((s0[i:i + (1 << 26)] - s1[i:i + (1 << 26)]).abs().max().item() for i in range(0, 1 << q, 1 << 26))
        bitid = torch.equal(s0, s1)
        norm = s1.abs().square().sum().item()
        del s0, s1
        torch.cuda.empty_cache()
        print(f"jit={jit} {name} q={q}: zero_skip 0 median {np.median(t[0]):.2f} ms {np.round(t[0], 2).tolist()} | "
              f"1 median {np.median(t[1]):.2f} ms {np.round(t[1], 2).tolist()} | max|d| {d:.2e} bit-identical {bitid} "
              f"norm {norm:.15f}", flush=True)
_native.set_option("zero_skip", 1)
