"""Interleaved A/B of one library option on the uncut simulator (NVRTC
kernels, jit = 3, compiled before timing): device time per simulate, and
max|delta| between the two settings' outputs (first 2^28 amplitudes).
    python tools/uncut_option_ab.py OPTION A B [workload ...]   (default cfg4a)
e.g. python tools/uncut_option_ab.py fuse 1 2 cfg4a"""
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
for name in sys.argv[4:] or ["cfg4a"]:
    spec = cb.BASELINE_CONFIGS[name]
    circ = cb.build_brickwall(spec)
    q = spec.q
    t = {va: [], vb: []}
    head = {}
    for g in (va, vb):
        _native.set_option(opt, g)
        sv = cb.simulate(circ, max_qubits=q)
        del sv
        _native.jit_wait(600)
    for rnd in range(6):
        for g in ((va, vb) if rnd % 2 == 0 else (vb, va)):
            _native.set_option(opt, g)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record()
            sv = cb.simulate(circ, max_qubits=q)
            b.record()
            b.synchronize()
            t[g].append(a.elapsed_time(b))
            if rnd == 0:
                head[g] = sv.device_tensor()[: 1 << min(q, 28)].clone()
            del sv
    d = (head[va] - head[vb]).abs().max().item()
    del head
    print(f"{name} q={q} {opt}: {va} median {np.median(t[va]):.2f} ms {np.round(t[va], 2).tolist()} | "
          f"{vb} median {np.median(t[vb]):.2f} ms {np.round(t[vb], 2).tolist()} | max|d| (2^28 head) {d:.2e}",
          flush=True)
_native.set_option(opt, old)
