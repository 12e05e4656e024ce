"""Interpreter vs NVRTC-specialised sweep kernels (sub stage and uncut)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2603_01443_b200 as cb  # noqa: E402
from paper_2603_01443_b200 import _native  # noqa: E402
from paper_2603_01443_b200.pipeline import preprocess, simulate_segments  # noqa: E402
from oracle import cutbench_oracle as orc  # noqa: E402


def timeit(fn, n=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / n


for jit in (0, 2):
    _native.set_option("jit", jit)
    for name in ("cfg2", "cfg4a", "cfg4b", "cfg5_q32_n2_c2"):
        spec = cb.BASELINE_CONFIGS[name]
        prep = preprocess(cb.build_brickwall(spec), spec.n)
        t0 = time.time()
        simulate_segments(prep)
        torch.cuda.synchronize()
        first = time.time() - t0
        print(f"jit={jit} sub {name}: {timeit(lambda: simulate_segments(prep)) * 1e3:.1f} us (first call {first:.2f} s)",
              flush=True)
    for name in ("cfg2", "cfg4a"):
        circ = cb.build_brickwall(cb.BASELINE_CONFIGS[name])
        t0 = time.time()
        sv = cb.simulate(circ)
        torch.cuda.synchronize()
        first = time.time() - t0
        ms = timeit(lambda: cb.simulate(circ, max_qubits=circ.num_qubits), n=2)
        print(f"jit={jit} uncut {name}: {ms:.2f} ms (first call {first:.2f} s)", flush=True)
        if name == "cfg2":
            ref = orc.simulate(circ.num_qubits, circ.kinds, circ.qa, circ.qb, circ.params)
            print("   max|d| vs oracle", float(np.abs(sv.amps - ref).max()), flush=True)
    print(_native.last_error(), flush=True)
