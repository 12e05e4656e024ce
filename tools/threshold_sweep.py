"""BASELINE cfg3 on the GPU: cut vs uncut end-to-end time at q=24, n=2,
d in {5, 10, 20}, c_total in 1..6, 3 seeds.

Emits the reference harness's CSV schema (`harness.py:41-45`: q, n, c_total,
D, G, t_pre, t_sub, t_merge, t_cut, t_orig, delta, reps, status,
schema_version) plus GPU columns (seed, max|d| cut vs uncut, merge GB/s).
Times are seconds; t_pre is host time, t_sub / t_merge / t_orig are CUDA-event
times; reps = repetitions averaged (after one warm-up), as in `measure`
(`harness.py:154-244`). Usage:

    python tools/threshold_sweep.py [reps] > profiles/rNN_threshold_q24.csv
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2603_01443_b200 as cb  # noqa: E402
from paper_2603_01443_b200 import engine  # noqa: E402
from paper_2603_01443_b200.merging import merge_chain_device  # noqa: E402
from paper_2603_01443_b200.pipeline import preprocess, simulate_segments  # noqa: E402

COLS = ["q", "n", "c_total", "D", "G", "t_pre", "t_sub", "t_merge", "t_cut", "t_orig", "delta", "reps",
        "status", "schema_version", "seed", "max_abs_diff", "merge_GBps"]


def ev():
    return torch.cuda.Event(enable_timing=True)


def point(spec, reps):
    circ = cb.build_brickwall(spec)
    q = spec.q
    out = torch.empty(1 << q, dtype=torch.complex128, device="cuda")
    ws = torch.empty(max(preprocess(circ, spec.n).chain.plan()[0], 1), dtype=torch.uint8, device="cuda")
    pre, sub, mer, orig = [], [], [], []
    uncut = None
    for r in range(reps + 1):  # r = 0 is the warm-up (program build + JIT)
        t0 = time.perf_counter()
        p = preprocess(circ, spec.n)
        t_pre = time.perf_counter() - t0
        e0, e1, e2 = ev(), ev(), ev()
        e0.record()
        batches = simulate_segments(p)
        e1.record()
        merge_chain_device(p.chain, batches, out=out, workspace=ws)
        e2.record()
        e2.synchronize()
        u0, u1 = ev(), ev()
        u0.record()
        uncut = cb.simulate(circ)
        u1.record()
        u1.synchronize()
        if r:
            pre.append(t_pre)
            sub.append(e0.elapsed_time(e1) / 1e3)
            mer.append(e1.elapsed_time(e2) / 1e3)
            orig.append(u0.elapsed_time(u1) / 1e3)
    diff = engine.max_abs_diff(cb.StateVec(q, device=out), uncut)
    t_pre, t_sub, t_merge, t_orig = (float(np.mean(x)) for x in (pre, sub, mer, orig))
    t_cut = t_pre + t_sub + t_merge
    return {"q": q, "n": spec.n, "c_total": spec.c_total, "D": spec.d, "G": circ.gate_count,
            "t_pre": t_pre, "t_sub": t_sub, "t_merge": t_merge, "t_cut": t_cut, "t_orig": t_orig,
            "delta": (t_cut - t_orig) / t_orig, "reps": reps, "status": "ok" if diff < 1e-10 else "MISMATCH",
            "schema_version": 1, "seed": spec.seed, "max_abs_diff": diff,
            "merge_GBps": (16 << q) / t_merge / 1e9}


def main():
    from paper_2603_01443_b200 import _native

    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    # NVRTC-specialised sweep kernels for both pipelines (compile outside the timers)
    _native.set_option("jit", int(sys.argv[2]) if len(sys.argv) > 2 else 2)
    print(",".join(COLS), flush=True)
    for spec in cb.generators.cfg3_grid():
        rec = point(spec, reps)
        print(",".join(f"{rec[c]:.6g}" if isinstance(rec[c], float) else str(rec[c]) for c in COLS), flush=True)


if __name__ == "__main__":
    main()
