"""Locate the cut-vs-uncut speedup boundary on the GPU (the BASELINE cfg3 goal
and the north_star's "reproduced cut-vs-uncut threshold curve on GPU").

For each (q, d) with n = 2 the cut count c grows until the cut pipeline's
end-to-end time t_cut = t_pre + t_sub + t_merge exceeds the uncut
simulator's t_orig (mean over seeds); c* = the largest c with t_cut < t_orig.
A least-squares line c* = slope * q + delta per depth is printed next to the
reference's theory (threshold_uniform, n = 2: slope 1/2, delta 0,
costmodel.py:102-116) and the paper's CPU fit (n = 2: c = 0.70 q - 7.30,
PAPER.md:777-783).

    python tools/threshold_boundary.py > profiles/rNN_boundary.csv
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2603_01443_b200 as cb  # noqa: E402
from paper_2603_01443_b200 import _native  # noqa: E402
from paper_2603_01443_b200.merging import merge_chain_device  # noqa: E402
from paper_2603_01443_b200.pipeline import preprocess, simulate_segments  # noqa: E402


def ev():
    return torch.cuda.Event(enable_timing=True)


def timed(spec, reps=2):
    circ = cb.build_brickwall(spec)
    q = spec.q
    out = torch.empty(1 << q, dtype=torch.complex128, device="cuda")
    ws = torch.empty(max(preprocess(circ, 2).chain.plan()[0], 1), dtype=torch.uint8, device="cuda")
    cut, orig = [], []
    for r in range(reps + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        p = preprocess(circ, 2)
        t_pre = time.perf_counter() - t0
        e0, e1 = ev(), ev()
        e0.record()
        merge_chain_device(p.chain, simulate_segments(p), out=out, workspace=ws)
        e1.record()
        e1.synchronize()
        u0, u1 = ev(), ev()
        u0.record()
        cb.simulate(circ, max_qubits=q)
        u1.record()
        u1.synchronize()
        if r:
            cut.append(t_pre + e0.elapsed_time(e1) / 1e3)
            orig.append(u0.elapsed_time(u1) / 1e3)
    del out, ws
    return float(np.mean(cut)), float(np.mean(orig))


def main():
    _native.set_option("jit", 2)
    qs = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "16,20,24,28").split(",")]
    ds = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "5,10,20").split(",")]
    seeds = (0,)
    print("q,d,c_total,t_cut,t_orig,delta,seeds", flush=True)
    best = {}
    for d in ds:
        for q in qs:
            cstar = 0
            for c in range(1, 15):
                vals = [timed(cb.BrickwallSpec(q, d, 2, c, s)) for s in seeds]
                t_cut = float(np.mean([v[0] for v in vals]))
                t_orig = float(np.mean([v[1] for v in vals]))
                delta = (t_cut - t_orig) / t_orig
                print(f"{q},{d},{c},{t_cut:.6g},{t_orig:.6g},{delta:.4f},{len(seeds)}", flush=True)
                if delta < 0:
                    cstar = c
                else:
                    break
            best[(q, d)] = cstar
    for d in ds:
        pts = [(q, best[(q, d)]) for q in qs]
        A = np.array([[q, 1.0] for q, _ in pts])
        y = np.array([c for _, c in pts], dtype=float)
        slope, icpt = np.linalg.lstsq(A, y, rcond=None)[0]
        print(f"# d={d}: c* = {[c for _, c in pts]} for q = {qs}; fit c* = {slope:.3f} q + {icpt:.2f} "
              f"(theory n=2: 0.5 q; paper CPU fit: 0.70 q - 7.30)", flush=True)


if __name__ == "__main__":
    main()
