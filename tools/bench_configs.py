"""Per-config measurements of the cut pipeline on one B200 (BASELINE.json
configs 1, 2, 4a, 4b, 5) with parity checks. Writes one JSON line per config.

    python tools/bench_configs.py [names...] > profiles/rNN_configs.jsonl

For each config: stage times (pre = host, sub / merge = CUDA events, median of
5 steps), merge kernel GB/s vs the measured HBM peak, the uncut simulator time
(where the full state fits next to the cut output), and a correctness check:
cut vs uncut on the device (max|d| and 1 - F) or, for the q=34 shard, sampled
amplitudes against the CPU oracle (done in the -m gpu tests, not here). "cfg5_q34_n2_c2_shard8" runs exactly one
GPU's share of the 8-GPU q=34 job (rows [0, 2^17/8) of the output).
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2603_01443_b200 as cb  # noqa: E402
from paper_2603_01443_b200 import engine  # noqa: E402
from paper_2603_01443_b200.merging import merge_chain_device  # noqa: E402
from paper_2603_01443_b200.pipeline import preprocess, simulate_segments  # noqa: E402

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0


def ev():
    return torch.cuda.Event(enable_timing=True)


def run(name, shard=1, steps=5):
    spec = cb.BASELINE_CONFIGS[name]
    circ = cb.build_brickwall(spec)
    q = spec.q
    prep = preprocess(circ, spec.n)
    ws_bytes, bond, qlow = prep.chain.plan()
    total = 1 << q
    end = total // shard
    out = torch.empty(end, dtype=torch.complex128, device="cuda")
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device="cuda")
    rec = {"config": name, "q": q, "n": spec.n, "c_total": spec.c_total, "d": spec.d, "bond": bond,
           "gates": circ.gate_count, "shard": f"1/{shard}", "out_bytes": end * 16}
    pre, sub, mer = [], [], []
    for i in range(steps + 2):
        t0 = time.perf_counter()
        p = preprocess(circ, spec.n)
        t_pre = time.perf_counter() - t0
        e0, e1, e2 = ev(), ev(), ev()
        e0.record()
        batches = simulate_segments(p)
        e1.record()
        merge_chain_device(p.chain, batches, out=out, out_range=(0, end), workspace=ws)
        e2.record()
        e2.synchronize()
        if i >= 2:
            pre.append(t_pre * 1e3)
            sub.append(e0.elapsed_time(e1))
            mer.append(e1.elapsed_time(e2))
    rec["stage_ms"] = {"pre": float(np.median(pre)), "sub": float(np.median(sub)),
                       "merge": float(np.median(mer))}
    fams = p.subs.segments
    in_bytes = sum(f.num_variants * (1 << f.num_qubits) * 16 for f in fams)
    merge_gbs = (16 * end + in_bytes) / (np.median(mer) * 1e-3) / 1e9
    rec["merge_GBps"] = merge_gbs
    rec["merge_frac_of_measured_hbm"] = merge_gbs / PEAK
    cut_ms = sum(rec["stage_ms"].values())
    rec["cut_amplitudes_per_s"] = end / (cut_ms * 1e-3)
    free = torch.cuda.mem_get_info()[0]
    if shard == 1 and free > total * 16 * 1.1:
        cut_sv = cb.StateVec(q, device=out)
        cb.simulate(circ, max_qubits=q)
        torch.cuda.synchronize()
        u0, u1 = ev(), ev()
        u0.record()
        uncut = cb.simulate(circ, max_qubits=q)
        u1.record()
        u1.synchronize()
        rec["uncut_ms"] = u0.elapsed_time(u1)
        rec["speedup_cut_vs_uncut"] = rec["uncut_ms"] / cut_ms
        rec["max_abs_diff_cut_vs_uncut"] = engine.max_abs_diff(cut_sv, uncut)
        re, im = engine.inner(uncut, cut_sv)
        n1, n2 = engine.inner(cut_sv, cut_sv)[0], engine.inner(uncut, uncut)[0]
        rec["one_minus_fidelity"] = 1 - (re * re + im * im) / (n1 * n2)
        del uncut
    else:
        rec["check"] = "see tests/test_gpu_parity.py::test_q34_shard_sampled_vs_oracle"
    del out, ws
    torch.cuda.empty_cache()
    return rec


def main():
    from paper_2603_01443_b200 import _native

    _native.set_option("jit", 2)
    names = sys.argv[1:] or ["cfg1", "cfg2", "cfg4a", "cfg4b", "cfg5_q32_n2_c2", "cfg5_q32_n2_c4",
                             "cfg5_q32_n4_c4", "cfg5_q34_n2_c2_shard8"]
    for name in names:
        shard = 1
        if name.endswith("_shard8"):
            name, shard = name[: -len("_shard8")], 8
        print(json.dumps(run(name, shard)), flush=True)


if __name__ == "__main__":
    main()
