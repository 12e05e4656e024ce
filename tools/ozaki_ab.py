"""A/B of int8 merge options, interleaved (min over rounds): every combination
of the given options at q=30 K=16/32/64 and q=32 K=16, time per product and
max|d| vs the FP64 3M kernel.
   python tools/ozaki_ab.py merge_ozaki_early=0,1 merge_ozaki_digits=7,8"""
import itertools
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_01443_b200 import _native  # noqa: E402
from paper_2603_01443_b200.merging import merge_terms_device  # noqa: E402

opts = [(a.split("=")[0], [int(v) for v in a.split("=")[1].split(",")]) for a in sys.argv[1:]]
combos = list(itertools.product(*[v for _, v in opts]))
ROUNDS = 3


def timed(fn, reps=8):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


peak = 6455.6e9
CASES = ((30, (16, 32, 64)), (32, (16,)))
if os.environ.get("OZ_CASES"):  # e.g. OZ_CASES="24:16,26:16,28:16"
    CASES = tuple((int(a), (int(b),)) for a, b in (c.split(":") for c in os.environ["OZ_CASES"].split(",")))
for q, Ks in CASES:
    out = torch.empty(1 << q, dtype=torch.complex128, device="cuda")
    g = torch.Generator(device="cuda").manual_seed(0)
    for K in Ks:
        hi = torch.randn(K, 1 << (q - q // 2), dtype=torch.complex128, device="cuda", generator=g) / 4
        lo = torch.randn(K, 1 << (q // 2), dtype=torch.complex128, device="cuda", generator=g) / 4
        idx = np.arange(K)
        coef = np.exp(1j * np.arange(K)) / np.sqrt(K)
        _native.set_option("merge_ozaki", 0)
        merge_terms_device(hi, lo, idx, idx, coef, out=out.view(1, -1))
        ref = out[: 1 << 26].clone()
        _native.set_option("merge_ozaki", 1)
        best = {c: 1e9 for c in combos}
        errs = {}
        for _ in range(ROUNDS):
            for c in combos:
                for (name, _), v in zip(opts, c):
                    _native.set_option(name, v)
                best[c] = min(best[c], timed(lambda: merge_terms_device(hi, lo, idx, idx, coef, out=out.view(1, -1))))
                errs[c] = (out[: 1 << 26] - ref).abs().max().item() / ref.abs().max().item()
        floor = 16 * (1 << q) / peak * 1e3
        print(f"q={q} K={K} | " + " | ".join(
            ",".join(f"{n}={v}" for (n, _), v in zip(opts, c)) + f": {best[c]:.4f} ms ({floor / best[c] * 100:.1f}%) err {errs[c]:.1e}"
            for c in combos), flush=True)
        del hi, lo
    del out
    torch.cuda.empty_cache()
