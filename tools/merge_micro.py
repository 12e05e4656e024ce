"""Merge kernel throughput vs K (terms) on synthetic n=2 inputs, 2^q output."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2603_01443_b200.merging import merge_terms_device  # noqa: E402

q = int(sys.argv[1]) if len(sys.argv) > 1 else 30
half = q // 2
peak = 6538.3
for K in (1, 2, 4, 8, 16, 32, 64):
    hi = torch.randn(K, 1 << (q - half), dtype=torch.complex128, device="cuda")
    lo = torch.randn(K, 1 << half, dtype=torch.complex128, device="cuda")
    out = torch.empty(1, 1 << q, dtype=torch.complex128, device="cuda")
    idx = np.arange(K)
    coef = np.exp(1j * np.arange(K))
    for _ in range(2):
        merge_terms_device(hi, lo, idx, idx, coef, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 5
    e0.record()
    for _ in range(n):
        merge_terms_device(hi, lo, idx, idx, coef, out=out)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / n
    gbs = (16 << q) / ms / 1e6
    tflops = 8 * K * (1 << q) / ms / 1e9
    print(f"q={q} K={K}: {ms:.3f} ms  {gbs:.0f} GB/s ({gbs / peak:.2f} of copy peak)  {tflops:.1f} FP64 TFLOP/s",
          flush=True)
    del hi, lo, out
