"""int8 tensor-core merge: persistent (merge_ozaki=1) vs short-lived unit CTAs
(merge_ozaki=2) for K = 16, 32 at q (default 30): time and max |diff| vs DFMA.
    python tools/ozaki_unit.py [q]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2603_01443_b200 import _native  # noqa: E402
from paper_2603_01443_b200.merging import merge_terms_device  # noqa: E402

q = int(sys.argv[1]) if len(sys.argv) > 1 else 30
half = q // 2
g = torch.Generator(device="cuda").manual_seed(0)
_native.set_option("merge_ozaki_min_k", 8)
for K in (8, 16, 32, 64):
    hi = torch.randn(K, 1 << (q - half), dtype=torch.complex128, device="cuda", generator=g) / 4
    lo = torch.randn(K, 1 << half, dtype=torch.complex128, device="cuda", generator=g) / 4
    out = torch.empty(1, 1 << q, dtype=torch.complex128, device="cuda")
    idx = np.arange(K)
    coef = np.exp(1j * np.arange(K)) / np.sqrt(K)
    ref = None
    for mode in (0, 1, 2):
        _native.set_option("merge_ozaki", mode)
        _native.set_option("merge_dmma", 0 if mode == 0 else 2)
        for _ in range(2):
            merge_terms_device(hi, lo, idx, idx, coef, out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            merge_terms_device(hi, lo, idx, idx, coef, out=out)
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / 5
        if mode == 0:
            ref = out.clone() if q <= 30 else None
            diff = 0.0
        else:
            diff = (out - ref).abs().max().item() if ref is not None else float("nan")
        print(f"q={q} K={K} merge_ozaki={mode}: {ms:.3f} ms {(16 << q) / ms / 1e6:.0f} GB/s max|d| {diff:.2e}",
              flush=True)
    del hi, lo, out, ref
    torch.cuda.empty_cache()
_native.set_option("merge_ozaki", 1)
_native.set_option("merge_ozaki_min_k", 16)
_native.set_option("merge_dmma", 2)
