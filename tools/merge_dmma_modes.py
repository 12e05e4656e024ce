"""Tensor-core merge variants at q (default 30/32): DFMA (merge_dmma=0), four
real GEMMs (1), three real GEMMs / 3M (2) for K = 8, 16, 32, 64 — time, the
achieved algorithmic FP64 rate (8 K flops per complex output for every
variant, so 3M can exceed the tensor peak) and max |diff| vs the DFMA result.

    python tools/merge_dmma_modes.py 30
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2603_01443_b200 import _native  # noqa: E402
from paper_2603_01443_b200.merging import merge_terms_device  # noqa: E402

q = int(sys.argv[1]) if len(sys.argv) > 1 else 30
half = q // 2
g = torch.Generator(device="cuda").manual_seed(0)
for K in (8, 16, 32, 64):
    hi = torch.randn(K, 1 << (q - half), dtype=torch.complex128, device="cuda", generator=g) / 4
    lo = torch.randn(K, 1 << half, dtype=torch.complex128, device="cuda", generator=g) / 4
    out = torch.empty(1, 1 << q, dtype=torch.complex128, device="cuda")
    ref = None
    idx = np.arange(K)
    coef = np.exp(1j * np.arange(K)) / np.sqrt(K)
    for mode in (0, 1, 2):
        _native.set_option("merge_dmma", mode)
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
        if mode == 0:
            ref = out.clone() if q <= 31 else out.cpu()
            diff = 0.0
        else:
            diff = max((out[0, i:i + (1 << 26)].to(ref.device) - ref[0, i:i + (1 << 26)]).abs().max().item()
                       for i in range(0, 1 << q, 1 << 26))
        tf = 8 * K * (1 << q) / ms / 1e9
        print(f"q={q} K={K} mode={mode}: {ms:.3f} ms  {(16 << q) / ms / 1e6:.0f} GB/s  {tf:.1f} TF/s(alg)  "
              f"maxdiff={diff:.2e}", flush=True)
    del hi, lo, out, ref
    torch.cuda.empty_cache()
_native.set_option("merge_dmma", 1)
