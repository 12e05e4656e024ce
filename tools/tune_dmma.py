"""Tensor-core merge staging budget (merge_smem_kb) x variant (merge_dmma 1/2, 3M warps 8/4)
at q=30 for K = 16, 32:  python tools/tune_dmma.py"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2603_01443_b200 import _native  # noqa: E402
from paper_2603_01443_b200.merging import merge_terms_device  # noqa: E402

q = 30
for K in (16, 32):
    hi = torch.randn(K, 1 << 15, dtype=torch.complex128, device="cuda") / 4
    lo = torch.randn(K, 1 << 15, dtype=torch.complex128, device="cuda") / 4
    out = torch.empty(1, 1 << q, dtype=torch.complex128, device="cuda")
    idx = np.arange(K)
    coef = np.exp(1j * np.arange(K)) / np.sqrt(K)
    for mode, warps in ((1, 8), (2, 8), (2, 4)):
        for kb in (48, 64, 96, 112):
            _native.set_option("merge_dmma", mode)
            _native.set_option("merge_dmma3_warps", warps)
            _native.set_option("merge_smem_kb", kb)
            merge_terms_device(hi, lo, idx, idx, coef, out=out)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                merge_terms_device(hi, lo, idx, idx, coef, out=out)
            e1.record()
            e1.synchronize()
            ms = e0.elapsed_time(e1) / 5
            print(f"K={K} mode={mode} warps={warps} smem_kb={kb}: {ms:.3f} ms  {8 * K * (1 << q) / ms / 1e9:.1f} TF/s(alg)",
                  flush=True)
