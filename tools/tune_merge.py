"""Merge kernel options at q=30, K=4 (cfg4a shape): streaming stores and row
groups per CTA."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2603_01443_b200 import _native  # noqa: E402
from paper_2603_01443_b200.merging import merge_terms_device  # noqa: E402

q = 30
K = 4
hi = torch.randn(K, 1 << 15, dtype=torch.complex128, device="cuda")
lo = torch.randn(K, 1 << 15, dtype=torch.complex128, device="cuda")
out = torch.empty(1, 1 << q, dtype=torch.complex128, device="cuda")
idx = np.arange(K)
coef = np.exp(1j * np.arange(K))
configs = [(s_, it) for s_ in (1, 0) for it in (0, 8, 16, 32, 64)]
for rnd in range(3):
    for stream, iters in configs:
        _native.set_option("merge_streaming", stream)
        _native.set_option("merge_iters", iters)
        for _ in range(2):
            merge_terms_device(hi, lo, idx, idx, coef, out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            merge_terms_device(hi, lo, idx, idx, coef, out=out)
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / 10
        print(f"round={rnd} streaming={stream} iters={iters}: {ms:.3f} ms {(16 << q) / ms / 1e6:.0f} GB/s",
              flush=True)
