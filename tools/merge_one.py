"""One merge_terms product (n = 2 shape) for profiling a single launch:
    python tools/merge_one.py Q K MERGE_DMMA [REPS]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2603_01443_b200 import _native  # noqa: E402
from paper_2603_01443_b200.merging import merge_terms_device  # noqa: E402

q, K, mode = (int(v) for v in sys.argv[1:4])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
_native.set_option("merge_dmma", mode)
half = q // 2
hi = torch.randn(K, 1 << (q - half), dtype=torch.complex128, device="cuda") / 4
lo = torch.randn(K, 1 << half, dtype=torch.complex128, device="cuda") / 4
out = torch.empty(1, 1 << q, dtype=torch.complex128, device="cuda")
idx = np.arange(K)
coef = np.exp(1j * np.arange(K)) / np.sqrt(K)
for _ in range(reps):
    merge_terms_device(hi, lo, idx, idx, coef, out=out)
torch.cuda.synchronize()
print("ok", q, K, mode)
