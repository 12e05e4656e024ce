"""One rank-K merge product at 2^q outputs (for ncu launch lists):
    python tools/merge_one.py q K [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_01443_b200.merging import merge_terms_device  # noqa: E402

q, K = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
out = torch.empty(1 << q, dtype=torch.complex128, device="cuda")
g = torch.Generator(device="cuda").manual_seed(0)
hi = torch.randn(K, 1 << (q - q // 2), dtype=torch.complex128, device="cuda", generator=g)
lo = torch.randn(K, 1 << (q // 2), dtype=torch.complex128, device="cuda", generator=g)
idx = np.arange(K)
for _ in range(reps):
    merge_terms_device(hi, lo, idx, idx, np.ones(K), out=out.view(1, -1))
torch.cuda.synchronize()
print("ok")
