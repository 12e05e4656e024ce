"""One int8 tcgen05 (Ozaki) merge launch, for ncu: python tools/oz_once.py K q [reps]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2603_01443_b200 import _native  # noqa: E402
from paper_2603_01443_b200.merging import merge_terms_device  # noqa: E402

K, q = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
half = q // 2
g = torch.Generator(device="cuda").manual_seed(0)
hi = torch.randn(K, 1 << (q - half), dtype=torch.complex128, device="cuda", generator=g) / 4
lo = torch.randn(K, 1 << half, dtype=torch.complex128, device="cuda", generator=g) / 4
out = torch.empty(1, 1 << q, dtype=torch.complex128, device="cuda")
_native.set_option("merge_ozaki", 1)
_native.set_option("merge_ozaki_min_k", 8)
idx = np.arange(K)
coef = np.exp(1j * np.arange(K)) / np.sqrt(K)
for _ in range(reps):
    merge_terms_device(hi, lo, idx, idx, coef, out=out)
torch.cuda.synchronize()
print("ok")
