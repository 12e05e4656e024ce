"""One int8 merge product at q=30 (for ncu --set full): K terms, digit base.
   python tools/ozaki_one.py K DIGITS"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_01443_b200 import _native  # noqa: E402
from paper_2603_01443_b200.merging import merge_terms_device  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 16
_native.set_option("merge_ozaki_digits", int(sys.argv[2]) if len(sys.argv) > 2 else 8)
q = 30
out = torch.empty(1 << q, dtype=torch.complex128, device="cuda")
g = torch.Generator(device="cuda").manual_seed(0)
hi = torch.randn(K, 1 << 15, dtype=torch.complex128, device="cuda", generator=g)
lo = torch.randn(K, 1 << 15, dtype=torch.complex128, device="cuda", generator=g)
idx = np.arange(K)
for _ in range(2):
    merge_terms_device(hi, lo, idx, idx, np.ones(K), out=out.view(1, -1))
torch.cuda.synchronize()
print("ok")
