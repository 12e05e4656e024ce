"""Merge kernels at small q (the threshold-study sizes): rank-K product into
2^q outputs, int8 tcgen05 (merge_ozaki=1/2) vs FP64 (merge_ozaki=0, the
DMMA/3M or DFMA kernel the library picks), event-timed per call incl. the
digit-prep launches.   python tools/merge_small_q.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_01443_b200 import _native  # noqa: E402
from paper_2603_01443_b200.merging import merge_terms_device  # noqa: E402


def timed(fn, reps=50):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps * 1e3


for q in (20, 22, 24, 26, 28):
    out = torch.empty(1 << q, dtype=torch.complex128, device="cuda")
    g = torch.Generator(device="cuda").manual_seed(0)
    row = []
    for K in (4, 8, 16, 32, 64):
        hi = torch.randn(K, 1 << (q - q // 2), dtype=torch.complex128, device="cuda", generator=g)
        lo = torch.randn(K, 1 << (q // 2), dtype=torch.complex128, device="cuda", generator=g)
        idx = np.arange(K)
        coef = np.ones(K)
        res = []
        for oz in (0, 1, 2):
            _native.set_option("merge_ozaki", oz)
            _native.set_option("merge_ozaki_min_k", 8)
            res.append(timed(lambda: merge_terms_device(hi, lo, idx, idx, coef, out=out.view(1, -1))))
        row.append(f"K={K}: fp64 {res[0]:.0f} / int8 {res[1]:.0f} / int8-unit {res[2]:.0f} us")
    _native.set_option("merge_ozaki", 1)
    _native.set_option("merge_ozaki_min_k", 16)
    floor = 16 * (1 << q) / 6455.6e9 * 1e6
    print(f"q={q} (HBM floor {floor:.0f} us) | " + " | ".join(row), flush=True)
