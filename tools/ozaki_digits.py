"""int8 tcgen05 merge: base-256 (7 diagonals) vs base-128 (8 diagonals) digit
schemes at q=30 (and q=32 K=16): time per product and max|d| vs the FP64
DFMA/3M kernels.   python tools/ozaki_digits.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_01443_b200 import _native  # noqa: E402
from paper_2603_01443_b200.merging import merge_terms_device  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


for q, Ks in ((30, (16, 32, 64)), (32, (16,))):
    out = torch.empty(1 << q, dtype=torch.complex128, device="cuda")
    g = torch.Generator(device="cuda").manual_seed(0)
    for K in Ks:
        hi = torch.randn(K, 1 << (q - q // 2), dtype=torch.complex128, device="cuda", generator=g) / 4
        lo = torch.randn(K, 1 << (q // 2), dtype=torch.complex128, device="cuda", generator=g) / 4
        idx = np.arange(K)
        coef = np.exp(1j * np.arange(K)) / np.sqrt(K)
        res = {}
        ref = None
        for name, oz, dig in (("fp64", 0, 8), ("int8_base128", 1, 7), ("int8_base256", 1, 8)):
            _native.set_option("merge_ozaki", oz)
            _native.set_option("merge_ozaki_digits", dig)
            ms = timed(lambda: merge_terms_device(hi, lo, idx, idx, coef, out=out.view(1, -1)))
            if ref is None:
                ref = out[: 1 << 26].clone()
                err = 0.0
            else:
                err = (out[: 1 << 26] - ref).abs().max().item() / ref.abs().max().item()
            res[name] = (ms, err)
        _native.set_option("merge_ozaki", 1)
        _native.set_option("merge_ozaki_digits", 8)
        floor = 16.0 * (1 << q) / 6548.2e9 * 1e3
        print(f"q={q} K={K} HBM floor {floor:.2f} ms | " + " | ".join(
            f"{k}: {v[0]:.3f} ms ({floor / v[0] * 100:.0f}% HBM) rel.err {v[1]:.1e}" for k, v in res.items()),
            flush=True)
        del hi, lo
    del out
    torch.cuda.empty_cache()
