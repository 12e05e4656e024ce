"""int8 tcgen05 merge epilogue forms: merge_ozaki_epi = 1 (output exponent in
the int64 -> double bias, 3 DADD per real output) vs 0 (fma + power-of-two
DMUL), both digit bases, q=30 K=16/32/64 and q=32 K=16: time per product and
max|d| vs the FP64 3M kernel.   python tools/ozaki_epi.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_01443_b200 import _native  # noqa: E402
from paper_2603_01443_b200.merging import merge_terms_device  # noqa: E402


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


peak = 6455.6e9
for q, Ks in ((30, (16, 32, 64)), (32, (16,))):
    out = torch.empty(1 << q, dtype=torch.complex128, device="cuda")
    g = torch.Generator(device="cuda").manual_seed(0)
    for K in Ks:
        hi = torch.randn(K, 1 << (q - q // 2), dtype=torch.complex128, device="cuda", generator=g) / 4
        lo = torch.randn(K, 1 << (q // 2), dtype=torch.complex128, device="cuda", generator=g) / 4
        idx = np.arange(K)
        coef = np.exp(1j * np.arange(K)) / np.sqrt(K)
        _native.set_option("merge_ozaki", 0)
        merge_terms_device(hi, lo, idx, idx, coef, out=out.view(1, -1))
        ref = out[: 1 << 26].clone()
        _native.set_option("merge_ozaki", 1)
        res = []
        for dig in (7, 8):
            for epi in (0, 1):
                _native.set_option("merge_ozaki_digits", dig)
                _native.set_option("merge_ozaki_epi", epi)
                ms = timed(lambda: merge_terms_device(hi, lo, idx, idx, coef, out=out.view(1, -1)))
                err = (out[: 1 << 26] - ref).abs().max().item() / ref.abs().max().item()
                res.append(f"base{1 << dig} epi{epi}: {ms:.3f} ms ({16 * (1 << q) / peak * 1e3 / ms * 100:.1f}%) err {err:.1e}")
        _native.set_option("merge_ozaki_digits", 7)
        _native.set_option("merge_ozaki_epi", 1)
        print(f"q={q} K={K} | " + " | ".join(res), flush=True)
        del hi, lo
    del out
    torch.cuda.empty_cache()
