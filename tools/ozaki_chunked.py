import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2603_01443_b200 import _native
from paper_2603_01443_b200.merging import merge_terms_device
q = 30; half = 15
for K in (128, 256):
    hi = torch.randn(K, 1 << half, dtype=torch.complex128, device='cuda') / 4
    lo = torch.randn(K, 1 << half, dtype=torch.complex128, device='cuda') / 4
    out = torch.empty(1, 1 << q, dtype=torch.complex128, device='cuda')
    idx = np.arange(K); coef = np.exp(1j * np.arange(K)) / np.sqrt(K)
    res = {}
    for oz in (1, 0):
        _native.set_option('merge_ozaki', oz)
        for _ in range(2): merge_terms_device(hi, lo, idx, idx, coef, out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3): merge_terms_device(hi, lo, idx, idx, coef, out=out)
        e1.record(); e1.synchronize()
        res[oz] = (e0.elapsed_time(e1) / 3, out.clone() if oz == 1 else None)
        if oz == 0:
            d = (res[1][1] - out).abs().max().item()
    _native.set_option('merge_ozaki', 1)
    print(f"K={K}: int8 {res[1][0]:.2f} ms, fp64 3M {res[0][0]:.2f} ms, max|d| {d:.2e}", flush=True)
    del hi, lo, out, res; torch.cuda.empty_cache()
