import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2603_01443_b200 import _native
from paper_2603_01443_b200.merging import merge_terms_device
for K in (16, 64):
  for q in range(20, 31, 2):
    half = q // 2
    hi = torch.randn(K, 1 << (q - half), dtype=torch.complex128, device='cuda') / 4
    lo = torch.randn(K, 1 << half, dtype=torch.complex128, device='cuda') / 4
    out = torch.empty(1, 1 << q, dtype=torch.complex128, device='cuda')
    idx = np.arange(K); coef = np.exp(1j * np.arange(K)) / np.sqrt(K)
    res = []
    for oz in (1, 0):
        _native.set_option('merge_ozaki', oz)
        for _ in range(3): merge_terms_device(hi, lo, idx, idx, coef, out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10): merge_terms_device(hi, lo, idx, idx, coef, out=out)
        e1.record(); e1.synchronize()
        res.append(e0.elapsed_time(e1) / 10)
    _native.set_option('merge_ozaki', 1)
    print(f"K={K} q={q}: ozaki {res[0]*1e3:9.1f} us   fp64 {res[1]*1e3:9.1f} us", flush=True)
