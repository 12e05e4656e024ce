import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2603_01443_b200 import _native
from paper_2603_01443_b200.merging import merge_terms_device
for q in (30, 32):
  half = q // 2
  for K in (16,):
    hi = torch.randn(K, 1 << (q - half), dtype=torch.complex128, device='cuda') / 4
    lo = torch.randn(K, 1 << half, dtype=torch.complex128, device='cuda') / 4
    out = torch.empty(1, 1 << q, dtype=torch.complex128, device='cuda')
    idx = np.arange(K); coef = np.exp(1j * np.arange(K)) / np.sqrt(K)
    for oz in (0, 1):
        _native.set_option('merge_ozaki', oz)
        for _ in range(2): merge_terms_device(hi, lo, idx, idx, coef, out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5): merge_terms_device(hi, lo, idx, idx, coef, out=out)
        e1.record(); e1.synchronize()
        print(f"q={q} K={K} ozaki={oz}: {e0.elapsed_time(e1)/5:.3f} ms", flush=True)
    del hi, lo, out; torch.cuda.empty_cache()
