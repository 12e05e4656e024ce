"""Do the FP64 vector (DFMA) and FP64 tensor (DMMA) pipes add up? The K-term
merge at q=30 split by rows between the DFMA kernel (merge_dmma=0) and the
3M tensor kernel (merge_dmma=2) on two streams, vs each alone.
    python tools/dual_pipe.py [K]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2603_01443_b200 import _native  # noqa: E402
from paper_2603_01443_b200.merging import merge_terms_device  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 16
q = 30
H = W = 1 << 15
hi = torch.randn(K, H, dtype=torch.complex128, device="cuda") / 4
lo = torch.randn(K, W, dtype=torch.complex128, device="cuda") / 4
out = torch.empty(1, 1 << q, dtype=torch.complex128, device="cuda")
idx = np.arange(K)
coef = np.exp(1j * np.arange(K)) / np.sqrt(K)
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()


def run(split):
    r = int(H * split) // 64 * 64
    ev = torch.cuda.Event()
    ev.record()
    sa.wait_event(ev)
    sb.wait_event(ev)
    if r > 0:
        _native.set_option("merge_dmma", 2)
        with torch.cuda.stream(sa):
            merge_terms_device(hi, lo, idx, idx, coef, out=out[:, : r * W], rows=(0, r), stream=sa)
    if r < H:
        _native.set_option("merge_dmma", 0)
        with torch.cuda.stream(sb):
            merge_terms_device(hi, lo, idx, idx, coef, out=out[:, r * W:], rows=(r, H), stream=sb)
    torch.cuda.current_stream().wait_stream(sa)
    torch.cuda.current_stream().wait_stream(sb)


for split in (1.0, 0.0, 0.8, 0.7, 0.6, 0.5):
    for _ in range(2):
        run(split)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        run(split)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"K={K} dmma-share={split:.1f}: {ms:.3f} ms  {8 * K * (1 << q) / ms / 1e9:.1f} TF/s(alg)", flush=True)
_native.set_option("merge_dmma", 2)
