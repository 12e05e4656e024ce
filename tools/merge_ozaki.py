"""int8 tcgen05 (Ozaki) merge vs the FP64 kernels: correctness against numpy at
small q, then time and max |diff| vs the DFMA kernel at q (default 30) for
K = 8, 16, 32, 64 (merge_ozaki on/off, merge_dmma 0 = DFMA, 2 = 3M).

    python tools/merge_ozaki.py 30
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2603_01443_b200 import _native  # noqa: E402
from paper_2603_01443_b200.merging import merge_terms_device  # noqa: E402


def modes(name):
    return {"dfma": (0, 0), "3m": (0, 2), "ozaki": (1, 2)}[name]


def set_mode(name):
    oz, dm = modes(name)
    _native.set_option("merge_ozaki", oz)
    _native.set_option("merge_ozaki_min_k", 8)
    _native.set_option("merge_dmma", dm)


# small-q check against numpy (every K, a row range, accumulate)
rng = np.random.default_rng(1)
for K in (8, 16, 32, 64):
    qh, ql = 6, 8
    hi = (rng.standard_normal((K, 1 << qh)) + 1j * rng.standard_normal((K, 1 << qh))) / 4
    lo = (rng.standard_normal((K, 1 << ql)) + 1j * rng.standard_normal((K, 1 << ql))) / 4
    hi[:, 3] = 0  # an all-zero row
    lo[2:, 5] *= 1e-9  # a badly scaled row
    coef = np.exp(1j * np.arange(K)) / np.sqrt(K)
    idx = np.arange(K)
    ref = np.einsum("t,th,tl->hl", coef, hi, lo).reshape(-1)
    set_mode("ozaki")
    out = torch.empty(1, 1 << (qh + ql), dtype=torch.complex128, device="cuda")
    merge_terms_device(torch.from_numpy(hi).cuda(), torch.from_numpy(lo).cuda(), idx, idx, coef, out=out)
    got = out.cpu().numpy().reshape(-1)
    err = np.abs(got - ref).max() / np.abs(ref).max()
    print(f"small K={K}: max rel err {err:.2e} (row 5 rel err "
          f"{np.abs(got.reshape(64, 256)[:, 5] - ref.reshape(64, 256)[:, 5]).max() / np.abs(ref.reshape(64, 256)[:, 5]).max():.2e})",
          flush=True)
    assert err < 1e-14, err

q = int(sys.argv[1]) if len(sys.argv) > 1 else 30
half = q // 2
g = torch.Generator(device="cuda").manual_seed(0)
for K in (8, 16, 32, 64):
    hi = torch.randn(K, 1 << (q - half), dtype=torch.complex128, device="cuda", generator=g) / 4
    lo = torch.randn(K, 1 << half, dtype=torch.complex128, device="cuda", generator=g) / 4
    out = torch.empty(1, 1 << q, dtype=torch.complex128, device="cuda")
    idx = np.arange(K)
    coef = np.exp(1j * np.arange(K)) / np.sqrt(K)
    ref = None
    for name in ("dfma", "3m", "ozaki"):
        set_mode(name)
        for _ in range(2):
            merge_terms_device(hi, lo, idx, idx, coef, out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 5
        e0.record()
        for _ in range(n):
            merge_terms_device(hi, lo, idx, idx, coef, out=out)
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / n
        if name == "dfma":
            ref = out.clone() if q <= 31 else out.cpu()
            diff = 0.0
            scale = max(out[0, i:i + (1 << 26)].abs().max().item() for i in range(0, 1 << q, 1 << 26))
        else:
            diff = max((out[0, i:i + (1 << 26)].to(ref.device) - ref[0, i:i + (1 << 26)]).abs().max().item()
                       for i in range(0, 1 << q, 1 << 26))
        print(f"q={q} K={K} {name:5s}: {ms:7.3f} ms  {(16 << q) / ms / 1e6:5.0f} GB/s  "
              f"{8 * K * (1 << q) / ms / 1e9:5.1f} TF/s(alg)  max|d|={diff:.2e} (max|out| {scale:.2e})", flush=True)
    del hi, lo, out, ref
    torch.cuda.empty_cache()
