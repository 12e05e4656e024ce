"""merge kernels (cs_merge_terms: DFMA and FP64-tensor-core DMMA variants)
against a plain numpy evaluation of out[s,h,l] = sum_t coef[s,t] hi[hidx][h] lo[lidx][l]
on random inputs: every K width incl. chunked K > 16 and non powers of two,
narrow and wide rows, row ranges, several slots, accumulate, complex64."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2603_01443_b200 import _native

    return torch, _native


def reference(hi, lo, hidx, lidx, coef, S, rows):
    K = len(hidx) // S
    r0, r1 = rows
    out = []
    for s in range(S):
        acc = np.zeros((r1 - r0, lo.shape[1]), np.complex128)
        for t in range(K):
            i = s * K + t
            acc += coef[i] * np.multiply.outer(hi[hidx[i], r0:r1], lo[lidx[i]])
        out.append(acc.ravel())
    return np.stack(out)


CASES = [  # (K, S, H, W, rows)
    (1, 1, 64, 256, None), (2, 1, 32, 8, None), (4, 1, 128, 4096, None), (4, 3, 16, 64, None),
    (8, 1, 256, 1024, None), (8, 2, 64, 256, (5, 60)), (16, 1, 128, 512, None), (16, 2, 40, 128, (3, 37)),
    (12, 1, 64, 256, None), (32, 1, 32, 128, None), (64, 1, 16, 256, None), (3, 1, 8, 2, None),
    (16, 1, 64, 2, None), (8, 1, 100, 4, None),
    # wide enough for the pipelined 3M kernel (16 warps x 16 / 8 columns), ragged rows
    (16, 2, 40, 256, (3, 37)), (32, 1, 20, 256, None), (8, 3, 24, 512, (1, 23)), (16, 1, 700, 512, None),
]


@pytest.mark.parametrize("dmma", [2, 1, 0])
@pytest.mark.parametrize("K,S,H,W,rows", CASES)
def test_merge_terms_vs_numpy(dev, K, S, H, W, rows, dmma):
    """The FP64 kernels (the int8 tensor-core path is switched off here and
    tested in test_gpu_ozaki.py)."""
    torch, native = dev
    from paper_2603_01443_b200.merging import merge_terms_device

    old_oz = native.get_option("merge_ozaki")
    native.set_option("merge_ozaki", 0)
    rng = np.random.default_rng(K * 1000 + W)
    nh, nl = max(2, K), max(2, K)
    hi = rng.normal(size=(nh, H)) + 1j * rng.normal(size=(nh, H))
    lo = rng.normal(size=(nl, W)) + 1j * rng.normal(size=(nl, W))
    hidx = rng.integers(0, nh, size=S * K)
    lidx = rng.integers(0, nl, size=S * K)
    coef = rng.normal(size=S * K) + 1j * rng.normal(size=S * K)
    rows = rows or (0, H)
    want = reference(hi, lo, hidx, lidx, coef, S, rows)
    old = native.get_option("merge_dmma")
    native.set_option("merge_dmma", dmma)
    try:
        got = merge_terms_device(torch.as_tensor(hi, device="cuda"), torch.as_tensor(lo, device="cuda"),
                                 hidx, lidx, coef, S=S, rows=rows).cpu().numpy()
    finally:
        native.set_option("merge_dmma", old)
        native.set_option("merge_ozaki", old_oz)
    scale = np.abs(want).max()
    assert np.abs(got - want).max() <= 1e-13 * max(1.0, scale) * K


def test_merge_accumulate_and_complex64(dev):
    torch, native = dev
    from paper_2603_01443_b200.merging import merge_terms_device

    rng = np.random.default_rng(3)
    hi = rng.normal(size=(8, 64)) + 1j * rng.normal(size=(8, 64))
    lo = rng.normal(size=(8, 512)) + 1j * rng.normal(size=(8, 512))
    idx = np.arange(8)
    coef = np.exp(1j * np.arange(8))
    base = rng.normal(size=(1, 64 * 512)) + 1j * rng.normal(size=(1, 64 * 512))
    out = torch.as_tensor(base.copy(), device="cuda")
    merge_terms_device(torch.as_tensor(hi, device="cuda"), torch.as_tensor(lo, device="cuda"), idx, idx, coef,
                       out=out, accumulate=True)
    want = base + reference(hi, lo, idx, idx, coef, 1, (0, 64))
    assert np.abs(out.cpu().numpy() - want).max() < 1e-12
    h32 = torch.as_tensor(hi.astype(np.complex64), device="cuda")
    l32 = torch.as_tensor(lo.astype(np.complex64), device="cuda")
    got = merge_terms_device(h32, l32, idx, idx, coef, dtype=np.complex64).cpu().numpy()
    assert got.dtype == np.complex64
    assert np.abs(got - reference(hi, lo, idx, idx, coef, 1, (0, 64))).max() < 1e-4


def test_dmma_kernel_is_used(dev):
    """The K=16 complex128 product goes through the tensor-core kernel (the
    library counts launches; the SASS check lives in profiles/)."""
    torch, native = dev
    from paper_2603_01443_b200.merging import merge_terms_device

    hi = torch.ones(16, 32, dtype=torch.complex128, device="cuda")
    lo = torch.ones(16, 256, dtype=torch.complex128, device="cuda")
    idx = np.arange(16)
    old = native.get_option("merge_ozaki")
    native.set_option("merge_ozaki", 0)
    try:
        n0 = native.launch_count()
        out = merge_terms_device(hi, lo, idx, idx, np.ones(16))
        assert native.launch_count() == n0 + 1
    finally:
        native.set_option("merge_ozaki", old)
    assert float(out.real.max().item()) == 16.0
