"""The int8 tensor-core merge (csrc/ozaki.cu: tcgen05.mma kind::i8, exact
FP64 splitting into 7 base-256 digits by default, or 8 base-128 digits) against numpy and against the FP64
DFMA kernel: every instantiated K (16, 32, 64) and chunked K (48, 128, 200),
row ranges (output shards), several slots, accumulate, all-zero and badly
scaled rows, ineligible shapes falling back to the FP64 kernels, and a
q=28 product. Tolerance: the FP64 kernels' own bound, |err| <= 1e-13 *
max|out| * K / 16 (measured: 1-2e-16 relative, below the 3M kernel's)."""
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


def run(torch, native, hi, lo, hidx, lidx, coef, S=1, rows=None, ozaki=1, out=None, accumulate=False, digits=8):
    from paper_2603_01443_b200.merging import merge_terms_device

    old = native.get_option("merge_ozaki"), native.get_option("merge_ozaki_digits"), \
        native.get_option("merge_ozaki_min_work")
    native.set_option("merge_ozaki", ozaki)
    native.set_option("merge_ozaki_digits", digits)
    native.set_option("merge_ozaki_min_work", 0)  # these products are small: take the int8 kernel anyway
    try:
        res = merge_terms_device(torch.as_tensor(hi, device="cuda"), torch.as_tensor(lo, device="cuda"),
                                 hidx, lidx, coef, S=S, rows=rows, out=out, accumulate=accumulate)
        torch.cuda.synchronize()
        return res
    finally:
        native.set_option("merge_ozaki", old[0])
        native.set_option("merge_ozaki_digits", old[1])
        native.set_option("merge_ozaki_min_work", old[2])


CASES = [  # (K, S, H, W, rows)
    (16, 1, 64, 256, None), (32, 1, 32, 128, None), (64, 1, 48, 512, None), (16, 2, 64, 128, (16, 48)),
    (48, 1, 32, 256, None), (128, 1, 16, 128, None), (200, 1, 16, 128, None), (64, 3, 32, 256, (0, 16)),
]


@pytest.mark.parametrize("digits", [8, 7], ids=["base256", "base128"])
@pytest.mark.parametrize("mode", [3, 2, 1], ids=["persistent", "unit-ctas", "auto"])
@pytest.mark.parametrize("K,S,H,W,rows", CASES)
def test_ozaki_vs_numpy_and_dfma(dev, K, S, H, W, rows, mode, digits):
    torch, native = dev
    rng = np.random.default_rng(K * 7 + W)
    nh = nl = max(2, K)
    hi = rng.normal(size=(nh, H)) + 1j * rng.normal(size=(nh, H))
    lo = rng.normal(size=(nl, W)) + 1j * rng.normal(size=(nl, W))
    hi[:, 3] = 0.0                 # an all-zero h row
    lo[:, 7] *= 1e-30              # a tiny l row
    lo[1:, 9] *= 1e-9              # a row whose entries span 9 decades
    hidx = rng.integers(0, nh, size=S * K)
    lidx = rng.integers(0, nl, size=S * K)
    coef = rng.normal(size=S * K) + 1j * rng.normal(size=S * K)
    rows = rows or (0, H)
    want = reference(hi, lo, hidx, lidx, coef, S, rows)
    n0 = native.launch_count()
    got = run(torch, native, hi, lo, hidx, lidx, coef, S=S, rows=rows, ozaki=mode, digits=digits).cpu().numpy()
    launches = native.launch_count() - n0
    dfma = run(torch, native, hi, lo, hidx, lidx, coef, S=S, rows=rows, ozaki=0).cpu().numpy()
    scale = np.abs(want).max()
    tol = 1e-13 * scale * max(1, K / 16)
    assert np.abs(got - want).max() <= tol
    assert np.abs(got - dfma).max() <= tol
    # the truncation level of the digit scheme: 2^-55 of max|a| max|b| per
    # kept diagonal (base 128) / 2^-49 (base 256), measured here against numpy
    term = np.abs(lo).max() * np.abs(hi).max() * np.abs(coef).max()
    assert np.abs(got - want).max() <= (4e-14 if digits == 8 else 1e-14) * term * max(1, K / 16)
    # the tiny row keeps its own relative accuracy (per-row power-of-two scaling)
    w2 = want.reshape(S, rows[1] - rows[0], W)
    g2 = got.reshape(S, rows[1] - rows[0], W)
    assert np.abs(g2[..., 7] - w2[..., 7]).max() <= 1e-13 * np.abs(w2[..., 7]).max() * max(1, K / 16)
    # one product = 3 launches (two digit-preparation kernels + the tcgen05 kernel) per slot and chunk
    chunks = {16: 1, 32: 1, 64: 1, 48: 2, 128: 2, 200: 5}[K]
    assert launches >= 3 * S * min(chunks, 2)


@pytest.mark.parametrize("mode", [3, 2, 1], ids=["persistent", "unit-ctas", "auto"])
def test_ozaki_accumulate(dev, mode):
    torch, native = dev
    rng = np.random.default_rng(5)
    K, H, W = 32, 32, 256
    hi = rng.normal(size=(K, H)) + 1j * rng.normal(size=(K, H))
    lo = rng.normal(size=(K, W)) + 1j * rng.normal(size=(K, W))
    idx = np.arange(K)
    coef = np.exp(1j * np.arange(K))
    base = rng.normal(size=(1, H * W)) + 1j * rng.normal(size=(1, H * W))
    out = torch.as_tensor(base.copy(), device="cuda")
    run(torch, native, hi, lo, idx, idx, coef, out=out, accumulate=True, ozaki=mode)
    want = base + reference(hi, lo, idx, idx, coef, 1, (0, H))
    assert np.abs(out.cpu().numpy() - want).max() < 1e-12


@pytest.mark.parametrize("H,W,rows", [(64, 64, None), (40, 256, None), (64, 256, (3, 40))])
def test_ineligible_shapes_fall_back(dev, H, W, rows):
    """lo_len not a multiple of 128 or a row range not a multiple of 16: the
    FP64 kernels run (one launch) and the result is the same."""
    torch, native = dev
    rng = np.random.default_rng(11)
    K = 16
    hi = rng.normal(size=(K, H)) + 1j * rng.normal(size=(K, H))
    lo = rng.normal(size=(K, W)) + 1j * rng.normal(size=(K, W))
    idx = np.arange(K)
    coef = np.ones(K)
    rows = rows or (0, H)
    n0 = native.launch_count()
    got = run(torch, native, hi, lo, idx, idx, coef, rows=rows).cpu().numpy()
    assert native.launch_count() - n0 == 1
    want = reference(hi, lo, idx, idx, coef, 1, rows)
    assert np.abs(got - want).max() <= 1e-13 * np.abs(want).max()


@pytest.mark.parametrize("mode", [3, 2, 1], ids=["persistent", "unit-ctas", "auto"])
def test_ozaki_large_product_vs_dfma(dev, mode):
    """q = 28 (14 | 14), K = 16: 4 GiB state, every tile of a full-size grid."""
    torch, native = dev
    g = torch.Generator(device="cuda").manual_seed(0)
    K = 16
    hi = torch.randn(K, 1 << 14, dtype=torch.complex128, device="cuda", generator=g)
    lo = torch.randn(K, 1 << 14, dtype=torch.complex128, device="cuda", generator=g)
    idx = np.arange(K)
    coef = np.exp(1j * np.arange(K)) / 4
    from paper_2603_01443_b200.merging import merge_terms_device

    old = native.get_option("merge_ozaki")
    native.set_option("merge_ozaki", mode)
    a = merge_terms_device(hi, lo, idx, idx, coef)
    native.set_option("merge_ozaki", 0)
    try:
        b = merge_terms_device(hi, lo, idx, idx, coef)
    finally:
        native.set_option("merge_ozaki", old)
    torch.cuda.synchronize()
    diff = (a - b).abs().max().item()
    scale = b.abs().max().item()
    assert diff <= 1e-15 * scale * K, (diff, scale)


@pytest.mark.parametrize("mode", [3, 2, 1], ids=["persistent", "unit-ctas", "auto"])
def test_ozaki_propagates_non_finite(dev, mode):
    """A NaN or Inf operand gives NaN outputs in its row/column (as the FP64
    kernels do), never a finite value made of saturated digits."""
    torch, native = dev
    rng = np.random.default_rng(3)
    K, H, W = 16, 32, 256
    hi = rng.normal(size=(K, H)) + 1j * rng.normal(size=(K, H))
    lo = rng.normal(size=(K, W)) + 1j * rng.normal(size=(K, W))
    lo[2, 5] = np.nan
    hi[4, 9] = np.inf
    idx = np.arange(K)
    coef = np.ones(K)
    got = run(torch, native, hi, lo, idx, idx, coef, ozaki=mode).cpu().numpy().reshape(H, W)
    assert np.isnan(got[:, 5]).all() and np.isnan(got[9, :]).all()
    mask = np.ones((H, W), bool)
    mask[:, 5] = False
    mask[9, :] = False
    assert np.isfinite(got[mask]).all()
    want = reference(hi, lo, idx, idx, coef, 1, (0, H)).reshape(H, W)
    assert np.abs(got[mask] - want[mask]).max() <= 1e-13 * np.abs(want[mask]).max()


def test_out_buffers_are_validated_before_native_calls(dev):
    """a wrong dtype / length / non-contiguous ``out`` raises
    ValidationError instead of letting a kernel write past the buffer."""
    torch, native = dev
    from paper_2603_01443_b200 import BrickwallSpec, build_brickwall, run_cut
    from paper_2603_01443_b200.errors import ValidationError
    from paper_2603_01443_b200.merging import merge_terms_device

    hi = torch.zeros(2, 16, dtype=torch.complex128, device="cuda")
    lo = torch.zeros(2, 128, dtype=torch.complex128, device="cuda")
    idx = np.arange(2)
    for bad in (torch.zeros(16 * 128, dtype=torch.complex64, device="cuda"),
                torch.zeros(16 * 128 - 1, dtype=torch.complex128, device="cuda"),
                torch.zeros(2 * 16 * 128, dtype=torch.complex128, device="cuda")[::2],
                torch.zeros(16 * 128, dtype=torch.complex128)):
        with pytest.raises(ValidationError):
            merge_terms_device(hi, lo, idx, idx, np.ones(2), out=bad)
    with pytest.raises(ValidationError):
        merge_terms_device(hi.to(torch.complex64), lo, idx, idx, np.ones(2))
    circ = build_brickwall(BrickwallSpec(8, 2, 2, 1, 0))
    for bad in (torch.zeros(256, dtype=torch.float64, device="cuda"),
                torch.zeros(128, dtype=torch.complex128, device="cuda")):
        with pytest.raises(ValidationError):
            run_cut(circ, 2, out=bad)
    from paper_2603_01443_b200.pipeline import run_cut_to_host

    with pytest.raises(ValidationError):
        run_cut_to_host(circ, 2, torch.zeros(256, dtype=torch.float64).view(torch.complex64))


def test_apply_gate_updates_a_held_host_array(dev):
    """Reference engine.py:171-181: apply_gate mutates the state in place, so
    an ``amps`` array obtained earlier sees the new amplitudes."""
    import paper_2603_01443_b200 as cb
    from paper_2603_01443_b200.circuits import h, x

    sv = cb.StateVec.zero_state(3)
    a = sv.amps
    cb.apply_gate(sv, h(0))
    r = 0.7071067811865475
    assert np.allclose(a, [r, r, 0, 0, 0, 0, 0, 0])
    b = sv.amps
    assert b is a
    from paper_2603_01443_b200.engine import apply_circuit

    apply_circuit(sv, cb.Circuit(3, (h(0), x(2))))
    assert np.allclose(a, [0, 0, 0, 0, 1, 0, 0, 0])
