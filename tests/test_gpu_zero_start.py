"""Zero-start tiles (Sweep::zero_tiles_log2, option zero_start_tiles): from
|0..0> a sweep launches only the tiles an earlier sweep could have made
non-zero, after one zeroing of the states. Results must be bit-identical to
launching every tile, for single states, variant batches (slotted cut
variants) and strided batches whose gaps belong to the caller."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_01443_b200 as cb
    from paper_2603_01443_b200 import _native, engine

    return torch, cb, _native, engine


def both(native, fn, windows=1):
    """fn() with zero-start tiles off and on, the tile-set policy pinned (the
    default cost-aware policy 3 applies only with zero-start tiles, so with
    `windows` = 1 both runs execute the same schedule)."""
    old = native.get_option("zero_start_tiles"), native.get_option("sweep_windows")
    try:
        native.set_option("sweep_windows", windows)
        native.set_option("zero_start_tiles", 0)
        a = fn()
        native.set_option("zero_start_tiles", 1)
        b = fn()
    finally:
        native.set_option("zero_start_tiles", old[0])
        native.set_option("sweep_windows", old[1])
    return a, b


@pytest.mark.parametrize("jit", [0, 2])
@pytest.mark.parametrize("q,d,tile_bits", [(22, 6, 10), (22, 8, 12), (24, 5, 6)])
def test_uncut_bit_identical(env, q, d, tile_bits, jit):
    torch, cb, native, engine = env
    circ = cb.build_brickwall(cb.BrickwallSpec(q, d, 2, 2, 1))
    old = native.get_option("tile_bits"), native.get_option("jit")
    native.set_option("tile_bits", tile_bits)
    native.set_option("jit", jit)
    try:
        a, b = both(native, lambda: engine.simulate(circ).device_tensor().clone())
    finally:
        native.set_option("tile_bits", old[0])
        native.set_option("jit", old[1])
    assert torch.equal(a, b)
    # the default schedule (cost-aware tile sets) agrees to rounding
    c = engine.simulate(circ).device_tensor()
    assert (c - a).abs().max().item() < 1e-12
    from oracle import cutbench_oracle as orc

    if q <= 22:
        ref = orc.simulate(q, circ.kinds, circ.qa, circ.qb, circ.params)
        assert np.abs(b.cpu().numpy() - ref).max() < 1e-10


def test_variant_batch_and_strided_gaps(env):
    torch, cb, native, engine = env
    circ = cb.build_brickwall(cb.BrickwallSpec(36, 4, 2, 6, 0))
    plan = cb.plan_cut(circ, 2)
    fam = cb.decompose(circ, plan).segments[0]  # 18 qubits x 64 variants: above the zero-start size floor
    nq, nv = fam.num_qubits, fam.num_variants
    old = native.get_option("tile_bits")
    native.set_option("tile_bits", 6)  # several sweeps on the 10-qubit segment
    try:
        def run():
            stride = (1 << nq) + 96
            buf = torch.full((nv * stride,), 7.0 + 3.0j, dtype=torch.complex128, device="cuda")
            states = buf.as_strided((nv, 1 << nq), (stride, 1))
            engine.run_table(states, nq, fam.template, slots=fam.slots, init_zero=True)
            torch.cuda.synchronize()
            return buf.cpu().numpy(), stride

        (a, stride), (b, _) = both(native, run)
    finally:
        native.set_option("tile_bits", old)
    assert np.array_equal(a, b)
    gaps = np.concatenate([b[v * stride + (1 << nq):(v + 1) * stride] for v in range(nv)])
    assert np.all(gaps == 7.0 + 3.0j), "zeroing touched the caller's memory between strided states"
    want = engine.simulate_family(fam).cpu().numpy()
    got = np.stack([b[v * stride:v * stride + (1 << nq)] for v in range(nv)])
    assert np.abs(got - want).max() < 1e-12
