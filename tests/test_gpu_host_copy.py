"""cs_copy_to_host (libcutsim): device -> host copies through the pinned
staging ring and the host copy threads for pageable destinations, the direct
path for pinned ones; and the pageable run_cut_to_host / StateVec.amps paths
built on it. Every byte is compared with torch's own copy."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch as t

    if not t.cuda.is_available():
        pytest.skip("no CUDA device")
    return t


@pytest.mark.parametrize("nbytes", [1, 4097, (64 << 20) - 8, (64 << 20) + 24, (200 << 20) + 16 * 3])
@pytest.mark.parametrize("pinned", [False, True], ids=["pageable", "pinned"])
def test_copy_to_host_matches_torch(torch, nbytes, pinned):
    from paper_2603_01443_b200 import _device, _native

    g = torch.Generator(device="cuda").manual_seed(nbytes)
    dev = torch.randint(0, 256, (nbytes,), dtype=torch.uint8, device="cuda", generator=g)
    want = dev.cpu().numpy()
    if pinned:
        host_t = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
        host = host_t.numpy()
    else:
        host = np.empty(nbytes, np.uint8)
    host[:] = 0
    _native.check(_native.load().cs_copy_to_host(host.ctypes.data, dev.data_ptr(), nbytes,
                                                 _device.stream_ptr()), "cs_copy_to_host")
    assert np.array_equal(host, want)


def test_copy_to_host_orders_after_queued_work(torch):
    """The staged copy starts after the work queued on the stream (a kernel
    still writing the source when the call is made)."""
    from paper_2603_01443_b200 import _device

    n = 48 << 20
    dev = torch.zeros(n // 16, dtype=torch.complex128, device="cuda")
    torch.cuda._sleep(50_000_000)
    dev.fill_(3 + 4j)
    got = _device.to_host(dev)
    assert got.dtype == np.complex128 and np.all(got == 3 + 4j)


def test_pageable_cut_to_host_and_amps_equal_device_state(torch):
    import paper_2603_01443_b200 as cb
    from paper_2603_01443_b200.pipeline import run_cut_to_host

    circ = cb.build_brickwall(cb.BrickwallSpec(24, 6, 2, 2, 5))
    dev = cb.run_cut(circ, 2)
    ref = dev.device_tensor().cpu().numpy()
    host = np.empty(1 << 24, np.complex128)
    run_cut_to_host(circ, 2, host)
    assert np.array_equal(host, ref)
    amps = dev.amps
    assert amps.flags.writeable and np.array_equal(amps, ref)
