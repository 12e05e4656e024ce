"""Device plumbing: PyTorch is used only to own CUDA memory and streams.

Tensors are allocated through torch's caching allocator and handed to the
C-ABI as raw pointers with the current torch stream. Nothing here computes.
"""
from __future__ import annotations

import numpy as np

from . import _native
from .errors import CapacityError, NativeUnavailableError, ValidationError

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as _t  # noqa: PLC0415  (heavy import, done lazily)

        _torch = _t
    return _torch


_CUDA_OK = False


def require_cuda():
    global _CUDA_OK
    t = torch()
    if _CUDA_OK:  # a visible device stays visible for the life of the process
        return t
    if not t.cuda.is_available():
        raise NativeUnavailableError(
            "no CUDA device is visible; the cut pipeline runs only on the sm_100a kernels "
            "(there is no CPU fallback)"
        )
    _native.load()
    _CUDA_OK = True
    return t


def code_of(dtype) -> int:
    dt = np.dtype(dtype)
    if dt == np.complex128:
        return _native.CS_C128
    if dt == np.complex64:
        return _native.CS_C64
    raise ValidationError(f"dtype must be complex128 or complex64, got {dt}")


def torch_dtype(dtype):
    t = torch()
    return t.complex128 if np.dtype(dtype) == np.complex128 else t.complex64


def stream_ptr(stream=None) -> int:
    if stream is not None:
        return int(stream.cuda_stream)
    # torch's current stream of the current device without building a Stream
    # object (the API path calls this per native call)
    t = torch()
    return int(t._C._cuda_getCurrentRawStream(t._C._cuda_getDevice()))


_TOTAL = {}


def _total_memory() -> int:
    t = torch()
    dev = t.cuda.current_device()
    if dev not in _TOTAL:
        _TOTAL[dev] = int(t.cuda.get_device_properties(dev).total_memory)
    return _TOTAL[dev]


def check_free(nbytes: int, what: str) -> None:
    """CapacityError if an allocation of nbytes cannot fit on the device.
    cudaMemGetInfo costs 0.3-10 ms per call (measured on the B200 box), so it
    is only consulted for allocations of 1 GiB or more that exceed half of
    what this process leaves of the device; smaller ones rely on torch's own
    out-of-memory error."""
    if nbytes < (1 << 30):
        return
    t = torch()
    # cheap bound first: device capacity minus what this process holds
    total = _total_memory()
    if nbytes < 0.5 * (total - t.cuda.memory_allocated()):
        return
    free, _total = t.cuda.mem_get_info()
    cached = t.cuda.memory_reserved() - t.cuda.memory_allocated()
    if nbytes > free + cached:
        raise CapacityError(f"{what} needs {nbytes / 2**30:.2f} GiB; "
                            f"{(free + cached) / 2**30:.2f} GiB free on the device")


def check_out(out, n_amps: int, dtype, what: str = "out", *, device: str = "cuda"):
    """Validate a caller-provided result buffer BEFORE its pointer reaches
    native code: a torch tensor on ``device`` of exactly ``n_amps`` elements
    of ``dtype``, contiguous. The kernels write n_amps * itemsize bytes, so a
    smaller or differently typed buffer would be written past its end."""
    t = torch()
    if not isinstance(out, t.Tensor):
        raise ValidationError(f"{what} must be a torch tensor, got {type(out).__name__}")
    if out.device.type != device:
        raise ValidationError(f"{what} must live on {device}, got {out.device}")
    if out.dtype != torch_dtype(dtype):
        raise ValidationError(f"{what} has dtype {out.dtype}, expected {torch_dtype(dtype)}")
    if out.numel() != n_amps:
        raise ValidationError(f"{what} has {out.numel()} elements, expected {n_amps}")
    if not out.is_contiguous():
        raise ValidationError(f"{what} must be contiguous")
    return out


def empty(n_states: int, nq: int, dtype=np.complex128, check_memory=True):
    """Uninitialised device batch [n_states, 2^nq]."""
    t = require_cuda()
    nbytes = n_states * (1 << nq) * np.dtype(dtype).itemsize
    if check_memory:
        check_free(nbytes, f"{n_states} state(s) of {nq} qubits")
    return t.empty((n_states, 1 << nq), dtype=torch_dtype(dtype), device="cuda")


def empty_shape(shape, dtype=np.complex128):
    """Uninitialised device tensor of an arbitrary shape (no capacity check)."""
    t = require_cuda()
    return t.empty(shape, dtype=torch_dtype(dtype), device="cuda")


def from_host(arr: np.ndarray, dtype=None):
    t = require_cuda()
    a = np.ascontiguousarray(arr, dtype=dtype or arr.dtype)
    return t.from_numpy(a).to("cuda", non_blocking=False)


_STAGED_MIN_BYTES = 16 << 20


def to_host(tensor, out: np.ndarray | None = None) -> np.ndarray:
    """Device tensor -> host numpy array (``out`` if given). Large contiguous
    copies go through libcutsim's cs_copy_to_host: pinned staging ring plus
    host copy threads for pageable destinations (the driver's own pageable
    path runs at ~20 GB/s)."""
    t = torch()
    tc = tensor.detach()
    nbytes = tc.numel() * tc.element_size()
    npdt = {t.complex128: np.complex128, t.complex64: np.complex64, t.float64: np.float64,
            t.float32: np.float32, t.uint8: np.uint8}.get(tc.dtype)
    if (npdt is not None and tc.is_cuda and tc.is_contiguous() and nbytes >= _STAGED_MIN_BYTES
            and (out is None or (out.flags.c_contiguous and out.nbytes == nbytes and out.flags.writeable
                                 and out.dtype == npdt))):
        host = out.reshape(-1) if out is not None else np.empty(tc.numel(), dtype=npdt)
        _native.check(_native.load().cs_copy_to_host(host.ctypes.data, tc.data_ptr(), nbytes, stream_ptr()),
                      "cs_copy_to_host")
        return out if out is not None else host.reshape(tuple(tc.shape))
    if out is not None:
        host = t.from_numpy(out.reshape(-1))
        host.copy_(tc.reshape(-1))
        return out
    return tc.cpu().numpy()
