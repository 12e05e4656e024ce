"""Native NCCL communicator of the multi-GPU paths (libcutsim's cs_nccl_*,
cs_allgather_states, cs_sendrecv; include/cutsim.h).

`NcclComm.create(rank, world, group)` makes one communicator per process
(one GPU each): rank 0 draws the NCCL unique id in C++, the id travels over
the existing torch.distributed group (any backend), every rank initialises
its communicator on its current device. The reference is single-process
(SURVEY.md §2), so there is no reference counterpart; this carries the one
exchange of the sharded cut pipeline (all-gather of subcircuit variant
states, parallel.run_cut_sharded) and the distributed uncut simulator's
half-shard swaps (distributed.simulate_distributed).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _device, _native


def _nccl_path() -> str | None:
    try:
        import nvidia.nccl

        for base in nvidia.nccl.__path__:
            cand = os.path.join(base, "lib", "libnccl.so.2")
            if os.path.exists(cand):
                return cand
    except ImportError:
        pass
    return None


class NcclComm:
    """One NCCL communicator of `world` ranks, this process being `rank`."""

    def __init__(self, handle: int, rank: int, world: int):
        self.handle = handle
        self.rank = rank
        self.world = world

    @classmethod
    def create(cls, rank: int, world: int, group=None) -> "NcclComm":
        import torch.distributed as dist

        torch = _device.require_cuda()
        lib = _native.load()
        # prefer the libnccl torch ships (already mapped in this process)
        _native.check(lib.cs_nccl_load(_nccl_path().encode() if _nccl_path() else None), "cs_nccl_load")
        uid = np.zeros(128, np.uint8)
        if rank == 0:
            _native.check(lib.cs_nccl_unique_id(_native.ptr(uid)), "cs_nccl_unique_id")
        if world > 1:
            box = [uid.tobytes()]
            dist.broadcast_object_list(box, src=0, group=group)
            uid = np.frombuffer(box[0], np.uint8).copy()
        handle = ctypes.c_void_p()
        _native.check(lib.cs_nccl_comm_init(world, rank, _native.ptr(uid), torch.cuda.current_device(),
                                            ctypes.byref(handle)), "cs_nccl_comm_init")
        return cls(handle.value, rank, world)

    def all_gather(self, recv, send) -> None:
        """recv (one contiguous buffer of world * send.numel() elements) gets
        every rank's `send`, rank-major."""
        nbytes = send.numel() * send.element_size()
        if recv.numel() * recv.element_size() != self.world * nbytes or not recv.is_contiguous():
            raise ValueError("all_gather: recv must be contiguous and hold world * send")
        _native.check(_native.load().cs_allgather_states(self.handle, send.data_ptr(), nbytes, recv.data_ptr(),
                                                         _device.stream_ptr()), "cs_allgather_states")

    def gather_parts(self, parts, send) -> None:
        """dist.all_gather-style entry: `parts` are consecutive equal views of
        one buffer (as gather_states allocates them)."""
        n = send.numel()
        base = parts[0]
        step = n * send.element_size()
        for i, p in enumerate(parts):
            if p.numel() != n or p.data_ptr() != base.data_ptr() + i * step:
                raise ValueError("gather_parts: parts must be consecutive views of one buffer")
        _native.check(_native.load().cs_allgather_states(self.handle, send.data_ptr(), step, base.data_ptr(),
                                                         _device.stream_ptr()), "cs_allgather_states")

    def sendrecv(self, send, recv, peer: int) -> None:
        nbytes = send.numel() * send.element_size()
        if recv.numel() * recv.element_size() != nbytes:
            raise ValueError("sendrecv: send and recv sizes differ")
        _native.check(_native.load().cs_sendrecv(self.handle, send.data_ptr(), recv.data_ptr(), nbytes, peer,
                                                 _device.stream_ptr()), "cs_sendrecv")

    def destroy(self) -> None:
        if self.handle:
            _native.check(_native.load().cs_nccl_comm_destroy(self.handle), "cs_nccl_comm_destroy")
            self.handle = None
