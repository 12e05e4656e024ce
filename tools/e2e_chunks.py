"""e2e leg (run_cut_to_host into pinned memory) vs the number of merge/copy
chunks, cfg4a.   python tools/e2e_chunks.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2603_01443_b200 as cb  # noqa: E402
from paper_2603_01443_b200 import _native  # noqa: E402
from paper_2603_01443_b200.pipeline import host_workspace_bytes, run_cut_to_host  # noqa: E402

_native.set_option("jit", 2)
spec = cb.BASELINE_CONFIGS["cfg4a"]
circ = cb.build_brickwall(spec)
host = torch.empty(1 << 30, dtype=torch.complex128, pin_memory=True)
for chunks in (4, 8, 16, 32, 64):
    ws = torch.empty(host_workspace_bytes(circ, 2, chunks=chunks), dtype=torch.uint8, device="cuda")
    run_cut_to_host(circ, 2, host, workspace=ws, chunks=chunks)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        run_cut_to_host(circ, 2, host, workspace=ws, chunks=chunks)
    torch.cuda.synchronize()
    t = (time.perf_counter() - t0) / 3
    print(f"chunks={chunks}: {t * 1e3:.1f} ms = {16 * (1 << 30) / t / 1e9:.1f} GB/s", flush=True)
    del ws
