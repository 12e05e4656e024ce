"""Sustained cfg4a steps: per-block step time over ~100 steps, a 3 s pause,
then more blocks; with the SM/memory clocks and throttle reasons sampled by
NVML in each block.   python tools/step_drift.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2603_01443_b200 as cb  # noqa: E402
from paper_2603_01443_b200 import _native  # noqa: E402

try:
    import pynvml  # noqa: E402

    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
except Exception:  # noqa: BLE001
    h = None


def sample():
    if h is None:
        return ""
    sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
    mem = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM)
    pw = pynvml.nvmlDeviceGetPowerUsage(h) / 1000
    r = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
    return f"sm {sm} MHz mem {mem} MHz {pw:.0f} W reasons 0x{r:x}"


_native.set_option("jit", 3)
spec = cb.BASELINE_CONFIGS["cfg4a"]
circ = cb.build_brickwall(spec)
q = spec.q
ws_bytes, _, _ = _native.cut_workspace(q, circ.table, [q // 2] * 2)
out = torch.empty(1 << q, dtype=torch.complex128, device="cuda")
ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
for _ in range(3):
    cb.run_cut(circ, 2, out=out, workspace=ws, max_qubits=q)
torch.cuda.synchronize()
_native.jit_wait(600)
for phase in ("run", "after 3 s pause"):
    if phase != "run":
        time.sleep(3)
    for blk in range(8):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            cb.run_cut(circ, 2, out=out, workspace=ws, max_qubits=q)
        b.record()
        time.sleep(0.01)
        s = sample()
        torch.cuda.synchronize()
        print(f"{phase} block {blk}: {a.elapsed_time(b) / 10 * 1e3:.1f} us/step  {s}", flush=True)
