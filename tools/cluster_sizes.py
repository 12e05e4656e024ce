"""Variant stage of the cut pipeline (cs_cut_run's sub stage, event-timed)
for cluster_max 4 / 8 / 16 and the per-launch kernels (cluster 0), NVRTC
kernels (jit 2).   python tools/cluster_sizes.py [workload]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_01443_b200 as cb  # noqa: E402
from paper_2603_01443_b200 import _native  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4a"
if len(sys.argv) > 2:
    _native.set_option("reg_bits", int(sys.argv[2]))
_native.set_option("jit", 2)
spec = cb.BASELINE_CONFIGS[name]
circ = cb.build_brickwall(spec)
out = torch.empty(1 << spec.q, dtype=torch.complex128, device="cuda")
for cl, cmax in ((0, 16), (1, 4), (1, 8), (1, 16)):
    _native.set_option("cluster", cl)
    _native.set_option("cluster_max", cmax)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    cb.run_cut(circ, spec.n, out=out, max_qubits=spec.q)
    ts = []
    for _ in range(10):
        cb.run_cut(circ, spec.n, out=out, events=evs, max_qubits=spec.q)
        torch.cuda.synchronize()
        ts.append(evs[0].elapsed_time(evs[1]) * 1e3)
    n0 = _native.launch_count()
    cb.run_cut(circ, spec.n, out=out, max_qubits=spec.q)
    print(f"{name} reg_bits={_native.get_option('reg_bits')} cluster={cl} cluster_max={cmax}: variant stage median {np.median(ts):.1f} us "
          f"(min {min(ts):.1f}), launches/step {_native.launch_count() - n0}", flush=True)
