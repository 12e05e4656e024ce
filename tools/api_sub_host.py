"""Host time per call of the variant stage entry points (no sync between
calls): cs_sim_families through pipeline.simulate_families, and the same
launches inside cs_cut_run.   python tools/api_sub_host.py [q] [c] [d]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2603_01443_b200 as cb  # noqa: E402
from paper_2603_01443_b200 import _native  # noqa: E402
from paper_2603_01443_b200.cutting import decompose, plan_cut  # noqa: E402
from paper_2603_01443_b200.pipeline import run_cut, simulate_families  # noqa: E402

q = int(sys.argv[1]) if len(sys.argv) > 1 else 24
c = int(sys.argv[2]) if len(sys.argv) > 2 else 4
d = int(sys.argv[3]) if len(sys.argv) > 3 else 10
jit = int(sys.argv[4]) if len(sys.argv) > 4 else 2
_native.set_option("jit", jit)
circ = cb.build_brickwall(cb.BrickwallSpec(q, d, 2, c, 0))
subs = decompose(circ, plan_cut(circ, 2))
for name, fn in (("simulate_families", lambda: simulate_families(subs.segments)),
                 ("run_cut (whole pipeline)", lambda: run_cut(circ, 2))):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(100):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{name:26s} host {1e6 * (t1 - t0) / 100:6.1f} us/call, with device drain {1e6 * (t2 - t0) / 100:6.1f} us/call")

# the native entry alone (prepared ctypes arguments, no Python wrapper)
import numpy as np  # noqa: E402

fams = subs.segments
nt = fams[0]._src[0]
_cuts, _counts, k, a, b, p, sl, _cid = nt
outs = [torch.empty((f.num_variants, 1 << f.num_qubits), dtype=torch.complex128, device="cuda") for f in fams]
ptr = _native.ptr
nq = np.array([f.num_qubits for f in fams], np.int32)
gcn = np.array([f._src[2] for f in fams], np.int64)
ns = np.array([f.num_variants for f in fams], np.int64)
ptrs = np.array([o.data_ptr() for o in outs], np.uint64)
args = (len(fams), ptr(nq), ptr(gcn), ptr(k), ptr(a), ptr(b), ptr(p), ptr(sl), ptr(ptrs), ptr(ns), 0, None)
lib = _native.load()
for name, fn in (("cs_sim_families (2 fams)", lambda: lib.cs_sim_families(*args)),
                 ("cs_sim_families (1 fam)", lambda: lib.cs_sim_families(1, *args[1:]))):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(200):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"{name:26s} host {1e6 * (t1 - t0) / 200:6.1f} us/call")
