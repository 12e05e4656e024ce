"""Host-time split of the drop-in API's family simulation at q=16 (the
reference suite's t_sub < t_orig law): Python argument preparation, the
cs_sim_families call, StateVec rows, and the launches it makes; against the
uncut simulate.   python tools/sub_host_split.py [c]"""
import gc
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2603_01443_b200 as cb  # noqa: E402
from paper_2603_01443_b200 import _device, _native, harness  # noqa: E402
from paper_2603_01443_b200.engine import StateVec  # noqa: E402

c = int(sys.argv[1]) if len(sys.argv) > 1 else 2
circ = harness.build(cb.BenchmarkSpec(q=16, n=2, blocks=c))
subs = cb.decompose(circ, cb.plan_cut(circ, 2))
fams = subs.segments
t = _device.torch()
lib = _native.load()


def split():
    nt = fams[0]._src[0]
    t0 = time.perf_counter_ns()
    outs = [t.empty((f.num_variants, 1 << f.num_qubits), dtype=t.complex128, device="cuda") for f in fams]
    t1 = time.perf_counter_ns()
    _cuts, _counts, k, a, b, p, sl, _cid = nt
    nq = np.array([f.num_qubits for f in fams], np.int32)
    gcn = np.array([f._src[2] for f in fams], np.int64)
    ns = np.array([f.num_variants for f in fams], np.int64)
    ptrs = np.array([o.data_ptr() for o in outs], np.uint64)
    ptr = _native.ptr
    args = (len(fams), ptr(nq), ptr(gcn), ptr(k), ptr(a), ptr(b), ptr(p), ptr(sl), ptr(ptrs), ptr(ns), 0,
            _device.stream_ptr())
    t2 = time.perf_counter_ns()
    n0 = _native.launch_count()
    rc = lib.cs_sim_families(*args)
    t3 = time.perf_counter_ns()
    nl = _native.launch_count() - n0
    assert rc == 0
    rows = [[StateVec.batch_row(f.num_qubits, o, v, np.complex128) for v in range(f.num_variants)]
            for f, o in zip(fams, outs)]
    t4 = time.perf_counter_ns()
    harness._sync()
    t5 = time.perf_counter_ns()
    del rows
    return np.array([t1 - t0, t2 - t1, t3 - t2, t4 - t3, t5 - t4, t5 - t0]) / 1e3, nl


def orig():
    t0 = time.perf_counter_ns()
    n0 = _native.launch_count()
    s = cb.simulate(circ)
    t1 = time.perf_counter_ns()
    nl = _native.launch_count() - n0
    harness._sync()
    t2 = time.perf_counter_ns()
    del s
    return np.array([t1 - t0, t2 - t1, t2 - t0]) / 1e3, nl


for _ in range(5):
    split()
    orig()
for collect in (False, True):
    a = []
    b = []
    for _ in range(40):
        harness._sync()
        r, nl = split()
        a.append(r)
        if collect:
            gc.collect()
        harness._sync()
        r2, nl2 = orig()
        b.append(r2)
        if collect:
            gc.collect()
    print(f"gc={collect} sub: empty/prep/native/rows/sync/total median us {np.median(a, axis=0).round(1)} launches {nl}")
    print(f"gc={collect} orig: call/sync/total median us {np.median(b, axis=0).round(1)} launches {nl2}", flush=True)
for jit in (0, 3):
    _native.set_option("jit", jit)
    for _ in range(5):
        split()
        orig()
    time.sleep(2)
    _native.jit_wait()
    a = [split()[0] for _ in range(30)]
    b = [orig()[0] for _ in range(30)]
    print(f"jit={jit}: sub {np.median(a, axis=0).round(1)} orig {np.median(b, axis=0).round(1)}", flush=True)
