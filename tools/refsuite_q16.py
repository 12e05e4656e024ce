"""The reference suite's t_sub < t_orig law at q=16 (pkg/tests/test_harness.py:258-264)
on the drop-in: measure() repeated, then a cProfile of one sub stage and one
uncut simulate after gc.collect().   python tools/refsuite_q16.py [runs]"""
import cProfile
import gc
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_01443_b200 as cb  # noqa: E402
from paper_2603_01443_b200 import harness  # noqa: E402

runs = int(sys.argv[1]) if len(sys.argv) > 1 else 8
for c in (2, 4, 6):
    rows = []
    for _ in range(runs):
        tb = cb.measure(cb.BenchmarkSpec(q=16, n=2, blocks=c), repetitions=3, discard_warmup=True)
        rows.append((tb.t_sub * 1e6, tb.t_orig * 1e6))
    fails = sum(s >= o for s, o in rows)
    print(f"c={c} fails {fails}/{runs}  (t_sub, t_orig) us: " + " ".join(f"({s:.0f},{o:.0f})" for s, o in rows), flush=True)

circ = harness.build(cb.BenchmarkSpec(q=16, n=2, blocks=2))
plan = cb.plan_cut(circ, 2)
subs = cb.decompose(circ, plan)
from paper_2603_01443_b200.pipeline import simulate_families  # noqa: E402


def sub_stage():
    harness._sync()
    t0 = time.perf_counter()
    b = simulate_families(subs.segments, max_qubits=30)
    t1 = time.perf_counter()
    harness._sync()
    return t1 - t0, time.perf_counter() - t0, b


def orig_stage():
    harness._sync()
    t0 = time.perf_counter()
    s = cb.simulate(circ)
    t1 = time.perf_counter()
    harness._sync()
    return t1 - t0, time.perf_counter() - t0, s


for f in (sub_stage, orig_stage):
    for _ in range(3):
        f()
    for collect in (False, True):
        hs, ts = [], []
        for _ in range(20):
            h, t, r = f()
            del r
            hs.append(h * 1e6)
            ts.append(t * 1e6)
            if collect:
                gc.collect()
        hs.sort()
        ts.sort()
        print(f"{f.__name__} gc={collect}: host-return median {hs[10]:.0f} us, synced median {ts[10]:.0f} us "
              f"(min {ts[0]:.0f}, max {ts[-1]:.0f})", flush=True)
    pr = cProfile.Profile()
    for _ in range(20):
        gc.collect()
        pr.enable()
        f()
        pr.disable()
    pstats.Stats(pr).sort_stats("cumtime").print_stats(14)
