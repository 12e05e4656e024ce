"""Random-configuration parity sweep on the GPU (not part of the test suite):
seeded U3 brick-walls with random (q, n, c_total, d); the one-call cut
pipeline and the drop-in API path against the GPU uncut simulator (every
config) and the CPU oracle (q <= 16). Exercises the int8 merge (K >= 16 on
eligible shapes), chain merges, zero-start tiles and cost-aware schedules.
    python tools/fuzz_parity.py [n_configs] [seed] [max_q]"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2603_01443_b200 as cb  # noqa: E402
from oracle import cutbench_oracle as orc  # noqa: E402
from paper_2603_01443_b200 import _native, engine  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 60
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 2026)
QMAX = int(sys.argv[3]) if len(sys.argv) > 3 else 24
_native.set_option("jit", 2)
worst = 0.0
t0 = time.time()
for i in range(N):
    n = int(rng.choice([2, 2, 3, 4]))
    q = int(rng.integers(max(4, 2 * n), QMAX + 1))
    q -= q % n
    d = int(rng.integers(1, 13))
    c = int(rng.integers(0, 9 if n == 2 else 11))
    seed = int(rng.integers(0, 1000))
    spec = cb.BrickwallSpec(q, d, n, c, seed)
    circ = cb.build_brickwall(spec)
    uncut = cb.simulate(circ)
    cut = cb.run_cut(circ, n)
    e1 = engine.max_abs_diff(cut, uncut)
    plan = cb.plan_cut(circ, n)
    subs = cb.decompose(circ, plan)
    states = [[engine.StateVec(f.num_qubits, device=b) for b in engine.simulate_family(f)] for f in subs.segments]
    api = cb.merge(cb.merge_input_from(subs, states))
    e2 = engine.max_abs_diff(api, uncut)
    e3 = 0.0
    if q <= 16:
        ref = orc.simulate(q, circ.kinds, circ.qa, circ.qb, circ.params)
        e3 = float(np.abs(uncut.amps - ref).max())
    err = max(e1, e2, e3)
    worst = max(worst, err)
    flag = "" if err < 1e-10 else "  <-- FAIL"
    print(f"{i:3d} q={q:2d} n={n} c={c:2d} d={d:2d} seed={seed:3d}: cut {e1:.1e} api {e2:.1e} oracle {e3:.1e}{flag}",
          flush=True)
print(f"worst {worst:.2e} over {N} configs in {time.time() - t0:.0f} s", "OK" if worst < 1e-10 else "FAIL")
