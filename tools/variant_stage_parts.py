"""Where the variant stage's time goes (cfg4a by default): event-timed device
time of one family batch alone, both families back to back on one stream, and
both through cs_sim_families (side streams, fork/join events).
    python tools/variant_stage_parts.py [workload]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_01443_b200 as cb  # noqa: E402
from paper_2603_01443_b200 import _native  # noqa: E402
from paper_2603_01443_b200.cutting import decompose, plan_cut  # noqa: E402
from paper_2603_01443_b200.engine import simulate_family  # noqa: E402
from paper_2603_01443_b200.pipeline import simulate_families  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4a"
_native.set_option("jit", 2)
spec = cb.BASELINE_CONFIGS[name]
circ = cb.build_brickwall(spec)
subs = decompose(circ, plan_cut(circ, spec.n))
fams = subs.segments


FILL = torch.empty(1 << 31, dtype=torch.uint8, device="cuda")


def timed(fn, reps=30, filler="sleep"):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        # a long-running filler first so the host launches are queued ahead
        # of the timed work: an idle spin, or a 2 GiB HBM write (as the merge
        # of the previous cut leaves the L2 full of dirty lines)
        if filler == "sleep":
            torch.cuda._sleep(200000)
        else:
            FILL.fill_(1)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return np.median(ts), min(ts)


for filler in ("sleep", "hbm-write"):
    for label, fn in (("family 0 alone", lambda: simulate_family(fams[0])),
                      ("family 1 alone", lambda: simulate_family(fams[1])),
                      ("both, one stream", lambda: [simulate_family(f) for f in fams]),
                      ("both, cs_sim_families", lambda: simulate_families(fams))):
        med, mn = timed(fn, filler=filler)
        print(f"{name} after {filler:9s} {label:24s} median {med:6.1f} us  min {mn:6.1f} us", flush=True)
