"""Where the host-side time of merge() goes (diagnostic): per-rep timings of
merge_input_from, mem_get_info, segment batches, the chain merge call and the
sync, for the staircase/brick-wall merge at small q."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2603_01443_b200 as cb  # noqa: E402
from paper_2603_01443_b200 import merging  # noqa: E402

q, c = (int(v) for v in sys.argv[1:3]) if len(sys.argv) > 2 else (20, 2)
circ = cb.build_brickwall(cb.BrickwallSpec(q, 10, 2, c, 0))
subs = cb.decompose(circ, cb.plan_cut(circ, 2))
fams = [cb.simulate_family(f) for f in subs.segments]
states = [[cb.StateVec(f.num_qubits, device=b[v]) for v in range(f.num_variants)]
          for f, b in zip(subs.segments, fams)]
for rep in range(12):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    mi = cb.merge_input_from(subs, states)
    t.append(time.perf_counter())
    torch.cuda.mem_get_info()
    t.append(time.perf_counter())
    batches = [merging.segment_batch(s, mi.segment_states[0][0].amps_dtype if hasattr(mi.segment_states[0][0], "amps_dtype") else __import__("numpy").complex128) for s in mi.segment_states]
    t.append(time.perf_counter())
    res = merging.merge_chain_device(mi.chain, batches)
    t.append(time.perf_counter())
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    del res
    print(rep, " ".join(f"{(b - a) * 1e3:.3f}" for a, b in zip(t, t[1:])), flush=True)
