"""Compare sweep engines (0: shared-memory tile, 1: register tile) on the
subcircuit stage and the uncut simulator."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2603_01443_b200 as cb  # noqa: E402
from paper_2603_01443_b200 import _native  # noqa: E402
from paper_2603_01443_b200.pipeline import preprocess, simulate_segments  # noqa: E402


def timeit(fn, n=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / n


for eng in (0, 1):
    _native.set_option("engine", eng)
    for tb in (0, 9, 10, 11, 12):
        _native.set_option("tile_bits", tb)
        for name in ("cfg2", "cfg4a", "cfg4b", "cfg5_q32_n2_c2"):
            spec = cb.BASELINE_CONFIGS[name]
            prep = preprocess(cb.build_brickwall(spec), spec.n)
            print(f"engine={eng} tile_bits={tb} sub {name}: {timeit(lambda: simulate_segments(prep)) * 1e3:.1f} us",
                  flush=True)
    _native.set_option("tile_bits", 0)
    for name in ("cfg2", "cfg4a"):
        circ = cb.build_brickwall(cb.BASELINE_CONFIGS[name])
        ms = timeit(lambda: cb.simulate(circ, max_qubits=circ.num_qubits), n=2)
        print(f"engine={eng} uncut {name}: {ms:.2f} ms", flush=True)
