"""Time the batched subcircuit stage under different tile/vb settings."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2603_01443_b200 as cb  # noqa: E402
from paper_2603_01443_b200 import _native  # noqa: E402
from paper_2603_01443_b200.pipeline import preprocess, simulate_segments  # noqa: E402


def timeit(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / n


for name in sys.argv[1:] or ["cfg4a", "cfg2", "cfg5_q32_n2_c2", "cfg4b"]:
    spec = cb.BASELINE_CONFIGS[name]
    circ = cb.build_brickwall(spec)
    prep = preprocess(circ, spec.n)
    for tb in (0, 8, 9, 10, 11):
        for vb in (0, 1, 2, 4):
            _native.set_option("tile_bits", tb)
            _native.set_option("vb", vb)
            try:
                ms = timeit(lambda: simulate_segments(prep))
            except Exception as exc:  # noqa: BLE001
                print(name, tb, vb, "ERR", exc)
                continue
            print(f"{name} tile_bits={tb} vb={vb}: {ms*1e3:.1f} us", flush=True)
    _native.set_option("tile_bits", 0)
    _native.set_option("vb", 0)
