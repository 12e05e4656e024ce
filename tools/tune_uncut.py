"""Time the uncut simulator under different sweep-kernel settings."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2603_01443_b200 as cb  # noqa: E402
from paper_2603_01443_b200 import _native  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4a"
circ = cb.build_brickwall(cb.BASELINE_CONFIGS[name])
q = circ.num_qubits
for minb in (2, 3, 4):
    for tb in (10, 11, 12):
        _native.set_option("sweep_minb", minb)
        _native.set_option("tile_bits", tb)
        try:
            sv = cb.simulate(circ, max_qubits=q)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            sv = cb.simulate(circ, max_qubits=q)
            e1.record()
            e1.synchronize()
            print(f"{name} minb={minb} tile_bits={tb}: {e0.elapsed_time(e1):.1f} ms", flush=True)
            del sv
        except Exception as exc:  # noqa: BLE001
            print(f"{name} minb={minb} tile_bits={tb}: ERR {exc}", flush=True)
