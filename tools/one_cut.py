import sys, torch
sys.path.insert(0, '.')
import paper_2603_01443_b200 as cb
from paper_2603_01443_b200 import _native
_native.set_option("jit", 3)
_native.set_option("cluster_loop", int(sys.argv[1]) if len(sys.argv) > 1 else 1)
spec = cb.BASELINE_CONFIGS["cfg4a"]
circ = cb.build_brickwall(spec)
out = torch.empty(1 << spec.q, dtype=torch.complex128, device="cuda")
for _ in range(3):
    cb.run_cut(circ, spec.n, out=out, max_qubits=spec.q)
    torch.cuda.synchronize()
    _native.jit_wait(600)
