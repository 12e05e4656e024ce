"""Per-repetition merge/sub stage samples of harness.measure at small q
(diagnostic of host-side noise):  python tools/diag_measure.py [JIT]"""
import sys
sys.path.insert(0, ".")
import paper_2603_01443_b200 as cb
from paper_2603_01443_b200 import _native, harness
_native.set_option("jit", int(sys.argv[1]) if len(sys.argv) > 1 else 2)
for q, c in [(24, 1), (24, 3), (20, 2), (16, 5)]:
    spec = cb.BrickwallSpec(q, 10, 2, c, 0)
    tb = harness.measure(spec, 5)
    print(q, c, [round(x * 1e3, 3) for x in tb.samples["merge"]], [round(x * 1e3, 3) for x in tb.samples["sub"]], flush=True)
