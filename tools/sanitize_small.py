"""Small runs of every hand-written kernel family for compute-sanitizer
(memcheck / racecheck / synccheck), each checked against the oracle:
  compute-sanitizer --tool memcheck python tools/sanitize_small.py
rsweep (register-tile sweeps, interpreter), sweep (shared-memory engine),
merge_kernel (DFMA), merge_dmma3 (FP64 tensor 3M, K=8), ozaki (int8
tcgen05: prep kernels + persistent and unit-CTA merge, both digit bases,
accumulate), NVRTC sweep kernels (value and param mode), the sharded call,
init/reductions/gather."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_01443_b200 as cb  # noqa: E402
from oracle import cutbench_oracle as orc  # noqa: E402
from paper_2603_01443_b200 import _native, engine  # noqa: E402
from paper_2603_01443_b200.merging import merge_terms_device  # noqa: E402
from paper_2603_01443_b200.pipeline import run_cut_sharded_native  # noqa: E402


def check(name, got, circ):
    ref = orc.simulate(circ.num_qubits, circ.kinds, circ.qa, circ.qb, circ.params)
    err = float(np.abs(got - ref).max())
    assert err < 1e-10, (name, err)
    print(f"{name}: max|d| {err:.1e}", flush=True)


c12 = cb.build_brickwall(cb.BrickwallSpec(12, 4, 2, 1, 0))
c14k8 = cb.build_brickwall(cb.BrickwallSpec(14, 4, 2, 3, 1))
c14k16 = cb.build_brickwall(cb.BrickwallSpec(14, 4, 2, 4, 2))
c16 = cb.build_brickwall(cb.BrickwallSpec(16, 4, 2, 2, 3))
for engine_id in (1, 0):
    _native.set_option("engine", engine_id)
    check(f"engine{engine_id} run_cut q12", cb.run_cut(c12, 2).amps, c12)
    check(f"engine{engine_id} simulate q16", cb.simulate(c16).amps, c16)
_native.set_option("engine", 1)
check("merge_dmma3 K=8", cb.run_cut(c14k8, 2).amps, c14k8)
for digits in (8, 7):
    for oz in (1, 2):
        _native.set_option("merge_ozaki_digits", digits)
        _native.set_option("merge_ozaki", oz)
        check(f"ozaki mode{oz} digits{digits} K=16", cb.run_cut(c14k16, 2).amps, c14k16)
_native.set_option("merge_ozaki", 1)
_native.set_option("merge_ozaki_digits", 8)
rng = np.random.default_rng(0)
K, H, W = 96, 32, 256  # chunked K: 64 + 32 with accumulate
hi = rng.normal(size=(K, H)) + 1j * rng.normal(size=(K, H))
lo = rng.normal(size=(K, W)) + 1j * rng.normal(size=(K, W))
idx = np.arange(K)
got = merge_terms_device(torch.as_tensor(hi, device="cuda"), torch.as_tensor(lo, device="cuda"), idx, idx,
                         np.ones(K)).cpu().numpy().reshape(H, W)
want = (hi.T @ lo)
assert np.abs(got - want).max() < 1e-11 * np.abs(want).max(), "ozaki accumulate"
print("ozaki K=96 (accumulate chunk): ok", flush=True)
for js in (1, 2):
    _native.set_option("jit", 2)
    _native.set_option("jit_struct", js)
    check(f"nvrtc jit_struct={js} run_cut q14", cb.run_cut(c14k8, 2).amps, c14k8)
    check(f"nvrtc jit_struct={js} simulate q16", cb.simulate(c16).amps, c16)
_native.set_option("jit", 0)
full = cb.run_cut(c16, 2).amps
sh = run_cut_sharded_native(c16, 2, rank=1, world=2)
assert np.array_equal(sh.amps, full[sh.begin:sh.end])
print("sharded call: ok", flush=True)
sv = cb.simulate(c12)
print("reductions:", engine.max_abs_diff(sv, sv), engine.inner(sv, sv), engine.gather(sv, [0, 5, 7])[:1])
print("SANITIZE RUN OK")
