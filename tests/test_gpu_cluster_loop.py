"""The ahead-of-time cluster-resident op-stream kernel (cluster.cu, option
cluster_loop = 2 forces it; the default runs it only while a new program's
NVRTC cluster kernel compiles) against the CPU oracle: every subcircuit
variant of 12..15-qubit segment families (cluster sizes 2..16, RB = 2 and 3),
cut slots, CX-controlled ops (staircase), complex64 (RB = 4), and the full
cut pipeline at q=30 sampled against the oracle's merged amplitudes."""
import numpy as np
import pytest

from oracle import cutbench_oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture
def cb():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_01443_b200 as pkg
    from paper_2603_01443_b200 import _native

    old = (_native.get_option("jit"), _native.get_option("cluster_loop"))
    _native.set_option("jit", 3)
    _native.set_option("cluster_loop", 2)
    yield pkg
    _native.set_option("jit", old[0])
    _native.set_option("cluster_loop", old[1])


def family_states(cb, circ, n, dtype):
    """Every segment family of ``circ`` simulated by the library (one batched
    call per family) and by the oracle, per variant."""
    from paper_2603_01443_b200 import _native
    from paper_2603_01443_b200.engine import simulate_family
    from paper_2603_01443_b200.pipeline import preprocess

    q = circ.num_qubits
    sizes = [q // n] * n
    k, qa, qb, p = circ.kinds, circ.qa, circ.qb, circ.params
    bgs, _, _ = orc.plan(k, qa, qb, sizes)
    prep = preprocess(circ, n)
    launches0 = _native.launch_count()
    out = []
    for s, fam in enumerate(prep.subs.segments):
        got = simulate_family(fam, dtype=dtype).cpu().numpy()
        want = [orc.simulate(sizes[s], *v) for v in orc.segment_variants(k, qa, qb, p, sizes, bgs, s)]
        out.append((got, np.stack(want)))
    return out, _native.launch_count() - launches0


@pytest.mark.parametrize("q,d,n,c,seed", [(24, 6, 2, 3, 1), (26, 5, 2, 4, 2), (28, 4, 2, 2, 3),
                                          (30, 10, 2, 2, 0), (39, 5, 3, 4, 4)])
def test_cluster_loop_families_match_oracle(cb, q, d, n, c, seed):
    circ = cb.build_brickwall(cb.BrickwallSpec(q, d, n, c, seed))
    fams, launches = family_states(cb, circ, n, np.complex128)
    for got, want in fams:
        assert got.shape == want.shape
        assert np.abs(got - want).max() < 1e-12
    assert launches == n  # one cluster kernel per family


def test_cluster_loop_controlled_gates(cb):
    circ = cb.build_staircase(cb.BenchmarkSpec(q=28, n=2, blocks=2))
    fams, _ = family_states(cb, circ, 2, np.complex128)
    for got, want in fams:
        assert np.abs(got - want).max() < 1e-12


def test_cluster_loop_complex64(cb):
    circ = cb.build_brickwall(cb.BrickwallSpec(28, 6, 2, 3, 5))
    fams, _ = family_states(cb, circ, 2, np.complex64)
    for got, want in fams:
        assert np.abs(got - want).max() < 1e-5


def test_cluster_loop_cut_pipeline_q30(cb):
    """The one-call pipeline (cs_cut_run) on cfg4a with the op-stream kernel
    against 4096 oracle-merged amplitudes, and against the NVRTC cluster
    kernel's result."""
    import torch

    from paper_2603_01443_b200 import _native

    spec = cb.BASELINE_CONFIGS["cfg4a"]
    circ = cb.build_brickwall(spec)
    q = spec.q
    out = torch.empty(1 << q, dtype=torch.complex128, device="cuda")
    cb.run_cut(circ, spec.n, out=out, max_qubits=q)
    rng = np.random.default_rng(11)
    idx = np.sort(rng.choice(1 << q, 4096, replace=False))
    got = out[torch.from_numpy(idx).cuda()].cpu().numpy()
    sizes = [q // spec.n] * spec.n
    k, qa, qb, p = circ.kinds, circ.qa, circ.qb, circ.params
    bgs, counts, _ = orc.plan(k, qa, qb, sizes)
    states = [[orc.simulate(sizes[s], *v) for v in orc.segment_variants(k, qa, qb, p, sizes, bgs, s)]
              for s in range(spec.n)]
    want = orc.sample_amplitudes(states, orc.merge_table(spec.n, bgs, sum(counts)), orc.coefficients(sum(counts)),
                                 sizes, idx)
    assert np.abs(got - want).max() < 1e-10
    _native.set_option("cluster_loop", 0)
    _native.set_option("jit", 2)
    ref = torch.empty_like(out)
    cb.run_cut(circ, spec.n, out=ref, max_qubits=q)
    assert (out - ref).abs().max().item() < 1e-15
