"""TEST INFRASTRUCTURE ONLY — the CPU oracle for the circuit-cutting path.

This package restates the reference algorithm (`cutbench`,
/root/reference/pkg/src/cutbench) on the CPU so the sm_100a product can be
checked against it. Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` legs may import it; the product package
never does (a test enforces that).

Pinning: `tests/golden/make_golden.py` runs the real reference in the build
container and commits its outputs as fixtures; `tests/test_oracle_golden.py`
checks this oracle against them (parity pinned for the reference gate set and
the cut tables; the U3 kernel is pinned by the dense-unitary oracle, the
linearity identity, term-replacement factorisation and cut == uncut).
"""
