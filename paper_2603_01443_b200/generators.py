"""Seeded U3 brick-wall circuit family of BASELINE.json (frozen here, once).

The reference has no parametrised gates (`circuits.py:25-33`, `SPEC.md:92`), so
this family is defined by this build, following SURVEY.md §8(d):

  rng = numpy.random.default_rng(seed)
  angles first:  u = rng.uniform(size=(d, q, 3));
                 theta = pi*u[...,0], phi = 2pi*u[...,1], lam = 2pi*u[...,2]
  then cuts:     for boundary k ascending: layers_k = sort(rng.integers(0, d, c_k))
  layer L:       U3 on qubits 0..q-1 ascending;
                 CZ(i, i+1) for i = L (mod 2) ascending, only inside a segment;
                 then the layer's boundary CZ(k*s-1, k*s), k ascending,
                 repeated by multiplicity (s = q/n).
  cut split:     c_total over n-1 boundaries as evenly as possible, the
                 remainder going to the lower boundaries ([1,1,0], [2,1,1], ...).

``one_qubit="clifford_t"`` builds the *shadow* of the same circuit: every U3
slot holds a reference gate chosen by floor(4*u[L,i,0]) -> (H, X, T, S). The
shadow runs unmodified through the reference package (parity tier A).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .circuits import (
    KIND_CZ,
    KIND_H,
    KIND_S,
    KIND_T,
    KIND_U3,
    KIND_X,
    Circuit,
    GateTable,
)
from .errors import ValidationError

SHADOW_KINDS = np.array([KIND_H, KIND_X, KIND_T, KIND_S], dtype=np.uint8)


def cut_distribution(n: int, c_total: int) -> list[int]:
    """Cuts per boundary: even split, remainder to the lower boundaries."""
    if n < 2:
        raise ValidationError(f"n must be >= 2, got {n}")
    if c_total < 0:
        raise ValidationError(f"c_total must be >= 0, got {c_total}")
    base, rem = divmod(c_total, n - 1)
    return [base + (1 if k < rem else 0) for k in range(n - 1)]


@dataclass(frozen=True)
class BrickwallSpec:
    q: int
    d: int
    n: int
    c_total: int
    seed: int = 0
    one_qubit: str = "u3"  # or "clifford_t" (reference-expressible shadow)

    def __post_init__(self):
        if self.q < 2 or self.n < 2 or self.q % self.n:
            raise ValidationError(
                f"need q >= 2, n >= 2 and n | q; got q={self.q}, n={self.n}"
            )
        if self.d < 1:
            raise ValidationError(f"depth must be >= 1, got {self.d}")
        if self.c_total < 0:
            raise ValidationError(f"c_total must be >= 0, got {self.c_total}")
        if self.one_qubit not in ("u3", "clifford_t"):
            raise ValidationError(f"one_qubit must be 'u3' or 'clifford_t', got {self.one_qubit}")

    @property
    def segment_size(self) -> int:
        return self.q // self.n

    @property
    def cuts_per_boundary(self) -> list[int]:
        return cut_distribution(self.n, self.c_total)


def draw(spec: BrickwallSpec):
    """The seeded draws, in the frozen order: (u[d,q,3], [layers_k ...])."""
    rng = np.random.default_rng(spec.seed)
    u = rng.uniform(size=(spec.d, spec.q, 3))
    layers = [np.sort(rng.integers(0, spec.d, size=ck)) for ck in spec.cuts_per_boundary]
    return u, layers


def build_brickwall(spec: BrickwallSpec) -> Circuit:
    q, d, s = spec.q, spec.d, spec.segment_size
    u, layers = draw(spec)
    theta = np.pi * u[..., 0]
    phi = 2.0 * np.pi * u[..., 1]
    lam = 2.0 * np.pi * u[..., 2]
    seg = np.arange(q) // s

    kinds, qa, qb, prm = [], [], [], []
    qubits = np.arange(q, dtype=np.int64)
    for L in range(d):
        if spec.one_qubit == "u3":
            kinds.append(np.full(q, KIND_U3, np.uint8))
            prm.append(np.stack([theta[L], phi[L], lam[L]], axis=1))
        else:
            pick = np.minimum((4.0 * u[L, :, 0]).astype(np.int64), 3)
            kinds.append(SHADOW_KINDS[pick])
            prm.append(np.zeros((q, 3)))
        qa.append(qubits)
        qb.append(np.full(q, -1, np.int64))
        i = np.arange(L % 2, q - 1, 2, dtype=np.int64)
        i = i[seg[i] == seg[i + 1]]
        kinds.append(np.full(i.size, KIND_CZ, np.uint8))
        qa.append(i)
        qb.append(i + 1)
        prm.append(np.zeros((i.size, 3)))
        cut_a = []
        for k, lay in enumerate(layers):
            mult = int(np.count_nonzero(lay == L))
            cut_a += [(k + 1) * s - 1] * mult
        if cut_a:
            ca = np.array(cut_a, dtype=np.int64)
            kinds.append(np.full(ca.size, KIND_CZ, np.uint8))
            qa.append(ca)
            qb.append(ca + 1)
            prm.append(np.zeros((ca.size, 3)))
    table = GateTable(np.concatenate(kinds), np.concatenate(qa), np.concatenate(qb),
                      np.concatenate(prm))
    return Circuit.from_table(q, table, validate=False)


# The BASELINE.json configurations, by name. cfg3 is a grid (d x c_total x seed).
BASELINE_CONFIGS = {
    "cfg1": BrickwallSpec(q=12, d=4, n=2, c_total=1, seed=0),
    "cfg2": BrickwallSpec(q=20, d=10, n=2, c_total=2, seed=0),
    "cfg4a": BrickwallSpec(q=30, d=10, n=2, c_total=2, seed=0),
    "cfg4b": BrickwallSpec(q=30, d=10, n=3, c_total=4, seed=0),
    "cfg5_q32_n2_c2": BrickwallSpec(q=32, d=10, n=2, c_total=2, seed=0),
    "cfg5_q32_n2_c4": BrickwallSpec(q=32, d=10, n=2, c_total=4, seed=0),
    "cfg5_q32_n4_c4": BrickwallSpec(q=32, d=10, n=4, c_total=4, seed=0),
    "cfg5_q34_n2_c2": BrickwallSpec(q=34, d=10, n=2, c_total=2, seed=0),
}


def cfg3_grid():
    for d in (5, 10, 20):
        for c in range(1, 7):
            for seed in (0, 1, 2):
                yield BrickwallSpec(q=24, d=d, n=2, c_total=c, seed=seed)
