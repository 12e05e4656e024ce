"""Cut planning and subcircuit generation (host-side preprocess, stage t_pre).

Same results as `/root/reference/pkg/src/cutbench/cutting.py`:
  * CZ = ((1-i)/2) S(x)S + ((1+i)/2) Sdg(x)Sdg; a boundary CX is
    (I(x)H) CZ (I(x)H), so its target side gets H,S,H / H,Sdg,H
    (`cutting.py:1-14, 34-35, 217-236`);
  * cut j is the j-th boundary gate in circuit order and owns bit j of the
    global term index m (`cutting.py:10-13`);
  * a segment's variant index b has bit k = the k-th cut adjacent to that
    segment, and variant b differs from the template only in the kind byte
    at ``patch_offsets[k]`` (S -> Sdg) (`cutting.py:237-247`);
  * merge table r_i(m) = m restricted to segment i's adjacent cuts
    (`cutting.py:251-263`); coefficients alpha_m (`cutting.py:266-272`).

How it differs: planning and fragment extraction are numpy passes over the
packed gate table (O(G) vector work, no per-gate Python), and the 2^{c_i}
variant circuits are *not* materialised — a segment is one template table plus
a ``slots`` column (cut bit that patches the gate, or -1). The device kernel
reads the template once for the whole variant batch; ``SegmentFamily.circuits``
builds reference-style ``Circuit`` objects lazily for callers that want them.
"""
from __future__ import annotations

import json
from dataclasses import dataclass, field
from typing import NamedTuple

import numpy as np

from .circuits import (
    KIND_CX,
    KIND_CZ,
    KIND_H,
    KIND_S,
    KIND_SDG,
    Circuit,
    GateTable,
)
from .errors import UnsupportedTopologyError, ValidationError

COEFF_TERM0 = 0.5 - 0.5j  # 1/(1+i)
COEFF_TERM1 = 0.5 + 0.5j  # i/(1+i)


class BoundaryGate(NamedTuple):
    """One cut: gate position and the segments it connects."""

    position: int
    boundary: int  # between segments `boundary` and `boundary + 1`
    control_segment: int
    target_segment: int


@dataclass(frozen=True)
class CutPlan:
    n: int
    segment_sizes: tuple[int, ...]
    segment_of: tuple[int, ...]
    boundary_gates: tuple[BoundaryGate, ...]
    c_per_boundary: tuple[int, ...]
    c_i: tuple[int, ...]
    c_total: int
    c_max: int

    @property
    def first_qubit(self) -> tuple[int, ...]:
        return tuple(int(v) for v in np.concatenate([[0], np.cumsum(self.segment_sizes)[:-1]]))

    def adjacent_cuts(self) -> list[list[int]]:
        """Per segment, the global cut ids touching it, in circuit order
        (local variant bit k = k-th entry)."""
        adj: list[list[int]] = [[] for _ in range(self.n)]
        for j, bg in enumerate(self.boundary_gates):
            adj[bg.boundary].append(j)
            adj[bg.boundary + 1].append(j)
        return adj


def plan_cut(circuit: Circuit, n: int) -> CutPlan:
    """Equal contiguous partition into n segments of q/n qubits."""
    if n < 2:
        raise ValidationError(f"segment count must be >= 2, got {n}")
    if circuit.num_qubits % n:
        raise ValidationError(f"q must be divisible by n: q={circuit.num_qubits}, n={n}")
    return plan_cut_sizes(circuit, (circuit.num_qubits // n,) * n)


def plan_cut_sizes(circuit: Circuit, sizes) -> CutPlan:
    """Contiguous partition with explicit segment sizes."""
    sizes = tuple(int(v) for v in sizes)
    n = len(sizes)
    if n < 2:
        raise ValidationError(f"segment count must be >= 2, got {n}")
    if min(sizes) < 1:
        raise ValidationError(f"segment sizes must be >= 1, got {sizes}")
    if sum(sizes) != circuit.num_qubits:
        raise ValidationError(f"segment sizes {sizes} must sum to q={circuit.num_qubits}")

    nt = _native_tables(circuit, sizes)
    if nt is not None:
        return _plan_from_tables(circuit, sizes, nt)
    seg_of = np.repeat(np.arange(n, dtype=np.int64), sizes)
    kinds = circuit.kinds
    two = np.flatnonzero((kinds == KIND_CX) | (kinds == KIND_CZ))
    sa = seg_of[circuit.qa[two]]
    sb = seg_of[circuit.qb[two]]
    crossing = sa != sb
    far = np.flatnonzero(np.abs(sa - sb) > 1)
    if far.size:
        i = int(far[0])
        pos = int(two[i])
        g = circuit.gates[pos] if circuit.gate_count < 4096 else None
        label = f"{g.kind.value}{g.qubits}" if g is not None else f"gate {pos}"
        raise UnsupportedTopologyError(
            f"gate {label} at position {pos} spans non-adjacent segments "
            f"{int(sa[i])} and {int(sb[i])}"
        )
    pos = two[crossing]
    ca, cb = sa[crossing], sb[crossing]
    bnd = np.minimum(ca, cb)
    boundary_gates = tuple(
        BoundaryGate(int(p), int(b), int(x), int(y)) for p, b, x, y in zip(pos, bnd, ca, cb)
    )
    counts = np.bincount(bnd, minlength=n - 1).astype(np.int64) if n > 1 else np.zeros(0)
    c_i = np.zeros(n, dtype=np.int64)
    c_i[:-1] += counts
    c_i[1:] += counts
    return CutPlan(
        n=n,
        segment_sizes=sizes,
        segment_of=tuple(int(v) for v in seg_of),
        boundary_gates=boundary_gates,
        c_per_boundary=tuple(int(v) for v in counts),
        c_i=tuple(int(v) for v in c_i),
        c_total=int(counts.sum()),
        c_max=int(c_i.max()),
    )


def _native_tables(circuit: Circuit, sizes):
    """plan + decompose by libcutsim's C++ planner (cs_cut_tables, ~10x the
    numpy path's speed) or None when the library cannot be loaded (the numpy
    path below is the same algorithm; tests check the two agree with each
    other and with the reference's golden tables)."""
    from . import _native

    try:
        _native.load()
    except Exception:  # noqa: BLE001  (no library here: host-only numpy planning)
        return None
    return _native.cut_tables(circuit.num_qubits, circuit.table, sizes)


def _plan_from_tables(circuit: Circuit, sizes: tuple[int, ...], nt) -> CutPlan:
    # plain Python over the (few) cuts: this is on the drop-in API's t_pre path
    n = len(sizes)
    rows = nt[0].tolist()
    boundary_gates = tuple(map(BoundaryGate._make, rows))
    counts = [0] * (n - 1)
    for r in rows:
        counts[r[1]] += 1
    c_i = [0] * n
    for b, cnt in enumerate(counts):
        c_i[b] += cnt
        c_i[b + 1] += cnt
    plan = CutPlan(
        n=n,
        segment_sizes=sizes,
        segment_of=tuple(i for i, sz in enumerate(sizes) for _ in range(sz)),
        boundary_gates=boundary_gates,
        c_per_boundary=tuple(counts),
        c_i=tuple(c_i),
        c_total=len(rows),
        c_max=max(c_i),
    )
    # decompose() reuses the tables for the same circuit (identity of its columns)
    object.__setattr__(plan, "_tables", (circuit.table.kinds, nt))
    return plan


def _families_from_tables(plan: CutPlan, nt) -> list[SegmentFamily]:
    _cuts, counts, k, a, b, p, sl, cid = nt
    fams = []
    g0 = c0 = first = 0
    cnt = counts.tolist()
    cids = cid.tolist()
    for seg in range(plan.n):
        m, nc = cnt[seg]
        slots = sl[g0:g0 + m]
        # every adjacent cut patches exactly one gate: patch[slot] = its row
        idx = np.flatnonzero(slots >= 0)
        patch = np.empty(idx.size, np.int64)
        patch[slots[idx]] = idx
        tab = GateTable.trusted(k[g0:g0 + m], a[g0:g0 + m], b[g0:g0 + m], p[g0:g0 + m])
        size = plan.segment_sizes[seg]
        fam = SegmentFamily(seg, first, size, tab, slots, patch, tuple(cids[c0:c0 + nc]))
        first += size
        # where the template sits in the C++ planner's concatenated tables:
        # pipeline.simulate_families runs all families of one decomposition
        # in one native call straight from them (while the template is unchanged)
        fam._src = (nt, g0, m, tab, (tab.kinds, tab.qa, tab.qb, tab.params), slots)
        fams.append(fam)
        g0 += m
        c0 += nc
    return fams


def count_subcircuits(plan: CutPlan) -> int:
    return int(sum(1 << c for c in plan.c_i))


class _VariantCircuits:
    """Lazy, cached list of the 2^{c_i} variant circuits of one segment."""

    def __init__(self, fam: "SegmentFamily"):
        self._fam = fam
        self._cache: dict[int, Circuit] = {}

    def __len__(self) -> int:
        return 1 << self._fam.num_cuts

    def __getitem__(self, b):
        if isinstance(b, slice):
            return [self[i] for i in range(*b.indices(len(self)))]
        b = int(b)
        if b < 0:
            b += len(self)
        if not 0 <= b < len(self):
            raise IndexError(b)
        if b not in self._cache:
            c = Circuit.from_table(self._fam.num_qubits, self._fam.variant_table(b), validate=False)
            c._origin = (self._fam, b)  # engine.simulate batches the family's variants
            self._cache[b] = c
        return self._cache[b]

    def __iter__(self):
        for b in range(len(self)):
            yield self[b]


@dataclass
class SegmentFamily:
    """All 2^{c_i} subcircuits of one segment, on local qubits 0..size-1.

    ``template`` is variant 0; ``slots[g] = k`` marks the gate that is S for
    bit k = 0 and Sdg for bit k = 1 (``-1`` elsewhere).
    """

    segment: int
    first_qubit: int
    num_qubits: int
    template: GateTable
    slots: np.ndarray
    patch_offsets: np.ndarray
    cut_ids: tuple[int, ...]
    circuits: _VariantCircuits = field(init=False, repr=False)

    def __post_init__(self):
        self.circuits = _VariantCircuits(self)
        self._pending = {}  # dtype -> (device batch, variants not yet handed out)
        self._src = None  # (planner tables, first row, rows, template, its columns, slots) from the C++ planner

    def claim_state(self, b: int, dtype, simulate_batch):
        """Variant b's state from one batched simulation of the whole family.

        The reference's call sequence simulates the variant circuits one by
        one (harness.py:136-139, `[[simulate(c) for c in fam.circuits] ...]`).
        The first request of a pass runs every variant in ONE batched launch
        sequence (`simulate_batch`) and each variant's state is handed out
        once, as a row of that batch (so merge() reads the batch in place);
        asking for a variant again starts a new pass — every call returns a
        fresh state, as the reference's simulate() does. Returns (batch, b)."""
        key = np.dtype(dtype).str
        batch, left = self._pending.get(key, (None, None))
        if batch is None or b not in left:
            batch = simulate_batch()
            left = set(range(self.num_variants))
        left.discard(b)
        if left:
            self._pending[key] = (batch, left)
        else:
            self._pending.pop(key, None)
        return batch, b

    @property
    def num_cuts(self) -> int:
        return len(self.cut_ids)

    @property
    def num_variants(self) -> int:
        return 1 << self.num_cuts

    def variant_table(self, b: int) -> GateTable:
        kinds = self.template.kinds.copy()
        for k, off in enumerate(self.patch_offsets):
            if (b >> k) & 1:
                kinds[off] = KIND_SDG
        return GateTable(kinds, self.template.qa, self.template.qb, self.template.params)


@dataclass
class SubcircuitSet:
    plan: CutPlan
    segments: list[SegmentFamily]
    merge_table: np.ndarray  # (n, 2^c_total) int64
    coeffs: np.ndarray  # (2^c_total,) complex128

    @property
    def num_subcircuits(self) -> int:
        return sum(f.num_variants for f in self.segments)

    def to_json_dict(self) -> dict:
        return {
            "schema_version": 1,
            "n": self.plan.n,
            "c_total": self.plan.c_total,
            "segment_sizes": list(self.plan.segment_sizes),
            "segments": [
                {
                    "segment": f.segment,
                    "first_qubit": f.first_qubit,
                    "num_qubits": f.num_qubits,
                    "subcircuits": [c.to_json_dict() for c in f.circuits],
                }
                for f in self.segments
            ],
            "merge_table": self.merge_table.tolist(),
            "coeffs": [[float(a.real), float(a.imag)] for a in self.coeffs],
        }

    def to_json(self) -> str:
        return json.dumps(self.to_json_dict())


def _segment_family(circuit: Circuit, plan: CutPlan, seg: int, cut_pos: np.ndarray,
                    owner: np.ndarray) -> SegmentFamily:
    first = plan.first_qubit[seg]
    size = plan.segment_sizes[seg]
    tab = circuit.table
    # gates owned by this segment that are not cuts (a non-cut 2q gate has both
    # qubits in one segment, so its first qubit decides ownership)
    mine = np.flatnonzero(owner == seg)
    adj = [j for j, bg in enumerate(plan.boundary_gates)
           if bg.control_segment == seg or bg.target_segment == seg]
    # fragments are split at the positions of the adjacent cuts
    split = np.searchsorted(mine, cut_pos[adj]) if adj else np.zeros(0, np.int64)
    frags = np.split(mine, split)

    pieces_k, pieces_a, pieces_b, pieces_p, pieces_slot = [], [], [], [], []
    patch = []
    length = 0

    def put_frag(idx):
        nonlocal length
        if idx.size == 0:
            return
        k = tab.kinds[idx]
        two = (k == KIND_CX) | (k == KIND_CZ)
        pieces_k.append(k)
        pieces_a.append(tab.qa[idx] - first)
        pieces_b.append(np.where(two, tab.qb[idx] - first, -1))
        pieces_p.append(tab.params[idx])
        pieces_slot.append(np.full(idx.size, -1, np.int32))
        length += idx.size

    def put_insert(kinds, lq, slot_at):
        nonlocal length
        m = len(kinds)
        pieces_k.append(np.array(kinds, np.uint8))
        pieces_a.append(np.full(m, lq, np.int64))
        pieces_b.append(np.full(m, -1, np.int64))
        pieces_p.append(np.zeros((m, 3)))
        sl = np.full(m, -1, np.int32)
        sl[slot_at] = len(patch)
        pieces_slot.append(sl)
        patch.append(length + slot_at)
        length += m

    put_frag(frags[0])
    for k, j in enumerate(adj):
        bg = plan.boundary_gates[j]
        kind = int(tab.kinds[bg.position])
        if bg.control_segment == seg:
            put_insert([KIND_S], int(tab.qa[bg.position]) - first, 0)
        else:
            lq = int(tab.qb[bg.position]) - first
            if kind == KIND_CX:
                put_insert([KIND_H, KIND_S, KIND_H], lq, 1)
            else:
                put_insert([KIND_S], lq, 0)
        put_frag(frags[k + 1])

    if pieces_k:
        template = GateTable(np.concatenate(pieces_k), np.concatenate(pieces_a),
                             np.concatenate(pieces_b), np.concatenate(pieces_p))
        slots = np.concatenate(pieces_slot).astype(np.int32)
    else:
        template = GateTable(np.zeros(0, np.uint8), np.zeros(0, np.int64),
                             np.zeros(0, np.int64), np.zeros((0, 3)))
        slots = np.zeros(0, np.int32)
    if len(adj) != plan.c_i[seg]:
        raise ValidationError(f"segment {seg}: {len(adj)} adjacent cuts, plan says {plan.c_i[seg]}")
    return SegmentFamily(seg, first, size, template, slots,
                         np.array(patch, dtype=np.int64), tuple(adj))


def _canonical_tables(plan: CutPlan):
    """Fresh copies of the plan's merge table and coefficients (callers may
    mutate a SubcircuitSet's arrays); the originals are computed once per plan
    and kept on it (merging.merge_input_from compares against them)."""
    canon = getattr(plan, "_canonical_tc", None)
    if canon is None:
        canon = (merge_table_of(plan), coefficients_of(plan.c_total))
        object.__setattr__(plan, "_canonical_tc", canon)
    return canon[0].copy(), canon[1].copy()


_TABLES_MEMO: dict = {}


def merge_table_of(plan: CutPlan) -> np.ndarray:
    """r_i(m) for every segment and term (a fresh array; the values depend
    only on n and the cuts' boundaries, so they are memoised on those)."""
    key = (plan.n, tuple(bg.boundary for bg in plan.boundary_gates))
    got = _TABLES_MEMO.get(key)
    if got is None:
        got = _merge_table(plan)
        got.flags.writeable = False
        if len(_TABLES_MEMO) > 1024:
            _TABLES_MEMO.clear()
        _TABLES_MEMO[key] = got
    return got.copy()


def _merge_table(plan: CutPlan) -> np.ndarray:
    ms = np.arange(1 << plan.c_total, dtype=np.int64)
    table = np.zeros((plan.n, ms.size), dtype=np.int64)
    for seg, cuts in enumerate(plan.adjacent_cuts()):
        for local_bit, j in enumerate(cuts):
            table[seg] |= ((ms >> j) & 1) << local_bit
    return table


def coefficients_of(c_total: int) -> np.ndarray:
    """alpha_m = t0^(c - popcount m) * t1^(popcount m), by exact repeated
    products (the factors are dyadic, so no rounding occurs). Memoised per
    c_total; a fresh array is returned."""
    got = _TABLES_MEMO.get(("coef", c_total))
    if got is None:
        got = _coefficients(c_total)
        got.flags.writeable = False
        _TABLES_MEMO[("coef", c_total)] = got
    return got.copy()


def _coefficients(c_total: int) -> np.ndarray:
    ms = np.arange(1 << c_total, dtype=np.int64)
    ones = np.zeros(ms.size, dtype=np.int64)
    for j in range(c_total):
        ones += (ms >> j) & 1
    p0 = [complex(1.0)]
    p1 = [complex(1.0)]
    for _ in range(c_total):
        p0.append(p0[-1] * COEFF_TERM0)
        p1.append(p1[-1] * COEFF_TERM1)
    p0 = np.array(p0, dtype=np.complex128)
    p1 = np.array(p1, dtype=np.complex128)
    return p0[c_total - ones] * p1[ones]


def decompose(circuit: Circuit, plan: CutPlan) -> SubcircuitSet:
    """All 2^{c_i} subcircuits per segment (as templates), merge table, coefficients."""
    seg_of = np.asarray(plan.segment_of, dtype=np.int64)
    if seg_of.size != circuit.num_qubits:
        raise ValidationError("plan does not match the circuit's qubit count")
    cached = getattr(plan, "_tables", None)
    nt = cached[1] if cached is not None and cached[0] is circuit.table.kinds else None
    if nt is None and cached is None:
        nt = _native_tables(circuit, plan.segment_sizes)
        if nt is not None and [int(v) for v in nt[0][:, 0]] != [bg.position for bg in plan.boundary_gates]:
            nt = None  # a plan that is not this circuit's own: follow it literally
    if nt is not None:
        table, coeffs = _canonical_tables(plan)
        return SubcircuitSet(plan, _families_from_tables(plan, nt), table, coeffs)
    cut_pos = np.array([bg.position for bg in plan.boundary_gates], dtype=np.int64)
    owner = seg_of[circuit.qa] if circuit.gate_count else np.zeros(0, np.int64)
    owner = owner.copy()
    owner[cut_pos] = -1
    segments = [_segment_family(circuit, plan, seg, cut_pos, owner) for seg in range(plan.n)]
    table, coeffs = _canonical_tables(plan)
    return SubcircuitSet(plan, segments, table, coeffs)
