"""Circuit IR: gate values, the packed gate table the kernels consume, and the
reference benchmark families.

Mirrors `/root/reference/pkg/src/cutbench/circuits.py`:
  * kind codes 0..6 are the reference's load-bearing dispatch values
    (`circuits.py:25-33`); this build adds ``KIND_U3 = 7`` with a per-gate
    ``params`` row (theta, phi, lambda), which the BASELINE configs need and the
    reference lacks;
  * qubit j is bit j of the amplitude index (qubit 0 = LSB); for CX/CZ the
    first qubit is the control (`circuits.py:67-75`);
  * ``Circuit`` keeps the packed table ``kinds:u8[G], qa:i64[G], qb:i64[G]``
    (`circuits.py:118-200`) plus ``params:f64[G,3]``.

Difference in *how*, not *what*: a ``Circuit`` built from a table (the cut
planner's subcircuits, the U3 generator) materialises its ``Gate`` tuple
lazily, so preprocessing never walks Python objects per gate.
"""
from __future__ import annotations

import json
import math
from dataclasses import dataclass
from enum import Enum, EnumMeta

import numpy as np

from .errors import ValidationError

KIND_H = 0
KIND_X = 1
KIND_T = 2
KIND_S = 3
KIND_SDG = 4
KIND_CX = 5
KIND_CZ = 6
KIND_U3 = 7

NUM_KINDS = 8


class _KindMeta(EnumMeta):
    """Iterating GateKind yields the reference's seven kinds (circuits.py:
    25-33: code written against the reference enumerates exactly those);
    the U3 extension stays reachable as GateKind.U3 / GateKind("U3")."""

    def __iter__(cls):
        return (m for m in super().__iter__() if m.name != "U3")

    def __len__(cls):
        return sum(1 for _ in cls.__iter__())


class GateKind(Enum, metaclass=_KindMeta):
    """Gate kinds; the value is the JSON wire string."""

    H = "H"
    X = "X"
    T = "T"
    S = "S"
    Sdg = "Sdg"
    CX = "CX"
    CZ = "CZ"
    U3 = "U3"

    @property
    def arity(self) -> int:
        return 2 if self in (GateKind.CX, GateKind.CZ) else 1

    @property
    def num_params(self) -> int:
        return 3 if self is GateKind.U3 else 0

    @property
    def code(self) -> int:
        return _CODE_OF[self]


_CODE_OF = {
    GateKind.H: KIND_H,
    GateKind.X: KIND_X,
    GateKind.T: KIND_T,
    GateKind.S: KIND_S,
    GateKind.Sdg: KIND_SDG,
    GateKind.CX: KIND_CX,
    GateKind.CZ: KIND_CZ,
    GateKind.U3: KIND_U3,
}
_KIND_OF_CODE = {code: kind for kind, code in _CODE_OF.items()}


def kind_from_code(code: int) -> GateKind:
    try:
        return _KIND_OF_CODE[int(code)]
    except KeyError as exc:
        raise ValidationError(f"unknown gate kind code {code}") from exc


@dataclass(frozen=True)
class Gate:
    """One gate application: kind, ordered qubits and (U3 only) angles."""

    kind: GateKind
    qubits: tuple[int, ...]
    params: tuple[float, ...] = ()

    def __post_init__(self):
        qs = tuple(int(q) for q in self.qubits)
        object.__setattr__(self, "qubits", qs)
        object.__setattr__(self, "params", tuple(float(v) for v in self.params))
        if len(qs) != self.kind.arity:
            raise ValidationError(
                f"{self.kind.value} acts on {self.kind.arity} qubit(s); got {len(qs)}"
            )
        if len(set(qs)) != len(qs):
            raise ValidationError(f"{self.kind.value} needs distinct qubits, got {qs}")
        if min(qs) < 0:
            raise ValidationError(f"negative qubit index in {qs}")
        if len(self.params) != self.kind.num_params:
            raise ValidationError(
                f"{self.kind.value} takes {self.kind.num_params} parameter(s); "
                f"got {len(self.params)}"
            )
        if self.params and not all(math.isfinite(v) for v in self.params):
            raise ValidationError(f"{self.kind.value} parameters must be finite")


def h(q: int) -> Gate:
    return Gate(GateKind.H, (q,))


def x(q: int) -> Gate:
    return Gate(GateKind.X, (q,))


def t(q: int) -> Gate:
    return Gate(GateKind.T, (q,))


def s(q: int) -> Gate:
    return Gate(GateKind.S, (q,))


def sdg(q: int) -> Gate:
    return Gate(GateKind.Sdg, (q,))


def cx(control: int, target: int) -> Gate:
    return Gate(GateKind.CX, (control, target))


def cz(a: int, b: int) -> Gate:
    return Gate(GateKind.CZ, (a, b))


def u3(q: int, theta: float, phi: float, lam: float) -> Gate:
    return Gate(GateKind.U3, (q,), (theta, phi, lam))


def u3_matrix(theta: float, phi: float, lam: float) -> np.ndarray:
    """OpenQASM-2 ``u3``: [[c, -e^{il} s], [e^{ip} s, e^{i(p+l)} c]], c,s of theta/2."""
    c, sn = math.cos(theta / 2.0), math.sin(theta / 2.0)
    return np.array(
        [
            [c, -complex(math.cos(lam), math.sin(lam)) * sn],
            [complex(math.cos(phi), math.sin(phi)) * sn,
             complex(math.cos(phi + lam), math.sin(phi + lam)) * c],
        ],
        dtype=np.complex128,
    )


class GateTable:
    """Structure-of-arrays view of a gate list (the kernel input)."""

    __slots__ = ("kinds", "qa", "qb", "params")

    def __init__(self, kinds, qa, qb, params=None):
        self.kinds = np.ascontiguousarray(kinds, dtype=np.uint8)
        self.qa = np.ascontiguousarray(qa, dtype=np.int64)
        self.qb = np.ascontiguousarray(qb, dtype=np.int64)
        g = self.kinds.shape[0]
        if params is None:
            params = np.zeros((g, 3), dtype=np.float64)
        self.params = np.ascontiguousarray(params, dtype=np.float64).reshape(g, 3)
        if not (self.qa.shape[0] == g and self.qb.shape[0] == g):
            raise ValidationError("gate table columns differ in length")

    @classmethod
    def trusted(cls, kinds, qa, qb, params) -> "GateTable":
        """Columns already of the kernel dtypes, contiguous and equally long
        (the C++ planner's output): no conversion pass."""
        t = cls.__new__(cls)
        t.kinds, t.qa, t.qb, t.params = kinds, qa, qb, params
        return t

    def __len__(self) -> int:
        return int(self.kinds.shape[0])


def validate_table(num_qubits: int, table: GateTable) -> None:
    """Vectorised range/arity checks, equivalent to the per-gate loop of the
    reference `_encode_and_check` (`circuits.py:185-200`)."""
    g = len(table)
    if g == 0:
        return
    k = table.kinds
    if int(k.max()) >= NUM_KINDS:
        raise ValidationError(f"unknown gate kind code {int(k.max())}")
    two = (k == KIND_CX) | (k == KIND_CZ)
    qa, qb = table.qa, table.qb
    if qa.min() < 0 or (two & (qb < 0)).any():
        raise ValidationError("negative qubit index in gate table")
    hi = np.where(two, np.maximum(qa, qb), qa)
    if int(hi.max()) >= num_qubits:
        bad = int(np.argmax(hi >= num_qubits))
        raise ValidationError(
            f"gate {kind_from_code(k[bad]).value} at position {bad} exceeds circuit "
            f"qubit count {num_qubits}"
        )
    if (two & (qa == qb)).any():
        raise ValidationError("two-qubit gate needs distinct qubits")
    if not np.isfinite(table.params).all():
        raise ValidationError("gate parameters must be finite")


def _encode(num_qubits: int, gates: tuple[Gate, ...]) -> GateTable:
    n = len(gates)
    kinds = np.empty(n, dtype=np.uint8)
    qa = np.empty(n, dtype=np.int64)
    qb = np.full(n, -1, dtype=np.int64)
    params = np.zeros((n, 3), dtype=np.float64)
    for i, g in enumerate(gates):
        qs = g.qubits
        if max(qs) >= num_qubits:
            raise ValidationError(
                f"gate {g.kind.value}{qs} exceeds circuit qubit count {num_qubits}"
            )
        kinds[i] = _CODE_OF[g.kind]
        qa[i] = qs[0]
        if len(qs) == 2:
            qb[i] = qs[1]
        if g.params:
            params[i] = g.params
    return GateTable(kinds, qa, qb, params)


def _decode(table: GateTable) -> tuple[Gate, ...]:
    out = []
    for i in range(len(table)):
        kind = _KIND_OF_CODE[int(table.kinds[i])]
        if kind.arity == 2:
            qs = (int(table.qa[i]), int(table.qb[i]))
        else:
            qs = (int(table.qa[i]),)
        prm = tuple(float(v) for v in table.params[i]) if kind.num_params else ()
        out.append(Gate(kind, qs, prm))
    return tuple(out)


class Circuit:
    """Ordered gate list over a fixed qubit count (immutable by convention).

    ``Circuit(num_qubits, gates)`` encodes Python gates; ``Circuit.from_table``
    wraps an already packed table and decodes ``gates`` only on first access.
    The ``_table`` keyword mirrors the reference's internal fast path
    (`circuits.py:129-138`): a ``(kinds, qa, qb)`` or ``(kinds, qa, qb, params)``
    tuple that is trusted to describe ``gates``.
    """

    __slots__ = ("num_qubits", "_gates", "_table", "_depth", "_origin")

    def __init__(self, num_qubits: int, gates=(), *, _table=None):
        if num_qubits < 0:
            raise ValidationError(f"num_qubits must be non-negative, got {num_qubits}")
        self.num_qubits = int(num_qubits)
        self._gates = tuple(gates)
        self._depth = None
        self._origin = None  # (SegmentFamily, variant) for decompose()'s lazy variant circuits
        if _table is not None:
            self._table = _table if isinstance(_table, GateTable) else GateTable(*_table)
            if self._gates and len(self._gates) != len(self._table):
                # the reference passes a table alongside the gate list; the
                # params column may be absent there, so re-derive it
                self._table = GateTable(self._table.kinds, self._table.qa, self._table.qb,
                                        _encode(self.num_qubits, self._gates).params)
        else:
            self._table = _encode(self.num_qubits, self._gates)
            if not self._gates:
                self._gates = ()

    @classmethod
    def from_table(cls, num_qubits: int, table: GateTable, *, validate: bool = True) -> "Circuit":
        obj = cls.__new__(cls)
        if num_qubits < 0:
            raise ValidationError(f"num_qubits must be non-negative, got {num_qubits}")
        obj.num_qubits = int(num_qubits)
        if validate:
            validate_table(obj.num_qubits, table)
        obj._table = table
        obj._gates = None
        obj._depth = None
        obj._origin = None
        return obj

    # -- packed table ---------------------------------------------------
    @property
    def table(self) -> GateTable:
        return self._table

    @property
    def kinds(self) -> np.ndarray:
        return self._table.kinds

    @property
    def qa(self) -> np.ndarray:
        return self._table.qa

    @property
    def qb(self) -> np.ndarray:
        return self._table.qb

    @property
    def params(self) -> np.ndarray:
        return self._table.params

    # -- gate view ----------------------------------------------------------
    @property
    def gates(self) -> tuple[Gate, ...]:
        if self._gates is None or (len(self._gates) == 0 and len(self._table) > 0):
            self._gates = _decode(self._table)
        return self._gates

    @property
    def gate_count(self) -> int:
        return len(self._table)

    def __len__(self) -> int:
        return len(self._table)

    @property
    def depth(self) -> int:
        if self._depth is None:
            self._depth = compute_depth(self)
        return self._depth

    def __eq__(self, other) -> bool:
        if not isinstance(other, Circuit) or other.num_qubits != self.num_qubits:
            return False
        a, b = self._table, other._table
        if len(a) != len(b):
            return False
        two = (a.kinds == KIND_CX) | (a.kinds == KIND_CZ)
        return bool(
            np.array_equal(a.kinds, b.kinds)
            and np.array_equal(a.qa, b.qa)
            and np.array_equal(np.where(two, a.qb, -1), np.where(two, b.qb, -1))
            and np.array_equal(a.params, b.params)
        )

    __hash__ = None

    def __repr__(self) -> str:
        return f"Circuit(num_qubits={self.num_qubits}, gates={self.gate_count})"

    # -- JSON ------------------------------------------------------------
    def to_json_dict(self) -> dict:
        out = []
        for g in self.gates:
            item = {"kind": g.kind.value, "qubits": list(g.qubits)}
            if g.params:
                item["params"] = list(g.params)
            out.append(item)
        return {"num_qubits": self.num_qubits, "gates": out}

    def to_json(self) -> str:
        return json.dumps(self.to_json_dict())

    @classmethod
    def from_json_dict(cls, data: dict) -> "Circuit":
        try:
            gates = [
                Gate(GateKind(g["kind"]), tuple(g["qubits"]), tuple(g.get("params", ())))
                for g in data["gates"]
            ]
            return cls(int(data["num_qubits"]), gates)
        except (KeyError, ValueError, TypeError) as exc:
            raise ValidationError(f"malformed circuit JSON: {exc}") from exc

    @classmethod
    def from_json(cls, text: str) -> "Circuit":
        return cls.from_json_dict(json.loads(text))


def compute_depth(circuit: Circuit) -> int:
    """Frontier-scheduled layer count (same rule as the reference,
    `circuits.py:203-213`)."""
    if circuit.num_qubits == 0:
        return 0
    front = np.zeros(circuit.num_qubits, dtype=np.int64)
    k, qa, qb = circuit.kinds, circuit.qa, circuit.qb
    depth = 0
    for i in range(len(k)):
        a = int(qa[i])
        if k[i] == KIND_CX or k[i] == KIND_CZ:
            b = int(qb[i])
            layer = 1 + max(front[a], front[b])
            front[a] = front[b] = layer
        else:
            layer = 1 + front[a]
            front[a] = layer
        if layer > depth:
            depth = int(layer)
    return depth


# ---------------------------------------------------------------------------
# Reference benchmark family (staircase, paper Fig. 2) — parity tier A.
# ---------------------------------------------------------------------------
MAX_PAD_EXPONENT = 7


@dataclass(frozen=True)
class BenchmarkSpec:
    """Staircase parameters; c_total = blocks * (n - 1) (`circuits.py:220-255`)."""

    q: int
    n: int
    blocks: int
    depth_pad_exponent: int | None = None

    def __post_init__(self):
        if self.q < 2:
            raise ValidationError(f"q must be >= 2, got {self.q}")
        if self.n < 2:
            raise ValidationError(f"n must be >= 2, got {self.n}")
        if self.q % self.n:
            raise ValidationError(f"q must be divisible by n: q={self.q}, n={self.n}")
        if self.blocks < 1:
            raise ValidationError(f"blocks must be >= 1, got {self.blocks}")
        p = self.depth_pad_exponent
        if p is not None and not (0 <= p <= MAX_PAD_EXPONENT):
            raise ValidationError(
                f"depth_pad_exponent must lie in [0, {MAX_PAD_EXPONENT}], got {p}"
            )

    @property
    def c_total(self) -> int:
        return self.blocks * (self.n - 1)


def _staircase_table(q: int, blocks: int) -> GateTable:
    # H on every qubit, then per block and per i: T(i) T(i+1) CX(i,i+1) T(i) T(i+1)
    i = np.arange(q - 1, dtype=np.int64)
    blk_k = np.tile(np.array([KIND_T, KIND_T, KIND_CX, KIND_T, KIND_T], np.uint8), q - 1)
    blk_a = np.stack([i, i + 1, i, i, i + 1], axis=1).ravel()
    blk_b = np.stack([-np.ones_like(i), -np.ones_like(i), i + 1, -np.ones_like(i),
                      -np.ones_like(i)], axis=1).ravel()
    kinds = np.concatenate([np.full(q, KIND_H, np.uint8)] + [blk_k] * blocks)
    qa = np.concatenate([np.arange(q, dtype=np.int64)] + [blk_a] * blocks)
    qb = np.concatenate([np.full(q, -1, np.int64)] + [blk_b] * blocks)
    return GateTable(kinds, qa, qb)


def build_staircase(spec: BenchmarkSpec) -> Circuit:
    if spec.depth_pad_exponent is not None:
        raise ValidationError("staircase generator: depth_pad_exponent must be absent")
    return Circuit.from_table(spec.q, _staircase_table(spec.q, spec.blocks), validate=False)


def build_depth_padded(spec: BenchmarkSpec) -> Circuit:
    """Staircase with 10^p alternating T,X on qubit 0 right after its H and the
    same appended on qubit q-1 (`circuits.py:269-282`)."""
    p = spec.depth_pad_exponent
    if p is None:
        raise ValidationError("depth-padded generator: depth_pad_exponent is required")
    base = _staircase_table(spec.q, spec.blocks)
    pad = 10**p
    alt = np.where(np.arange(pad) % 2 == 0, KIND_T, KIND_X).astype(np.uint8)
    kinds = np.concatenate([base.kinds[:1], alt, base.kinds[1:], alt])
    qa = np.concatenate([base.qa[:1], np.zeros(pad, np.int64), base.qa[1:],
                         np.full(pad, spec.q - 1, np.int64)])
    qb = np.concatenate([base.qb[:1], np.full(pad, -1, np.int64), base.qb[1:],
                         np.full(pad, -1, np.int64)])
    return Circuit.from_table(spec.q, GateTable(kinds, qa, qb), validate=False)


def build_benchmark(spec: BenchmarkSpec) -> Circuit:
    if spec.depth_pad_exponent is None:
        return build_staircase(spec)
    return build_depth_padded(spec)
