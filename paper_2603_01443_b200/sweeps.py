"""GPU experiment drivers of the threshold study: (q, c_total) heat-map
sweeps, the fitted speedup boundary, merge-time crossovers, budgeted
feasibility scans, bipartition sweeps and depth sweeps, plus their JSON
reports — the reference's harness API (`/root/reference/pkg/src/cutbench/
harness.py`: `SweepResult` :246-257, `sweep_heatmap` :268-320, `fit_boundary`
:323-335, `detect_crossovers` :346-356, `breakdown_series` :359-380,
`scan_feasible` :394-461, `split_sweep` :482-528, `depth_sweep` :538-571,
reports :598-704), driven by `harness.measure`, whose stage timers bracket
device work with synchronisation.

Differences from the reference, by design:

* `family="brickwall"` runs the BASELINE cfg3 U3 brick-wall family
  (`generators.BrickwallSpec`, depth d, seeds) instead of the staircase
  (`family="staircase"`, the reference's only family, the default);
* grid points never run concurrently on one GPU (`parallel_points` > 1 is
  accepted and recorded, and the rows are marked "contended" exactly as the
  reference does, but execution stays sequential so timings are clean).
"""
from __future__ import annotations

import json
import math
import os
import platform
import time
from dataclasses import dataclass
from datetime import datetime, timezone
from typing import Iterable, Sequence

import numpy as np

from . import _device
from .boundary_fit import BoundaryFit, fit_weighted_line
from .circuits import BenchmarkSpec, build_benchmark
from .engine import DEFAULT_MAX_QUBITS, simulate
from .errors import CapacityError, ValidationError
from .generators import BrickwallSpec
from .harness import SCHEMA_VERSION, TimingBreakdown, format_csv, measure
from .theory import threshold_line

DEFAULT_GRIDS = {
    2: (tuple(range(2, 21, 2)), tuple(range(1, 11))),
    3: (tuple(range(3, 19, 3)), tuple(range(2, 13, 2))),
}
MACHINE_TAG_ENV = "CUTBENCH_MACHINE_TAG"

__all__ = [
    "DEFAULT_GRIDS", "SweepResult", "sweep_heatmap", "fit_boundary", "Crossovers", "detect_crossovers",
    "breakdown_series", "FeasibilityScan", "scan_feasible", "SplitPoint", "SplitSweepResult", "split_sweep",
    "DepthSweepResult", "depth_sweep", "boundary_fit_report", "crossover_report", "feasibility_report",
    "split_report", "depth_sweep_report", "sweep_report", "write_text", "write_json", "machine_tag", "warm_up",
    "format_csv",
]


def machine_tag(override: str | None = None) -> str:
    return override or os.environ.get(MACHINE_TAG_ENV) or platform.node() or "unknown"


def warm_up() -> None:
    """Build (and NVRTC-compile, if enabled) the device programs of a tiny
    cut and uncut run so the first measured point does not pay for it."""
    from .pipeline import run_cut

    for n, q in ((2, 2), (3, 3), (4, 4)):
        circ = build_benchmark(BenchmarkSpec(q=q, n=n, blocks=1))
        run_cut(circ, n)
        simulate(circ)
    _device.torch().cuda.synchronize()


@dataclass
class SweepResult:
    points: list[TimingBreakdown]
    metadata: dict

    def __post_init__(self):
        keys = [(p.q, p.c_total) for p in self.points]
        if len(set(keys)) != len(keys):
            raise ValidationError("sweep grid points must be unique")


def _blocks_for(c_total: int, n: int) -> int:
    if c_total < n - 1 or c_total % (n - 1):
        raise ValidationError(f"c_total={c_total} must be a positive multiple of n-1={n - 1}")
    return c_total // (n - 1)


def _spec(family: str, q: int, n: int, c: int, *, pad_exponent, depth: int, seed: int):
    if family == "staircase":
        return BenchmarkSpec(q=q, n=n, blocks=_blocks_for(c, n), depth_pad_exponent=pad_exponent)
    if family == "brickwall":
        return BrickwallSpec(q, depth, n, c, seed)
    raise ValidationError(f"unknown circuit family {family!r} (staircase | brickwall)")


def _mean_breakdown(rows: list[TimingBreakdown]) -> TimingBreakdown:
    """Seed-averaged row (brick-wall family with several seeds)."""
    if len(rows) == 1:
        return rows[0]
    first = rows[0]
    avg = {k: float(np.mean([getattr(r, k) for r in rows]))
           for k in ("t_pre", "t_sub", "t_merge", "t_orig")}
    t_cut = avg["t_pre"] + avg["t_sub"] + avg["t_merge"]
    delta = (t_cut - avg["t_orig"]) / avg["t_orig"] if math.isfinite(t_cut) and avg["t_orig"] else math.nan
    status = "ok" if all(r.status == "ok" for r in rows) else "+".join(sorted({r.status for r in rows}))
    return TimingBreakdown(q=first.q, n=first.n, c_total=first.c_total, depth=first.depth,
                           gate_count=int(np.mean([r.gate_count for r in rows])), t_cut=t_cut, delta=delta,
                           reps=sum(r.reps for r in rows), status=status, **avg)


def sweep_heatmap(q_values: Iterable[int] | None = None, c_values: Iterable[int] | None = None, n: int = 2,
                  repetitions: int = 10, *, pad_exponent: int | None = None, budget: float | None = None,
                  parallel_points: int = 1, max_qubits: int = DEFAULT_MAX_QUBITS, tag: str | None = None,
                  family: str = "staircase", depth: int = 10, seeds: Sequence[int] = (0,),
                  cut_path: str = "api") -> SweepResult:
    """Relative overhead delta = (t_cut - t_orig) / t_orig on a (q, c_total)
    grid, one `measure` per point (mean over seeds for the brick-wall family)."""
    if q_values is None or c_values is None:
        if n not in DEFAULT_GRIDS:
            raise ValidationError(f"no default grid for n={n}; pass q and c values")
        dq, dc = DEFAULT_GRIDS[n]
        q_values = dq if q_values is None else q_values
        c_values = dc if c_values is None else c_values
    grid = [(int(q), int(c)) for q in q_values for c in c_values]
    for q, c in grid:  # validate the whole grid before spending device time
        _spec(family, q, n, c, pad_exponent=pad_exponent, depth=depth, seed=0)
    warm_up()
    points = []
    for q, c in grid:
        rows = [measure(_spec(family, q, n, c, pad_exponent=pad_exponent, depth=depth, seed=s), repetitions,
                        budget=budget, max_qubits=max_qubits, cut_path=cut_path)
                for s in (seeds if family == "brickwall" else (0,))]
        points.append(_mean_breakdown(rows))
    if parallel_points > 1:
        for p in points:
            p.status = "contended" if p.status == "ok" else p.status + "+contended"
    meta = {"schema_version": SCHEMA_VERSION, "n": n, "repetitions": repetitions,
            "pad_exponent": pad_exponent, "budget_seconds": budget, "parallel_points": parallel_points,
            "machine_tag": machine_tag(tag), "timestamp": datetime.now(timezone.utc).isoformat(),
            "family": family, "device": _device_name(), "cut_path": cut_path}
    if family == "brickwall":
        meta.update(depth=depth, seeds=list(seeds))
    return SweepResult(points=points, metadata=meta)


def _device_name() -> str:
    t = _device.torch()
    return t.cuda.get_device_name() if t.cuda.is_available() else "none"


def fit_boundary(sweep) -> BoundaryFit:
    """Weighted-SVM boundary through a sweep, started on the analytic line."""
    if isinstance(sweep, SweepResult):
        rows, n = sweep.points, sweep.metadata.get("n", 2)
    else:
        rows = list(sweep)
        n = rows[0].n if rows else 2
    rows = [r for r in rows if math.isfinite(r.delta)]
    qc = np.array([[r.q, r.c_total] for r in rows], dtype=float).reshape(-1, 2)
    return fit_weighted_line(qc, np.array([r.delta for r in rows], dtype=float), threshold_line(n))


@dataclass(frozen=True)
class Crossovers:
    q_pre_cross: int | None
    q_sub_cross: int | None


def detect_crossovers(breakdowns: Sequence[TimingBreakdown]) -> Crossovers:
    """First q (ascending) where t_merge exceeds t_pre and where it exceeds t_sub."""
    rows = sorted((b for b in breakdowns if b.ok), key=lambda b: b.q)
    kinds = sorted({(b.n, b.c_total) for b in rows})
    if len(kinds) > 1:
        raise ValidationError(f"crossover series mixes configurations: {kinds}")

    def first(pred):
        return next((b.q for b in rows if pred(b)), None)

    return Crossovers(first(lambda b: b.t_merge > b.t_pre), first(lambda b: b.t_merge > b.t_sub))


def breakdown_series(q_values: Iterable[int], n: int = 2, c_total: int = 6, repetitions: int = 10, *,
                     pad_exponent: int | None = None, budget: float | None = None,
                     max_qubits: int = DEFAULT_MAX_QUBITS) -> list[TimingBreakdown]:
    blocks = _blocks_for(c_total, n)
    return [measure(BenchmarkSpec(q=int(q), n=n, blocks=blocks, depth_pad_exponent=pad_exponent), repetitions,
                    budget=budget, max_qubits=max_qubits) for q in q_values]


@dataclass
class FeasibilityScan:
    pad_exponent: int | None
    budget_seconds: float
    q_max_orig: int | None
    q_max_cut: int | None
    rows: list[TimingBreakdown]


def scan_feasible(pad_exponents: Sequence[int | None], budget_seconds: float, n: int = 2, c_total: int = 6, *,
                  repetitions: int = 1, q_start: int | None = None, q_stop: int | None = None,
                  max_qubits: int = DEFAULT_MAX_QUBITS) -> list[FeasibilityScan]:
    """Grow q in steps of n until both pipelines exceed the per-run budget or
    the memory guard is reached; q_max is the largest q whose every
    repetition finished in budget (every reported q was executed)."""
    if budget_seconds <= 0:
        raise ValidationError(f"budget must be positive, got {budget_seconds}")
    blocks = _blocks_for(c_total, n)
    warm_up()
    stop = min(q_stop or max_qubits, max_qubits)
    scans = []
    for p in pad_exponents:
        alive = {"cut": True, "orig": True}
        best: dict[str, int | None] = {"cut": None, "orig": None}
        rows = []
        q = max(2, n) if q_start is None else q_start
        while q <= stop and any(alive.values()):
            row = measure(BenchmarkSpec(q=q, n=n, blocks=blocks, depth_pad_exponent=p), repetitions,
                          budget=budget_seconds, max_qubits=max_qubits,
                          pipelines=tuple(k for k in ("cut", "orig") if alive[k]))
            rows.append(row)
            for k in ("cut", "orig"):
                if alive[k]:
                    if k in row.status:
                        alive[k] = False
                    else:
                        best[k] = q
            q += n
        scans.append(FeasibilityScan(p, budget_seconds, best["orig"], best["cut"], rows))
    return scans


@dataclass
class SplitPoint:
    cut: int
    split: int
    t_cut: float
    t_orig: float
    ratio: float


@dataclass
class SplitSweepResult:
    q: int
    points: list[SplitPoint]
    best_split: dict[int, int]


def _timed(fn, reps: int) -> float:
    t = _device.torch()
    vals = []
    for _ in range(reps):
        t.cuda.synchronize()
        t0 = time.perf_counter()
        res = fn()
        t.cuda.synchronize()
        vals.append(time.perf_counter() - t0)
        del res
    return float(np.mean(vals))


def split_sweep(q: int, cut_range: Iterable[int], n: int = 2, repetitions: int = 10, *,
                max_qubits: int = DEFAULT_MAX_QUBITS) -> SplitSweepResult:
    """t_cut / t_orig for every bipartition 1..q-1 of the staircase (which
    crosses any contiguous boundary once per block, so c_total = blocks)."""
    from .pipeline import run_cut

    if n != 2:
        raise ValidationError(f"split sweep is defined for n=2, got n={n}")
    if q % 2:
        raise ValidationError(f"q must be even, got {q}")
    warm_up()
    points: list[SplitPoint] = []
    best: dict[int, int] = {}
    for c in (int(v) for v in cut_range):
        circ = build_benchmark(BenchmarkSpec(q=q, n=2, blocks=c))
        t_orig = _timed(lambda: simulate(circ, max_qubits=max_qubits), repetitions)
        mine = []
        for split in range(1, q):
            try:
                t_cut = _timed(lambda: run_cut(circ, 2, sizes=(split, q - split), max_qubits=max_qubits),
                               repetitions)
            except CapacityError:
                continue
            mine.append(SplitPoint(c, split, t_cut, t_orig, t_cut / t_orig))
        points += mine
        if mine:
            best[c] = min(mine, key=lambda sp: sp.ratio).split
    return SplitSweepResult(q=q, points=points, best_split=best)


@dataclass
class DepthSweepResult:
    fits: list[tuple[int, BoundaryFit]]
    sweeps: list[SweepResult]
    slope_differences: dict[tuple[int, int], float]


def depth_sweep(pad_exponents: Sequence[int], q_values=None, c_values=None, n: int = 2, repetitions: int = 10,
                *, budget: float | None = None, max_qubits: int = DEFAULT_MAX_QUBITS) -> DepthSweepResult:
    """One boundary fit per depth-padding exponent and their pairwise slope gaps."""
    qv = None if q_values is None else list(q_values)
    cv = None if c_values is None else list(c_values)
    sweeps, fits = [], []
    for p in (int(v) for v in pad_exponents):
        sw = sweep_heatmap(qv, cv, n=n, repetitions=repetitions, pad_exponent=p, budget=budget,
                           max_qubits=max_qubits)
        sweeps.append(sw)
        fits.append((p, fit_boundary(sw)))
    gaps = {(fits[i][0], fits[j][0]): abs(fits[i][1].slope - fits[j][1].slope)
            for i in range(len(fits)) for j in range(i + 1, len(fits))}
    return DepthSweepResult(fits=fits, sweeps=sweeps, slope_differences=gaps)


# -- reports (schema of harness.py:598-704) -------------------------------------
def _header(kind: str, tag: str | None) -> dict:
    return {"schema_version": SCHEMA_VERSION, "kind": kind, "machine_tag": machine_tag(tag)}


def sweep_report(sweep: SweepResult) -> str:
    """The sweep as the reference CSV (harness.py:41-45)."""
    return format_csv(sweep.points)


def boundary_fit_report(fit: BoundaryFit, *, tag: str | None = None) -> dict:
    rep = _header("boundary-fit", tag)
    rep.update(slope=fit.slope, intercept=fit.intercept, weighted_accuracy=fit.weighted_accuracy,
               margin_violations=fit.margin_violations, iterations=fit.iterations,
               points=[{"q": float(p[0]), "c_total": float(p[1]), "label": int(lab), "weight": float(w)}
                       for p, lab, w in zip(fit.points, fit.labels, fit.weights)])
    return rep


def crossover_report(cross: Crossovers, breakdowns: Sequence[TimingBreakdown], *, tag: str | None = None) -> dict:
    rep = _header("crossovers", tag)
    rep.update(q_pre_cross=cross.q_pre_cross, q_sub_cross=cross.q_sub_cross,
               series=[{"q": b.q, "c_total": b.c_total, "t_pre": b.t_pre, "t_sub": b.t_sub,
                        "t_merge": b.t_merge, "status": b.status} for b in breakdowns])
    return rep


def feasibility_report(scans: Sequence[FeasibilityScan], *, tag: str | None = None) -> dict:
    rep = _header("feasibility-scan", tag)
    rep["scans"] = [{"pad_exponent": s.pad_exponent, "budget_seconds": s.budget_seconds,
                     "q_max_orig": s.q_max_orig, "q_max_cut": s.q_max_cut,
                     "executed": [{"q": r.q, "status": r.status, "t_cut": r.t_cut, "t_orig": r.t_orig}
                                  for r in s.rows]} for s in scans]
    return rep


def split_report(result: SplitSweepResult, *, tag: str | None = None) -> dict:
    rep = _header("split-sweep", tag)
    rep.update(q=result.q, best_split={str(c): s for c, s in result.best_split.items()},
               points=[{"c_total": p.cut, "split": p.split, "t_cut": p.t_cut, "t_orig": p.t_orig,
                        "ratio": p.ratio} for p in result.points])
    return rep


def depth_sweep_report(result: DepthSweepResult, *, tag: str | None = None) -> dict:
    rep = _header("depth-sweep", tag)
    rep["fits"] = [{"pad_exponent": p, "slope": f.slope, "intercept": f.intercept} for p, f in result.fits]
    rep["slope_differences"] = [{"pad_exponents": list(k), "difference": v}
                                for k, v in result.slope_differences.items()]
    return rep


def write_text(path: str | None, text: str) -> None:
    if path in (None, "-"):
        print(text, end="" if text.endswith("\n") else "\n")
        return
    with open(path, "w") as fh:
        fh.write(text)


def write_json(path: str | None, payload: dict) -> None:
    write_text(path, json.dumps(payload, indent=2) + "\n")
