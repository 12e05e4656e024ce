"""Stage-timed measurement of the cut pipeline vs the uncut simulator.

Mirrors the timing contract of `/root/reference/pkg/src/cutbench/harness.py`
(`TimingBreakdown` :62-89, `_cut_once` :125-145, `_orig_once` :148-151,
`measure` :154-244, CSV schema :41-45): t_pre = plan_cut + decompose (host),
t_sub = every subcircuit simulation, t_merge = merge_input_from + merge,
t_cut = t_pre + t_sub + t_merge (phase-sum identity), t_orig = uncut
simulate, delta = (t_cut - t_orig) / t_orig; R repetitions, mean and sample
std, budgets recorded as "timeout-*" status data.

On the GPU every stage boundary synchronises the device, so each stage time
is the wall time of its work (kernels included). The sweep drivers, the
boundary fit and the reports built on `measure` live in `sweeps.py`.
"""
from __future__ import annotations

import gc
import math

import numpy as np
import time
from dataclasses import dataclass, field
from io import StringIO
from typing import Sequence

from . import _device
from .circuits import BenchmarkSpec, Circuit, build_benchmark
from .cutting import decompose, plan_cut
from .engine import DEFAULT_MAX_QUBITS, simulate, simulate_family
from .errors import BudgetExceededError, ValidationError
from .generators import BrickwallSpec, build_brickwall
from .merging import merge, merge_input_from

SCHEMA_VERSION = 1
CSV_COLUMNS = (
    "q", "n", "c_total", "D", "G",
    "t_pre", "t_sub", "t_merge", "t_cut", "t_orig",
    "delta", "reps", "status", "schema_version",
)


@dataclass
class TimingBreakdown:
    q: int
    n: int
    c_total: int
    depth: int
    gate_count: int
    t_pre: float
    t_sub: float
    t_merge: float
    t_cut: float
    t_orig: float
    delta: float
    reps: int
    status: str
    blocks: int = 0
    pad_exponent: int | None = None
    t_pre_std: float = math.nan
    t_sub_std: float = math.nan
    t_merge_std: float = math.nan
    t_orig_std: float = math.nan
    samples: dict = field(default_factory=dict, repr=False)

    @property
    def ok(self) -> bool:
        return not self.status.startswith("timeout")


def _sync():
    _device.torch().cuda.synchronize()


def build(spec) -> Circuit:
    if isinstance(spec, BrickwallSpec):
        return build_brickwall(spec)
    if isinstance(spec, BenchmarkSpec):
        return build_benchmark(spec)
    raise ValidationError(f"unknown spec type {type(spec).__name__}")


def _cut_once_native(circuit: Circuit, n: int, *, max_qubits: int, deadline: float | None):
    """The same three stages through the one-call pipeline (cs_cut_run):
    t_pre = its C++ plan/decompose, t_sub / t_merge = CUDA events around the
    batched variant sweeps and the merge (the call synchronises)."""
    from .pipeline import StageTimes, run_cut

    if deadline is not None and time.monotonic() > deadline:
        raise BudgetExceededError("cut pipeline exceeded its budget before starting")
    times = StageTimes()
    merged = run_cut(circuit, n, max_qubits=max_qubits, timers=times)
    if deadline is not None and time.monotonic() > deadline:
        raise BudgetExceededError("cut pipeline exceeded its budget")
    return times.pre, times.sub, times.merge, merged


def _cut_once(circuit: Circuit, n: int, *, max_qubits: int, deadline: float | None, batched: bool = True):
    """One timed pass of the cut pipeline: (t_pre, t_sub, t_merge, state)."""
    _sync()
    t0 = time.perf_counter()
    plan = plan_cut(circuit, n)
    subs = decompose(circuit, plan)
    t_pre = time.perf_counter() - t0
    if deadline is not None and time.monotonic() > deadline:
        raise BudgetExceededError("cut pipeline exceeded its budget during preprocessing")
    t0 = time.perf_counter()
    if batched:
        from .engine import StateVec

        states = []
        if deadline is None:
            # every family in one batched launch sequence, families concurrently
            # on side streams (pipeline.simulate_families)
            from .pipeline import simulate_families

            batches = simulate_families(subs.segments, max_qubits=max_qubits)
        else:
            batches = [simulate_family(fam, deadline=deadline, max_qubits=max_qubits) for fam in subs.segments]
        for fam, batch in zip(subs.segments, batches):
            nq, dt = fam.num_qubits, np.complex128
            states.append([StateVec.batch_row(nq, batch, v, dt) for v in range(fam.num_variants)])
    else:
        states = [[simulate(c, max_qubits=max_qubits, deadline=deadline) for c in fam.circuits]
                  for fam in subs.segments]
    _sync()
    t_sub = time.perf_counter() - t0
    t0 = time.perf_counter()
    merged = merge(merge_input_from(subs, states), max_qubits=max_qubits, deadline=deadline)
    _sync()
    t_merge = time.perf_counter() - t0
    return t_pre, t_sub, t_merge, merged


def _orig_once(circuit: Circuit, *, max_qubits: int, deadline: float | None):
    _sync()
    t0 = time.perf_counter()
    state = simulate(circuit, max_qubits=max_qubits, deadline=deadline)
    _sync()
    return time.perf_counter() - t0, state


def _mean_std(values: Sequence[float], skip: int):
    vals = values[skip:] if len(values) > skip else values
    if not vals:
        return math.nan, math.nan
    mean = sum(vals) / len(vals)
    if len(vals) < 2:
        return mean, 0.0
    return mean, math.sqrt(sum((v - mean) ** 2 for v in vals) / (len(vals) - 1))


def measure(spec, repetitions: int = 10, *, budget: float | None = None,
            max_qubits: int = DEFAULT_MAX_QUBITS, discard_warmup: bool = False,
            pipelines: tuple[str, ...] = ("cut", "orig"), cut_path: str = "api") -> TimingBreakdown:
    """Measure one configuration: phase-timed cut pipeline plus uncut baseline
    (same protocol as the reference `measure`, harness.py:154-244).
    cut_path "api": the drop-in Python API stage by stage (plan_cut +
    decompose, simulate per family, merge_input_from + merge), as the
    reference times itself; "native": the same stages inside one
    cs_cut_run call (C++ preprocess, event-timed device stages)."""
    if cut_path not in ("api", "native"):
        raise ValidationError(f"cut_path must be 'api' or 'native', got {cut_path!r}")
    cut_once = _cut_once if cut_path == "api" else _cut_once_native
    if repetitions < 1:
        raise ValidationError(f"repetitions must be >= 1, got {repetitions}")
    unknown = set(pipelines) - {"cut", "orig"}
    if unknown:
        raise ValidationError(f"unknown pipelines: {sorted(unknown)}")
    circuit = build(spec)
    _device.require_cuda()
    samples: dict[str, list[float]] = {"pre": [], "sub": [], "merge": [], "orig": []}
    cut_timeout = orig_timeout = False
    # the first call of each pipeline builds (and, with the "jit" option,
    # NVRTC-compiles) its device programs: run both once untimed, as the
    # reference's warm_up() keeps numba compilation out of its timers
    # (harness.py:95-111)
    if "cut" in pipelines:
        try:
            cut_once(circuit, spec.n, max_qubits=max_qubits, deadline=None)
        except BudgetExceededError:
            pass
    if "orig" in pipelines and (budget is None or circuit.num_qubits <= 26):
        _orig_once(circuit, max_qubits=max_qubits, deadline=None)
    for _ in range(repetitions):
        if "cut" in pipelines and not cut_timeout:
            deadline = time.monotonic() + budget if budget is not None else None
            try:
                t_pre, t_sub, t_merge, merged = cut_once(circuit, spec.n, max_qubits=max_qubits,
                                                          deadline=deadline)
                samples["pre"].append(t_pre)
                samples["sub"].append(t_sub)
                samples["merge"].append(t_merge)
                del merged
            except BudgetExceededError:
                cut_timeout = True
            gc.collect()
        if "orig" in pipelines and not orig_timeout:
            deadline = time.monotonic() + budget if budget is not None else None
            try:
                t_orig, state = _orig_once(circuit, max_qubits=max_qubits, deadline=deadline)
                samples["orig"].append(t_orig)
                del state
            except BudgetExceededError:
                orig_timeout = True
            gc.collect()
    skip = 1 if discard_warmup else 0
    t_pre, pre_std = _mean_std(samples["pre"], skip)
    t_sub, sub_std = _mean_std(samples["sub"], skip)
    t_merge, merge_std = _mean_std(samples["merge"], skip)
    t_orig, orig_std = _mean_std(samples["orig"], skip)
    if "cut" not in pipelines or cut_timeout:
        t_pre = t_sub = t_merge = math.nan
    if "orig" not in pipelines or orig_timeout:
        t_orig = math.nan
    t_cut = t_pre + t_sub + t_merge
    delta = (t_cut - t_orig) / t_orig if math.isfinite(t_cut) and math.isfinite(t_orig) else math.nan
    timed_out = [name for name, flag in (("cut", cut_timeout), ("orig", orig_timeout)) if flag]
    status = "timeout-" + "+".join(timed_out) if timed_out else "ok"
    return TimingBreakdown(
        q=spec.q, n=spec.n, c_total=spec.c_total, depth=circuit.depth, gate_count=circuit.gate_count,
        t_pre=t_pre, t_sub=t_sub, t_merge=t_merge, t_cut=t_cut, t_orig=t_orig, delta=delta,
        reps=repetitions, status=status, blocks=getattr(spec, "blocks", 0),
        pad_exponent=getattr(spec, "depth_pad_exponent", None), t_pre_std=pre_std, t_sub_std=sub_std,
        t_merge_std=merge_std, t_orig_std=orig_std, samples=samples,
    )


def format_csv(rows: Sequence[TimingBreakdown]) -> str:
    """The reference CSV schema (harness.py:41-45, 583-593)."""
    buf = StringIO()
    buf.write(",".join(CSV_COLUMNS) + "\n")
    for r in rows:
        vals = [r.q, r.n, r.c_total, r.depth, r.gate_count, r.t_pre, r.t_sub, r.t_merge, r.t_cut, r.t_orig,
                r.delta, r.reps, r.status, SCHEMA_VERSION]
        buf.write(",".join(f"{v:.9g}" if isinstance(v, float) else str(v) for v in vals) + "\n")
    return buf.getvalue()
