#!/usr/bin/env python
"""Benchmark of the B200 circuit-cutting path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one pass of the cut pipeline over the BASELINE cfg4a circuit
(q=30, d=10, n=2 (15|15), c_total=2, seeded U3 brick-wall, complex128):
host preprocess (plan_cut + decompose) -> batched subcircuit simulation
(sm_100a sweep kernel) -> chain merge writing the 16 GiB state once
(sm_100a merge kernel). ``value`` = 2^30 amplitudes x steps / device time
with the output resident in HBM; ``e2e`` = the same through the public API
delivering the state into pinned HOST memory (device->host copy in the
timed region). Multi-GPU (torchrun): the output is sharded by its high
amplitude bits, subcircuit variants are split across ranks and all-gathered
over NCCL; value is whole-job (strong scaling, total work fixed).

``--impl reference`` times the reference algorithm's CPU implementation
(the C restatement of the reference numba kernels in oracle/, all host
threads) on a bounded sample of the same workload, extrapolated to the
same metric.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "End-to-end cut-sim amplitudes/s at q=30; merge % of HBM roofline; stage ms"
UNIT = "amplitudes/s"
WORKLOAD = "cfg4a"


DFMA_PEAK_TF = 36.5  # measured on this B200 pool (tools/fp64_peak.cu)


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md)"


def load_traffic():
    """dram bytes read+write per merge launch from the committed ncu capture."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return d.get("merge_kernel", {}).get("dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


def load_dram_pct():
    """ncu's dram throughput (% of its DRAM peak) for the committed capture of
    the same merge launch, for reading `frac` (which is against the measured
    read+write copy rate) next to the DRAM-peak view."""
    path = os.path.join(ROOT, "profiles", "r01_ncu_full.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return float(d["merge_kernel"][0]["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"])
    except (OSError, ValueError, KeyError, IndexError, TypeError):
        return None


class ClockSampler:
    """SM clocks and throttle reasons sampled every few ms during the timed
    region (NVML through nvidia_ml_py; nvidia-smi as a fallback)."""

    REASONS = {  # NVML clocks-event-reason bits
        0x0000000000000004: "sw_power_cap",
        0x0000000000000008: "hw_slowdown",
        0x0000000000000020: "sw_thermal_slowdown",
        0x0000000000000040: "hw_thermal_slowdown",
        0x0000000000000080: "hw_power_brake_slowdown",
    }

    def __init__(self, index: int, interval: float = 0.005):
        self.index = index
        self.interval = interval
        self.samples = []
        self._stop = threading.Event()
        self._thr = None
        self._nvml = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001
            self._nvml = None
            self.max_mhz = None

    def _sample_nvml(self):
        nv = self._nvml
        sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
        try:
            bits = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
        except AttributeError:
            bits = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
        return sm, bits

    def _run(self):
        while not self._stop.is_set():
            try:
                if self._nvml is not None:
                    sm, bits = self._sample_nvml()
                    self.samples.append((float(sm), [n for b, n in self.REASONS.items() if bits & b]))
                else:
                    out = subprocess.run(
                        ["nvidia-smi", "-i", str(self.index),
                         "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                         "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits"],
                        capture_output=True, text=True, timeout=5)
                    v = [x.strip() for x in out.stdout.strip().split(",")]
                    if len(v) == 6:
                        self.max_mhz = float(v[1])
                        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
                        self.samples.append((float(v[0]), [names[i] for i in range(4) if v[2 + i] == "Active"]))
            except Exception:  # noqa: BLE001
                return
            self._stop.wait(self.interval)

    def __enter__(self):
        self._thr = threading.Thread(target=self._run, daemon=True)
        self._thr.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._thr:
            self._thr.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"], "samples": 0}
        sm = [s for s, _ in self.samples]
        reasons = sorted({r for _, rs in self.samples for r in rs})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(self.samples), "source": "nvml" if self._nvml else "nvidia-smi"}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------------------
# CPU reference arm: the C restatement of the reference kernels (oracle/)
# ---------------------------------------------------------------------------
def cpu_sample(spec, threads: int, row_fraction: float):
    """Time preprocess + all subcircuit simulations + a row sample of the merge
    with the reference's algorithm on the host; extrapolate to the full step."""
    from oracle import cutbench_oracle as orc
    from oracle import oracle_c
    from paper_2603_01443_b200.generators import build_brickwall

    circ = build_brickwall(spec)
    k, qa, qb, p = circ.kinds, circ.qa, circ.qb, circ.params
    q, n = spec.q, spec.n
    sizes = [q // n] * n
    t0 = time.perf_counter()
    bgs, counts, _ = orc.plan(k, qa, qb, sizes)
    variants = [orc.segment_variants(k, qa, qb, p, sizes, bgs, s) for s in range(n)]
    tab = orc.merge_table(n, bgs, sum(counts))
    co = orc.coefficients(sum(counts))
    t_pre = time.perf_counter() - t0
    t0 = time.perf_counter()
    states = [[oracle_c.simulate(sizes[s], *v, threads=threads) for v in variants[s]] for s in range(n)]
    t_sub = time.perf_counter() - t0
    rows_total = 1 << sizes[1]
    rows = max(1, int(rows_total * row_fraction))
    _acc, t_m = oracle_c.merge_rows(states, tab, co, (0, rows), threads=threads)
    t_merge = t_m * rows_total / rows
    return {"t_pre": t_pre, "t_sub": t_sub, "t_merge": t_merge,
            "value": (1 << q) / (t_pre + t_sub + t_merge), "rows": rows, "rows_total": rows_total}


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    from oracle import oracle_c
    from paper_2603_01443_b200.generators import BASELINE_CONFIGS

    spec = BASELINE_CONFIGS[WORKLOAD]
    # all host threads this process may use (torchrun sets OMP_NUM_THREADS=1
    # for its workers; the C port passes num_threads explicitly)
    try:
        host_threads = len(os.sched_getaffinity(0))
    except AttributeError:
        host_threads = os.cpu_count() or oracle_c.max_threads()
    threads = host_threads if args.threads <= 0 else args.threads
    frac = args.row_fraction
    for _ in range(args.warmup):
        cpu_sample(spec, threads, frac / 8)
    vals, steps = [], []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        r = cpu_sample(spec, threads, frac)
        vals.append(r["value"])
        steps.append(r)
    wall = time.perf_counter() - t0
    value = float(np.mean(vals))
    ms = 1e3 * (1 << spec.q) / value
    sample = (f"per step: full preprocess + all {sum(1 << c for c in [spec.c_total] * spec.n)} "
              f"subcircuit states + merge rows [0, {steps[0]['rows']}) of {steps[0]['rows_total']} "
              f"(fraction {frac}); merge time extrapolated by row count")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{WORKLOAD}: q=30 d=10 n=2 c_total=2 seed=0 (U3 brick-wall)",
                   "q": spec.q, "n": spec.n, "c_total": spec.c_total, "d": spec.d},
        "stage_ms": {"pre": 1e3 * np.mean([s["t_pre"] for s in steps]),
                     "sub": 1e3 * np.mean([s["t_sub"] for s in steps]),
                     "merge": 1e3 * np.mean([s["t_merge"] for s in steps])},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": sample, "wall_s": wall},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def run_ours(args):
    import torch

    import paper_2603_01443_b200 as cb
    from paper_2603_01443_b200 import _native
    from paper_2603_01443_b200.generators import BASELINE_CONFIGS
    from paper_2603_01443_b200.parallel import run_cut_sharded
    from paper_2603_01443_b200.pipeline import host_workspace_bytes, preprocess, run_cut_to_host

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    comm = None
    if world > 1:
        # the pipeline's one exchange goes through libcutsim's NCCL binding
        from paper_2603_01443_b200.comm import NcclComm

        comm = NcclComm.create(rank, world)
    spec = BASELINE_CONFIGS[WORKLOAD]
    circ = cb.build_brickwall(spec)
    q = spec.q
    total = 1 << q
    stream = torch.cuda.current_stream()
    # NVRTC-specialise the sweep programs on first use: compiled during the
    # warm-up steps, outside the timed region (as the reference's warm_up()
    # keeps numba JIT out of its timers, harness.py:95-111)
    _native.set_option("jit", 0 if args.no_jit else 2)
    peak, peak_src = load_peaks()

    # shard geometry and preallocated output / workspace
    prep0 = preprocess(circ, spec.n)
    ws_bytes, qlow, _c = _native.cut_workspace(q, circ.table, [q // spec.n] * spec.n)
    bond = prep0.chain.plan()[1]
    from paper_2603_01443_b200.parallel import shard_range

    begin, end = shard_range(q, world, rank, qlow)
    out = torch.empty(end - begin, dtype=torch.complex128, device="cuda")
    workspace = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device="cuda")

    merge_ms = []

    def step(record=False):
        if world == 1:
            # one native call: C++ preprocess -> batched variant sweeps -> chain merge
            evs = None
            if record:
                evs = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            cb.run_cut(circ, spec.n, out=out, workspace=workspace, events=evs)
            if record:
                merge_ms.append((evs[1], evs[2]))
        else:
            timers = {} if record else None
            res, _ = run_cut_sharded(circ, spec.n, rank=rank, world=world, out=out, merge_events=timers,
                                     comm=comm)
            if record:
                merge_ms.append((timers["start"], timers["end"]))
            del res

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = _native.launch_count()
    ev_start = torch.cuda.Event(enable_timing=True)
    ev_end = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        ev_start.record(stream)
        for _ in range(args.steps):
            step(record=True)
        ev_end.record(stream)
        torch.cuda.synchronize()
    launches = _native.launch_count() - launches0
    elapsed = ev_start.elapsed_time(ev_end) / 1e3
    if dist:
        tt = torch.tensor([elapsed], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        elapsed = float(tt.item())
        dist.barrier()
    torch.cuda.synchronize()
    value = total * args.steps / elapsed
    ms_per_step = 1e3 * elapsed / args.steps

    # stage breakdown (separate, synchronised pass; not the headline)
    times = cb.StageTimes()
    stage = {"pre": None, "sub": None, "merge": None}
    if world == 1:
        acc = {"pre": [], "sub": [], "merge": []}
        for _ in range(3):
            cb.run_cut(circ, spec.n, out=out, workspace=workspace, timers=times)
            acc["pre"].append(times.pre)
            acc["sub"].append(times.sub)
            acc["merge"].append(times.merge)
        stage = {k: 1e3 * float(np.median(v)) for k, v in acc.items()}

    # the uncut simulator on the same circuit (the cut-vs-uncut comparison point)
    uncut_ms = None
    uncut = None
    if world == 1 and not args.no_uncut:
        cb.simulate(circ)  # builds (and JIT-compiles) the uncut program
        torch.cuda.synchronize()
        u0 = torch.cuda.Event(enable_timing=True)
        u1 = torch.cuda.Event(enable_timing=True)
        u0.record(stream)
        sv = cb.simulate(circ)
        u1.record(stream)
        u1.synchronize()
        uncut_ms = u0.elapsed_time(u1)
        del sv
        torch.cuda.empty_cache()
        # per-sweep HBM rate and FP64 use of the uncut simulator.
        # Started from |0..0>, sweep k launches only its 2^z_k tiles that can be
        # non-zero (the state is zeroed once: 16 B per amplitude written), so the
        # algorithmic traffic is 32 B per amplitude of the launched tiles.
        plan = json.loads(_native.sweep_plan_json(q, circ.table))
        n_sweeps = len(plan["sweeps"])
        sparse = _native.get_option("zero_start_tiles") == 1
        n_dense = 0
        amps_swept = 0
        dense_amps = 0
        for sw in plan["sweeps"]:
            ents, i, nd = sw["entries"], 0, 0
            while i < len(ents):  # a slotted op occupies two entries
                nd += ents[i]["type"] == 0
                i += 2 if ents[i]["slot"] >= 0 else 1
            tiles = 1 << (sw["z"] if sparse else q - sw["T"])
            amps = tiles << sw["T"]
            n_dense += nd
            amps_swept += amps
            dense_amps += nd * amps
        t = uncut_ms / 1e3
        traffic = 32.0 * amps_swept + (16.0 * total if sparse else 0.0)
        uncut = {"ms": uncut_ms, "sweeps": n_sweeps, "dense_ops": n_dense,
                 "sweeps_full_equivalent": amps_swept / total,
                 "hbm_gbs": traffic / t / 1e9,
                 "hbm_frac": traffic / t / 1e9 / peak,
                 "fp64_tflops_alg": 16.0 * dense_amps / t / 1e12,
                 "fp64_frac_of_dfma_peak": 16.0 * dense_amps / t / 1e12 / DFMA_PEAK_TF,
                 "note": "32 B/amplitude per launched tile per sweep (read+write) + the 16 B/amplitude zeroing; "
                         "only the tiles that can be non-zero from |0..0> are launched (z per sweep); "
                         "8 FMA (16 flop) per amplitude per dense 2x2 op; DFMA peak 36.5 TF/s measured "
                         "with tools/fp64_peak.cu"}

    # the same merge with more cut terms (cfg5 c=4 / threshold region): the
    # int8 tcgen05 kernel (exact FP64 splitting) vs the FP64 tensor-core 3M
    # kernel, on the preallocated output (informational, not the headline)
    int8_merge = None
    if world == 1 and not args.no_uncut:
        from paper_2603_01443_b200.merging import merge_terms_device

        g = torch.Generator(device="cuda").manual_seed(0)
        int8_merge = {}
        for K in (16, 64):
            hi = torch.randn(K, 1 << (q - q // 2), dtype=torch.complex128, device="cuda", generator=g) / 4
            lo = torch.randn(K, 1 << (q // 2), dtype=torch.complex128, device="cuda", generator=g) / 4
            idx = np.arange(K)
            coef = np.exp(1j * np.arange(K)) / np.sqrt(K)
            res = {}
            for name, oz in (("int8_tcgen05", 1), ("fp64_dmma_3m", 0)):
                _native.set_option("merge_ozaki", oz)
                merge_terms_device(hi, lo, idx, idx, coef, out=out.view(1, -1))
                torch.cuda.synchronize()
                m0 = torch.cuda.Event(enable_timing=True)
                m1 = torch.cuda.Event(enable_timing=True)
                m0.record(stream)
                for _ in range(3):
                    merge_terms_device(hi, lo, idx, idx, coef, out=out.view(1, -1))
                m1.record(stream)
                m1.synchronize()
                res[name] = m0.elapsed_time(m1) / 3
            _native.set_option("merge_ozaki", 1)
            t = res["int8_tcgen05"] / 1e3
            int8_merge[f"K{K}"] = {"ms": res["int8_tcgen05"], "fp64_dmma_3m_ms": res["fp64_dmma_3m"],
                                   "out_gbs": 16.0 * total / t / 1e9,
                                   "fp64_tflops_alg": 8.0 * K * total / t / 1e12}
            del hi, lo
        int8_merge["note"] = ("q=30 rank-K product out[h][l] = sum_t c_t hi_t[h] lo_t[l] (n=2 merge with K cut "
                              "terms) into the 16 GiB output: int8 tcgen05.mma with 8 base-128 digits per FP64 "
                              "operand (max|d| vs DFMA ~1e-16) vs the FP64 tensor-core 3M kernel; 8K flop per "
                              "output algorithmic")

    # roofline of the dominant kernel (merge) from the timed region
    roofline = None
    if merge_ms:
        dur = float(np.mean([a.elapsed_time(b) for a, b in merge_ms])) / 1e3
        fams = prep0.subs.segments
        in_bytes = sum(f.num_variants * (1 << f.num_qubits) * 16 for f in fams)
        alg = 16 * (end - begin) + in_bytes
        achieved = alg / dur / 1e9
        roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak, "traffic": load_traffic(), "kernel": "merge_kernel",
                    "algorithmic_bytes_per_launch": alg, "avg_launch_ms": dur * 1e3,
                    "peak_source": peak_src, "ncu_dram_pct_of_peak": load_dram_pct()}

    # e2e through the public API into pinned host memory (N=1)
    e2e = None
    if world == 1 and not args.no_e2e:
        host = torch.empty(total, dtype=torch.complex128, pin_memory=True)
        del out
        torch.cuda.empty_cache()
        hws = torch.empty(host_workspace_bytes(circ, spec.n), dtype=torch.uint8, device="cuda")
        for _ in range(max(1, min(args.warmup, 2))):
            run_cut_to_host(circ, spec.n, host, workspace=hws)
        torch.cuda.synchronize()
        e_steps = max(1, min(args.steps, args.e2e_steps))
        t0 = time.perf_counter()
        for _ in range(e_steps):
            run_cut_to_host(circ, spec.n, host, workspace=hws)
        torch.cuda.synchronize()
        t_e2e = (time.perf_counter() - t0) / e_steps
        g_bytes = int(sum(a.nbytes for a in (circ.kinds, circ.qa, circ.qb, circ.params)))
        # the bound of this leg: a plain pinned device->host copy of the same bytes
        del hws
        chunk = torch.empty(total // 8, dtype=torch.complex128, device="cuda")
        c0 = torch.cuda.Event(enable_timing=True)
        c1 = torch.cuda.Event(enable_timing=True)
        host_view = host[: chunk.numel()]
        host_view.copy_(chunk, non_blocking=True)
        c0.record(stream)
        for _ in range(4):
            host_view.copy_(chunk, non_blocking=True)
        c1.record(stream)
        c1.synchronize()
        d2h_gbs = 4 * chunk.numel() * 16 / (c0.elapsed_time(c1) / 1e3) / 1e9
        e2e = {"value": total / t_e2e, "unit": UNIT, "h2d_bytes_per_step": g_bytes,
               "d2h_bytes_per_step": total * 16, "ms_per_step": t_e2e * 1e3, "steps": e_steps,
               "path": "run_cut_to_host -> cs_cut_run_to_host (C-ABI, host buffer): chunked merge "
                       "overlapped with D2H into pinned host memory",
               "bound": {"kind": "pcie_d2h", "measured_copy_gbs": d2h_gbs,
                         "achieved_gbs": total * 16 / t_e2e / 1e9,
                         "frac": total * 16 / t_e2e / 1e9 / d2h_gbs}}
        del host, chunk

    # e2e at N > 1 (or --sharded-e2e at N = 1): every rank runs the sharded
    # pipeline (parallel.run_cut_sharded: its variant slice, the NCCL
    # all-gather, its output rows) and copies its shard into pinned host memory
    # over its own PCIe link; time = max over ranks, value = whole job
    if (world > 1 or args.sharded_e2e) and not args.no_e2e:
        if comm is None:  # --sharded-e2e at one rank: a world-1 NCCL communicator
            from paper_2603_01443_b200.comm import NcclComm

            comm = NcclComm.create(rank, world)
        if "out" not in locals() or out is None:
            out = torch.empty(end - begin, dtype=torch.complex128, device="cuda")
        host = torch.empty(end - begin, dtype=torch.complex128, pin_memory=True)
        g_bytes = int(sum(a.nbytes for a in (circ.kinds, circ.qa, circ.qb, circ.params)))

        def e2e_step():
            res, _ = run_cut_sharded(circ, spec.n, rank=rank, world=world, out=out, comm=comm)
            host.copy_(res, non_blocking=True)
            torch.cuda.synchronize()
            del res

        for _ in range(max(1, min(args.warmup, 2))):
            e2e_step()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        e_steps = max(1, min(args.steps, args.e2e_steps))
        t0 = time.perf_counter()
        for _ in range(e_steps):
            e2e_step()
        t_rank = (time.perf_counter() - t0) / e_steps
        if dist:
            tt = torch.tensor([t_rank], device="cuda", dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t_rank = float(tt.item())
        e2e = {"value": total / t_rank, "unit": UNIT, "h2d_bytes_per_step": g_bytes * world,
               "d2h_bytes_per_step": total * 16, "ms_per_step": t_rank * 1e3, "steps": e_steps,
               "path": (f"parallel.run_cut_sharded on {world} rank(s) (variant slices, NCCL all-gather, "
                        f"output rows [{begin}, {end}) per rank) + device->host copy of each shard into "
                        "pinned host memory over the rank's own PCIe link; max over ranks")}
        del host

    # CPU baseline (the oracle port, 1 thread = the reference's protocol), rank 0, N=1
    cpu = None
    if world == 1 and not args.no_cpu:
        try:
            r = cpu_sample(spec, 1, args.row_fraction)
            cpu = {"value": r["value"], "unit": UNIT, "cores": 1, "kind": "port",
                   "sample": (f"oracle C port (reference loop structure), 1 thread: full preprocess, all "
                              f"subcircuit states, merge rows [0,{r['rows']}) of {r['rows_total']} "
                              f"extrapolated"),
                   "stage_ms": {"pre": r["t_pre"] * 1e3, "sub": r["t_sub"] * 1e3,
                                "merge": r["t_merge"] * 1e3},
                   "host_cpus": os.cpu_count()}
        except Exception as exc:  # noqa: BLE001  (baseline is informational)
            cpu = {"value": None, "unit": UNIT, "cores": 1, "kind": "port", "sample": f"failed: {exc}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded U3 brick-wall, SURVEY.md §8(d)); output resident in HBM",
            "config": {"workload": f"{WORKLOAD}: q=30 d=10 n=2 (15|15) c_total=2 seed=0 complex128",
                       "q": q, "n": spec.n, "c_total": spec.c_total, "d": spec.d, "bond": bond,
                       "parallelism": f"output-shard{world}",
                       "l2": "no flush: each step writes the 16 GiB output (>> 126 MB L2)"},
            "stage_ms": stage,
            "uncut_ms": uncut_ms,
            "uncut": uncut,
            "int8_merge": int8_merge,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": clocks.summary(),
            "gpu_launches": launches,
            "jit": _native.get_option("jit"),
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--threads", type=int, default=0, help="reference arm host threads (0 = all)")
    ap.add_argument("--row-fraction", type=float, default=1 / 16,
                    help="merge rows sampled by the CPU legs")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--sharded-e2e", action="store_true",
                    help="N=1: measure e2e through the sharded (multi-GPU) path instead (its test at one rank)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-uncut", action="store_true")
    ap.add_argument("--no-jit", action="store_true", help="interpreter sweep kernels only")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
