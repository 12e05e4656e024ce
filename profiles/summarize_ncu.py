"""Summarise ncu captures brought back in gpurun_out/ into profiles/ (run here,
no GPU needed):  python profiles/summarize_ncu.py <tag> <rep> [<rep>...]
Writes profiles/<tag>_ncu_full.json; tags starting with "r" (the round's
bench capture of the merge kernel) also refresh profiles/ncu_summary.json,
which bench.py reads for the roofline's `traffic`."""
import csv
import io
import json
import os
import subprocess
import sys

KEYS = [
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second", "lts__t_bytes.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__average_warp_latency_issue_stalled_barrier",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__cluster_dim_x",
    "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
]

UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
              "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for row in rows[2:]:
        d = {"kernel": row[hdr.index("Kernel Name")]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                val = row[i].replace(",", "")
                try:
                    v = float(val) * UNIT_SCALE.get(units[i], 1.0)
                except ValueError:
                    v = val
                d[k] = v
        res.append(d)
    return res


def main():
    tag, reps = sys.argv[1], sys.argv[2:]
    here = os.path.dirname(os.path.abspath(__file__))
    summary = {}
    for rep in reps:
        for d in raw(rep):
            name = d["kernel"].split("(")[0].split("<")[0].replace("void ", "").strip()
            summary.setdefault(name, []).append(d)
    with open(os.path.join(here, f"{tag}_ncu_full.json"), "w") as fh:
        json.dump(summary, fh, indent=1)
    agg = {}
    for name, lst in summary.items():
        b = [x.get("dram__bytes_read.sum", 0) + x.get("dram__bytes_write.sum", 0) for x in lst]
        agg[name] = {"dram_bytes_per_launch": sum(b) / len(b), "launches_captured": len(lst),
                     "duration_s": sum(x.get("gpu__time_duration.sum", 0) for x in lst) / len(lst)}
    if tag.startswith("r") and "_" not in tag:
        with open(os.path.join(here, "ncu_summary.json"), "w") as fh:
            json.dump({"round": tag, **agg}, fh, indent=1)
    print(json.dumps(agg, indent=1))


if __name__ == "__main__":
    main()
