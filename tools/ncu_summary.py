"""Summarise ncu --set full captures into profiles/ JSON.

    python tools/ncu_summary.py OUT.json NAME=path.ncu-rep [NAME=path.ncu-rep ...]
    (path may also be the raw-page CSV exported on the box: ncu -i REP --page raw --csv)

Keeps the metrics the docs cite: duration, DRAM bytes, pipe utilisation
(FMA / ALU / tensor), issue activity, the top stall reasons and the global
atomic / reduction counts (must be 0 on the product path).
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed_op_global_red.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_atom.sum",
    "l1tex__t_requests_pipe_lsu_mem_global_op_red.sum", "sass__inst_executed_local_loads",
]
STALLS = ["long_scoreboard", "math_pipe_throttle", "wait", "not_selected", "short_scoreboard", "dispatch_stall",
          "barrier", "branch_resolving", "no_instruction", "mio_throttle", "lg_throttle"]


def summarise(rep):
    # a .ncu-rep, or the CSV of its raw page (ncu -i REP --page raw --csv), exported on the box
    if rep.endswith(".csv"):
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
    res = {k: list(d[k]) for k in KEYS if k in d}
    res["stalls_per_issue"] = {
        s: float(d["smsp__average_warps_issue_stalled_%s_per_issue_active.ratio" % s][0])
        for s in STALLS if "smsp__average_warps_issue_stalled_%s_per_issue_active.ratio" % s in d}
    return res


def main():
    out = sys.argv[1]
    res = {}
    for arg in sys.argv[2:]:
        name, rep = arg.split("=", 1)
        res[name] = summarise(rep)
        res[name]["source"] = rep.split("/")[-1]
    json.dump(res, open(out, "w"), indent=1)


if __name__ == "__main__":
    main()
