"""Measured DRAM bytes and L2 atomics per kernel vs the access models.

Run on the GPU box (one shape per ncu process):

    for s in kat-s kat-b; do
      ncu --clock-control none --csv --log-file gpurun_out/access_$s.csv \\
          --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,\\
smsp__sass_inst_executed_op_global_red.sum,lts__t_requests_op_red.sum,lts__t_requests_op_atom.sum \\
          python tools/access_ncu.py run --shape $s
    done
    python tools/access_ncu.py summarize gpurun_out/access_kat-s.csv gpurun_out/access_kat-b.csv \\
        > profiles/r1/access_model_vs_ncu.json

`run` launches K1, K2+K3 and K4 (fp32, FAST) once each on seeded N(0,1)
inputs, after one untimed warm pass of each.  `summarize` takes the LAST launch
of every kernel name and sets it beside `paper_2505_13813_b200.access`'s
device model and the reference's element-access model (x element size).
"""
import csv
import json
import os
import sys
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SHAPES = {"kat-t": (8 * 197, 192), "kat-s": (128 * 197, 1536), "kat-b": (256 * 197, 3072)}
GROUPS = 8


def run(shape):
    import torch
    from paper_2505_13813_b200 import ops
    rows, d = SHAPES[shape]
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(rows, d, device="cuda", generator=g)
    u = torch.randn(rows, d, device="cuda", generator=g)
    a = torch.randn(GROUPS, 6, device="cuda", generator=g)
    b = torch.randn(GROUPS, 4, device="cuda", generator=g)
    for _ in range(2):
        ops.rational_forward(x, a, b)
        ops.rational_backward(x, u, a, b)
        ops.rational_backward_atomic(x, u, a, b)
    torch.cuda.synchronize()
    print(json.dumps({"shape": shape, "rows": rows, "d": d, "groups": GROUPS}))


def _kernel_family(name):
    for key, fam in (("k_bwd_atomic", "K4"), ("k_bwd_reduce", "K3"), ("k_bwd", "K2"), ("k_fwd", "K1")):
        if key in name:
            return fam
    return None


def _read_csv(path):
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    per = OrderedDict()  # (launch id) -> {metric: value, name}
    for r in csv.DictReader(lines):
        k = r["ID"]
        e = per.setdefault(k, {"name": r["Kernel Name"]})
        v = r["Metric Value"].replace(",", "")
        unit = r.get("Metric Unit", "")
        try:
            val = float(v)
        except ValueError:
            continue
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
                 "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}.get(unit, 1)
        e[r["Metric Name"]] = val * scale
    return list(per.values())


def summarize(paths):
    from paper_2505_13813_b200 import access
    out = {"_note": ("ncu --clock-control none, one launch per kernel (the last of each name), fp32 FAST, "
                     "seeded N(0,1). model_bytes: paper_2505_13813_b200.access.device_traffic; "
                     "reference_bytes: the reference's element-access model (pkg/src/grkan/access.py:89-126, "
                     "block 256) x 4 B. dram = dram__bytes_read.sum + dram__bytes_write.sum; "
                     "red_thread_ops = smsp__sass_inst_executed_op_global_red.sum x 32 (full warps)."),
           "shapes": {}}
    for path in paths:
        shape = os.path.basename(path).split("access_")[-1].rsplit(".", 1)[0]
        rows, d = SHAPES[shape]
        last = OrderedDict()
        for launch in _read_csv(path):
            fam = _kernel_family(launch["name"])
            if fam:
                last[fam] = launch
        res = {}
        for op, fams in (("fwd", ["K1"]), ("bwd", ["K2", "K3"]), ("bwd_atomic", ["K4"])):
            m = access.device_traffic(rows, d, GROUPS, "fp32", op)
            got = [last[f] for f in fams if f in last]
            dram = sum(l.get("dram__bytes_read.sum", 0) + l.get("dram__bytes_write.sum", 0) for l in got)
            red = sum(l.get("smsp__sass_inst_executed_op_global_red.sum", 0) for l in got)
            res[op] = {
                "kernels": [l["name"].split("(")[0] for l in got],
                "us": sum(l.get("gpu__time_duration.sum", 0) for l in got),
                "dram_bytes": dram,
                "model_bytes": m.total_bytes,
                "dram_over_model": dram / m.total_bytes if m.total_bytes else None,
                "reference_accesses": m.reference_accesses,
                "reference_bytes": m.reference_bytes,
                "model_atomics": m.atomics,
                "red_thread_ops": red * 32,
                "l2_red_requests": sum(l.get("lts__t_requests_op_red.sum", 0) for l in got),
                "l2_atom_requests": sum(l.get("lts__t_requests_op_atom.sum", 0) for l in got),
            }
        out["shapes"][shape] = {"rows": rows, "d": d, "groups": GROUPS, "elements": rows * d, **res}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(sys.argv[sys.argv.index("--shape") + 1])
    else:
        summarize(sys.argv[2:])
