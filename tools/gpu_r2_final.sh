# Round-2 evidence on the current build: the driver's sequence (GPU tests, smoke, default
# bench line), bf16 / KAT-S / fused-step lines, the reference arm, launch lists with DRAM
# bytes, and ncu --set full captures of the dominant kernels.  usage: bash tools/gpu_r2_final.sh TAG
TAG=${1:-r2z}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu_${TAG}.txt 2>&1
lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/gpu_${TAG}.txt
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_${TAG}.txt 2>&1; tail -1 gpurun_out/pytest_gpu_${TAG}.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.txt 2>&1; tail -1 gpurun_out/smoke_${TAG}.txt
timeout 900 python bench.py > gpurun_out/bench_${TAG}_fp32.json 2> gpurun_out/bench_${TAG}_fp32.err; cut -c1-200 gpurun_out/bench_${TAG}_fp32.json
for cfg in kat-b kat-s; do for dt in fp32 bf16; do for fs in "" "--fused-step"; do
  timeout 300 python bench.py --config $cfg --dtype $dt $fs --no-cpu-baseline > gpurun_out/bench_${TAG}_${cfg}_${dt}${fs}.json 2>/dev/null
  python - <<PY
import json
d = json.load(open("gpurun_out/bench_${TAG}_${cfg}_${dt}${fs}.json")); k = d["kernels"]
print("${cfg} ${dt} ${fs}", "value %.3e ms %.4f roofline %.3f" % (d["value"], d["ms_per_step"], d["roofline"]["frac"]),
      "fwd %s bwd %s" % (k.get("fwd_us"), k.get("bwd_us")), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
PY
done; done; done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_${TAG}_reference.json 2> gpurun_out/bench_${TAG}_reference.err; cut -c1-200 gpurun_out/bench_${TAG}_reference.json
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv"
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --strategy blocked"
for cfg in kat-b kat-s; do for dt in fp32 bf16; do
  timeout 600 ncu $M --log-file gpurun_out/launches_${TAG}_${cfg}_${dt}.csv $B --config $cfg --dtype $dt > /dev/null 2>&1
done; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${TAG}_default.csv python bench.py --steps 2 --warmup 3 > /dev/null 2>&1
F="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --strategy blocked"
# full captures are exported to CSV on the box (raw page + SASS source page) and the
# .ncu-rep removed: gpurun copies back at most 64 MiB
cap() {  # name kernel-regex extra-args
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$2" -s 3 -c 1 -o gpurun_out/prof_${TAG}_$1 $F $3 > /dev/null 2>&1
  ncu -i gpurun_out/prof_${TAG}_$1.ncu-rep --page raw --csv > gpurun_out/prof_${TAG}_$1_raw.csv 2>/dev/null
  ncu -i gpurun_out/prof_${TAG}_$1.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/prof_${TAG}_$1_sass.csv.gz
  rm -f gpurun_out/prof_${TAG}_$1.ncu-rep
}
cap bwd_fp32 k_bwd_staged ""
cap bwd_bf16 k_bwd_staged "--dtype bf16"
cap fwd_fp32 k_fwd ""
cap fwd_bf16 k_fwd "--dtype bf16"
ls -la gpurun_out | grep $TAG
