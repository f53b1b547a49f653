# Round-2 evidence on one GPU: the driver's round-end sequence (GPU tests, smoke, default
# bench line), the bf16 / KAT-S / fused-step lines, the reference arm, the ncu launch
# list of the default bench command and full captures of the backward kernels.
# usage: bash tools/gpu_r2_evidence.sh TAG
TAG=${1:-r2}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu_${TAG}.txt 2>&1
lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/gpu_${TAG}.txt
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_${TAG}.txt 2>&1; tail -3 gpurun_out/pytest_gpu_${TAG}.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.txt 2>&1; tail -1 gpurun_out/smoke_${TAG}.txt
timeout 900 python bench.py > gpurun_out/bench_${TAG}_fp32.json 2> gpurun_out/bench_${TAG}_fp32.err; cut -c1-300 gpurun_out/bench_${TAG}_fp32.json
for cfg in kat-b kat-s; do for dt in fp32 bf16; do
  timeout 300 python bench.py --config $cfg --dtype $dt --no-cpu-baseline > gpurun_out/bench_${TAG}_${cfg}_${dt}.json 2>/dev/null
  timeout 300 python bench.py --config $cfg --dtype $dt --fused-step --no-cpu-baseline > gpurun_out/bench_${TAG}_${cfg}_${dt}_fused.json 2>/dev/null
  python - <<EOF
import json
for f in ("gpurun_out/bench_${TAG}_${cfg}_${dt}.json", "gpurun_out/bench_${TAG}_${cfg}_${dt}_fused.json"):
    try:
        d = json.load(open(f)); k = d["kernels"]
        print(f.split("/")[-1], "value %.3e ms %.4f roofline %.3f" % (d["value"], d["ms_per_step"], d["roofline"]["frac"]),
              "fwd %s bwd %s" % (k.get("fwd_us"), k.get("bwd_us")), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
    except Exception as e:
        print(f, "failed", e)
EOF
done; done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_${TAG}_reference.json 2> gpurun_out/bench_${TAG}_reference.err; cut -c1-300 gpurun_out/bench_${TAG}_reference.json
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${TAG}_fp32.csv $B > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${TAG}_bf16.csv $B --dtype bf16 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_bwd_staged" -s 3 -c 1 -o gpurun_out/prof_${TAG}_bwd_bf16 $B --dtype bf16 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_bwd_staged" -s 3 -c 1 -o gpurun_out/prof_${TAG}_bwd_fp32 $B > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_bwd_staged" -s 3 -c 1 -o gpurun_out/prof_${TAG}_fstep_bf16 $B --dtype bf16 --fused-step > /dev/null 2>&1
ls -la gpurun_out | grep $TAG
