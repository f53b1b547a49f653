# FFMA2 operand-form microbenchmark; bench lines across run_bench's workload surface (groups, degrees).
TAG=${1:-r2h}
mkdir -p gpurun_out
./tools/micro/ffma2_ops > gpurun_out/ffma2_ops_${TAG}.txt 2>&1; cat gpurun_out/ffma2_ops_${TAG}.txt
for dt in fp32 bf16; do
  for g in 1 16 64; do
    timeout 300 python bench.py --config kat-b --groups $g --dtype $dt --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_${TAG}_g${g}_${dt}.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/bench_${TAG}_g${g}_${dt}.json')); k=d['kernels']; print('g$g $dt', 'bwd=%.1fus(%.3f)'%(k['bwd_us'],k['bwd_frac']), 'fwd=%.1fus(%.3f)'%(k['fwd_us'],k['fwd_frac']), d['clocks']['sm_mhz'])"
  done
  timeout 300 python bench.py --config kat-b --num-coeffs 4 --den-coeffs 2 --dtype $dt --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_${TAG}_deg32_${dt}.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/bench_${TAG}_deg32_${dt}.json')); k=d['kernels']; print('deg(3,2) $dt', 'bwd=%.1fus(%.3f)'%(k['bwd_us'],k['bwd_frac']), 'fwd=%.1fus(%.3f)'%(k['fwd_us'],k['fwd_frac']), d['clocks']['sm_mhz'])"
done
