# Full GPU suite on the current build; KAT-S bf16 with the table forced on/off; bench lines
# across run_bench's workload surface at KAT-B E (groups 1/16/64, degrees (3,2)).
TAG=${1:-r2f}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_${TAG}.txt 2>&1; tail -3 gpurun_out/pytest_gpu_${TAG}.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.txt 2>&1; tail -1 gpurun_out/smoke_${TAG}.txt
for lut in 1 0; do
  GRKAN_LUT=$lut timeout 300 python bench.py --config kat-s --dtype bf16 --steps 50 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_${TAG}_kat-s_bf16_lut${lut}.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/bench_${TAG}_kat-s_bf16_lut${lut}.json')); k=d['kernels']; print('kat-s bf16 lut=$lut fwd %.1f bwd %.1f (%.3f) value %.3e' % (k['fwd_us'], k['bwd_us'], k['bwd_frac'], d['value']))"
done
for dt in fp32 bf16; do
  for g in 1 16 64; do
    timeout 300 python bench.py --config kat-b --groups $g --dtype $dt --steps 30 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_${TAG}_g${g}_${dt}.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/bench_${TAG}_g${g}_${dt}.json')); k=d['kernels']; print('g$g $dt', 'bwd=%.1fus(%.3f)'%(k['bwd_us'],k['bwd_frac']), 'fwd=%.1fus(%.3f)'%(k['fwd_us'],k['fwd_frac']), 'value %.3e frac %.3f'%(d['value'], d['roofline']['frac']), d['clocks']['sm_mhz'])"
  done
  timeout 300 python bench.py --config kat-b --num-coeffs 4 --den-coeffs 2 --dtype $dt --steps 30 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_${TAG}_deg32_${dt}.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/bench_${TAG}_deg32_${dt}.json')); k=d['kernels']; print('deg(3,2) $dt', 'bwd=%.1fus(%.3f)'%(k['bwd_us'],k['bwd_frac']), 'fwd=%.1fus(%.3f)'%(k['fwd_us'],k['fwd_frac']), 'value %.3e'%d['value'], d['clocks']['sm_mhz'])"
done
