# Round 2 first check: GPU suite, smoke, fp32/bf16 bench lines (KAT-B, KAT-S).
TAG=${1:-r2a}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' 2>&1 | tail -2
timeout 1800 python -m pytest tests -q -m gpu -x ${PYTEST_ARGS} > gpurun_out/pytest_gpu_${TAG}.txt 2>&1; tail -15 gpurun_out/pytest_gpu_${TAG}.txt
for cfg in kat-b kat-s; do for dt in fp32 bf16; do
  timeout 600 python bench.py --config $cfg --dtype $dt --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench_${TAG}_${cfg}_${dt}.json 2> gpurun_out/bench_${TAG}_${cfg}_${dt}.err
  python -c "import json; d=json.load(open('gpurun_out/bench_${TAG}_${cfg}_${dt}.json')); k=d['kernels']; print('$cfg $dt', 'Gelem/s=%.1f'%(d['value']/1e9), 'fwd=%.1fus(%.3f)'%(k['fwd_us'],k['fwd_frac']), 'bwd=%.1fus(%.3f)'%(k['bwd_us'],k['bwd_frac']), 'clk', d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'), 'e2e', d['e2e']['value']/1e9, d['e2e'].get('reference_api',{}).get('ms_per_step'))" || tail -5 gpurun_out/bench_${TAG}_${cfg}_${dt}.err
done; done
