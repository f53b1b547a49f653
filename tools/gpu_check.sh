# usage: [NCU=1] [PYTEST=0] bash tools/gpu_check.sh TAG
TAG=${1:-run}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' 2>&1 | tail -3
if [ "${PYTEST:-1}" = "1" ]; then timeout 1500 python -m pytest tests -x -q -m gpu ${PYTEST_ARGS} 2>&1 | tail -25; fi
bench() {  # name env dtype mode
  env $2 timeout 600 python bench.py --steps 20 --warmup 5 --dtype $3 --mode $4 --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench_${TAG}_$1.json 2>gpurun_out/bench_${TAG}_$1.err
  python -c "import json,sys; d=json.load(open('gpurun_out/bench_${TAG}_$1.json')); k=d['kernels']; print('$1', 'Gelem/s=%.1f'%(d['value']/1e9), 'fwd=%.1fus(%.3f)'%(k['fwd_us'],k['fwd_frac']), 'bwd=%.1fus(%.3f)'%(k['bwd_us'],k['bwd_frac']), 'clk', d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))" || tail -5 gpurun_out/bench_${TAG}_$1.err
}
bench fp32_fast GRKAN_STAGED=1 fp32 fast
bench bf16_fast GRKAN_STAGED=1 bf16 fast
bench fp32_exact GRKAN_STAGED=1 fp32 exact
bench bf16_exact GRKAN_STAGED=1 bf16 exact
bench fp32_fast_direct GRKAN_STAGED=0 fp32 fast
bench bf16_fast_direct GRKAN_STAGED=0 bf16 fast
if [ -n "$NCU" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_bwd" -s 3 -c 1 -o gpurun_out/prof_bwd_${TAG} python bench.py --steps 4 --warmup 3 --no-cpu-baseline --e2e-steps 1 ${NCU_ARGS} > gpurun_out/ncu_bwd_${TAG}.log 2>&1; tail -2 gpurun_out/ncu_bwd_${TAG}.log
fi
