# usage: bash tools/gpu_quick.sh TAG [pytest-args]  -- parity tests + fp32/bf16 FAST benches
TAG=${1:-q}; shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu "$@" 2>&1 | tail -4
for dt in fp32 bf16; do
  timeout 300 python bench.py --steps 20 --warmup 5 --dtype $dt --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_${TAG}_$dt.json 2>gpurun_out/bench_${TAG}_$dt.err
  python -c "import json; d=json.load(open('gpurun_out/bench_${TAG}_$dt.json')); k=d['kernels']; print('$TAG $dt', 'Gelem/s=%.1f'%(d['value']/1e9), 'fwd=%.1fus(%.3f)'%(k['fwd_us'],k['fwd_frac']), 'bwd=%.1fus(%.3f)'%(k['bwd_us'],k['bwd_frac']), d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))" || tail -3 gpurun_out/bench_${TAG}_$dt.err
done
