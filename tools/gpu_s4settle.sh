# Fresh box: GPU tests, smoke, then the default line after a 20 s idle wait (the driver's order plus a pause):
# does the first line's ~6% HBM deficit come from background work left by the previous processes?
TAG=${1:-s4s1}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_${TAG}.txt 2>&1; tail -1 gpurun_out/pytest_gpu_${TAG}.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.txt 2>&1; tail -1 gpurun_out/smoke_${TAG}.txt
nvidia-smi --query-gpu=utilization.gpu,utilization.memory --format=csv,noheader; sleep 20; nvidia-smi --query-gpu=utilization.gpu,utilization.memory --format=csv,noheader
for i in 1 2; do
  timeout 900 python bench.py > gpurun_out/bench_${TAG}_default_$i.json 2> gpurun_out/bench_${TAG}_default_$i.err
  python -c "import json; d=json.load(open('gpurun_out/bench_${TAG}_default_$i.json')); k=d['kernels']; c=d['clocks']; print('run $i value %.3e fwd %.1f bwd %.1f' % (d['value'], k['fwd_us'], k['bwd_us']), c['sm_mhz'], c.get('mem_mhz'), c['reasons'], c.get('temp_c'))"
done
