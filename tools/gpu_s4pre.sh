# Fresh box: GPU tests, smoke, then the first default line with 16 GB mapped / touched / released first,
# then a plain default line.
TAG=${1:-s4p1}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_${TAG}.txt 2>&1; tail -1 gpurun_out/pytest_gpu_${TAG}.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.txt 2>&1; tail -1 gpurun_out/smoke_${TAG}.txt
i=0
for pre in 16 0 16; do i=$((i+1))
  GRKAN_BENCH_PREALLOC_GB=$pre timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_${TAG}_$i.json 2> gpurun_out/bench_${TAG}_$i.err
  python -c "import json; d=json.load(open('gpurun_out/bench_${TAG}_$i.json')); k=d['kernels']; c=d['clocks']; print('run $i prealloc $pre value %.3e fwd %.1f bwd %.1f' % (d['value'], k['fwd_us'], k['bwd_us']), c['sm_mhz'], c.get('mem_mhz'), c['reasons'])"
done
