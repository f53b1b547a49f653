# Same box: NVML polling during the timed region on / off (GRKAN_BENCH_NVML_POLL=0), and after a CPU-heavy run.
TAG=${1:-s4n}
mkdir -p gpurun_out
i=0
for p in 0 1 0 1; do i=$((i+1))
  GRKAN_BENCH_NVML_POLL=$p timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_${TAG}_$i.json 2> gpurun_out/bench_${TAG}_$i.err
  python -c "import json; d=json.load(open('gpurun_out/bench_${TAG}_$i.json')); k=d['kernels']; c=d['clocks']; print('run $i poll $p value %.3e fwd %.1f bwd %.1f' % (d['value'], k['fwd_us'], k['bwd_us']), c['sm_mhz'], c.get('samples'), c['reasons'])"
done
