# Same (slow-state) box: the default line with its CPU-baseline leg, then a line without it.
TAG=${1:-s4c}
mkdir -p gpurun_out
for i in 1 2; do
  if [ $i = 1 ]; then X=""; else X="--no-cpu-baseline"; fi
  timeout 900 python bench.py $X > gpurun_out/bench_${TAG}_$i.json 2> gpurun_out/bench_${TAG}_$i.err
  python -c "import json; d=json.load(open('gpurun_out/bench_${TAG}_$i.json')); k=d['kernels']; c=d['clocks']; print('run $i $X value %.3e fwd %.1f bwd %.1f' % (d['value'], k['fwd_us'], k['bwd_us']), c['sm_mhz'], c['reasons'])"
done
