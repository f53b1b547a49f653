# Fresh box: smoke, then the default line (CPU reference leg now before the GPU measurement) twice.
TAG=${1:-s4o}
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.txt 2>&1; tail -1 gpurun_out/smoke_${TAG}.txt
for i in 1 2; do
  timeout 900 python bench.py > gpurun_out/bench_${TAG}_$i.json 2> gpurun_out/bench_${TAG}_$i.err
  python -c "import json; d=json.load(open('gpurun_out/bench_${TAG}_$i.json')); k=d['kernels']; c=d['clocks']; print('run $i value %.3e fwd %.1f bwd %.1f cpu %.3e' % (d['value'], k['fwd_us'], k['bwd_us'], d['cpu_baseline']['value']), c['sm_mhz'], c['reasons'])"
done
