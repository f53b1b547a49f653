# First heavy run on a box is slower (fp32 KAT-B: ~3.02e11 vs 3.22e11 for the next runs, same temperatures):
# is it transient?  Smoke, then the default line with a 3 s warm-up first, then the default (150 ms) twice.
TAG=${1:-s4w}
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.txt 2>&1; tail -1 gpurun_out/smoke_${TAG}.txt
i=0
for w in 3 0.15 0.15 3; do i=$((i+1))
  GRKAN_BENCH_WARM_S=$w timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_${TAG}_$i.json 2> gpurun_out/bench_${TAG}_$i.err
  python -c "import json; d=json.load(open('gpurun_out/bench_${TAG}_$i.json')); k=d['kernels']; c=d['clocks']; print('run $i warm $w value %.3e fwd %.1f bwd %.1f' % (d['value'], k['fwd_us'], k['bwd_us']), c['sm_mhz'], c['reasons'], c.get('temp_c'))"
done
