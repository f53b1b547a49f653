# Per-step event count: bench lines (timed region with one event per step) at KAT-B/KAT-S fp32/bf16.
TAG=${1:-r2z}
mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests/test_bench_contract.py > gpurun_out/pytest_${TAG}.txt 2>&1; tail -1 gpurun_out/pytest_${TAG}.txt
for rep in 1 2; do for cfg in kat-b kat-s; do for dt in fp32 bf16; do
  timeout 300 python bench.py --config $cfg --dtype $dt --steps 100 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_${TAG}_${cfg}_${dt}.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/bench_${TAG}_${cfg}_${dt}.json')); k=d['kernels']; print('$cfg $dt value %.3e ms %.4f (fwd %.1f + bwd %.1f = %.1f) step frac %.3f' % (d['value'], d['ms_per_step'], k['fwd_us'], k['bwd_us'], k['fwd_us']+k['bwd_us'], d['hbm_gbs']/d['roofline']['peak']), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done; done; done
