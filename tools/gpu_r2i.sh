TAG=${1:-r2i}
mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests/test_gpu_fused_step.py tests/test_gpu_parity.py tests/test_gpu_api.py > gpurun_out/pytest_${TAG}.txt 2>&1; tail -5 gpurun_out/pytest_${TAG}.txt
for cfg in kat-b kat-s; do for dt in fp32 bf16; do
  timeout 300 python bench.py --config $cfg --dtype $dt --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_${TAG}_${cfg}_${dt}.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/bench_${TAG}_${cfg}_${dt}.json')); k=d['kernels']; f=k['fused_step']; print('$cfg $dt two-pass %.1f Gel/s (%.3f of HBM, fwd %.1f bwd %.1f us) | fused %.1f us %.1f Gel/s frac(4sE) %.3f frac(5sE) %.3f' % (d['value']/1e9, d['hbm_gbs']/d['roofline']['peak'], k['fwd_us'], k['bwd_us'], f['us'], f['elements_per_s']/1e9, f['frac'], f['gbs_fwd_plus_bwd_bytes']/d['roofline']['peak']), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  timeout 300 python bench.py --config $cfg --dtype $dt --fused-step --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_${TAG}_${cfg}_${dt}_fused.json 2>gpurun_out/bench_${TAG}_fused.err
  python -c "import json; d=json.load(open('gpurun_out/bench_${TAG}_${cfg}_${dt}_fused.json')); print('$cfg $dt --fused-step value %.1f Gel/s ms %.4f roofline %.3f' % (d['value']/1e9, d['ms_per_step'], d['roofline']['frac']))" || tail -3 gpurun_out/bench_${TAG}_fused.err
done; done
