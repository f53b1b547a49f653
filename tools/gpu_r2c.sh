# Round 2 check c: bf16 backward variants (lean FAST math, 1-CTA geometry, compute-only probes) + spawn test under pytest.
TAG=${1:-r2c}
mkdir -p gpurun_out
for v in default lean cw16 leancw16 lean3 probe leanprobe; do
  if [ "$v" = default ]; then L=""; else L="GRKAN_LIB=tools/variants/$v/libgrkan_b200.so"; fi
  for cfg in kat-b kat-s; do
    env $L timeout 300 python bench.py --config $cfg --steps 30 --warmup 5 --dtype bf16 --no-cpu-baseline --e2e-steps 1 > /tmp/vb.json 2>/tmp/vb.err
    python -c "import json; d=json.load(open('/tmp/vb.json')); k=d['kernels']; print('$v $cfg bf16', 'bwd=%.1fus(%.3f)'%(k['bwd_us'],k['bwd_frac']), 'fwd=%.1fus(%.3f)'%(k['fwd_us'],k['fwd_frac']), d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 /tmp/vb.err
  done
  env $L timeout 300 python bench.py --config kat-b --steps 30 --warmup 5 --dtype fp32 --no-cpu-baseline --e2e-steps 1 > /tmp/vb.json 2>/tmp/vb.err
  python -c "import json; d=json.load(open('/tmp/vb.json')); k=d['kernels']; print('$v kat-b fp32', 'bwd=%.1fus(%.3f)'%(k['bwd_us'],k['bwd_frac']), 'fwd=%.1fus(%.3f)'%(k['fwd_us'],k['fwd_frac']))" || tail -3 /tmp/vb.err
done
GRKAN_BENCH_TRACE_AFTER=100 timeout 600 python -m pytest -q -m gpu tests/test_bench_contract.py > gpurun_out/pytest_${TAG}_contract.txt 2>&1; tail -30 gpurun_out/pytest_${TAG}_contract.txt
