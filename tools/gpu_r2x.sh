TAG=${1:-r2x}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_${TAG}.txt 2>&1; tail -3 gpurun_out/pytest_gpu_${TAG}.txt
for cfg in kat-b kat-s kat-t; do
  timeout 300 python bench.py --config $cfg --dtype bf16 --steps 100 --no-cpu-baseline --e2e-steps 1 > /tmp/ab.json 2>/tmp/ab.err
  python -c "import json; d=json.load(open('/tmp/ab.json')); k=d['kernels']; print('$cfg bf16 fwd %.1f bwd %.1f (%.3f) value %.3e' % (k['fwd_us'], k['bwd_us'], k['bwd_frac'], d['value']), d['clocks']['sm_mhz'])"
done
