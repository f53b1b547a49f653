TAG=${1:-r2chk}
mkdir -p gpurun_out
timeout 2400 python -m pytest -q -m gpu tests > gpurun_out/pytest_gpu_${TAG}.txt 2>&1; tail -1 gpurun_out/pytest_gpu_${TAG}.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for dt in fp32 bf16; do
  timeout 300 python bench.py --dtype $dt --steps 100 --no-cpu-baseline --e2e-steps 1 > /tmp/ab.json 2>/dev/null
  python -c "import json; d=json.load(open('/tmp/ab.json')); k=d['kernels']; print('kat-b $dt value %.3e fwd %.1f bwd %.1f (%.3f)' % (d['value'], k['fwd_us'], k['bwd_us'], k['bwd_frac']), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
