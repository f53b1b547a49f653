# Three-array bf16 table: tests + bf16 lines (+ deterministic collective line).
TAG=${1:-r2aa}
mkdir -p gpurun_out
timeout 1500 python -m pytest -q -m gpu tests/test_gpu_lut.py tests/test_gpu_deterministic.py tests/test_gpu_fused_step.py tests/test_gpu_parity.py tests/test_gpu_tma.py tests/test_gpu_access_instr.py > gpurun_out/pytest_${TAG}.txt 2>&1; tail -3 gpurun_out/pytest_${TAG}.txt
for rep in 1 2; do for cfg in kat-b kat-s; do
  timeout 300 python bench.py --config $cfg --dtype bf16 --steps 100 --no-cpu-baseline --e2e-steps 1 > /tmp/ab.json 2>/dev/null
  python -c "import json; d=json.load(open('/tmp/ab.json')); k=d['kernels']; print('$cfg bf16 value %.3e fwd %.1f bwd %.1f (%.3f) step %.3f' % (d['value'], k['fwd_us'], k['bwd_us'], k['bwd_frac'], d['hbm_gbs']/d['roofline']['peak']), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done; done
timeout 300 python bench.py --config kat-b --dtype bf16 --steps 50 --no-cpu-baseline --e2e-steps 1 --collective deterministic > /tmp/ab.json 2>/dev/null
python -c "import json; d=json.load(open('/tmp/ab.json')); k=d['kernels']; print('kat-b bf16 deterministic value %.3e fwd %.1f bwd %.1f' % (d['value'], k['fwd_us'], k['bwd_us']))"
