# Flattened backward partition A/B (GRKAN_FLAT=1 default vs 0) + parity subset.
TAG=${1:-r2v}
mkdir -p gpurun_out
timeout 1500 python -m pytest -q -m gpu tests/test_gpu_parity.py tests/test_gpu_tma.py tests/test_gpu_lut.py tests/test_gpu_deterministic.py tests/test_gpu_fused_step.py tests/test_gpu_api.py tests/test_gpu_access_instr.py > gpurun_out/pytest_${TAG}.txt 2>&1; tail -3 gpurun_out/pytest_${TAG}.txt
one() {  # env cfg dtype extra
  env $1 timeout 300 python bench.py --config $2 --dtype $3 --steps 100 --no-cpu-baseline --e2e-steps 1 $4 > /tmp/ab.json 2>/tmp/ab.err
  python -c "import json; d=json.load(open('/tmp/ab.json')); k=d['kernels']; print('$1 $2 $3 $4 fwd %.1f bwd %.1f (%.3f) value %.3e' % (k['fwd_us'], k['bwd_us'], k['bwd_frac'], d['value']), d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 /tmp/ab.err
}
for rep in 1 2; do for f in 1 0; do
  one GRKAN_FLAT=$f kat-b fp32; one GRKAN_FLAT=$f kat-b bf16; one GRKAN_FLAT=$f kat-s fp32; one GRKAN_FLAT=$f kat-s bf16
  one GRKAN_FLAT=$f kat-b fp32 "--groups 64"; one GRKAN_FLAT=$f kat-b bf16 "--groups 64"
done; done 2>&1 | tee gpurun_out/ab_${TAG}.txt
