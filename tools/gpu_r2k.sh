# Fixed (3,2) register-direct instantiations: golden parity + lines.
TAG=${1:-r2k}
mkdir -p gpurun_out
timeout 1200 python -m pytest -q -m gpu tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_gpu_combine.py tests/test_gpu_access_instr.py > gpurun_out/pytest_${TAG}.txt 2>&1; tail -3 gpurun_out/pytest_${TAG}.txt
one() {  # env cfg dtype extra
  env $1 timeout 300 python bench.py --config $2 --dtype $3 --steps 50 --no-cpu-baseline --e2e-steps 1 $4 > /tmp/ab.json 2>/tmp/ab.err
  python -c "import json; d=json.load(open('/tmp/ab.json')); k=d['kernels']; print('$1 $2 $3 $4 fwd %.1f (%.3f) bwd %.1f (%.3f) value %.3e step %.3f' % (k['fwd_us'], k['fwd_frac'], k['bwd_us'], k['bwd_frac'], d['value'], d['hbm_gbs']/d['roofline']['peak']), d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 /tmp/ab.err
  cp /tmp/ab.json gpurun_out/bench_${TAG}_$2_$3$(echo $4 | tr -d ' -').json 2>/dev/null
}
{
one X=1 kat-b fp32 "--num-coeffs 4 --den-coeffs 2"
one X=1 kat-b bf16 "--num-coeffs 4 --den-coeffs 2"
} 2>&1 | tee gpurun_out/ab_${TAG}.txt
