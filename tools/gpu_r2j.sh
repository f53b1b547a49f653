# 3-D tensor-map boxes (bf16 backward at any row length): tests + A/B.
TAG=${1:-r2j}
mkdir -p gpurun_out
timeout 1200 python -m pytest -q -m gpu tests/test_gpu_tma.py tests/test_gpu_lut.py tests/test_gpu_parity.py tests/test_gpu_fused_step.py tests/test_gpu_deterministic.py > gpurun_out/pytest_${TAG}.txt 2>&1; tail -3 gpurun_out/pytest_${TAG}.txt
one() {  # env cfg dtype extra
  env $1 timeout 300 python bench.py --config $2 --dtype $3 --steps 50 --no-cpu-baseline --e2e-steps 1 $4 > /tmp/ab.json 2>/tmp/ab.err
  python -c "import json; d=json.load(open('/tmp/ab.json')); k=d['kernels']; print('$1 $2 $3 $4 fwd %.1f (%.3f) bwd %.1f (%.3f) value %.3e step %.3f' % (k['fwd_us'], k['fwd_frac'], k['bwd_us'], k['bwd_frac'], d['value'], d['hbm_gbs']/d['roofline']['peak']), d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 /tmp/ab.err
}
for rep in 1 2; do for t in 1 0; do
  one GRKAN_TMA2D=$t kat-b bf16
  one GRKAN_TMA2D=$t kat-s bf16
done; done 2>&1 | tee gpurun_out/ab_${TAG}.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_bwd_staged" -s 3 -c 1 -o gpurun_out/prof_${TAG}_bwd_bf16 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --dtype bf16 > /dev/null 2>&1
ls gpurun_out | grep $TAG
