# bf16 table v2 (SoA, packed slot arithmetic, lane-pair accumulator slots): parity + A/B + ncu.
TAG=${1:-r2e}
mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests/test_gpu_lut.py tests/test_gpu_deterministic.py tests/test_gpu_parity.py -k "lut or bf16 or deterministic or golden" > gpurun_out/pytest_${TAG}.txt 2>&1; tail -3 gpurun_out/pytest_${TAG}.txt
for rep in 1 2; do for lut in 1 0; do
  GRKAN_LUT=$lut timeout 300 python bench.py --config kat-b --dtype bf16 --steps 50 --no-cpu-baseline --e2e-steps 1 > /tmp/ab.json 2>/tmp/ab.err
  python -c "import json; d=json.load(open('/tmp/ab.json')); k=d['kernels']; print('lut=$lut kat-b bf16 fwd %.1f bwd %.1f (%.3f) value %.3e' % (k['fwd_us'], k['bwd_us'], k['bwd_frac'], d['value']), d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 /tmp/ab.err
done; done 2>&1 | tee gpurun_out/ab_${TAG}.txt
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --dtype bf16"
GRKAN_LUT=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_bwd_staged" -s 3 -c 1 -o gpurun_out/prof_${TAG}_bwd_bf16_lut $B > /dev/null 2>&1
ls gpurun_out | grep $TAG
