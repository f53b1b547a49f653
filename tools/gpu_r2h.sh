# Tensor-map copies for the FP32-math bf16 forward too; A/B lines; ncu of the y-table forward.
TAG=${1:-r2h}
mkdir -p gpurun_out
timeout 1200 python -m pytest -q -m gpu tests/test_gpu_tma.py tests/test_gpu_lut.py tests/test_gpu_parity.py > gpurun_out/pytest_${TAG}.txt 2>&1; tail -3 gpurun_out/pytest_${TAG}.txt
one() {  # env cfg dtype extra
  env $1 timeout 300 python bench.py --config $2 --dtype $3 --steps 50 --no-cpu-baseline --e2e-steps 1 $4 > /tmp/ab.json 2>/tmp/ab.err
  python -c "import json; d=json.load(open('/tmp/ab.json')); k=d['kernels']; print('$1 $2 $3 $4 fwd %.1f (%.3f) bwd %.1f (%.3f) value %.3e step %.3f' % (k['fwd_us'], k['fwd_frac'], k['bwd_us'], k['bwd_frac'], d['value'], d['hbm_gbs']/d['roofline']['peak']), d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 /tmp/ab.err
}
for t in 1 0; do
  one GRKAN_TMA2D=$t kat-s bf16
  one GRKAN_TMA2D=$t kat-b bf16 "--groups 16"
  one GRKAN_TMA2D=$t kat-b bf16 "--groups 64"
  one GRKAN_TMA2D=$t kat-t bf16
  one GRKAN_TMA2D=$t kat-t fp32
done 2>&1 | tee gpurun_out/ab_${TAG}_tma.txt
one GRKAN_FWD_LUT=0 kat-b bf16 | tee -a gpurun_out/ab_${TAG}_tma.txt
one GRKAN_FWD_LUT=0 kat-s fp32 | tee -a gpurun_out/ab_${TAG}_tma.txt
GRKAN_FWD_LUT=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_fwd_lut" -s 3 -c 1 -o gpurun_out/prof_${TAG}_fwd_lut python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --dtype bf16 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_fwd_staged" -s 3 -c 1 -o gpurun_out/prof_${TAG}_fwd_staged python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --dtype bf16 > /dev/null 2>&1
ls gpurun_out | grep $TAG
