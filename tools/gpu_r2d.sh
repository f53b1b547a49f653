# A/B: consumer-warp geometry variants (tools/variants/w16, w12s5) x bf16 table on/off;
# ncu of the default build's bf16 backward (suspend-hint waits).  usage: bash tools/gpu_r2d.sh TAG
TAG=${1:-r2d}
mkdir -p gpurun_out
one() {  # lib lut cfg dtype
  if [ "$1" = default ]; then L=""; else L="GRKAN_LIB=tools/variants/$1/libgrkan_b200.so"; fi
  env $L GRKAN_LUT=$2 timeout 300 python bench.py --config $3 --dtype $4 --steps 50 --no-cpu-baseline --e2e-steps 1 > /tmp/ab.json 2>/tmp/ab.err
  python -c "import json; d=json.load(open('/tmp/ab.json')); k=d['kernels']; print('$1 lut=$2 $3 $4 fwd %.1f bwd %.1f (%.3f) value %.3e' % (k['fwd_us'], k['bwd_us'], k['bwd_frac'], d['value']), d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 /tmp/ab.err
}
for lib in default w16 w12s5; do
  for cfg in kat-b kat-s; do
    one $lib 1 $cfg bf16
    one $lib 0 $cfg bf16
    one $lib 0 $cfg fp32
  done
done 2>&1 | tee gpurun_out/ab_${TAG}.txt
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --dtype bf16"
GRKAN_LUT=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_bwd_staged" -s 3 -c 1 -o gpurun_out/prof_${TAG}_bwd_bf16_hint $B > /dev/null 2>&1
GRKAN_LUT=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_bwd_staged" -s 3 -c 1 -o gpurun_out/prof_${TAG}_bwd_bf16_lut_hint $B > /dev/null 2>&1
ls gpurun_out | grep $TAG
