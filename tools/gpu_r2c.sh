# A/B: mbarrier suspend-time hint (default build) vs none (tools/variants/nohint), and the
# bf16 x-factor table on/off.  usage: bash tools/gpu_r2c.sh TAG
TAG=${1:-r2c}
mkdir -p gpurun_out
one() {  # lib lut cfg dtype
  if [ "$1" = default ]; then L=""; else L="GRKAN_LIB=tools/variants/$1/libgrkan_b200.so"; fi
  env $L GRKAN_LUT=$2 timeout 300 python bench.py --config $3 --dtype $4 --steps 50 --no-cpu-baseline --e2e-steps 1 > /tmp/ab.json 2>/tmp/ab.err
  python -c "import json; d=json.load(open('/tmp/ab.json')); k=d['kernels']; print('$1 lut=$2 $3 $4 fwd %.1f bwd %.1f (%.3f) value %.3e' % (k['fwd_us'], k['bwd_us'], k['bwd_frac'], d['value']), d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 /tmp/ab.err
}
for rep in 1 2; do
for lib in default nohint; do
  for cfg in kat-b kat-s; do
    one $lib 1 $cfg bf16
    one $lib 0 $cfg bf16
    one $lib 0 $cfg fp32
  done
done
done 2>&1 | tee gpurun_out/ab_${TAG}.txt
