# fp32 geometry A/B: 2 x 8 (default) vs 1 x 16 consumer warps, KAT-B and KAT-S, interleaved.
TAG=${1:-r2o}
mkdir -p gpurun_out
one() {  # lib cfg dtype
  if [ "$1" = default ]; then L=""; else L="GRKAN_LIB=tools/variants/$1/libgrkan_b200.so"; fi
  env $L timeout 300 python bench.py --config $2 --dtype $3 --steps 100 --no-cpu-baseline --e2e-steps 1 > /tmp/ab.json 2>/tmp/ab.err
  python -c "import json; d=json.load(open('/tmp/ab.json')); k=d['kernels']; print('$1 $2 $3 fwd %.1f bwd %.1f (%.3f) value %.3e' % (k['fwd_us'], k['bwd_us'], k['bwd_frac'], d['value']), d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 /tmp/ab.err
}
for rep in 1 2 3; do for lib in default w16b; do one $lib kat-b fp32; one $lib kat-s fp32; done; done 2>&1 | tee gpurun_out/ab_${TAG}.txt
