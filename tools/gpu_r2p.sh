# Geometry x stage-copy A/B: 2 x 8 vs 1 x 16 consumer warps, per-row copies vs tensor-map boxes.
TAG=${1:-r2p}
mkdir -p gpurun_out
one() {  # lib env cfg dtype
  if [ "$1" = default ]; then L=""; else L="GRKAN_LIB=tools/variants/$1/libgrkan_b200.so"; fi
  env $L $2 timeout 300 python bench.py --config $3 --dtype $4 --steps 100 --no-cpu-baseline --e2e-steps 1 > /tmp/ab.json 2>/tmp/ab.err
  python -c "import json; d=json.load(open('/tmp/ab.json')); k=d['kernels']; print('$1 $2 $3 $4 fwd %.1f bwd %.1f (%.3f) value %.3e' % (k['fwd_us'], k['bwd_us'], k['bwd_frac'], d['value']), d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 /tmp/ab.err
}
for rep in 1 2; do
  for cfg in kat-b kat-s; do for dt in fp32 bf16; do
    one default GRKAN_TMA2D=1 $cfg $dt
    one default GRKAN_TMA2D=2 $cfg $dt
    one w16b GRKAN_TMA2D=1 $cfg $dt
    one w16b GRKAN_TMA2D=2 $cfg $dt
  done; done
done 2>&1 | tee gpurun_out/ab_${TAG}.txt
