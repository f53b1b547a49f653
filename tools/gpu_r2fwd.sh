# bf16 forward geometry A/B (variants f4/f8/f16 from tools/build_variant.py) at KAT-B and KAT-S.
TAG=${1:-r2fwd}
mkdir -p gpurun_out
one() {  # lib cfg
  if [ "$1" = default ]; then L=""; else L="GRKAN_LIB=tools/variants/$1/libgrkan_b200.so"; fi
  env $L timeout 300 python bench.py --config $2 --dtype bf16 --steps 100 --no-cpu-baseline --e2e-steps 1 > /tmp/ab.json 2>/tmp/ab.err
  python -c "import json; d=json.load(open('/tmp/ab.json')); k=d['kernels']; print('$1 $2 bf16 fwd %.1f (%.3f) bwd %.1f value %.3e' % (k['fwd_us'], k['fwd_frac'], k['bwd_us'], d['value']), d['clocks']['sm_mhz'])" || tail -3 /tmp/ab.err
}
for rep in 1 2; do for lib in default f4 f8 f16; do one $lib kat-b; one $lib kat-s; done; done 2>&1 | tee gpurun_out/ab_${TAG}.txt
