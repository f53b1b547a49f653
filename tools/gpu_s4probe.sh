# Per-CTA timeline of the staged backward (tools/probe_times.py) at KAT-S / KAT-B, fp32 / bf16.
TAG=${1:-s4p}
mkdir -p gpurun_out
python tools/build_variant.py probe GRKAN_PROBE_TIMES=1 > gpurun_out/build_probe.txt 2>&1 || { tail gpurun_out/build_probe.txt; exit 1; }
for c in kat-s kat-b; do for d in fp32 bf16; do
  GRKAN_LIB=tools/variants/probe/libgrkan_b200.so timeout 300 python tools/probe_times.py --config $c --dtype $d --dump gpurun_out/probe_${TAG}_${c}_${d}.json
done; done 2>&1 | tee gpurun_out/probe_${TAG}.txt
# A/B: bf16 table as float2 pairs (GRKAN_LUT_PAIRED=1) vs two arrays
python tools/build_variant.py pair GRKAN_LUT_PAIRED=1 > gpurun_out/build_pair.txt 2>&1 || { tail gpurun_out/build_pair.txt; exit 1; }
one() {  # lib cfg dtype
  env $1 timeout 300 python bench.py --config $2 --dtype $3 --steps 100 --no-cpu-baseline --e2e-steps 1 > /tmp/ab.json 2>/tmp/ab.err
  python -c "import json; d=json.load(open('/tmp/ab.json')); k=d['kernels']; print('$1 $2 $3 value %.3e fwd %.1f bwd %.1f (%.3f)' % (d['value'], k['fwd_us'], k['bwd_us'], k['bwd_frac']), d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 /tmp/ab.err
}
for rep in 1 2; do for lib in GRKAN_LIB= GRKAN_LIB=tools/variants/pair/libgrkan_b200.so; do
  one $lib kat-b bf16; one $lib kat-s bf16
done; done 2>&1 | tee gpurun_out/ab_pair_${TAG}.txt
