# A/B: first-wave share of the staged backward at 2 CTAs per SM (GRKAN_SKEW, 1/64 units; 64 = even).
TAG=${1:-s4s}
mkdir -p gpurun_out
one() {  # env cfg dtype extra
  env $1 timeout 300 python bench.py --config $2 --dtype $3 --steps 100 --no-cpu-baseline --e2e-steps 1 $4 > /tmp/ab.json 2>/tmp/ab.err
  python -c "import json; d=json.load(open('/tmp/ab.json')); k=d['kernels']; print('$1 $2 $3 $4 value %.3e fwd %.1f bwd %.1f (%.3f)' % (d['value'], k['fwd_us'], k['bwd_us'], k['bwd_frac']), d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 /tmp/ab.err
}
for rep in 1 2; do for w in 64 72 80 88 96; do
  one GRKAN_SKEW=$w kat-s fp32; one GRKAN_SKEW=$w kat-b fp32 "--groups 16"
done; done 2>&1 | tee gpurun_out/ab_skew_${TAG}.txt
python tools/build_variant.py probe GRKAN_PROBE_TIMES=1 > gpurun_out/build_probe.txt 2>&1 || { tail gpurun_out/build_probe.txt; exit 1; }
for w in 64 80 88; do
  GRKAN_SKEW=$w GRKAN_LIB=tools/variants/probe/libgrkan_b200.so timeout 300 python tools/probe_times.py --config kat-s --dtype fp32 --dump gpurun_out/probe_${TAG}_w${w}.json
done 2>&1 | tee gpurun_out/probe_${TAG}.txt
