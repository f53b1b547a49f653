# Wide backward geometry chosen per shape (default build) vs GRKAN_WIDE=0; full GPU suite.
TAG=${1:-r2q}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_${TAG}.txt 2>&1; tail -3 gpurun_out/pytest_gpu_${TAG}.txt
one() {  # env cfg dtype
  env $1 timeout 300 python bench.py --config $2 --dtype $3 --steps 100 --no-cpu-baseline --e2e-steps 1 > /tmp/ab.json 2>/tmp/ab.err
  python -c "import json; d=json.load(open('/tmp/ab.json')); k=d['kernels']; print('$1 $2 $3 fwd %.1f bwd %.1f (%.3f) value %.3e step %.3f' % (k['fwd_us'], k['bwd_us'], k['bwd_frac'], d['value'], d['hbm_gbs']/d['roofline']['peak']), d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 /tmp/ab.err
}
for rep in 1 2; do for w in X=1 GRKAN_WIDE=0; do
  one $w kat-b fp32; one $w kat-b bf16; one $w kat-s fp32; one $w kat-s bf16
done; done 2>&1 | tee gpurun_out/ab_${TAG}.txt
