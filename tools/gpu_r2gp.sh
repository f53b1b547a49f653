# Two groups per wide CTA (GRKAN_GPC default 2) vs one: tests + A/B.
TAG=${1:-r2gp}
mkdir -p gpurun_out
timeout 2400 python -m pytest -q -m gpu tests > gpurun_out/pytest_gpu_${TAG}.txt 2>&1; tail -3 gpurun_out/pytest_gpu_${TAG}.txt
one() {  # env cfg dtype extra
  env $1 timeout 300 python bench.py --config $2 --dtype $3 --steps 100 --no-cpu-baseline --e2e-steps 1 $4 > /tmp/ab.json 2>/tmp/ab.err
  python -c "import json; d=json.load(open('/tmp/ab.json')); k=d['kernels']; print('$1 $2 $3 $4 value %.3e fwd %.1f bwd %.1f (%.3f)' % (d['value'], k['fwd_us'], k['bwd_us'], k['bwd_frac']), d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 /tmp/ab.err
}
for rep in 1 2; do for gp in 2 1; do
  one GRKAN_GPC=$gp kat-b fp32; one GRKAN_GPC=$gp kat-b bf16; one GRKAN_GPC=$gp kat-s bf16; one GRKAN_GPC=$gp kat-b bf16 "--groups 16"
done; done 2>&1 | tee gpurun_out/ab_${TAG}.txt
