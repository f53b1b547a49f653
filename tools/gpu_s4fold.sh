# GPU suite (incl. test_gpu_fold) + A/B: K3 folded into K2 (default) vs launched (GRKAN_FOLD=0).
TAG=${1:-s4k}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fold.py -q -x > gpurun_out/pytest_fold_${TAG}.txt 2>&1; tail -3 gpurun_out/pytest_fold_${TAG}.txt
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_${TAG}.txt 2>&1; tail -3 gpurun_out/pytest_gpu_${TAG}.txt
one() {  # env cfg dtype extra
  env $1 timeout 300 python bench.py --config $2 --dtype $3 --steps 100 --no-cpu-baseline --e2e-steps 1 $4 > /tmp/ab.json 2>/tmp/ab.err
  python -c "import json; d=json.load(open('/tmp/ab.json')); k=d['kernels']; print('$1 $2 $3 $4 value %.3e ms %.4f fwd %.1f (%.3f) bwd %.1f (%.3f) fused %.1f' % (d['value'], d['ms_per_step'], k['fwd_us'], k['fwd_frac'], k['bwd_us'], k['bwd_frac'], k['fused_step']['us']), d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 /tmp/ab.err
}
for rep in 1 2; do for f in 1 0; do
  one GRKAN_FOLD=$f kat-s fp32; one GRKAN_FOLD=$f kat-s bf16; one GRKAN_FOLD=$f kat-b bf16; one GRKAN_FOLD=$f kat-b fp32
done; done 2>&1 | tee gpurun_out/ab_fold_${TAG}.txt
