# Same-box bisection of a bench-sequence slowdown: libraries built from earlier commits (tools/basebuild/*) vs current.
TAG=${1:-s4ab2}
mkdir -p gpurun_out
one() {  # env cfg dtype
  env $1 timeout 300 python bench.py --config $2 --dtype $3 --steps 100 --no-cpu-baseline --e2e-steps 1 > /tmp/ab.json 2>/tmp/ab.err
  python -c "import json; d=json.load(open('/tmp/ab.json')); k=d['kernels']; print('$1 $2 $3 value %.3e ms %.4f fwd %.1f (%.3f) bwd %.1f (%.3f)' % (d['value'], d['ms_per_step'], k['fwd_us'], k['fwd_frac'], k['bwd_us'], k['bwd_frac']), d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 /tmp/ab.err
}
nvidia-smi --query-gpu=name,serial --format=csv,noheader
for rep in 1 2; do for lib in GRKAN_LIB=tools/basebuild/libgrkan_b200.so GRKAN_LIB=tools/basebuild/4c28996/libgrkan_b200.so GRKAN_LIB=tools/basebuild/38c2cfd/libgrkan_b200.so GRKAN_LIB= "GRKAN_LIB= GRKAN_ZST=0"; do
  one "$lib" kat-b bf16; one "$lib" kat-s fp32
done; done 2>&1 | tee gpurun_out/ab_base_${TAG}.txt
