# Diagnose the self-spawned 2-rank bench on a 1-GPU box: all-thread stack dumps after 90 s.
TAG=${1:-diag}
mkdir -p gpurun_out
for i in 1 2; do
  GRKAN_BENCH_TRACE_AFTER=90 timeout 200 python bench.py --gpus 2 --config kat-t --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --dist-backend gloo > gpurun_out/spawn_${TAG}_$i.out 2> gpurun_out/spawn_${TAG}_$i.err
  echo "run $i rc=$?"; grep -c '^{' gpurun_out/spawn_${TAG}_$i.out
done
