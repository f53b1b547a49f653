TAG=${1:-r2m}
mkdir -p gpurun_out
for i in 1 2 3 4; do
  GRKAN_BENCH_TRACE_AFTER=150 timeout 240 python bench.py --gpus 2 --config kat-t --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --dist-backend gloo > gpurun_out/spawn_${TAG}_$i.out 2> gpurun_out/spawn_${TAG}_$i.err
  echo "run $i rc=$? lines=$(grep -c '^{' gpurun_out/spawn_${TAG}_$i.out)"
done
for c in deterministic p2p; do
  GRKAN_BENCH_TRACE_AFTER=150 timeout 240 python bench.py --gpus 2 --config kat-t --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --dist-backend gloo --collective $c > gpurun_out/spawn_${TAG}_$c.out 2> gpurun_out/spawn_${TAG}_$c.err
  echo "$c rc=$? lines=$(grep -c '^{' gpurun_out/spawn_${TAG}_$c.out)"
done
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_${TAG}.txt 2>&1; tail -3 gpurun_out/pytest_gpu_${TAG}.txt
