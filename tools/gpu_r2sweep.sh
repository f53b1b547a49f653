# Config 5 stress sweep on the round-2 kernels (5 passes, 3 above 1e8; CPU reference to 1e7).
TAG=${1:-r2sw}
mkdir -p gpurun_out
timeout 3000 python tools/stress_sweep.py --passes 5 --max-passes-e 1e8 --cpu-max-e 1e7 > gpurun_out/stress_sweep_${TAG}.jsonl 2> gpurun_out/stress_sweep_${TAG}.err
echo rc=$?; wc -l gpurun_out/stress_sweep_${TAG}.jsonl; tail -3 gpurun_out/stress_sweep_${TAG}.err
