# End-of-session check on one GPU: the driver's round-end sequence (GPU tests, smoke,
# default bench line) plus the bf16 line and the reference arm.  usage: bash tools/gpu_final.sh TAG
TAG=${1:-final}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_${TAG}.txt 2>&1; tail -1 gpurun_out/pytest_gpu_${TAG}.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.txt 2>&1; tail -1 gpurun_out/smoke_${TAG}.txt
timeout 900 python bench.py > gpurun_out/bench_${TAG}_fp32.json 2> gpurun_out/bench_${TAG}_fp32.err; cut -c1-400 gpurun_out/bench_${TAG}_fp32.json
timeout 900 python bench.py --dtype bf16 --no-cpu-baseline > gpurun_out/bench_${TAG}_bf16.json 2> gpurun_out/bench_${TAG}_bf16.err; cut -c1-200 gpurun_out/bench_${TAG}_bf16.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_${TAG}_reference.json 2> gpurun_out/bench_${TAG}_reference.err; cut -c1-200 gpurun_out/bench_${TAG}_reference.json
