# usage: bash tools/gpu_prof_bf16.sh TAG -- microbenchmarks + ncu full captures of the bf16 kernels
TAG=${1:-prof}
mkdir -p gpurun_out
./tools/micro/pipe_mix > gpurun_out/pipe_mix_${TAG}.txt 2>&1; cat gpurun_out/pipe_mix_${TAG}.txt
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --dtype bf16"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_bwd_staged" -s 3 -c 1 -o gpurun_out/prof_${TAG}_bwd_bf16 $B > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_fwd" -s 3 -c 1 -o gpurun_out/prof_${TAG}_fwd_bf16 $B > /dev/null 2>&1
ls -la gpurun_out | grep $TAG
