# usage: bash tools/gpu_prof.sh TAG  -- ncu captures of the hot kernels (fp32 + bf16)
TAG=${1:-prof}
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_bwd_staged|k_bwd_main" -s 3 -c 1 -o gpurun_out/prof_${TAG}_bwd_fp32 $B > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_bwd_staged|k_bwd_main" -s 3 -c 1 -o gpurun_out/prof_${TAG}_bwd_bf16 $B --dtype bf16 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_fwd" -s 3 -c 1 -o gpurun_out/prof_${TAG}_fwd_fp32 $B > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_fwd" -s 3 -c 1 -o gpurun_out/prof_${TAG}_fwd_bf16 $B --dtype bf16 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_${TAG}.csv $B > /dev/null 2>&1
ls gpurun_out | grep $TAG
