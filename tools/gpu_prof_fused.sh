# ncu captures of the fused layer-backward kernel at both KAT-B layer shapes
TAG=${1:-fz}
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_linear_bwd_fused" -s 2 -c 1 -o gpurun_out/prof_${TAG}_fc2 python tools/bench_fused.py --reps 3 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_linear_bwd_fused" -s 10 -c 1 -o gpurun_out/prof_${TAG}_fc1 python tools/bench_fused.py --reps 3 > /dev/null 2>&1
ls -la gpurun_out | grep $TAG
