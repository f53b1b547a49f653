# Round evidence: default bench line, bf16 line, reference arm, ncu launch list + full captures.
# usage (on the GPU box via gpurun): bash tools/gpu_evidence.sh TAG
TAG=${1:-r1}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv,noheader
timeout 900 python bench.py > gpurun_out/bench_${TAG}_default.json 2> gpurun_out/bench_${TAG}_default.err; cat gpurun_out/bench_${TAG}_default.json
timeout 900 python bench.py --dtype bf16 --no-cpu-baseline > gpurun_out/bench_${TAG}_bf16.json 2>&1; cut -c1-300 gpurun_out/bench_${TAG}_bf16.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_${TAG}_reference.json 2>&1; cat gpurun_out/bench_${TAG}_reference.json
lscpu | grep -E "Model name|^CPU\(s\)|Thread|Core|Socket" > gpurun_out/host_cpu_${TAG}.txt
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 12 -c 15 --csv --log-file gpurun_out/launches_${TAG}.csv $B > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_bwd_staged" -s 2 -c 1 -o gpurun_out/prof_${TAG}_bwd_fp32 $B > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_fwd" -s 2 -c 1 -o gpurun_out/prof_${TAG}_fwd_fp32 $B > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_bwd_reduce" -s 2 -c 1 -o gpurun_out/prof_${TAG}_reduce_fp32 $B > /dev/null 2>&1
ls -la gpurun_out | grep ${TAG}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_bwd_staged" -s 2 -c 1 -o gpurun_out/prof_${TAG}_bwd_bf16 $B --dtype bf16 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 12 -c 15 --csv --log-file gpurun_out/launches_${TAG}_bf16.csv $B --dtype bf16 > /dev/null 2>&1
ls -la gpurun_out | grep ${TAG}
timeout 600 python bench.py --config kat-b-train --steps 10 --warmup 3 > gpurun_out/train_${TAG}.json 2>&1
timeout 600 python bench.py --config kat-b-train --steps 10 --warmup 3 --fused-mlp > gpurun_out/train_${TAG}_fused.json 2>&1
timeout 600 python tools/bench_fused.py > gpurun_out/fused_${TAG}.jsonl 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 --collective deterministic > gpurun_out/bench_${TAG}_det.json 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 --collective p2p > gpurun_out/bench_${TAG}_p2p.json 2>&1
timeout 300 python tools/pcie_bw.py > gpurun_out/pcie_${TAG}.json 2>&1
ls -la gpurun_out | grep ${TAG}
