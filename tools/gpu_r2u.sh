# KAT-B training step (config 4) and the fused layer backward on the round-2 build.
TAG=${1:-r2u}
mkdir -p gpurun_out
timeout 900 python bench.py --config kat-b-train --steps 20 --warmup 5 > gpurun_out/train_${TAG}.json 2> gpurun_out/train_${TAG}.err; cut -c1-300 gpurun_out/train_${TAG}.json; tail -2 gpurun_out/train_${TAG}.err
timeout 900 python bench.py --config kat-b-train --fused-mlp --steps 20 --warmup 5 > gpurun_out/train_${TAG}_fused.json 2> gpurun_out/train_${TAG}_fused.err; cut -c1-300 gpurun_out/train_${TAG}_fused.json
timeout 900 python tools/bench_fused.py > gpurun_out/bench_fused_${TAG}.jsonl 2> gpurun_out/bench_fused_${TAG}.err; cat gpurun_out/bench_fused_${TAG}.jsonl | cut -c1-300; tail -2 gpurun_out/bench_fused_${TAG}.err
