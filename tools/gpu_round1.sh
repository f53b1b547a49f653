set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
mkdir -p gpurun_out
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' 2>&1 | tail -20
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -40
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; tail -5 gpurun_out/bench1.err; cat gpurun_out/bench1.json
timeout 600 python bench.py --steps 20 --warmup 5 --dtype bf16 --no-cpu-baseline > gpurun_out/bench1_bf16.json 2>&1; cat gpurun_out/bench1_bf16.json
timeout 600 python bench.py --steps 20 --warmup 5 --mode exact --no-cpu-baseline > gpurun_out/bench1_exact.json 2>&1; cat gpurun_out/bench1_exact.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1; head -c 3000 gpurun_out/launches.csv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bwd_main -s 3 -c 1 -o gpurun_out/prof_bwd python bench.py --steps 4 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_bwd.log 2>&1; tail -3 gpurun_out/ncu_bwd.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fwd -s 3 -c 1 -o gpurun_out/prof_fwd python bench.py --steps 4 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_fwd.log 2>&1; tail -3 gpurun_out/ncu_fwd.log
ls -la gpurun_out
