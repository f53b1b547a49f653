TAG=${1:-r2e}
mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests/test_gpu_host.py tests/test_gpu_api.py > gpurun_out/pytest_${TAG}.txt 2>&1; tail -5 gpurun_out/pytest_${TAG}.txt
timeout 600 python bench.py --config kat-b --dtype fp32 --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench_${TAG}_katb_fp32.json 2> gpurun_out/bench_${TAG}_katb_fp32.err
python -c "import json; d=json.load(open('gpurun_out/bench_${TAG}_katb_fp32.json')); print('shim', d['e2e'].get('reference_api')); print('e2e', d['e2e']['value'], d['e2e']['ms_per_step'])" || tail -5 gpurun_out/bench_${TAG}_katb_fp32.err
timeout 600 python tools/host_probe.py 2>&1 | head -3
