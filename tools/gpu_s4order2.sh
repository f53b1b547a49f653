# Fresh box, the driver's round-end order: GPU tests, smoke, the default line (CPU leg first now).
TAG=${1:-s4o2}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_${TAG}.txt 2>&1; tail -1 gpurun_out/pytest_gpu_${TAG}.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.txt 2>&1; tail -1 gpurun_out/smoke_${TAG}.txt
timeout 900 python bench.py > gpurun_out/bench_${TAG}_1.json 2> gpurun_out/bench_${TAG}_1.err
python -c "import json; d=json.load(open('gpurun_out/bench_${TAG}_1.json')); k=d['kernels']; c=d['clocks']; print('default value %.3e fwd %.1f bwd %.1f roofline %.3f' % (d['value'], k['fwd_us'], k['bwd_us'], d['roofline']['frac']), c['sm_mhz'], c['reasons'])"
