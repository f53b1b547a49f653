# Round 2 check d: new GPU tests (instrumentation, layer fixtures, combine, host pipeline), bf16 ILP variants, shim probe.
TAG=${1:-r2d}
mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests/test_gpu_access_instr.py tests/test_gpu_layer.py tests/test_gpu_combine.py tests/test_gpu_host.py > gpurun_out/pytest_${TAG}_new.txt 2>&1; tail -25 gpurun_out/pytest_${TAG}_new.txt
for v in default ilp ilpprobe gnp4 gnp1 probe; do
  if [ "$v" = default ]; then L=""; else L="GRKAN_LIB=tools/variants/$v/libgrkan_b200.so"; fi
  for cfg in kat-b kat-s; do
    env $L timeout 300 python bench.py --config $cfg --steps 30 --warmup 5 --dtype bf16 --no-cpu-baseline --e2e-steps 1 > /tmp/vb.json 2>/tmp/vb.err
    python -c "import json; d=json.load(open('/tmp/vb.json')); k=d['kernels']; print('$v $cfg bf16', 'bwd=%.1fus(%.3f)'%(k['bwd_us'],k['bwd_frac']), 'fwd=%.1fus(%.3f)'%(k['fwd_us'],k['fwd_frac']), d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 /tmp/vb.err
  done
done
timeout 600 python tools/host_probe.py > gpurun_out/host_probe_${TAG}.jsonl 2>&1; cat gpurun_out/host_probe_${TAG}.jsonl
