TAG=${1:-r2f}
mkdir -p gpurun_out
for v in default estrin estrinprobe probe; do
  if [ "$v" = default ]; then L=""; else L="GRKAN_LIB=tools/variants/$v/libgrkan_b200.so"; fi
  for cfg in kat-b kat-s; do for dt in bf16 fp32; do
    env $L timeout 300 python bench.py --config $cfg --steps 30 --warmup 5 --dtype $dt --no-cpu-baseline --e2e-steps 1 > /tmp/vb.json 2>/tmp/vb.err
    python -c "import json; d=json.load(open('/tmp/vb.json')); k=d['kernels']; print('$v $cfg $dt', 'bwd=%.1fus(%.3f)'%(k['bwd_us'],k['bwd_frac']), 'fwd=%.1fus(%.3f)'%(k['fwd_us'],k['fwd_frac']), d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 /tmp/vb.err
  done; done
done
GRKAN_LIB=tools/variants/estrin/libgrkan_b200.so timeout 900 python -m pytest -q -m gpu tests/test_gpu_parity.py -x > gpurun_out/pytest_${TAG}_estrin_parity.txt 2>&1; tail -3 gpurun_out/pytest_${TAG}_estrin_parity.txt
