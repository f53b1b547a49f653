# A/B library variants built by tools/build_variant.py: bash tools/gpu_variants.sh v1 v2 ...  ("default" = in-tree build)
for v in "$@"; do
  if [ "$v" = default ]; then L=""; else L="GRKAN_LIB=tools/variants/$v/libgrkan_b200.so"; fi
  for dt in fp32 bf16; do
    env $L timeout 300 python bench.py --steps 20 --warmup 5 --dtype $dt --no-cpu-baseline --e2e-steps 1 > /tmp/vb.json 2>/tmp/vb.err
    python -c "import json; d=json.load(open('/tmp/vb.json')); k=d['kernels']; print('$v $dt', 'bwd=%.1fus(%.3f)'%(k['bwd_us'],k['bwd_frac']), 'fwd=%.1fus(%.3f)'%(k['fwd_us'],k['fwd_frac']))" || tail -3 /tmp/vb.err
  done
done
