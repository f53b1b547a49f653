for v in ${DET_VARIANTS:-default det256 det512}; do
  if [ "$v" = default ]; then L=""; else L="GRKAN_LIB=tools/variants/$v/libgrkan_b200.so"; fi
  for dt in fp32 bf16; do
  env $L timeout 300 python bench.py --steps 20 --warmup 5 --dtype $dt --no-cpu-baseline --e2e-steps 1 --collective deterministic 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print('$v $dt', round(k['bwd_us'],1), round(k['collective_us'],1))"
  done
done
