# A/B fused-kernel variants: bash tools/gpu_fused_variants.sh v1 v2 ...
for v in "$@"; do
  if [ "$v" = default ]; then L=""; else L="GRKAN_LIB=tools/variants/$v/libgrkan_b200.so"; fi
  env $L timeout 300 python tools/bench_fused.py --reps 20 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    print('$v', d['direction'], d['shape'][:30], 'fused=%.1fus unfused=%.1fus x%.2f' % (d['fused_us'], d['unfused_us'], d['speedup']))"
done
