# fp32 KAT-B backward geometry vs power: default bench lines alternating wide / 2x8, clocks and power.
TAG=${1:-r2pw}
mkdir -p gpurun_out
for rep in 1 2 3; do for w in 1 0; do
  GRKAN_WIDE=$w timeout 300 python bench.py --no-cpu-baseline --e2e-steps 1 > /tmp/ab.json 2>/dev/null
  python -c "import json; d=json.load(open('/tmp/ab.json')); k=d['kernels']; c=d['clocks']; print('wide=$w value %.3e fwd %.1f bwd %.1f' % (d['value'], k['fwd_us'], k['bwd_us']), c['sm_mhz'], c['reasons'], 'P_inst_med %.0f max %.0f' % (c.get('power_inst_w_median') or 0, c.get('power_inst_w_max') or 0))"
done; done 2>&1 | tee gpurun_out/ab_${TAG}.txt
