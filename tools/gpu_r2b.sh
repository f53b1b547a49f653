# Round 2 check b: host-pipeline tests, shim e2e, spawn-hang diagnosis, bf16 backward variants, ncu source capture.
TAG=${1:-r2b}
mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests/test_gpu_host.py tests/test_gpu_api.py -k "host or staged or concurrent" > gpurun_out/pytest_${TAG}_host.txt 2>&1; tail -5 gpurun_out/pytest_${TAG}_host.txt
# shim (reference API) e2e, fp32 KAT-B
timeout 600 python bench.py --config kat-b --dtype fp32 --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench_${TAG}_katb_fp32.json 2> gpurun_out/bench_${TAG}_katb_fp32.err
python -c "import json; d=json.load(open('gpurun_out/bench_${TAG}_katb_fp32.json')); print('shim', d['e2e'].get('reference_api'))" || tail -5 gpurun_out/bench_${TAG}_katb_fp32.err
# spawn hang: dump stacks after 60 s
GRKAN_BENCH_TRACE_AFTER=60 timeout 150 python bench.py --gpus 2 --config kat-t --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --dist-backend gloo > gpurun_out/spawn_${TAG}.out 2> gpurun_out/spawn_${TAG}.err; echo "spawn rc=$?"; tail -c 3000 gpurun_out/spawn_${TAG}.err
for v in default cw6 cw4 cw12 guard; do
  if [ "$v" = default ]; then L=""; else L="GRKAN_LIB=tools/variants/$v/libgrkan_b200.so"; fi
  for cfg in kat-b kat-s; do
    env $L timeout 300 python bench.py --config $cfg --steps 30 --warmup 5 --dtype bf16 --no-cpu-baseline --e2e-steps 1 > /tmp/vb.json 2>/tmp/vb.err
    python -c "import json; d=json.load(open('/tmp/vb.json')); k=d['kernels']; print('$v $cfg bf16', 'bwd=%.1fus(%.3f)'%(k['bwd_us'],k['bwd_frac']), 'fwd=%.1fus(%.3f)'%(k['fwd_us'],k['fwd_frac']), d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 /tmp/vb.err
  done
  env $L timeout 300 python bench.py --config kat-b --steps 30 --warmup 5 --dtype fp32 --no-cpu-baseline --e2e-steps 1 > /tmp/vb.json 2>/tmp/vb.err
  python -c "import json; d=json.load(open('/tmp/vb.json')); k=d['kernels']; print('$v kat-b fp32', 'bwd=%.1fus(%.3f)'%(k['bwd_us'],k['bwd_frac']), 'fwd=%.1fus(%.3f)'%(k['fwd_us'],k['fwd_frac']))" || tail -3 /tmp/vb.err
done
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --dtype bf16"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_bwd_staged" -s 3 -c 1 -o gpurun_out/prof_${TAG}_bwd_bf16 $B > /dev/null 2>&1
ls gpurun_out | grep prof_${TAG}
