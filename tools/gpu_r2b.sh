# bf16 x-factor table (LUT) A/B: parity tests, KAT-B/KAT-S bf16 lines with and
# without the table, an ncu capture of the table kernel; plus a stack dump of the
# self-spawned 2-rank bench.  usage: bash tools/gpu_r2b.sh TAG
TAG=${1:-r2b}
mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests/test_gpu_lut.py tests/test_gpu_deterministic.py "tests/test_gpu_parity.py" -k "lut or bf16 or deterministic or golden" > gpurun_out/pytest_${TAG}.txt 2>&1; tail -3 gpurun_out/pytest_${TAG}.txt
for cfg in kat-b kat-s; do for lut in 1 0; do
  GRKAN_LUT=$lut timeout 300 python bench.py --config $cfg --dtype bf16 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_${TAG}_${cfg}_lut${lut}.json 2>gpurun_out/bench_${TAG}.err
  python -c "import json; d=json.load(open('gpurun_out/bench_${TAG}_${cfg}_lut${lut}.json')); k=d['kernels']; print('$cfg lut=$lut value %.3e ms %.4f fwd %.1f bwd %.1f bwd_frac %.3f' % (d['value'], d['ms_per_step'], k['fwd_us'], k['bwd_us'], k['bwd_frac']), d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 gpurun_out/bench_${TAG}.err
done; done
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --dtype bf16"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_bwd_staged" -s 3 -c 1 -o gpurun_out/prof_${TAG}_bwd_bf16_lut $B > /dev/null 2>&1
GRKAN_BENCH_TRACE_AFTER=150 timeout 240 python bench.py --gpus 2 --config kat-t --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --dist-backend gloo > gpurun_out/spawn_${TAG}.out 2> gpurun_out/spawn_${TAG}.err; echo "spawn rc=$?"; tail -c 600 gpurun_out/spawn_${TAG}.out
ls -la gpurun_out | grep $TAG
