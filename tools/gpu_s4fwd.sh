# bf16 / fp32 forward and backward vs batch (fixed-cost fit) and forward variants (staged / direct, box copies).
TAG=${1:-s4f}
mkdir -p gpurun_out
one() {  # env cfg dtype extra
  env $1 timeout 300 python bench.py --config $2 --dtype $3 --steps 100 --no-cpu-baseline --e2e-steps 1 $4 > /tmp/ab.json 2>/tmp/ab.err
  python -c "import json; d=json.load(open('/tmp/ab.json')); k=d['kernels']; print('$1 $2 $3 $4 value %.3e fwd %.1f (%.3f) bwd %.1f (%.3f)' % (d['value'], k['fwd_us'], k['fwd_frac'], k['bwd_us'], k['bwd_frac']), d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 /tmp/ab.err
}
{
for b in 32 64 128 256; do one X=1 kat-b bf16 "--batch $b"; one X=1 kat-b fp32 "--batch $b"; done
for rep in 1 2; do
  one GRKAN_STAGED_FWD=1 kat-s bf16; one GRKAN_STAGED_FWD=0 kat-s bf16; one GRKAN_TMA2D=2 kat-s bf16
  one GRKAN_STAGED_FWD=1 kat-b bf16; one GRKAN_STAGED_FWD=0 kat-b bf16; one GRKAN_TMA2D=2 kat-b bf16
  one GRKAN_STAGED_FWD=1 kat-s fp32; one "GRKAN_WIDE=1 GRKAN_TMA2D=2" kat-s fp32
done
} 2>&1 | tee gpurun_out/ab_fwd_${TAG}.txt
