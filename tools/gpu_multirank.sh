# Two ranks sharing one GPU (gloo for the torch.distributed plumbing): exercises bench.py's
# N > 1 path -- per-rank shards, barrier + max-over-ranks timing, the three da/db
# collectives, incl. the CUDA-IPC peer exchange across two processes.
mkdir -p gpurun_out
for c in ${COLLECTIVES:-allreduce deterministic p2p}; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port $((29500 + RANDOM % 1000)) bench.py --gpus 2 --steps 10 --warmup 3 --dist-backend gloo \
    --collective $c --no-cpu-baseline --e2e-steps 1 > gpurun_out/multirank_$c.json 2> gpurun_out/multirank_$c.err
  echo "$c rc=$?"; tail -c 600 gpurun_out/multirank_$c.json; grep -i "error\|Traceback" gpurun_out/multirank_$c.err | head -5
done
# the DDP training step (config 4 path) with two ranks, KAT-T
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port $((29500 + RANDOM % 1000)) bench.py --config kat-t-train --gpus 2 --steps 5 --warmup 3 \
  --dist-backend gloo > gpurun_out/multirank_train.json 2> gpurun_out/multirank_train.err
echo "train rc=$?"
# strong scaling: global B=256 split over the two ranks
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port $((29500 + RANDOM % 1000)) bench.py --gpus 2 --steps 10 --warmup 3 --dist-backend gloo \
  --scaling strong --no-cpu-baseline --e2e-steps 1 > gpurun_out/multirank_strong.json 2> gpurun_out/multirank_strong.err
echo "strong rc=$?"
