#!/bin/bash
# Usage (GPU box): TAG=r2n bash tools/r2_emulate.sh — the default bench (config 3 +
# the per-config table) as the driver's scaling run would launch it, with N
# ranks sharing GPU 0 (--emulate: correctness of the N > 1 flow only).
TAG=${TAG:-r2}
mkdir -p gpurun_out
for n in 2 4 8; do
  timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr 127.0.0.1 \
    --master-port $((29700 + n)) bench.py --gpus $n --steps 3 --warmup 3 --emulate \
    > gpurun_out/${TAG}_emulated_n$n.json 2> gpurun_out/${TAG}_emulated_n$n.err
  echo "n=$n rc=$?"
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr 127.0.0.1 \
    --master-port $((29800 + n)) bench.py --impl reference --gpus $n --steps 3 --warmup 3 \
    > gpurun_out/${TAG}_emulated_reference_n$n.json 2> gpurun_out/${TAG}_emulated_reference_n$n.err
  echo "reference n=$n rc=$?"
done
