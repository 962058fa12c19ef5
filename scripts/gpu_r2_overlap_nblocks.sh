#!/bin/bash
# Overlap-pipeline exposed sync at N=4 vs the side-stream mean's CTA count.
mkdir -p gpurun_out
P=29710
for NB in 128 32 8; do
  P=$((P+1))
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $P \
    bench.py --gpus 4 --steps 20 --warmup 5 --no-cpu-baseline --no-virtual --legs overlap,fused --nblocks $NB \
    > gpurun_out/overlap_nb$NB.log 2>&1
  echo "nb=$NB rc=$?"
done
