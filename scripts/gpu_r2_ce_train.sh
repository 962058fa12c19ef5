#!/bin/bash
# Training legs at N=4 and N=2: overlap on the SM mean vs overlap on the copy-engine mean.
mkdir -p gpurun_out
PORT=29850
for P in 4 2; do
  for rep in 1 2; do
    PORT=$((PORT+1))
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port $PORT \
      bench.py --gpus $P --steps 20 --warmup 5 --no-cpu-baseline --no-virtual --legs overlap,overlap_ce,fused \
      > gpurun_out/ce_train_n${P}_$rep.log 2>&1
    echo "P=$P rep=$rep rc=$?"
  done
done
