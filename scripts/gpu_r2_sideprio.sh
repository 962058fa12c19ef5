#!/bin/bash
# Overlap-pipeline exposure vs the side stream's priority (N=4), and the side-stream
# wait at the boundary (timeline) — is the mean starved by forward/backward?
mkdir -p gpurun_out
PORT=29890
for PR in 0 -1; do
  PORT=$((PORT+1))
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $PORT \
    bench.py --gpus 4 --steps 20 --warmup 5 --no-cpu-baseline --no-virtual --legs overlap,overlap_sm,fused \
    --side-priority $PR > gpurun_out/sideprio_n4_$PR.log 2>&1
  echo "prio=$PR rc=$?"
done
