#!/bin/bash
# Copy-engine mean: multi-GPU parity, then the all-reduce sweep (SM one-shot/two-shot vs
# CE vs NCCL) at P=2 and P=4.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multigpu.py -x -q -k "copy_engine" > gpurun_out/ce_test.log 2>&1
echo "test rc=$?"
tail -3 gpurun_out/ce_test.log
PORT=29810
for P in 4 2; do
  PORT=$((PORT+1))
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port $PORT \
    tools/micro_sweep.py --sizes-mb 4,16,64,102.228128,256,1024 --nblocks 32,128 --algos twoshot,ce --fused-algos "" \
    > gpurun_out/ce_sweep_p$P.jsonl 2> gpurun_out/ce_sweep_p$P.err
  echo "sweep P=$P rc=$?"
done
