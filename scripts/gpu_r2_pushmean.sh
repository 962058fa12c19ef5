#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multigpu.py -x -q -k "allreduce or copy_engine or worker_round" > gpurun_out/pm_test.log 2>&1; echo "test rc=$? $(tail -1 gpurun_out/pm_test.log)"
PORT=29950
for P in 4 3 2; do
  PORT=$((PORT+1))
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port $PORT \
    tools/micro_sweep.py --sizes-mb 16,64,102.228128,256,1024 --nblocks 128,296 --algos twoshot,push,ce --fused-algos "" \
    > gpurun_out/pm_sweep_p$P.jsonl 2> gpurun_out/pm_sweep_p$P.err
  echo "sweep P=$P rc=$?"
done
