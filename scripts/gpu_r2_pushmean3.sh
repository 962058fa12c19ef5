#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_multigpu.py -x -q -k "allreduce or copy_engine or fault or adaptive or graph_replay or worker_round" > gpurun_out/pm3_test.log 2>&1; echo "tests rc=$? $(tail -1 gpurun_out/pm3_test.log)"
PORT=29960
for P in 4 3; do
  PORT=$((PORT+1))
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port $PORT \
    tools/micro_sweep.py --sizes-mb 4,16,64,102.228128,256,1024 --nblocks 128 --algos twoshot,push,ce --fused-algos "auto" \
    > gpurun_out/pm3_sweep_p$P.jsonl 2> gpurun_out/pm3_sweep_p$P.err
  echo "sweep P=$P rc=$?"
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29969 tools/push_mean_trace.py 2>/dev/null > gpurun_out/pm3_trace.jsonl
