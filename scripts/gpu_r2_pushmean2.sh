#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_multigpu.py tests/test_gpu_p2p_one_gpu.py -x -q > gpurun_out/pm2_test.log 2>&1; echo "tests rc=$? $(tail -1 gpurun_out/pm2_test.log)"
PORT=29970
for P in 4 3; do
  PORT=$((PORT+1))
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port $PORT \
    tools/micro_sweep.py --sizes-mb 4,16,64,102.228128,256,1024 --nblocks 128 --algos oneshot,twoshot,push,ce --fused-algos "auto" \
    > gpurun_out/pm2_sweep_p$P.jsonl 2> gpurun_out/pm2_sweep_p$P.err
  echo "sweep P=$P rc=$?"
done
PORT=$((PORT+1))
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $PORT \
  bench.py --gpus 4 --steps 20 --warmup 5 --no-cpu-baseline --no-virtual --legs overlap,overlap_sm,overlap_ce,fused \
  > gpurun_out/pm2_train_n4.log 2>&1
echo "train rc=$?"
