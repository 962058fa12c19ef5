#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_multigpu.py tests/test_gpu_p2p_one_gpu.py -x -q > gpurun_out/ce2_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/ce2_tests.log
PORT=29870
for P in 4 3; do
  PORT=$((PORT+1))
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port $PORT \
    bench.py --gpus $P --steps 20 --warmup 5 --no-cpu-baseline --no-virtual --legs overlap,overlap_sm,overlap_ce,fused \
    > gpurun_out/ce2_train_n$P.log 2>&1
  echo "train P=$P rc=$?"
done
PORT=$((PORT+1))
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 3 --master-addr 127.0.0.1 --master-port $PORT \
  tools/micro_sweep.py --sizes-mb 16,102.228128,256,1024 --nblocks 128 --algos twoshot,ce --fused-algos "" \
  > gpurun_out/ce_sweep_p3.jsonl 2> gpurun_out/ce_sweep_p3.err
echo "sweep P=3 rc=$?"
