#!/bin/bash
# Round-end multi-GPU validation: pytest -m gpu on 4 GPUs, the driver's bench at N=2 and
# N=4 with their reference arms (driver flags), an external nvidia-smi sampler running.
mkdir -p gpurun_out
timeout 2000 python -m pytest tests -m gpu -q > gpurun_out/h_gpu4.log 2>&1; echo "gpu4 rc=$? $(tail -1 gpurun_out/h_gpu4.log)"
nvidia-smi --query-gpu=clocks.sm --format=csv -lms 200 > gpurun_out/h_smi.csv 2>&1 &
SMI=$!
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for N in 2 4; do
  timeout 900 $TR --nproc-per-node $N --master-port 2991$N bench.py --impl reference --gpus $N --steps 20 --warmup 5 > gpurun_out/h_ref_n$N.json 2> gpurun_out/h_ref_n$N.err; echo "ref n$N rc=$?"
  timeout 1500 $TR --nproc-per-node $N --master-port 2992$N bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/h_n$N.json 2> gpurun_out/h_n$N.err; echo "n$N rc=$?"
done
kill $SMI
