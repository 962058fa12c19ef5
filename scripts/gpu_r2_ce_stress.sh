#!/bin/bash
# CE mean + torch.optim front end under repetition: the multi-GPU CE test 5x at world 4,
# the whole multi-GPU suite once more, and the training legs at N=4 once.
mkdir -p gpurun_out/stress_ce
for i in 1 2 3 4 5; do
  timeout 600 python -m pytest tests/test_gpu_multigpu.py -x -q -k "copy_engine or torch_optim" > gpurun_out/stress_ce/ce_$i.log 2>&1
  echo "ce run $i rc=$? $(tail -1 gpurun_out/stress_ce/ce_$i.log)"
done
timeout 1500 python -m pytest tests/test_gpu_multigpu.py tests/test_gpu_torch_optim.py -q > gpurun_out/stress_ce/multigpu.log 2>&1
echo "multigpu rc=$? $(tail -1 gpurun_out/stress_ce/multigpu.log)"
