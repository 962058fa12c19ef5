#!/bin/bash
mkdir -p gpurun_out/stress_final
for i in 1 2; do
  timeout 900 python -m pytest tests/test_gpu_multigpu.py -x -q > gpurun_out/stress_final/multigpu_$i.log 2>&1
  echo "pass $i rc=$? $(tail -1 gpurun_out/stress_final/multigpu_$i.log)"
done
