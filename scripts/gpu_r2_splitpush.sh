#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_multigpu.py tests/test_gpu_p2p_one_gpu.py -x -q > gpurun_out/sp_test.log 2>&1; echo "tests rc=$? $(tail -1 gpurun_out/sp_test.log)"
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for N in 4 3 4; do
  P=$((29700 + RANDOM % 200))
  timeout 900 $TR --nproc-per-node $N --master-port $P bench.py --gpus $N --steps 20 --warmup 5 --no-train --no-cpu-baseline > gpurun_out/sp_n$N.json 2> /dev/null
  python - $N <<'PY'
import json,sys
for l in open(f"gpurun_out/sp_n{sys.argv[1]}.json"):
    if l.startswith("{"):
        d=json.loads(l); k=d["sync_kernels"]["fused_round"]
        print("N", sys.argv[1], "ms/step", round(d["ms_per_step"],4), "avg", round(k["avg_ms"],4), "iso", round(k["isolated_ms"],4), "frac", round(d["roofline"]["frac"],3))
PY
done
