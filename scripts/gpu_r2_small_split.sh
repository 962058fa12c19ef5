#!/bin/bash
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for M in resnet18 mobilenet_v2; do
  for N in 4 3; do
    P=$((29600 + RANDOM % 200))
    timeout 600 $TR --nproc-per-node $N --master-port $P bench.py --gpus $N --model $M --steps 50 --warmup 10 --no-train --no-cpu-baseline --no-virtual > gpurun_out/small_${M}_n$N.json 2>/dev/null
    python - $M $N <<'PY'
import json,sys
for l in open(f"gpurun_out/small_{sys.argv[1]}_n{sys.argv[2]}.json"):
    if l.startswith("{"):
        d=json.loads(l); k=d["sync_kernels"]["fused_round"]
        print(json.dumps({"model": sys.argv[1], "N": int(sys.argv[2]), "ms_per_step": round(d["ms_per_step"],4), "isolated_ms": round(k.get("isolated_ms",0),4), "algo": d["config"].get("fused_round_algo")}))
PY
  done
done
