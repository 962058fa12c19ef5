#!/bin/bash
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for NB in 222 296 444 148; do
  P=$((29500 + RANDOM % 100))
  timeout 600 $TR --nproc-per-node 4 --master-port $P bench.py --gpus 4 --steps 50 --warmup 10 --no-train --no-cpu-baseline --no-virtual --fused-nblocks $NB > gpurun_out/fnb_$NB.json 2>/dev/null
  python - $NB <<'PY'
import json,sys
for l in open(f"gpurun_out/fnb_{sys.argv[1]}.json"):
    if l.startswith("{"):
        d=json.loads(l); k=d["sync_kernels"]["fused_round"]
        print(json.dumps({"fused_nblocks": int(sys.argv[1]), "ms_per_step": round(d["ms_per_step"],4), "isolated_ms": round(k.get("isolated_ms",0),4)}))
PY
done
