#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multigpu.py -x -q -k "graph_replay" > gpurun_out/sp2_test.log 2>&1; echo "tests rc=$? $(tail -1 gpurun_out/sp2_test.log)"
nvidia-smi --query-gpu=clocks.sm --format=csv -lms 200 > /dev/null 2>&1 &
SMI=$!
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1500 $TR --nproc-per-node 4 --master-port 29881 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/sp2_n4.json 2> gpurun_out/sp2_n4.err; echo "n4 rc=$?"
timeout 900 $TR --nproc-per-node 4 --master-port 29882 bench.py --gpus 4 --steps 20 --warmup 5 --no-train --no-cpu-baseline --sync-graph > gpurun_out/sp2_n4_graph.json 2> /dev/null; echo "n4 graph rc=$?"
kill $SMI
for f in sp2_n4 sp2_n4_graph; do python - $f <<'PY'
import json,sys
for l in open(f"gpurun_out/{sys.argv[1]}.json"):
    if l.startswith("{"):
        d=json.loads(l); k=d["sync_kernels"]["fused_round"]
        print(sys.argv[1], "ms/step", round(d["ms_per_step"],4), "iso", round(k.get("isolated_ms",0),4), "frac", round(d["roofline"]["frac"],3), "e2e", round(d["e2e"]["value"]))
        t=d.get("training")
        if t: print({kk:round(t[kk]["exposed_sync_ms_per_step"],3) for kk in t if isinstance(t[kk],dict) and "exposed_sync_ms_per_step" in t[kk]})
        print(d.get("allreduce_isolated_ms"))
PY
done
