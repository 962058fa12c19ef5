# programmatic dependent launch on every plain sync-kernel launch: full suite (2 GPUs) + per-round timing
set -x
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pdl_all2.log 2>&1; echo all rc=$?
tail -1 gpurun_out/pdl_all2.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29631 tools/graph_trace_probe.py 2>/dev/null | grep '"rank": 0' > gpurun_out/gtp_pdl_n2.jsonl; echo p2 rc=$?
ALGO=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29632 tools/graph_trace_probe.py 2>/dev/null | grep '"rank": 0' > gpurun_out/gtp_pdl_n2_k7.jsonl; echo p2b rc=$?
cat gpurun_out/gtp_pdl_n2*.jsonl
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 --no-train --no-cpu-baseline > gpurun_out/pdl_n1.json 2> gpurun_out/pdl_n1.err; echo n1 rc=$?
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 --no-train --no-cpu-baseline --pipeline overlap --no-sync-graph --no-virtual > gpurun_out/pdl_n1_ov.json 2>> gpurun_out/pdl_n1.err; echo n1ov rc=$?
