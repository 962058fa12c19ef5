set -x
timeout 900 python -m pytest tests/test_gpu_guardbands.py -x -q > gpurun_out/guard.log 2>&1; echo guard rc=$?
tail -3 gpurun_out/guard.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 tools/overlap_timeline.py > gpurun_out/timeline_p2.jsonl 2> gpurun_out/timeline_p2.err; echo tl rc=$?
tail -3 gpurun_out/timeline_p2.err
cat gpurun_out/timeline_p2.jsonl
