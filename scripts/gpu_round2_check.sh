# round-2 check on one GPU: smoke, the new graph-replay tests, then the whole -m gpu suite
set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 900 python -m pytest tests/test_gpu_sync_graph.py tests/test_gpu_optimizer.py -x -q > gpurun_out/t1.log 2>&1; echo t1 rc=$?
tail -3 gpurun_out/t1.log
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_all.log 2>&1; echo all rc=$?
tail -3 gpurun_out/gpu_all.log
