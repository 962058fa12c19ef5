set -x
timeout 600 python -m pytest tests/test_gpu_multigpu.py -x -q -k "graph_replay" > gpurun_out/mg_graph.log 2>&1; echo g rc=$?
tail -30 gpurun_out/mg_graph.log | grep -E "Error|error|assert|passed|failed" | head -10
timeout 900 python -m pytest tests/test_gpu_sync_graph.py tests/test_gpu_fused.py tests/test_gpu_guardbands.py -x -q > gpurun_out/t_sg.log 2>&1; echo sg rc=$?
tail -2 gpurun_out/t_sg.log
