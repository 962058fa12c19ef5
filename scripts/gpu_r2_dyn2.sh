set -x
timeout 900 python -m pytest tests/test_gpu_sync_graph.py tests/test_gpu_guardbands.py -x -q > gpurun_out/t_sg2.log 2>&1; echo sg rc=$?
tail -1 gpurun_out/t_sg2.log
timeout 600 python -m pytest tests/test_gpu_multigpu.py -x -q -k "graph_replay" > gpurun_out/mg_graph2.log 2>&1; echo g rc=$?
tail -1 gpurun_out/mg_graph2.log
for i in 1 2; do
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 --no-train --no-cpu-baseline --no-virtual > gpurun_out/d_n1_$i.json 2> gpurun_out/d_n1.err; echo n1 rc=$?
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 --no-train --no-cpu-baseline --no-virtual --no-sync-graph > gpurun_out/de_n1_$i.json 2>> gpurun_out/d_n1.err; echo n1e rc=$?
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2"
timeout 600 $TR --master-port 2956$i bench.py --gpus 2 --steps 20 --warmup 5 --no-train > gpurun_out/d_n2_$i.json 2> gpurun_out/d_n2.err; echo n2 rc=$?
timeout 600 $TR --master-port 2957$i bench.py --gpus 2 --steps 20 --warmup 5 --no-train --no-sync-graph > gpurun_out/de_n2_$i.json 2>> gpurun_out/d_n2.err; echo n2e rc=$?
done
