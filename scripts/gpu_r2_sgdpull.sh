# the one-pass overlap boundary (lasgd_sgd_pull): whole suite on 2 GPUs, then the overlap leg's exposed sync at N=2
set -x
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/sp_all2.log 2>&1; echo all rc=$?
tail -1 gpurun_out/sp_all2.log
timeout 900 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2 --master-port 29691 bench.py --gpus 2 --steps 20 --warmup 5 --no-virtual --legs fused,overlap,overlap_adaptive > gpurun_out/sp_n2.json 2> gpurun_out/sp_n2.err; echo n2 rc=$?
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 --no-virtual --no-cpu-baseline --legs fused,overlap > gpurun_out/sp_n1.json 2> gpurun_out/sp_n1.err; echo n1 rc=$?
