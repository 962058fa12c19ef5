# NVLS (tolerance-mode in-switch mean) on 4 GPUs: the multi-GPU suite, then the overlap pipeline on it in training
set -x
timeout 1500 python -m pytest tests/test_gpu_multigpu.py -x -q > gpurun_out/nv4_mg.log 2>&1; echo mg rc=$?
tail -1 gpurun_out/nv4_mg.log
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29761 bench.py --gpus 4 --steps 20 --warmup 5 --legs fused,overlap,overlap_nvls --nvls-leg > gpurun_out/nv4_bench.json 2> gpurun_out/nv4_bench.err; echo b rc=$?
tail -3 gpurun_out/nv4_bench.err
