# 2-GPU check: the multi-GPU suites (bucketed SGD-AR included), then bench at N=1 and N=2
set -x
timeout 1200 python -m pytest tests/test_gpu_multigpu.py -x -q > gpurun_out/mg2.log 2>&1; echo mg rc=$?
tail -3 gpurun_out/mg2.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bn1.json 2> gpurun_out/bn1.err; echo bn1 rc=$?
tail -3 gpurun_out/bn1.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/bn2.json 2> gpurun_out/bn2.err; echo bn2 rc=$?
tail -3 gpurun_out/bn2.err
