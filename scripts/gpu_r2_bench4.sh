# N=4 bench (driver's command line) + its reference arm; then the multi-GPU suites at world 4
set -x
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/r2_n4.json 2> gpurun_out/r2_n4.err; echo n4 rc=$?
tail -3 gpurun_out/r2_n4.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29522 bench.py --impl reference --gpus 4 --steps 20 --warmup 5 > gpurun_out/r2_ref_n4.json 2> gpurun_out/r2_ref_n4.err; echo ref4 rc=$?
timeout 1500 python -m pytest tests/test_gpu_multigpu.py -x -q > gpurun_out/mg4.log 2>&1; echo mg4 rc=$?
tail -2 gpurun_out/mg4.log
