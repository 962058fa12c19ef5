# 4 GPUs: whole GPU suite, then bench N=2 and N=4 (sync path + virtual kernels, no training)
set -x
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/c4_all.log 2>&1; echo all rc=$?
tail -1 gpurun_out/c4_all.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for N in 2 4; do
  timeout 600 $TR --nproc-per-node $N --master-port 2966$N bench.py --gpus $N --steps 20 --warmup 5 --no-train > gpurun_out/c4_n$N.json 2> gpurun_out/c4_n$N.err; echo n$N rc=$?
  timeout 600 $TR --nproc-per-node $N --master-port 2967$N bench.py --gpus $N --steps 20 --warmup 5 --no-train --sync-graph > gpurun_out/c4_g$N.json 2> gpurun_out/c4_g$N.err; echo g$N rc=$?
done
