# multi-rank graph replay on 4 GPUs: full GPU suite at world 4, bench N=2/N=4 graph vs eager (sync path only)
set -x
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/all4.log 2>&1; echo all rc=$?
tail -2 gpurun_out/all4.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for N in 2 4; do
  timeout 600 $TR --nproc-per-node $N --master-port 2953$N bench.py --gpus $N --steps 20 --warmup 5 --no-train > gpurun_out/g_n$N.json 2> gpurun_out/g_n$N.err; echo g$N rc=$?
  timeout 600 $TR --nproc-per-node $N --master-port 2954$N bench.py --gpus $N --steps 20 --warmup 5 --no-train --no-sync-graph > gpurun_out/e_n$N.json 2> gpurun_out/e_n$N.err; echo e$N rc=$?
done
