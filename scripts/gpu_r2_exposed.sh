# exposed-sync resolution run: every training leg interleaved, 20 repetitions x 5 steps
N=${1:-2}
set -x
if [ "$N" = "1" ]; then
  timeout 1500 python bench.py --gpus 1 --steps 200 --warmup 20 --train-reps 20 --train-block 5 > gpurun_out/exposed_n1.json 2> gpurun_out/exposed_n1.err
else
  timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus $N --steps 200 --warmup 20 --train-reps 20 --train-block 5 > gpurun_out/exposed_n$N.json 2> gpurun_out/exposed_n$N.err
fi
echo rc=$?
tail -3 gpurun_out/exposed_n$N.err
