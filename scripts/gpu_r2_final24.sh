# the driver's bench at N=2 and N=4 (default flags)
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for N in 2 4; do
  timeout 1500 $TR --nproc-per-node $N --master-port 2980$N bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/g2_n$N.json 2> gpurun_out/g2_n$N.err; echo n$N rc=$?
done
