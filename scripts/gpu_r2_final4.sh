# round-end check on 4 GPUs: multi-GPU suites 3x (stress), then the driver's bench at N=2 and N=4 with reference arms
set -x
for i in 1 2 3; do
  timeout 1200 python -m pytest tests/test_gpu_multigpu.py tests/test_gpu_cli.py -x -q > gpurun_out/st4_$i.log 2>&1; echo stress$i rc=$?
  tail -1 gpurun_out/st4_$i.log
done
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for N in 2 4; do
  timeout 900 $TR --nproc-per-node $N --master-port 2970$N bench.py --impl reference --gpus $N --steps 20 --warmup 5 > gpurun_out/fin_ref_n$N.json 2> gpurun_out/fin_ref_n$N.err; echo ref$N rc=$?
  timeout 1500 $TR --nproc-per-node $N --master-port 2971$N bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/fin_n$N.json 2> gpurun_out/fin_n$N.err; echo n$N rc=$?
done
