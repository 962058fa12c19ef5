# BASELINE configs[1], [3]: ResNet-18 (CIFAR) and MobileNetV2 flat buffers, sync path at N=1/2/4 (no training legs)
set -x
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for M in mobilenet_v2 resnet18; do
  timeout 600 python bench.py --model $M --gpus 1 --steps 50 --warmup 5 --no-train --no-cpu-baseline --no-virtual > gpurun_out/sm_${M}_n1.json 2>/dev/null; echo $M n1 rc=$?
  for N in 2 4; do
    timeout 600 $TR --nproc-per-node $N --master-port 2978$N bench.py --model $M --gpus $N --steps 50 --warmup 5 --no-train > gpurun_out/sm_${M}_n$N.json 2>/dev/null; echo $M n$N rc=$?
  done
done
