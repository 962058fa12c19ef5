# MobileNetV2 sync path vs the fused round's CTA count at N=2 / N=4
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
P=29790
for N in 2 4; do for NB in 74 148 296; do
  P=$((P+1))
  timeout 600 $TR --nproc-per-node $N --master-port $P bench.py --model mobilenet_v2 --gpus $N --steps 100 --warmup 10 --no-train --fused-nblocks $NB 2>/dev/null | grep "^{" | python -c "import sys,json; d=json.loads(sys.stdin.read()); print($N, $NB, d['config']['fused_round_algo'], round(d['ms_per_step'],4))"
done; done
