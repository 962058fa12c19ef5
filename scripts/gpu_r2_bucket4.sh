# exposed sync of the bucketed SGD-AR vs DDP at 4 GPUs for bucket CTA budgets / algorithms,
# and the eager per-round time at N=2 / N=4 (publish_done with a device-scope per-CTA fence)
set -x
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4"
P=29600
for C in 64 32 128; do
  P=$((P+1))
  timeout 900 $TR --master-port $P bench.py --gpus 4 --steps 5 --warmup 3 --no-virtual --legs sgd_ar_bucketed,ddp_nccl --bucket-ctas $C > gpurun_out/bk_c$C.json 2> gpurun_out/bk_c$C.err; echo c$C rc=$?
done
for N in 2 4; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2962$N tools/graph_trace_probe.py 2>/dev/null | grep '"rank": 0' > gpurun_out/gtp_fence_n$N.jsonl; echo p$N rc=$?
done
cat gpurun_out/gtp_fence_n*.jsonl
