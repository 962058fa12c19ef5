# side-stream all-reduce CTA budget vs the overlap pipeline's exposed sync at N=4
set -x
P=29770
for NB in 128 32 16; do
  P=$((P+1))
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $P bench.py --gpus 4 --steps 5 --warmup 3 --no-virtual --legs overlap,overlap_nvls --nvls-leg --nblocks $NB > gpurun_out/bud_$NB.json 2> gpurun_out/bud_$NB.err; echo nb$NB rc=$?
done
