# everything on a 4-GPU box: smoke, the whole GPU suite (world 4), bench N=1 (driver command line)
set -x
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/af_smoke.log 2>&1; echo smoke rc=$?
timeout 3000 python -m pytest tests -m gpu -q > gpurun_out/af_gpu4.log 2>&1; echo gpu rc=$?
tail -1 gpurun_out/af_gpu4.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/af_n1.json 2> gpurun_out/af_n1.err; echo n1 rc=$?
