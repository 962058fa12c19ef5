# the driver's round-end sequence on one GPU: smoke, pytest -m gpu, bench N=1 + reference arm
set -x
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo smoke rc=$?
tail -1 gpurun_out/f_smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/f_gpu1.log 2>&1; echo gpu rc=$?
tail -1 gpurun_out/f_gpu1.log
nvidia-smi --query-gpu=clocks.sm --format=csv -lms 200 > gpurun_out/f_smi.csv 2>&1 &
SMI=$!
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/f_ref_n1.json 2> gpurun_out/f_ref_n1.err; echo ref rc=$?
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/f_n1.json 2> gpurun_out/f_n1.err; echo n1 rc=$?
kill $SMI
