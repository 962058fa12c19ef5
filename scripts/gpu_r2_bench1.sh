# N=1 bench at the driver's command with an external nvidia-smi sampler (as the driver runs it),
# then the flat-alignment A/B of the training step
set -x
nvidia-smi --query-gpu=clocks.sm --format=csv -lms 200 > gpurun_out/ext_smi.csv 2>&1 &
SMI=$!
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_n1.json 2> gpurun_out/r2_n1.err; echo n1 rc=$?
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_ref_n1.json 2> gpurun_out/r2_ref_n1.err; echo ref rc=$?
kill $SMI
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 --flat-align 4 --no-virtual --no-cpu-baseline > gpurun_out/r2_n1_align4.json 2> gpurun_out/r2_n1_align4.err; echo a4 rc=$?
tail -2 gpurun_out/r2_n1.err
