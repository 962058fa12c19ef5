# round-2 ncu evidence (one GPU): launch list of the N=1 sync-path bench, --set full of the
# round-2 kernels (report reduced to CSV pages on the box: the .ncu-rep exceeds the 64 MiB
# copy-back), plus the K1 copy-variant probe
set -x
./tools/copy_probe > gpurun_out/copy_probe.jsonl 2>&1
B="python bench.py --steps 20 --warmup 5 --kernels-only --no-cpu-baseline --no-virtual"
$B > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02_bench_n1.csv $B > gpurun_out/ncu_bench.log 2>&1
echo launches rc=$?
python tools/profile_r02.py > gpurun_out/plain_prof.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'k_sgd_dyn|k_push|k_twoshot|k_oneshot' -o /tmp/prof_r02 python tools/profile_r02.py > gpurun_out/ncu_prof.log 2>&1
echo full rc=$?
ncu -i /tmp/prof_r02.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__grid_size,sm__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum > gpurun_out/prof_r02_raw.csv 2>&1
ncu -i /tmp/prof_r02.ncu-rep --page details --csv > gpurun_out/prof_r02_details.csv 2>&1
ncu -i /tmp/prof_r02.ncu-rep --page source --csv -k regex:k_sgd_dyn -c 1 > gpurun_out/prof_r02_source_sgd_dyn.csv 2>&1
ls -la gpurun_out/
du -sh gpurun_out
