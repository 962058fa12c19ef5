# compute-sanitizer over the virtual-rank suites (one tool per call: memcheck or synccheck / racecheck)
TOOL=${1:-memcheck}
set -x
timeout 2400 compute-sanitizer --tool $TOOL --target-processes all --error-exitcode 99 --log-file gpurun_out/sanitizer_$TOOL.%p.log \
  python -m pytest tests/test_gpu_fused.py tests/test_gpu_collective.py tests/test_gpu_kernels.py tests/test_gpu_sync_graph.py -q -x \
  -k "not 1gib and not resnet50_size" > gpurun_out/sanitizer_$TOOL.pytest.log 2>&1
echo rc=$?
tail -3 gpurun_out/sanitizer_$TOOL.pytest.log
cat gpurun_out/sanitizer_$TOOL.*.log | grep -E "ERROR SUMMARY|========= [A-Z]" | sort | uniq -c | head -20
