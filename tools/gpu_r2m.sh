mkdir -p gpurun_out
TAG=${TAG:-r2m}
timeout 1500 python -m pytest tests/test_conv_stats_gpu.py tests/test_w16_gpu.py tests/test_engine_gpu.py tests/test_engine_c2_gpu.py tests/test_profiler_gpu.py -q -rs -x > gpurun_out/tests_${TAG}.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/tests_${TAG}.log; grep -E "^(FAILED|ERROR)|^E " gpurun_out/tests_${TAG}.log | head -20
