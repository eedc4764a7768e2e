mkdir -p gpurun_out
TAG=${TAG:-r2g}
timeout 900 python -m pytest tests/test_w16_gpu.py tests/test_kernels_gpu.py tests/test_kernels_c2_gpu.py -x -q > gpurun_out/tests_${TAG}.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/tests_${TAG}.log
timeout 600 python tools/conv_bench.py --resnet50 > gpurun_out/conv_table_${TAG}.txt 2>&1
echo "conv table rc=$?"; cat gpurun_out/conv_table_${TAG}.txt
