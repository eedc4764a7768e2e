mkdir -p gpurun_out
TAG=${TAG:-r2l}
timeout 1200 python -m pytest tests/test_w16_gpu.py tests/test_engine_gpu.py tests/test_kernels_gpu.py -q -rs > gpurun_out/tests_${TAG}.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/tests_${TAG}.log; grep -E "^FAILED" gpurun_out/tests_${TAG}.log
for a in "googlenet 4 64" "mobilenet_v2 4 64" "vgg16 4 64 --fuse"; do timeout 600 python tools/conv_shapes_check.py $a 2>&1 | tail -1; done
