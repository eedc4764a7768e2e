# kernel tests with hang protection, the ResNet-50 conv table, then fresh catalogs if the tests pass
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_kernels_gpu.py -q -x 2>&1 | tail -15
rc=${PIPESTATUS[0]}
timeout 300 python tools/conv_bench.py --resnet50 --variants splitk --iters 5 2>&1 | tee gpurun_out/conv_table.log | tail -30
if [ "${CATALOG:-0}" = 1 ]; then bash tools/gpu_catalog.sh; fi
