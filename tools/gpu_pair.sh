# pair variant: kernel tests with hang protection, then the ResNet-50 conv table for splitk vs pair
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_kernels_gpu.py -q -x 2>&1 | tail -4
timeout 400 python tools/conv_bench.py --resnet50 --variants splitk,pair --iters 5 2>&1 | tee gpurun_out/conv_table_pair.log | tail -40
