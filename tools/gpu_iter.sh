# quick GPU iteration: layout probe, kernel numerics, conv micro-bench
mkdir -p gpurun_out
timeout 120 python tools/gemm_probe.py > gpurun_out/probe.log 2>&1; echo "probe rc=$?"
tail -30 gpurun_out/probe.log
timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q 2>&1 | tail -15
timeout 300 python tools/conv_bench.py --variants implicit,tf32x3 > gpurun_out/conv_bench.log 2>&1; echo "bench rc=$?"
cat gpurun_out/conv_bench.log
