# ncu evidence for the round: launch list of one bench step + full capture of the top kernel.
mkdir -p gpurun_out
TAG=${TAG:-r1}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
  --log-file gpurun_out/launches_${TAG}.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-graph > gpurun_out/ncu_bench_${TAG}.log 2>&1
echo "launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_ -c 1 \
  -o gpurun_out/gemm_fwd_${TAG} -f python tools/conv_bench.py --only l2_3x3_128 --passes fwd --variants splitk --iters 1 > gpurun_out/ncu_gemm_fwd_${TAG}.log 2>&1
echo "gemm fwd rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_ -c 1 \
  -o gpurun_out/gemm_wgrad_${TAG} -f python tools/conv_bench.py --only l1_3x3_64 --passes wgrad --variants splitk --iters 1 > gpurun_out/ncu_gemm_wgrad_${TAG}.log 2>&1
echo "gemm wgrad rc=$?"
timeout 600 ncu --set full --clock-control none -k regex:bn_ -c 2 \
  -o gpurun_out/bn_${TAG} -f python -m pytest tests/test_kernels_gpu.py -m gpu -q -k batchnorm > gpurun_out/ncu_bn_${TAG}.log 2>&1
echo "bn rc=$?"
ls -la gpurun_out
