mkdir -p gpurun_out
TAG=${TAG:-r2n}
timeout 1500 python -m pytest tests/test_engine_gpu.py tests/test_profiler_gpu.py tests/test_dp_engine_gpu.py tests/test_kernels_gpu.py -q -rs > gpurun_out/tests_${TAG}.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/tests_${TAG}.log; grep -E "^(FAILED|ERROR)" gpurun_out/tests_${TAG}.log | head -20
bash tools/gpu_catalogs_r2c.sh > gpurun_out/catalogs_${TAG}.log 2>&1
for job in "vgg16 176 224 --fused" "vgg16 176 224 --fused --split"; do
  timeout 1500 python tools/profile_catalog.py $job > /dev/null 2>&1; echo "$job rc=$?"
done
cp profiles/catalog_*.json gpurun_out/catalogs/
