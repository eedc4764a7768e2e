mkdir -p gpurun_out
TAG=${TAG:-r2o}
timeout 900 python -m pytest tests/test_conv_stats_gpu.py -q -x > gpurun_out/tests_${TAG}.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/tests_${TAG}.log
bash tools/gpu_catalogs_r2c.sh > gpurun_out/catalogs_${TAG}.log 2>&1
for job in "vgg16 176 224 --fused" "vgg16 176 224 --fused --split"; do
  timeout 1500 python tools/profile_catalog.py $job > /dev/null 2>&1; echo "$job rc=$?"
done
cp profiles/catalog_*.json gpurun_out/catalogs/
