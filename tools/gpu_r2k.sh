# VGG-16 with conv+ReLU fused: catalogs (unsplit and split) + the new GPU tests.
mkdir -p gpurun_out/catalogs
TAG=${TAG:-r2k}
timeout 900 python -m pytest tests/test_engine_gpu.py tests/test_w16_gpu.py -q -rs -k "vgg or prefetch or w16" > gpurun_out/tests_${TAG}.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/tests_${TAG}.log
for job in "vgg16 176 224 --fused" "vgg16 176 224 --fused --split"; do
  name=$(echo $job | tr ' ' '_' | tr -d '-')
  timeout 1500 python tools/profile_catalog.py $job > gpurun_out/cat_${name}.log 2>&1
  echo "$job rc=$?"
done
cp profiles/catalog_vgg16_fused*.json gpurun_out/catalogs/
timeout 600 python tools/conv_shapes_check.py googlenet 4 64 > gpurun_out/shapes_googlenet_${TAG}.txt 2>&1
tail -40 gpurun_out/shapes_googlenet_${TAG}.txt
timeout 120 tools/bin/tma_bw_probe > gpurun_out/tma_bw_${TAG}.txt 2>&1; cat gpurun_out/tma_bw_${TAG}.txt
