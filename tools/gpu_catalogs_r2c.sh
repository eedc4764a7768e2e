# Re-measure every benchmark catalog with the pre-split-weight conv path (graph params_bytes
# now include the bf16 weight planes, so every catalog and schedule is re-made).
set -x
mkdir -p gpurun_out/catalogs
for job in "resnet50 184 224 --fused" "resnet50 184 224 --fused --split" "resnet50 184 224" \
           "vgg16 176 224" "vgg16 176 224 --split" "mobilenet_v2 272 224 --fused" \
           "googlenet 320 224 --fused" "unet 11 416x608 --fused"; do
  name=$(echo $job | tr ' ' '_' | tr -d '-')
  timeout 1500 python tools/profile_catalog.py $job > gpurun_out/cat_${name}.log 2>&1
  echo "$job rc=$?"
  cp profiles/catalog_*.json gpurun_out/catalogs/
done
tail -n 1 gpurun_out/cat_*.log
