# Re-measure every benchmark catalog with the round-2 kernels (R3 profiler, monet_profile_variant).
set -x
python tools/profile_catalog.py resnet50 184 224 --fused > gpurun_out/cat_r50f.log 2>&1
python tools/profile_catalog.py resnet50 184 224 --fused --split > gpurun_out/cat_r50fs.log 2>&1
python tools/profile_catalog.py vgg16 176 224 > gpurun_out/cat_vgg.log 2>&1
python tools/profile_catalog.py vgg16 176 224 --split > gpurun_out/cat_vggs.log 2>&1
python tools/profile_catalog.py mobilenet_v2 272 224 --fused > gpurun_out/cat_mb.log 2>&1
python tools/profile_catalog.py googlenet 320 224 --fused > gpurun_out/cat_gn.log 2>&1
python tools/profile_catalog.py unet 11 416x608 --fused > gpurun_out/cat_unet.log 2>&1
mkdir -p gpurun_out/catalogs && cp profiles/catalog_*.json gpurun_out/catalogs/
tail -n 2 gpurun_out/cat_*.log
