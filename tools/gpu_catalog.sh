# re-measure the catalogs (fused + unfused ResNet-50 b184 224) on the device
mkdir -p gpurun_out
timeout 900 python tools/profile_catalog.py --fused > gpurun_out/profile_fused.log 2>&1; echo "fused rc=$?"; tail -2 gpurun_out/profile_fused.log
timeout 900 python tools/profile_catalog.py > gpurun_out/profile_plain.log 2>&1; echo "plain rc=$?"; tail -2 gpurun_out/profile_plain.log
cp profiles/catalog_resnet50_fused_b184_224.json profiles/catalog_resnet50_b184_224.json gpurun_out/
