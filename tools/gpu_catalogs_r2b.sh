# Re-measure the catalogs whose stem uses the fprop tap view (splitk forward variant).
python tools/profile_catalog.py resnet50 184 224 --fused > gpurun_out/cat_r50f.log 2>&1
python tools/profile_catalog.py resnet50 184 224 --fused --split > gpurun_out/cat_r50fs.log 2>&1
python tools/profile_catalog.py mobilenet_v2 272 224 --fused > gpurun_out/cat_mb.log 2>&1
python tools/profile_catalog.py googlenet 320 224 --fused > gpurun_out/cat_gn.log 2>&1
mkdir -p gpurun_out/catalogs && cp profiles/catalog_*.json gpurun_out/catalogs/
tail -n 1 gpurun_out/cat_*.log
