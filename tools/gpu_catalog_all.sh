# re-measure every frozen catalog on the device (ResNet-50 fused/plain, VGG-16, MobileNet-V2, GoogLeNet, UNet)
mkdir -p gpurun_out
set -x
timeout 900 python tools/profile_catalog.py --fused > gpurun_out/prof_r50f.log 2>&1
timeout 900 python tools/profile_catalog.py > gpurun_out/prof_r50.log 2>&1
timeout 900 python tools/profile_catalog.py vgg16 176 224 --fused > gpurun_out/prof_vgg.log 2>&1
timeout 900 python tools/profile_catalog.py mobilenet_v2 272 224 --fused > gpurun_out/prof_mbv2.log 2>&1
timeout 900 python tools/profile_catalog.py googlenet 320 224 --fused > gpurun_out/prof_gnet.log 2>&1
timeout 900 python tools/profile_catalog.py unet 11 416x608 --fused > gpurun_out/prof_unet.log 2>&1
cp profiles/catalog_*.json gpurun_out/
