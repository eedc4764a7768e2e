# Round-2 bench lines for the other BASELINE configs (C3 VGG-16 / UNet, C4 MobileNet-V2 / GoogLeNet).
mkdir -p gpurun_out/bench_r2
run() { tag=$1; shift; timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/bench_r2/$tag.json 2> gpurun_out/bench_r2/$tag.err; echo "$tag rc=$?"; }
for b in 6.5 7 8 10; do run vgg16_fused_split_${b}gib --arch vgg16 --batch 176 --split --budget-gib $b; done
for b in 6 8 10; do run googlenet_${b}gib --arch googlenet --batch 320 --budget-gib $b; done
for b in 6 8 10; do run mobilenet_v2_${b}gib --arch mobilenet_v2 --batch 272 --budget-gib $b; done
for b in 6 8 10; do run unet_${b}gib --arch unet --batch 11 --image 416x608 --budget-gib $b; done
