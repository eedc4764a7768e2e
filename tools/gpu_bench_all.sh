# every config's bench lines: ResNet-50 (C2) 8/6/10, VGG-16 (C3) 10/9, MobileNet-V2 (C4) 10/8/6
mkdir -p gpurun_out
for b in 8 6 10; do
  timeout 600 python bench.py --steps 5 --warmup 3 --budget-gib $b $( [ $b != 8 ] && echo --no-cpu-baseline ) > gpurun_out/bench_${b}gib.json 2> gpurun_out/bench_${b}gib.err
  echo "resnet50 budget $b rc=$?"
done
bash tools/gpu_bench_vgg.sh
bash tools/gpu_bench_c4.sh
ARCH=googlenet B=320 bash tools/gpu_bench_c4.sh
ARCH=unet B=11 IMG=416x608 bash tools/gpu_bench_c4.sh
