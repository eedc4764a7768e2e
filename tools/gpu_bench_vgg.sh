# config C3: VGG-16 b176 224^2 at 10 and 9 GiB (exact-ILP schedules, measured catalog)
mkdir -p gpurun_out
for b in 10 9; do
  timeout 900 python bench.py --arch vgg16 --batch 176 --steps 3 --warmup 3 --budget-gib $b $( [ $b != 10 ] && echo --no-cpu-baseline ) > gpurun_out/bench_vgg16_${b}gib.json 2> gpurun_out/bench_vgg16_${b}gib.err
  echo "budget $b rc=$?"; tail -3 gpurun_out/bench_vgg16_${b}gib.err
done
