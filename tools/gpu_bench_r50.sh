mkdir -p gpurun_out
for b in 8 6 10; do
  timeout 600 python bench.py --steps 5 --warmup 3 --budget-gib $b $( [ $b != 8 ] && echo --no-cpu-baseline ) > gpurun_out/bench_${b}gib.json 2> gpurun_out/bench_${b}gib.err
  echo "resnet50 budget $b rc=$?"; tail -2 gpurun_out/bench_${b}gib.err
done
