# bench line at the three BASELINE budgets (6 / 8 / 10 GiB) + GPU tests
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for b in 8 6 10; do
  timeout 600 python bench.py --steps 5 --warmup 3 --budget-gib $b $( [ $b != 8 ] && echo --no-cpu-baseline ) > gpurun_out/bench_${b}gib.json 2> gpurun_out/bench_${b}gib.err
  echo "budget $b rc=$?"; tail -2 gpurun_out/bench_${b}gib.err
done
