# Round-2 evidence: bench line, launch list with per-launch DRAM bytes, skipped-test listing.
mkdir -p gpurun_out
TAG=${TAG:-r2a}
python -m pytest tests -m gpu -q -rs -k "dp_engine or profiler" 2>&1 | grep -E "SKIP|passed|failed" > gpurun_out/skips_${TAG}.log
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/launches_${TAG}.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-graph --no-overhead-run > gpurun_out/ncu_bench_${TAG}.log 2>&1
echo "launches rc=$?"
