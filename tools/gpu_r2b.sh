# Round-2 state after re-planning with the round-2 catalogs: headline parity, bench lines, conv table, ncu.
mkdir -p gpurun_out
TAG=${TAG:-r2b}
timeout 900 python -m pytest tests/test_engine_c2_gpu.py tests/test_kernels_c2_gpu.py -q -rs > gpurun_out/c2tests_${TAG}.log 2>&1
echo "c2 tests rc=$?"
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
echo "bench rc=$?"
timeout 600 python bench.py --steps 10 --warmup 3 --split --no-cpu-baseline > gpurun_out/bench_split_${TAG}.json 2> gpurun_out/bench_split_${TAG}.err
echo "bench split rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_${TAG}.json 2> gpurun_out/bench_ref_${TAG}.err
echo "bench ref rc=$?"
timeout 600 python tools/conv_bench.py --resnet50 > gpurun_out/conv_table_${TAG}.txt 2>&1
echo "conv table rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
  --log-file gpurun_out/launches_${TAG}.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-graph --no-overhead-run > gpurun_out/ncu_bench_${TAG}.log 2>&1
echo "launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_ -c 1 \
  -o gpurun_out/gemm_fwd_${TAG} -f python tools/conv_bench.py --only l2_3x3_128 --passes fwd --variants splitk --iters 1 > gpurun_out/ncu_gemm_fwd_${TAG}.log 2>&1
echo "gemm fwd rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_ -c 1 \
  -o gpurun_out/gemm_wgrad_${TAG} -f python tools/conv_bench.py --only l1_3x3_64 --passes wgrad --variants splitk --iters 1 > gpurun_out/ncu_gemm_wgrad_${TAG}.log 2>&1
echo "gemm wgrad rc=$?"
for l in l2_3x3_128 l1_3x3_64; do for ps in fwd dgrad wgrad; do timeout 60 python tools/gemm_waits.py $l $ps; done; done > gpurun_out/waits_${TAG}.txt 2>&1
