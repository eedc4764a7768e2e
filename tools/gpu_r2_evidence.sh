# Round-2 evidence: GPU suite, ResNet-50 bench lines (8 / 6 / 10 GiB, split graph at 6 GiB),
# reference arm, --no-graph dispatch cost, launch list and full ncu captures of the top kernels.
mkdir -p gpurun_out
TAG=${TAG:-r2j}
timeout 1500 python -m pytest tests -m gpu -q -rs --timeout 900 > gpurun_out/gputests_${TAG}.log 2>&1
echo "gpu tests rc=$?"; tail -2 gpurun_out/gputests_${TAG}.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
echo "bench rc=$?"
for b in 6 10; do
  timeout 600 python bench.py --steps 10 --warmup 3 --budget-gib $b --no-cpu-baseline > gpurun_out/bench_${TAG}_${b}gib.json 2> gpurun_out/bench_${TAG}_${b}gib.err
  echo "bench ${b} rc=$?"
done
timeout 600 python bench.py --steps 10 --warmup 3 --budget-gib 6 --split --no-cpu-baseline > gpurun_out/bench_${TAG}_split_6gib.json 2> gpurun_out/bench_${TAG}_split_6gib.err
echo "bench split 6 rc=$?"
timeout 600 python bench.py --steps 5 --warmup 3 --no-graph --no-cpu-baseline --no-overhead-run > gpurun_out/bench_${TAG}_nograph.json 2> gpurun_out/bench_${TAG}_nograph.err
echo "bench nograph rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_${TAG}.json 2> gpurun_out/bench_ref_${TAG}.err
echo "bench ref rc=$?"
timeout 600 python tools/conv_bench.py --resnet50 > gpurun_out/conv_table_${TAG}.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/launches_${TAG}.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-graph --no-overhead-run > gpurun_out/ncu_bench_${TAG}.log 2>&1
echo "launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_ -c 1 \
  -o gpurun_out/gemm_fwd_${TAG} -f python tools/conv_bench.py --only l2_3x3_128 --passes fwd --variants splitk --iters 1 > gpurun_out/ncu_gemm_fwd_${TAG}.log 2>&1
echo "gemm fwd rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_ -c 1 \
  -o gpurun_out/gemm_wgrad_${TAG} -f python tools/conv_bench.py --only l2_3x3_128 --passes wgrad --variants splitk --iters 1 > gpurun_out/ncu_gemm_wgrad_${TAG}.log 2>&1
echo "gemm wgrad rc=$?"
timeout 600 ncu --set full --clock-control none -k regex:"bnrelu|relu_fwd|bn_reduce|bnaddrelu" -c 8 \
  -o gpurun_out/local_${TAG} -f python tools/local_bench.py > gpurun_out/ncu_local_${TAG}.log 2>&1
echo "local rc=$?"
