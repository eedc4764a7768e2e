# ncu evidence for the round: launch list of one bench step + full captures of the top kernels.
mkdir -p gpurun_out
TAG=${TAG:-r1}
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
timeout 600 ncu --set full --clock-control none -k regex:"bnrelu|relu_fwd|bn_reduce" -c 6 \
  -o gpurun_out/local_${TAG} -f python tools/local_bench.py > gpurun_out/ncu_local_${TAG}.log 2>&1
echo "local rc=$?"
for l in l2_3x3_128 l4_3x3_512; do for ps in fwd dgrad wgrad; do timeout 60 python tools/gemm_waits.py $l $ps; done; done > gpurun_out/waits_${TAG}.txt 2>&1
ls -la gpurun_out
