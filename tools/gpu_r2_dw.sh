# Round-2 depthwise-conv rework and re-planned UNet / MobileNet schedules: GPU suite, bench lines,
# one MobileNet launch list.
mkdir -p gpurun_out/bench_r2dw
TAG=${TAG:-r2dw}
timeout 1800 python -m pytest tests -m gpu -q -rs --timeout 900 > gpurun_out/gputests_${TAG}.log 2>&1
echo "gpu tests rc=$?"; tail -2 gpurun_out/gputests_${TAG}.log; grep -E "^(FAILED|ERROR)" gpurun_out/gputests_${TAG}.log
run() { tag=$1; shift; timeout 900 python bench.py --steps 10 --warmup 3 "$@" > gpurun_out/bench_r2dw/$tag.json 2> gpurun_out/bench_r2dw/$tag.err; echo "$tag rc=$?"; }
for b in 6 8 10; do run mobilenet_v2_${b}gib --arch mobilenet_v2 --batch 272 --budget-gib $b --no-cpu-baseline; done
run unet_6gib --arch unet --batch 11 --image 416x608 --budget-gib 6 --no-cpu-baseline
run resnet50_8gib
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/launches_mb_${TAG}.csv \
  python bench.py --arch mobilenet_v2 --batch 272 --budget-gib 8 --steps 1 --warmup 3 --no-cpu-baseline --no-graph --no-overhead-run > gpurun_out/ncu_mb_${TAG}.log 2>&1
echo "launches rc=$?"
