# Round-2 final evidence (BN statistics from the conv epilogue, re-planned schedules):
# GPU suite, ResNet-50 bench lines, ablation lines, other configs, reference arm, ncu.
mkdir -p gpurun_out/bench_r2f
TAG=${TAG:-r2f}
timeout 1800 python -m pytest tests -m gpu -q -rs --timeout 900 > gpurun_out/gputests_${TAG}.log 2>&1
echo "gpu tests rc=$?"; tail -2 gpurun_out/gputests_${TAG}.log; grep -E "^(FAILED|ERROR)" gpurun_out/gputests_${TAG}.log
run() { tag=$1; shift; timeout 900 python bench.py --steps 10 --warmup 3 "$@" > gpurun_out/bench_r2f/$tag.json 2> gpurun_out/bench_r2f/$tag.err; echo "$tag rc=$?"; }
run resnet50_8gib
run resnet50_6gib --budget-gib 6 --no-cpu-baseline
run resnet50_10gib --budget-gib 10 --no-cpu-baseline
run resnet50_split_6gib --budget-gib 6 --split --no-cpu-baseline
for m in none conv out int; do run resnet50_8gib_abl-$m --ablation $m --no-cpu-baseline; done
for b in 6.5 7 8 10; do run vgg16_fused_split_${b}gib --arch vgg16 --batch 176 --split --budget-gib $b --no-cpu-baseline; done
for b in 6 8 10; do run googlenet_${b}gib --arch googlenet --batch 320 --budget-gib $b --no-cpu-baseline; done
for b in 6 8 10; do run mobilenet_v2_${b}gib --arch mobilenet_v2 --batch 272 --budget-gib $b --no-cpu-baseline; done
for b in 6 8 10; do run unet_${b}gib --arch unet --batch 11 --image 416x608 --budget-gib $b --no-cpu-baseline; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_r2f/reference.json 2> gpurun_out/bench_r2f/reference.err
echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/launches_${TAG}.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-graph --no-overhead-run > gpurun_out/ncu_bench_${TAG}.log 2>&1
echo "launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_ -c 1 \
  -o gpurun_out/gemm_fwd_${TAG} -f python tools/conv_bench.py --only l2_3x3_128 --passes fwd --variants splitk --iters 1 > /dev/null 2>&1
echo "gemm fwd rc=$?"
