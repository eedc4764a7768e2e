# Stride-1 depthwise dgrad as a flipped forward, MobileNet re-planned:
# affected GPU tests, bench lines.
TAG=${TAG:-r2dw2}; mkdir -p gpurun_out/bench_$TAG
timeout 1500 python -m pytest tests/test_conv_stats_gpu.py tests/test_kernels_gpu.py tests/test_engine_gpu.py tests/test_engine_c2_gpu.py -m gpu -q -rs --timeout 900 > gpurun_out/gputests_${TAG}.log 2>&1
echo "gpu tests rc=$?"; tail -1 gpurun_out/gputests_${TAG}.log; grep -E "^(FAILED|ERROR)" gpurun_out/gputests_${TAG}.log
run() { tag=$1; shift; timeout 900 python bench.py --steps 10 --warmup 3 "$@" > gpurun_out/bench_$TAG/$tag.json 2> gpurun_out/bench_$TAG/$tag.err; echo "$tag rc=$?"; }
for b in 6 8 10; do run mobilenet_v2_${b}gib --arch mobilenet_v2 --batch 272 --budget-gib $b --no-cpu-baseline; done
run resnet50_8gib
run resnet50_6gib_split --budget-gib 6 --split --no-cpu-baseline
