# Round-2 closing check after the depthwise grid reorder: full GPU suite, smoke(), MobileNet bench lines.
TAG=${TAG:-r2f2}; mkdir -p gpurun_out/bench_$TAG
timeout 1800 python -m pytest tests -m gpu -q -rs --timeout 900 > gpurun_out/gputests_${TAG}.log 2>&1
echo "gpu tests rc=$?"; tail -1 gpurun_out/gputests_${TAG}.log; grep -E "^(FAILED|ERROR)" gpurun_out/gputests_${TAG}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
python tools/dw_bench.py 2>&1 | tail -1
run() { tag=$1; shift; timeout 900 python bench.py --steps 10 --warmup 3 "$@" > gpurun_out/bench_$TAG/$tag.json 2> gpurun_out/bench_$TAG/$tag.err; echo "$tag rc=$?"; }
for b in 6 8 10; do run mobilenet_v2_${b}gib --arch mobilenet_v2 --batch 272 --budget-gib $b --no-cpu-baseline; done
