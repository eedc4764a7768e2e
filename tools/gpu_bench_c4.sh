# config C4: MobileNet-V2 b272 224^2 at 10/8/6 GiB (measured catalog, frozen schedules)
mkdir -p gpurun_out
ARCH=${ARCH:-mobilenet_v2}; B=${B:-272}; IMG=${IMG:-224}
for b in ${BUDGETS:-10 8 6}; do
  timeout 900 python bench.py --arch $ARCH --batch $B --image $IMG --steps 5 --warmup 3 --budget-gib $b --no-cpu-baseline > gpurun_out/bench_${ARCH}_${b}gib.json 2> gpurun_out/bench_${ARCH}_${b}gib.err
  echo "$ARCH budget $b rc=$?"; tail -3 gpurun_out/bench_${ARCH}_${b}gib.err
done
