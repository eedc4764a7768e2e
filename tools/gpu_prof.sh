# ncu --set full of one conv pass: LAYER PASS VARIANT TAG
mkdir -p gpurun_out
L=${1:-l2_3x3_128}; P=${2:-fwd}; V=${3:-implicit}; T=${4:-x}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_ -c 1 \
  -o gpurun_out/prof_${T} -f python tools/conv_bench.py --only $L --passes $P --variants $V --iters 1 > gpurun_out/prof_${T}.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/prof_${T}.log
