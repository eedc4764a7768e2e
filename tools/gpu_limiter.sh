# GEMM limiter sweep (debug build): time each conv pass with pipeline stages skipped.
mkdir -p gpurun_out
TAG=${TAG:-r2c}
for m in 0 1 3 4 8 12 7 15; do
  MONET_DBG_MODE=$m timeout 120 python tools/gemm_limiter.py l2_3x3_128 fwd l2_3x3_128 dgrad l2_3x3_128 wgrad \
    l1_3x3_64 fwd l1_3x3_64 wgrad l3_1x1_1024_256 fwd l4_3x3_512 wgrad l1_1x1_64_256 fwd
done > gpurun_out/limiter_${TAG}.txt 2>&1
cat gpurun_out/limiter_${TAG}.txt
