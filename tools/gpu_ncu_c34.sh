# ncu evidence for the C3/C4 kernels (dwconv, fused BN+ReLU6, dropout, concat)
mkdir -p gpurun_out
TAG=${TAG:-r1j}
timeout 300 python tools/local_bench2.py > gpurun_out/local2_${TAG}.txt 2>&1; cat gpurun_out/local2_${TAG}.txt
timeout 900 ncu --set full --clock-control none \
  -k regex:"dwconv|bnrelu_apply|bnrelu_bwd_apply|bn_reduce|dropout|channel_copy" -c 16 \
  -o gpurun_out/local2_${TAG} -f python tools/local_bench2.py > gpurun_out/ncu_local2_${TAG}.log 2>&1
echo "ncu rc=$?"
