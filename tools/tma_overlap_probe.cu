// Probe: does a TMA tiled tensor map accept OVERLAPPING strides, and does it load
// the strided-conv wgrad "tap view" correctly?  (debug tool)
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/bin/tma_overlap_probe tools/tma_overlap_probe.cu
// View over a zero-padded NHWC input xp[N][Hp][Wp][C] for a conv with S x R taps
// and stride 2: element (sc, q, r, p, n) = xp[n][2p + r][2q + s][c] with sc = s*C + c,
// i.e. dims {S*C, Q, R, P, N} and byte strides {2*C*4, Wp*C*4, 2*Wp*C*4, Hp*Wp*C*4}
// (q's stride is smaller than the sc extent: the rows of the box overlap in memory).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe_kernel(const __grid_constant__ CUtensorMap tmap, float* out, int q0, int r0, int p0, int n0,
                             int bytes) {
  __shared__ alignas(1024) float buf[8192];
  __shared__ alignas(8) uint64_t bar;
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) buf[i] = -7.f;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(bytes));
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, "
        "%6}], [%7];" ::"r"(smem_u32(buf)),
        "l"(&tmap), "r"(0), "r"(q0), "r"(r0), "r"(p0), "r"(n0), "r"(smem_u32(&bar))
        : "memory");
    asm volatile(
        "{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}" ::"r"(
            smem_u32(&bar)));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < bytes / 4; i += blockDim.x) out[i] = buf[i];
}

int main() {
  const int N = 2, C = 4, R = 7, S = 7, P = 3, Q = 4, Hp = 2 * P + R - 1, Wp = 2 * Q + S - 1;
  const int BQ = 8, BR = 4;  // box: {S*C, BQ, BR, 1, 1}; q >= Q and r >= R fall out of bounds
  std::vector<float> hx((size_t)N * Hp * Wp * C);
  for (int n = 0; n < N; ++n)
    for (int h = 0; h < Hp; ++h)
      for (int w = 0; w < Wp; ++w)
        for (int c = 0; c < C; ++c) hx[((n * Hp + h) * Wp + w) * C + c] = 1 + n * 10000 + h * 100 + w + c * 0.1f;
  float *dx, *dout;
  cudaMalloc(&dx, hx.size() * 4);
  cudaMalloc(&dout, 8192 * 4);
  cudaMemcpy(dx, hx.data(), hx.size() * 4, cudaMemcpyHostToDevice);
  PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &qr);
  if (!encode) {
    printf("no entry point\n");
    return 1;
  }
  alignas(64) CUtensorMap tm;
  cuuint64_t dims[5] = {(cuuint64_t)S * C, (cuuint64_t)Q, (cuuint64_t)R, (cuuint64_t)P, (cuuint64_t)N};
  cuuint64_t strides[4] = {(cuuint64_t)2 * C * 4, (cuuint64_t)Wp * C * 4, (cuuint64_t)2 * Wp * C * 4,
                           (cuuint64_t)Hp * Wp * C * 4};
  cuuint32_t box[5] = {(cuuint32_t)S * C, BQ, BR, 1, 1};
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult res = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, dx, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode(overlapping strides) -> %d\n", (int)res);
  if (res != CUDA_SUCCESS) return 2;
  const int bytes = S * C * BQ * BR * 4;
  int bad = 0, total = 0;
  const int cases[][4] = {{0, 0, 0, 0}, {0, 4, 1, 1}, {0, 0, 2, 1}, {0, 4, 2, 0}};
  for (auto& cs : cases) {
    const int q0 = cs[0], r0 = cs[1], p0 = cs[2], n0 = cs[3];
    probe_kernel<<<1, 256>>>(tm, dout, q0, r0, p0, n0, bytes);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> ho(bytes / 4);
    cudaMemcpy(ho.data(), dout, bytes, cudaMemcpyDeviceToHost);
    for (int rb = 0; rb < BR; ++rb)
      for (int qb = 0; qb < BQ; ++qb)
        for (int sc = 0; sc < S * C; ++sc) {
          const int r = r0 + rb, q = q0 + qb, s = sc / C, c = sc % C;
          float want = 0.f;
          if (r < R && q < Q) want = hx[((n0 * Hp + 2 * p0 + r) * Wp + 2 * q + s) * C + c];
          const float got = ho[(rb * BQ + qb) * S * C + sc];
          ++total;
          if (got != want) {
            if (bad < 8) printf("  mismatch r%d q%d s%d c%d: got %.1f want %.1f\n", r, q, s, c, got, want);
            ++bad;
          }
        }
    printf("case q0=%d r0=%d p0=%d n0=%d: %s, %d/%d mismatches\n", q0, r0, p0, n0, cudaGetErrorString(e), bad, total);
  }
  printf(bad ? "FAIL\n" : "PASS\n");
  return bad ? 1 : 0;
}
