// Standalone probe of TMA im2col / tiled tensor-map semantics on sm_100a (debug tool).
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tma_probe tools/tma_probe.cu && ./tma_probe
// Loads one im2col box of x[N][H][W][C] (values encode (n, h, w, c)) into shared
// memory and prints which source pixel each box row came from, for several
// corner / offset settings, so the coordinate order conventions can be pinned.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe_kernel(const __grid_constant__ CUtensorMap tmap, float* out, int c0, int w0, int h0, int n0,
                             int off_w, int off_h, int bytes) {
  __shared__ alignas(1024) float buf[32 * 64];
  __shared__ alignas(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(bytes));
    const uint16_t ow = (uint16_t)off_w, oh = (uint16_t)off_h;
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
        "%5}], [%6], {%7, %8};" ::"r"(smem_u32(buf)),
        "l"(&tmap), "r"(c0), "r"(w0), "r"(h0), "r"(n0), "r"(smem_u32(&bar)), "h"(ow), "h"(oh)
        : "memory");
    asm volatile(
        "{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}" ::"r"(
            smem_u32(&bar)));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < bytes / 4; i += blockDim.x) out[i] = buf[i];
}

int main(int argc, char** argv) {
  const int N = 2, H = 5, W = 7, C = argc > 1 ? atoi(argv[1]) : 32;
  const int CH = argc > 2 ? atoi(argv[2]) : C;
  std::vector<float> hx(N * H * W * C);
  for (int n = 0; n < N; ++n)
    for (int h = 0; h < H; ++h)
      for (int w = 0; w < W; ++w)
        for (int c = 0; c < C; ++c) hx[((n * H + h) * W + w) * C + c] = 1 + n * 1000 + h * 100 + w * 10 + c * 0.01f;
  float *dx, *dout;
  cudaMalloc(&dx, hx.size() * 4);
  cudaMalloc(&dout, 32 * 64 * 4);
  cudaMemcpy(dx, hx.data(), hx.size() * 4, cudaMemcpyHostToDevice);

  PFN_cuTensorMapEncodeIm2col_v12000 encode = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", (void**)&encode, cudaEnableDefault, &q);
  if (!encode) {
    printf("no entry point\n");
    return 1;
  }
  struct Case {
    int lo0, lo1, up0, up1, es1, es2, c0, w0, h0, n0, ow, oh;
    const char* what;
  };
  Case cases[] = {
      {-1, -1, -1, -1, 1, 1, 0, -1, -1, 0, 0, 0, "3x3 pad1 stride1, start (w-1,h-1), offs 0,0"},
      {-1, -1, -1, -1, 1, 1, 0, -1, -1, 0, 1, 0, "same, offs (1,0)"},
      {-1, -1, -1, -1, 1, 1, 0, -1, -1, 0, 0, 1, "same, offs (0,1)"},
      {-1, -1, -1, -1, 2, 2, 0, -1, -1, 0, 0, 0, "stride 2 (elementStrides w,h = 2)"},
      {-1, 0, -1, 0, 1, 1, 0, -1, 0, 0, 0, 0, "lower/upper {-1, 0}: W range 7 if index0 = W"},
      {-1, -1, -1, -1, 1, 1, 0, -1, -1, 0, 2, 2, "offs (2,2)"},
  };
  for (const Case& cs : cases) {
    cudaGetLastError();
    alignas(64) CUtensorMap tm;
    cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
    cuuint64_t strides[3] = {(cuuint64_t)C * 4, (cuuint64_t)W * C * 4, (cuuint64_t)H * W * C * 4};
    int lo[2] = {cs.lo0, cs.lo1}, up[2] = {cs.up0, cs.up1};
    cuuint32_t es[4] = {1, (cuuint32_t)cs.es1, (cuuint32_t)cs.es2, 1};
    CUresult r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, dx, dims, strides, lo, up, CH, 24, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("== %s  (encode rc=%d)\n", cs.what, (int)r);
    if (r != CUDA_SUCCESS) continue;
    cudaMemset(dout, 0xff, 32 * 64 * 4);
    probe_kernel<<<1, 128>>>(tm, dout, cs.c0, cs.w0, cs.h0, cs.n0, cs.ow, cs.oh, 24 * CH * 4);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("kernel error %s\n", cudaGetErrorString(e));
      continue;
    }
    std::vector<float> ho(24 * CH);
    cudaMemcpy(ho.data(), dout, ho.size() * 4, cudaMemcpyDeviceToHost);
    for (int p = 0; p < 24; p += 7) {
      float v = ho[p * CH];
      if (v == 0) {
        printf("  px%2d: zero\n", p);
      } else {
        int iv = (int)(v - 1 + 0.5f);
        printf("  px%2d: n%d h%d w%d  (c1 %.2f)\n", p, iv / 1000, (iv / 100) % 10, (iv / 10) % 10, ho[p * CH + 1]);
      }
    }
  }
  return 0;
}
