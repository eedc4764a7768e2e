// Microbenchmark of tcgen05.mma issue rate on sm_100a (debug tool).
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/bin/mma_probe tools/mma_probe.cu && tools/bin/mma_probe
// One CTA per SM issues back-to-back kind::f16 (bf16) 128xNx16 MMAs into one
// TMEM accumulator (operand contents irrelevant) and reports clocks per MMA
// and the implied dense TFLOP/s, for A from shared memory (ss) and from TMEM (ts).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc(uint32_t addr) {  // K-major SWIZZLE_128B, SBO 1024
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) mma_rate(int iters, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  uint8_t* a = sm;             // 128 x 64 bf16 (16 KB)
  uint8_t* b = sm + 16384;     // N x 64 bf16
  const int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0) {
    const uint32_t d_tmem = tmem;            // accumulator: columns [0, N)
    const uint32_t a_tmem = tmem + 256;      // A operand in TMEM (ts form): 8 columns per k16
    const uint64_t ad = desc(smem_u32(a)), bd = desc(smem_u32(b));
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t acc = i > 0;
      if (TS) {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
                     "r"(a_tmem + (i & 3) * 8), "l"(bd + (uint64_t)((i & 3) * 2)), "r"(idesc), "r"(acc));
      } else {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
                     "l"(ad + (uint64_t)((i & 3) * 2)), "l"(bd + (uint64_t)((i & 3) * 2)), "r"(idesc), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                 : "memory");
    asm volatile("{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}" ::"r"(
        smem_u32(&bar)));
    t1 = clock64();
    cycles[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int N, bool TS>
void run(const char* name) {
  const int iters = 20000, grid = 148;
  long long* d;
  cudaMalloc(&d, grid * sizeof(long long));
  const int smem = 16384 + N * 128 + 1024;
  cudaFuncSetAttribute(mma_rate<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  mma_rate<N, TS><<<grid, 128, smem>>>(100, d);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  mma_rate<N, TS><<<grid, 128, smem>>>(iters, d);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < grid; ++i) avg += h[i];
  avg /= grid;
  const double flops = 2.0 * 128 * N * 16 * iters * grid;
  printf("%-10s N=%3d  %6.1f clk/MMA  %7.1f TFLOP/s (event %.3f ms) %s\n", name, N, avg / iters, flops / (ms * 1e-3) / 1e12,
         ms, cudaGetErrorString(err));
  cudaFree(d);
}

int main() {
  run<128, false>("ss");
  run<128, true>("ts");
  run<256, false>("ss");
  run<256, true>("ts");
  run<64, true>("ts");
  return 0;
}
