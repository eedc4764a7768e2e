// TMA delivery-rate probe on sm_100a (debug tool): how fast do the operand box shapes the
// bf16x3 GEMM uses arrive in shared memory, with nothing consuming them?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/bin/tma_bw_probe tools/tma_bw_probe.cu
//   tools/bin/tma_bw_probe
// One CTA per SM; one thread streams boxes into a ring of slots (mbarrier per slot,
// re-issued as soon as a slot's previous load has landed), walking an NHWC fp32 tensor
// [pixels][C] from a per-CTA start.  Reports chip-wide GB/s for L2-resident (32 MB) and
// HBM-sized (1 GB) tensors.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

struct Job {
  int mode;       // 0 tiled 2D {c, pixel}, 1 im2col (3x3 window offsets cycling)
  int bc, bp;     // box: channels x pixels
  int nbox;       // boxes per slot (channel offsets bc apart)
  int slots;
  int C, pixels;  // tensor
  int H, W;       // im2col image dims (pixels = N*H*W)
  int nq;         // issuing threads (lane 0 of warps 0..nq-1), each with its own ring of slots
  int lane_stride;  // > 0: the issuers are lanes 0, ls, 2*ls, ... of warp 0 instead
};

__global__ void __launch_bounds__(128, 1) probe(const __grid_constant__ CUtensorMap m, Job j, int iters,
                                                 unsigned long long* cycles) {
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char* base = smem + ((1024 - (smem_u32(smem) & 1023)) & 1023);
  const int slot_bytes = j.bc * j.bp * 4 * j.nbox * (j.mode == 2 ? 2 : 1);
  uint64_t* bars0 = reinterpret_cast<uint64_t*>(base + j.nq * j.slots * slot_bytes);
  if (threadIdx.x == 0) {
    for (int s = 0; s < j.nq * j.slots; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars0[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int q = j.lane_stride ? (threadIdx.x < 32 && threadIdx.x % j.lane_stride == 0 ? threadIdx.x / j.lane_stride : 99)
                              : threadIdx.x / 32;
  if ((!j.lane_stride && (threadIdx.x & 31) != 0) || q >= j.nq) return;
  uint64_t* bars = bars0 + q * j.slots;
  base += q * j.slots * slot_bytes;
  const long long t0 = clock64();
  const int per_cta = j.pixels / (gridDim.x * j.nq);
  const int cta = blockIdx.x * j.nq + q;
  int p0 = cta * per_cta;
  int cgrp = 0, tap = 0;
  for (int i = 0; i < iters; ++i) {
    const int s = i % j.slots;
    if (i >= j.slots) {
      const uint32_t ph = ((i / j.slots) - 1) & 1;
      asm volatile(
          "{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W;\n\t}" ::"r"(
              smem_u32(&bars[s])),
          "r"(ph));
    }
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bars[s])), "r"(slot_bytes));
    const uint32_t dst = smem_u32(base + s * slot_bytes);
    for (int b = 0; b < j.nbox; ++b) {
      const int c = (cgrp * j.nbox + b) * j.bc;
      if (j.mode == 2) {
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
            "%4}], [%5];" ::"r"(dst + b * j.bc * j.bp * 8),
            "l"(&m), "r"(0), "r"(p0), "r"(c / 32), "r"(smem_u32(&bars[s]))
            : "memory");
      } else if (j.mode == 0) {
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
            "[%4];" ::"r"(dst + b * j.bc * j.bp * 4),
            "l"(&m), "r"(c), "r"(p0), "r"(smem_u32(&bars[s]))
            : "memory");
      } else {
        const int w = p0 % j.W, t = p0 / j.W, h = t % j.H, n = t / j.H;
        const uint16_t ow = (uint16_t)(tap % 3), oh = (uint16_t)(tap / 3);
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
            "%5}], [%6], {%7, %8};" ::"r"(dst + b * j.bc * j.bp * 4),
            "l"(&m), "r"(c), "r"(w - 1), "r"(h - 1), "r"(n), "r"(smem_u32(&bars[s])), "h"(ow), "h"(oh)
            : "memory");
      }
    }
    // walk: channel groups, then (im2col) taps, then pixels
    if (++cgrp * j.nbox * j.bc >= j.C) {
      cgrp = 0;
      if (j.mode == 0 || ++tap == 9) {
        tap = 0;
        p0 += j.bp;
        if (p0 + j.bp > (cta + 1) * per_cta) p0 = cta * per_cta;
      }
    }
  }
  for (int s = 0; s < j.slots && s < iters; ++s) {
    const int last = iters - 1 - ((iters - 1 - s) % j.slots);
    const uint32_t ph = (last / j.slots) & 1;
    asm volatile(
        "{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W;\n\t}" ::"r"(
            smem_u32(&bars[s])),
        "r"(ph));
  }
  atomicMax(cycles, (unsigned long long)(clock64() - t0));
}

int main() {
  PFN_cuTensorMapEncodeTiled_v12000 enc_t = nullptr;
  PFN_cuTensorMapEncodeIm2col_v12000 enc_i = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc_t, cudaEnableDefault, &q);
  cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", (void**)&enc_i, cudaEnableDefault, &q);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* buf;
  const size_t big = 1ull << 30;
  cudaMalloc(&buf, big);
  cudaMemset(buf, 0, big);
  unsigned long long* cyc;
  cudaMalloc(&cyc, 8);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  struct Case {
    const char* name;
    int mode, bc, bp, nbox, slots, C;
    CUtensorMapSwizzle sw;
    int nq;
    int ls = 0;
  } cases[] = {
      {"tiled {32c,128p} 16K x4 q1", 0, 32, 128, 1, 4, 128, CU_TENSOR_MAP_SWIZZLE_128B, 1},
      {"tiled {32c,128p} 16K x4 q2 warps", 0, 32, 128, 1, 4, 128, CU_TENSOR_MAP_SWIZZLE_128B, 2},
      {"tiled {32c,128p} 16K x4 q2 lanes", 0, 32, 128, 1, 4, 128, CU_TENSOR_MAP_SWIZZLE_128B, 2, 16},
      {"tiled {32c,128p} 16K x3 q4 lanes", 0, 32, 128, 1, 3, 128, CU_TENSOR_MAP_SWIZZLE_128B, 4, 8},
      {"im2col {128c,32p} NONE 16K x4 q2 warps", 1, 128, 32, 1, 4, 128, CU_TENSOR_MAP_SWIZZLE_NONE, 2},
      {"im2col {128c,32p} NONE 16K x3 q4 warps", 1, 128, 32, 1, 3, 128, CU_TENSOR_MAP_SWIZZLE_NONE, 4},
      {"im2col {128c,32p} NONE 16K x3 q4 lanes", 1, 128, 32, 1, 3, 128, CU_TENSOR_MAP_SWIZZLE_NONE, 4, 8},
      {"tiled {128c,32p} NONE 16K x4 q2 warps", 0, 128, 32, 1, 4, 128, CU_TENSOR_MAP_SWIZZLE_NONE, 2},
      {"tiled {128c,32p} NONE 16K x3 q4 warps", 0, 128, 32, 1, 3, 128, CU_TENSOR_MAP_SWIZZLE_NONE, 4},
  };
  for (size_t bytes : {size_t(32) << 20}) {
    for (const Case& k : cases) {
      const int H = 56, W = 56;
      const int pixels = (int)(bytes / 4 / k.C) / (H * W) * (H * W);
      CUtensorMap m;
      CUresult r;
      if (k.mode == 2) {
        cuuint64_t dims[3] = {32, (cuuint64_t)pixels, (cuuint64_t)k.C / 32};
        cuuint64_t strides[2] = {(cuuint64_t)k.C * 4, 128};
        cuuint32_t box[3] = {32, (cuuint32_t)k.bp, 2}, es[3] = {1, 1, 1};
        r = enc_t(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  k.sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      } else if (k.mode == 0) {
        cuuint64_t dims[2] = {(cuuint64_t)k.C, (cuuint64_t)pixels};
        cuuint64_t strides[1] = {(cuuint64_t)k.C * 4};
        cuuint32_t box[2] = {(cuuint32_t)k.bc, (cuuint32_t)k.bp}, es[2] = {1, 1};
        r = enc_t(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  k.sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      } else {
        cuuint64_t dims[4] = {(cuuint64_t)k.C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)(pixels / (H * W))};
        cuuint64_t strides[3] = {(cuuint64_t)k.C * 4, (cuuint64_t)W * k.C * 4, (cuuint64_t)H * W * k.C * 4};
        int lo[2] = {-1, -1}, up[2] = {-1, -1};
        cuuint32_t es[4] = {1, 1, 1, 1};
        r = enc_i(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, buf, dims, strides, lo, up, k.bc, k.bp, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, k.sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      }
      if (r != CUDA_SUCCESS) {
        printf("%-46s encode failed (%d)\n", k.name, (int)r);
        continue;
      }
      Job j{k.mode, k.bc, k.bp, k.nbox, k.slots, k.C, pixels, H, W, k.nq, k.ls};
      const int slot_bytes = k.bc * k.bp * 4 * k.nbox * (k.mode == 2 ? 2 : 1);
      const int smem = k.nq * k.slots * slot_bytes + 1024 + 8 * k.nq * k.slots;
      const int iters = 4000;
      probe<<<sms, 128, smem>>>(m, j, 200, cyc);  // warm
      cudaMemset(cyc, 0, 8);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      probe<<<sms, 128, smem>>>(m, j, iters, cyc);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      cudaError_t e = cudaGetLastError();
      const double gbs = (double)sms * k.nq * iters * slot_bytes / (ms * 1e-3) / 1e9;
      printf("%-46s %5s  %7.1f GB/s  (%d B/slot, %d slots)%s\n", k.name, bytes > (64u << 20) ? "HBM" : "L2", gbs,
             slot_bytes, k.slots, e != cudaSuccess ? cudaGetErrorString(e) : "");
    }
  }
  return 0;
}
