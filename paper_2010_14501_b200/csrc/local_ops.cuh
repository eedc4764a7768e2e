// HBM-bound memory-efficient local operators on NHWC fp32 tensors
// (SURVEY.md §2.2 K4-K13): sign-bitmask ReLU, training BatchNorm with
// input- and output-activated backwards, residual add / gradient
// pass-through, maxpool with an 8-bit window index, global average pool,
// softmax cross-entropy, SGD with momentum.
//
// Mask layout (fixed once): bit b of uint32 word w <-> element
// 32*w + b of the tensor in its physical NHWC order; tail bits are zero.
#pragma once
#include "common.cuh"

namespace monet {

constexpr int kEwThreads = 256;

// ------------------------------------------------------------------ ReLU
// y = max(x, 0) (NaN -> 0, matching mask bit x > 0); optional packed mask.
// kSix (ReLU6 = hardtanh(0, 6), MobileNet-V2): y = min(max(x, 0), 6) and the
// mask bit is the gradient gate 0 < x < 6.
// Each thread handles 8 consecutive elements (two float4) -> one byte of mask;
// 4 consecutive lanes assemble one 32-bit word with shuffles.
template <bool kSix>
MONET_DEV bool relu_gate(float v) {
  return kSix ? (v > 0.f && v < 6.f) : v > 0.f;
}
template <bool kSix>
MONET_DEV float relu_val(float v) {
  return kSix ? (v > 0.f ? fminf(v, 6.f) : 0.f) : (v > 0.f ? v : 0.f);
}
template <bool kSix = false>
__global__ void relu_fwd_kernel(const float* __restrict__ x, float* y, uint32_t* __restrict__ mask,
                                long long n) {
  const long long n8 = (n + 7) / 8;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i - threadIdx.x % 32 < n8; i += stride) {
    // whole warp iterates together (mask assembly uses shuffles)
    const bool active = i < n8;
    uint32_t byte = 0;
    if (active) {
      const long long e0 = i * 8;
      if (e0 + 8 <= n) {
        float4 a = *reinterpret_cast<const float4*>(x + e0);
        float4 b = *reinterpret_cast<const float4*>(x + e0 + 4);
        byte = relu_gate<kSix>(a.x) | (relu_gate<kSix>(a.y) << 1) | (relu_gate<kSix>(a.z) << 2) |
               (relu_gate<kSix>(a.w) << 3) | (relu_gate<kSix>(b.x) << 4) | (relu_gate<kSix>(b.y) << 5) |
               (relu_gate<kSix>(b.z) << 6) | (relu_gate<kSix>(b.w) << 7);
        a.x = relu_val<kSix>(a.x);
        a.y = relu_val<kSix>(a.y);
        a.z = relu_val<kSix>(a.z);
        a.w = relu_val<kSix>(a.w);
        b.x = relu_val<kSix>(b.x);
        b.y = relu_val<kSix>(b.y);
        b.z = relu_val<kSix>(b.z);
        b.w = relu_val<kSix>(b.w);
        *reinterpret_cast<float4*>(y + e0) = a;
        *reinterpret_cast<float4*>(y + e0 + 4) = b;
      } else {
        for (long long e = e0; e < n; ++e) {
          float v = x[e];
          byte |= (uint32_t)relu_gate<kSix>(v) << (e - e0);
          y[e] = relu_val<kSix>(v);
        }
      }
    }
    if (mask != nullptr) {
      uint32_t word = byte << (8 * (threadIdx.x & 3));
      word |= __shfl_xor_sync(0xffffffffu, word, 1);
      word |= __shfl_xor_sync(0xffffffffu, word, 2);
      if (active && (threadIdx.x & 3) == 0) mask[i / 4] = word;
    }
  }
}

// dx (=|+=) dy * bit; bit from the packed mask.
__global__ void relu_bwd_mask_kernel(const uint32_t* __restrict__ mask, const float* __restrict__ dy, float* dx,
                                     long long n, int accumulate) {
  const long long n8 = (n + 7) / 8;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n8;
       i += (long long)gridDim.x * blockDim.x) {
    const uint32_t byte = (__ldg(mask + i / 4) >> (8 * (i & 3))) & 0xFFu;
    const long long e0 = i * 8;
    if (e0 + 8 <= n) {
      float4 a = *reinterpret_cast<const float4*>(dy + e0);
      float4 b = *reinterpret_cast<const float4*>(dy + e0 + 4);
      a.x = (byte & 1) ? a.x : 0.f;
      a.y = (byte & 2) ? a.y : 0.f;
      a.z = (byte & 4) ? a.z : 0.f;
      a.w = (byte & 8) ? a.w : 0.f;
      b.x = (byte & 16) ? b.x : 0.f;
      b.y = (byte & 32) ? b.y : 0.f;
      b.z = (byte & 64) ? b.z : 0.f;
      b.w = (byte & 128) ? b.w : 0.f;
      if (accumulate) {
        float4 c = *reinterpret_cast<const float4*>(dx + e0);
        float4 d = *reinterpret_cast<const float4*>(dx + e0 + 4);
        a.x += c.x; a.y += c.y; a.z += c.z; a.w += c.w;
        b.x += d.x; b.y += d.y; b.z += d.z; b.w += d.w;
      }
      *reinterpret_cast<float4*>(dx + e0) = a;
      *reinterpret_cast<float4*>(dx + e0 + 4) = b;
    } else {
      for (long long e = e0; e < n; ++e) {
        float v = ((byte >> (e - e0)) & 1) ? dy[e] : 0.f;
        dx[e] = accumulate ? dx[e] + v : v;
      }
    }
  }
}

// dx (=|+=) dy * [s > 0] where s is the ReLU input or output (same sign test);
// kSix: [0 < s < 6] (ReLU6 input or output: the same gate).
template <bool kSix = false>
__global__ void relu_bwd_sign_kernel(const float* __restrict__ s, const float* __restrict__ dy, float* dx,
                                     long long n, int accumulate) {
  const long long n4 = n / 4;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4;
       i += (long long)gridDim.x * blockDim.x) {
    float4 v = *reinterpret_cast<const float4*>(s + 4 * i);
    float4 g = *reinterpret_cast<const float4*>(dy + 4 * i);
    g.x = relu_gate<kSix>(v.x) ? g.x : 0.f;
    g.y = relu_gate<kSix>(v.y) ? g.y : 0.f;
    g.z = relu_gate<kSix>(v.z) ? g.z : 0.f;
    g.w = relu_gate<kSix>(v.w) ? g.w : 0.f;
    if (accumulate) {
      float4 c = *reinterpret_cast<const float4*>(dx + 4 * i);
      g.x += c.x; g.y += c.y; g.z += c.z; g.w += c.w;
    }
    *reinterpret_cast<float4*>(dx + 4 * i) = g;
  }
  if (blockIdx.x == 0 && threadIdx.x < (n & 3)) {
    long long e = n4 * 4 + threadIdx.x;
    float v = relu_gate<kSix>(s[e]) ? dy[e] : 0.f;
    dx[e] = accumulate ? dx[e] + v : v;
  }
}

// ------------------------------------------------------------------ elementwise
// y = a + b  (residual join)
__global__ void add_kernel(const float* __restrict__ a, const float* __restrict__ b, float* y, long long n) {
  const long long n4 = n / 4;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4;
       i += (long long)gridDim.x * blockDim.x) {
    float4 u = *reinterpret_cast<const float4*>(a + 4 * i);
    float4 v = *reinterpret_cast<const float4*>(b + 4 * i);
    *reinterpret_cast<float4*>(y + 4 * i) = make_float4(u.x + v.x, u.y + v.y, u.z + v.z, u.w + v.w);
  }
  if (blockIdx.x == 0 && threadIdx.x < (n & 3)) {
    long long e = n4 * 4 + threadIdx.x;
    y[e] = a[e] + b[e];
  }
}

// Fused residual join + ReLU: z = max(a + b, 0)
__global__ void addrelu_kernel(const float* __restrict__ a, const float* __restrict__ b, float* z, long long n) {
  const long long n4 = n / 4;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4;
       i += (long long)gridDim.x * blockDim.x) {
    const float4 u = *reinterpret_cast<const float4*>(a + 4 * i);
    const float4 v = *reinterpret_cast<const float4*>(b + 4 * i);
    *reinterpret_cast<float4*>(z + 4 * i) = make_float4(fmaxf(u.x + v.x, 0.f), fmaxf(u.y + v.y, 0.f),
                                                        fmaxf(u.z + v.z, 0.f), fmaxf(u.w + v.w, 0.f));
  }
  if (blockIdx.x == 0 && threadIdx.x < (n & 3)) {
    const long long e = n4 * 4 + threadIdx.x;
    z[e] = fmaxf(a[e] + b[e], 0.f);
  }
}

// Its backward: g = dz * [gate > 0] with the gate from the output z (s1 = z,
// s2 = nullptr) or recomputed from the inputs (s1 + s2 = a + b); both input
// gradients in one pass, each stored or accumulated.
__global__ void addrelu_bwd_kernel(const float* __restrict__ s1, const float* __restrict__ s2,
                                   const float* __restrict__ dz, float* da, int acc_a, float* db, int acc_b,
                                   long long n) {
  const long long n4 = n / 4;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4;
       i += (long long)gridDim.x * blockDim.x) {
    float4 t = *reinterpret_cast<const float4*>(s1 + 4 * i);
    if (s2) {
      const float4 u = *reinterpret_cast<const float4*>(s2 + 4 * i);
      t.x += u.x; t.y += u.y; t.z += u.z; t.w += u.w;
    }
    float4 g = *reinterpret_cast<const float4*>(dz + 4 * i);
    g.x = t.x > 0.f ? g.x : 0.f;
    g.y = t.y > 0.f ? g.y : 0.f;
    g.z = t.z > 0.f ? g.z : 0.f;
    g.w = t.w > 0.f ? g.w : 0.f;
    float4 oa = g, ob = g;
    if (acc_a) {
      const float4 c = *reinterpret_cast<const float4*>(da + 4 * i);
      oa.x += c.x; oa.y += c.y; oa.z += c.z; oa.w += c.w;
    }
    if (acc_b) {
      const float4 c = *reinterpret_cast<const float4*>(db + 4 * i);
      ob.x += c.x; ob.y += c.y; ob.z += c.z; ob.w += c.w;
    }
    *reinterpret_cast<float4*>(da + 4 * i) = oa;
    *reinterpret_cast<float4*>(db + 4 * i) = ob;
  }
  if (blockIdx.x == 0 && threadIdx.x < (n & 3)) {
    const long long e = n4 * 4 + threadIdx.x;
    const float t = s2 ? s1[e] + s2[e] : s1[e];
    const float g = t > 0.f ? dz[e] : 0.f;
    da[e] = acc_a ? da[e] + g : g;
    db[e] = acc_b ? db[e] + g : g;
  }
}

// dx (=|+=) scale * dy
__global__ void scale_acc_kernel(const float* __restrict__ dy, float* dx, long long n, float scale, int accumulate) {
  const long long n4 = n / 4;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4;
       i += (long long)gridDim.x * blockDim.x) {
    float4 g = *reinterpret_cast<const float4*>(dy + 4 * i);
    g.x *= scale; g.y *= scale; g.z *= scale; g.w *= scale;
    if (accumulate) {
      float4 c = *reinterpret_cast<const float4*>(dx + 4 * i);
      g.x += c.x; g.y += c.y; g.z += c.z; g.w += c.w;
    }
    *reinterpret_cast<float4*>(dx + 4 * i) = g;
  }
  if (blockIdx.x == 0 && threadIdx.x < (n & 3)) {
    long long e = n4 * 4 + threadIdx.x;
    float v = scale * dy[e];
    dx[e] = accumulate ? dx[e] + v : v;
  }
}

// ------------------------------------------------------------------ BatchNorm

// The BN affine map of one element, y = ((x - mean) * invstd) * gamma + beta, with its
// rounding pinned: subtract, multiply, then one fused multiply-add.  Every forward apply,
// replay and recomputed ReLU gate evaluates exactly this, so the gate a backward
// recomputes is the forward's sign bit for bit -- and the CPU oracle reproduces it
// (oracle/cpu_executor.py:_bn_pre).
MONET_DEV float bn_aff(float x, float m, float s, float g, float b) {
  return __fmaf_rn(__fmul_rn(__fsub_rn(x, m), s), g, b);
}
// Per-channel reduction over rows of an NHWC [rows, C] matrix.  Each block
// owns a contiguous range of rows; a thread owns channel quad q and rows
// r0 + rpi*j.  Partial sums go to ws[block][2][C] and are combined in fp64
// by bn_finalize (deterministic: fixed block count and order).
struct BnLayout {
  int tpr;  // threads per row (channel quads handled concurrently)
  int qpt;  // quads per thread
  int rpi;  // rows per iteration of a block
};

__host__ __device__ inline BnLayout bn_layout(int C) {
  BnLayout L;
  int cq = C / 4;
  L.tpr = cq <= kEwThreads ? cq : kEwThreads;
  L.qpt = (cq + L.tpr - 1) / L.tpr;
  L.rpi = kEwThreads / L.tpr;
  return L;
}

// mode 0: sum x, sum x^2           (forward statistics)
// mode 1: sum dy, sum dy*xhat      (backward, xhat = (x-mean)*invstd)
// mode 2: sum dy, sum dy*xhat      (backward, xhat = (y-beta)/gamma)
// mode 3: as mode 1 with dy = dz * [gamma*xhat + beta > 0]  (fused BN+ReLU
//         backward from x; p2 / p3 = gamma / beta)
// mode 4: as mode 3 with the ReLU6 gate [0 < gamma*xhat + beta < 6]  (fused BN+ReLU6)
// mode 5: as mode 1 with dy = dz * [z > 0], z = p4  (fused BN+add+ReLU, gate from its output)
// mode 6: as mode 1 with dy = dz * [gamma*xhat + beta + skip > 0], skip = p4 (gate from its inputs)
// mode 7: sum (x - x0), sum (x - x0)^2 with the pivot x0 = the channel's value in row 0: the
//         shifted statistics bn_finalize_fwd turns into mean and variance without the
//         E[x^2] - mean^2 cancellation when |mean| >> std
__global__ void bn_reduce_kernel(int mode, const float* __restrict__ x, const float* __restrict__ dy,
                                 const float* __restrict__ p0, const float* __restrict__ p1, long long rows, int C,
                                 float* __restrict__ ws, const float* __restrict__ p2 = nullptr,
                                 const float* __restrict__ p3 = nullptr, const float* __restrict__ p4 = nullptr) {
  const BnLayout L = bn_layout(C);
  const int t = threadIdx.x;
  const int rsub = t / L.tpr;
  const int qbase = t % L.tpr;
  const long long rows_per_block = (rows + gridDim.x - 1) / gridDim.x;
  const long long r_begin = blockIdx.x * rows_per_block;
  const long long r_end = min(rows, r_begin + rows_per_block);
  __shared__ float red[2][kEwThreads * 4];
  for (int qi = 0; qi < L.qpt; ++qi) {
    const int q = qbase + qi * L.tpr;
    float s1[4] = {0.f, 0.f, 0.f, 0.f}, s2[4] = {0.f, 0.f, 0.f, 0.f};
    if (rsub < L.rpi && q < C / 4) {
      float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a, ga = a, be = a;
      const bool sums = mode == 0 || mode == 7;  // one input tensor, plain (shifted) sums
      if (mode == 7) a = *reinterpret_cast<const float4*>(x + 4 * q);  // pivot: row 0
      if (!sums) {
        a = *reinterpret_cast<const float4*>(p0 + 4 * q);  // mean | beta
        b = *reinterpret_cast<const float4*>(p1 + 4 * q);  // invstd | 1/gamma
      }
      if (mode == 3 || mode == 4 || mode == 6) {
        ga = *reinterpret_cast<const float4*>(p2 + 4 * q);
        be = *reinterpret_cast<const float4*>(p3 + 4 * q);
      }
      auto acc = [&](const float4& v, float4 g, const float4& e) {
        if (mode == 5) {  // gate from the fused op's output z = e
          g.x = e.x > 0.f ? g.x : 0.f;
          g.y = e.y > 0.f ? g.y : 0.f;
          g.z = e.z > 0.f ? g.z : 0.f;
          g.w = e.w > 0.f ? g.w : 0.f;
        } else if (mode == 6) {  // gate recomputed from x and the skip input e (forward's formula)
          g.x = (__fadd_rn(bn_aff(v.x, a.x, b.x, ga.x, be.x), e.x) > 0.f) ? g.x : 0.f;
          g.y = (__fadd_rn(bn_aff(v.y, a.y, b.y, ga.y, be.y), e.y) > 0.f) ? g.y : 0.f;
          g.z = (__fadd_rn(bn_aff(v.z, a.z, b.z, ga.z, be.z), e.z) > 0.f) ? g.z : 0.f;
          g.w = (__fadd_rn(bn_aff(v.w, a.w, b.w, ga.w, be.w), e.w) > 0.f) ? g.w : 0.f;
        } else if (mode >= 3 && mode <= 4) {  // the ReLU's gradient gate, recomputed with the forward's formula
          const bool six = mode == 4;
          auto gate = [six](float u) { return six ? (u > 0.f && u < 6.f) : u > 0.f; };
          g.x = gate(bn_aff(v.x, a.x, b.x, ga.x, be.x)) ? g.x : 0.f;
          g.y = gate(bn_aff(v.y, a.y, b.y, ga.y, be.y)) ? g.y : 0.f;
          g.z = gate(bn_aff(v.z, a.z, b.z, ga.z, be.z)) ? g.z : 0.f;
          g.w = gate(bn_aff(v.w, a.w, b.w, ga.w, be.w)) ? g.w : 0.f;
        }
        if (sums) {
          const float d0 = v.x - a.x, d1 = v.y - a.y, d2 = v.z - a.z, d3 = v.w - a.w;
          s1[0] += d0; s1[1] += d1; s1[2] += d2; s1[3] += d3;
          s2[0] += d0 * d0; s2[1] += d1 * d1; s2[2] += d2 * d2; s2[3] += d3 * d3;
        } else {
          float h0 = (v.x - a.x) * b.x, h1 = (v.y - a.y) * b.y, h2 = (v.z - a.z) * b.z, h3 = (v.w - a.w) * b.w;
          s1[0] += g.x; s1[1] += g.y; s1[2] += g.z; s1[3] += g.w;
          s2[0] += g.x * h0; s2[1] += g.y * h1; s2[2] += g.z * h2; s2[3] += g.w * h3;
        }
      };
      const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
      long long r = r_begin + rsub;
      if (sums) {  // statistics read one tensor: eight rows in flight to cover the latency
        for (; r + 7 * L.rpi < r_end; r += 8 * L.rpi) {
          float4 v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) v[u] = *reinterpret_cast<const float4*>(x + (r + u * L.rpi) * C + 4 * q);
#pragma unroll
          for (int u = 0; u < 8; ++u) acc(v[u], z4, z4);
        }
      } else if (mode < 5) {  // two tensors (x, dy): eight rows in flight as well
        for (; r + 7 * L.rpi < r_end; r += 8 * L.rpi) {
          float4 v[8], g[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const long long off = (r + u * L.rpi) * C + 4 * q;
            v[u] = *reinterpret_cast<const float4*>(x + off);
            g[u] = *reinterpret_cast<const float4*>(dy + off);
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) acc(v[u], g[u], z4);
        }
      }
      // four rows in flight per thread (same accumulation order as one at a time)
      for (; r + 3 * L.rpi < r_end; r += 4 * L.rpi) {
        float4 v[4], g[4], e[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const long long off = (r + u * L.rpi) * C + 4 * q;
          v[u] = *reinterpret_cast<const float4*>(x + off);
          g[u] = sums ? z4 : *reinterpret_cast<const float4*>(dy + off);
          e[u] = (mode == 5 || mode == 6) ? *reinterpret_cast<const float4*>(p4 + off) : z4;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) acc(v[u], g[u], e[u]);
      }
      for (; r < r_end; r += L.rpi) {
        const long long off = r * C + 4 * q;
        acc(*reinterpret_cast<const float4*>(x + off), sums ? z4 : *reinterpret_cast<const float4*>(dy + off),
            (mode == 5 || mode == 6) ? *reinterpret_cast<const float4*>(p4 + off) : z4);
      }
    }
    // combine the rpi row-subgroups of each channel quad in shared memory
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      red[0][t * 4 + c] = s1[c];
      red[1][t * 4 + c] = s2[c];
    }
    __syncthreads();
    if (rsub == 0 && q < C / 4) {
      for (int c = 0; c < 4; ++c) {
        float a1 = 0.f, a2 = 0.f;
        for (int j = 0; j < L.rpi; ++j) {
          a1 += red[0][(j * L.tpr + qbase) * 4 + c];
          a2 += red[1][(j * L.tpr + qbase) * 4 + c];
        }
        ws[(long long)blockIdx.x * 2 * C + 4 * q + c] = a1;
        ws[(long long)blockIdx.x * 2 * C + C + 4 * q + c] = a2;
      }
    }
    __syncthreads();
  }
}

// Sum the per-block partials of channel c with one warp: lane l adds blocks
// l, l+32, ... in fp64, then a fixed xor tree combines the lanes -- the same
// order on every run (deterministic) and ~nblocks/32 loads per lane.
__device__ __forceinline__ void bn_warp_sum(const float* __restrict__ ws, int nblocks, int C, int c, double& s1,
                                            double& s2) {
  const int lane = threadIdx.x & 31;
  s1 = 0.0;
  s2 = 0.0;
  // eight blocks' loads in flight per lane before the (unchanged, in-order) fp64 adds: the
  // loop was a chain of dependent L2 round trips (~10 us per finalize launch)
  for (int b0 = lane; b0 < nblocks; b0 += 32 * 8) {
    float a1[8], a2[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int b = b0 + 32 * u;
      a1[u] = b < nblocks ? ws[(long long)b * 2 * C + c] : 0.f;
      a2[u] = b < nblocks ? ws[(long long)b * 2 * C + C + c] : 0.f;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (b0 + 32 * u < nblocks) {
        s1 += a1[u];
        s2 += a2[u];
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    s2 += __shfl_xor_sync(0xffffffffu, s2, o);
  }
}

// forward: mean/invstd from the shifted sums of bn_reduce mode 7 (pivot x0 = row 0 of x);
// running-stat update (momentum, unbiased var).  One warp per channel (launch C warps).
__global__ void bn_finalize_fwd_kernel(const float* __restrict__ ws, int nblocks, long long rows, int C, float eps,
                                       float momentum, int update_running, float* mean_out, float* invstd_out,
                                       float* running_mean, float* running_var, const float* __restrict__ x) {
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (c >= C) return;
  double s1, s2;
  bn_warp_sum(ws, nblocks, C, c, s1, s2);
  if ((threadIdx.x & 31) != 0) return;
  const double shift = s1 / (double)rows;  // mean - x0
  double mean = (double)x[c] + shift;
  double var = s2 / (double)rows - shift * shift;
  if (var < 0.0) var = 0.0;
  mean_out[c] = (float)mean;
  invstd_out[c] = (float)(1.0 / sqrt(var + (double)eps));
  if (update_running) {
    double unbiased = rows > 1 ? var * (double)rows / (double)(rows - 1) : var;
    running_mean[c] = (float)((1.0 - momentum) * running_mean[c] + momentum * mean);
    running_var[c] = (float)((1.0 - momentum) * running_var[c] + momentum * unbiased);
  }
}

// backward: dgamma = sum dy*xhat, dbeta = sum dy (parameter grads overwrite),
// and the per-channel affine form of the input gradient
//   dx = k*dy + cb*v + cc,  k = gamma*invstd,  xhat = (v - p0)*p1,
//   cb = -k*p1*S2/M,  cc = -k*S1/M + k*p1*p0*S2/M        (S1 = sum dy, S2 = sum dy*xhat)
// so the apply pass is two FMAs per element.  cb / cc overwrite coef_b / coef_c.
__global__ void bn_finalize_bwd_kernel(const float* __restrict__ ws, int nblocks, int C, long long rows,
                                       const float* __restrict__ p0, const float* __restrict__ p1,
                                       const float* __restrict__ gamma, const float* __restrict__ invstd,
                                       float* coef_b, float* coef_c, float* dgamma, float* dbeta) {
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (c >= C) return;
  double s1, s2;
  bn_warp_sum(ws, nblocks, C, c, s1, s2);
  if ((threadIdx.x & 31) != 0) return;
  if (dgamma) dgamma[c] = (float)s2;
  if (dbeta) dbeta[c] = (float)s1;
  const double k = (double)gamma[c] * (double)invstd[c];
  const double inv_m = 1.0 / (double)rows;
  const double a0 = p0[c], a1 = p1[c];
  coef_b[c] = (float)(-k * a1 * s2 * inv_m);
  coef_c[c] = (float)(-k * s1 * inv_m + k * a1 * a0 * s2 * inv_m);
}

// The apply passes below stream float4 groups of an NHWC [rows, C] tensor with a grid-stride
// loop that keeps kEwUnroll independent 16-B loads per input in flight per thread (issued
// before any of them is used): one load at a time leaves ~32 KB per SM in flight, below what
// HBM3e needs to reach its bandwidth (profiles/ncu_r2.md: bnrelu_apply 4.4 TB/s -> ...).
constexpr int kEwUnroll = 4;

#define MONET_EW_LOOP_BEGIN(n4)                                                             \
  const long long ew_stride_ = (long long)gridDim.x * blockDim.x;                            \
  for (long long ew_i0_ = blockIdx.x * (long long)blockDim.x + threadIdx.x; ew_i0_ < (n4); \
       ew_i0_ += kEwUnroll * ew_stride_) {
#define MONET_EW_IDX(u) (ew_i0_ + (long long)(u) * ew_stride_)
#define MONET_EW_LOOP_END }

MONET_DEV float4 ld4(const float* p, long long i) { return __ldcs(reinterpret_cast<const float4*>(p) + i); }
MONET_DEV float4 ldc4(const float* p, int q) { return __ldg(reinterpret_cast<const float4*>(p) + q); }
MONET_DEV void st4(float* p, long long i, float4 v) { reinterpret_cast<float4*>(p)[i] = v; }

// y = (x - mean) * invstd * gamma + beta   (train and replay share this kernel,
// so a recompute with saved statistics is bit-identical to the first forward)
__global__ void bn_apply_kernel(const float* __restrict__ x, float* y, const float* __restrict__ mean,
                                const float* __restrict__ invstd, const float* __restrict__ gamma,
                                const float* __restrict__ beta, long long rows, int C) {
  const int cq = C / 4;
  const long long n4 = rows * cq;
  MONET_EW_LOOP_BEGIN(n4)
  float4 v[kEwUnroll];
#pragma unroll
  for (int u = 0; u < kEwUnroll; ++u)
    if (MONET_EW_IDX(u) < n4) v[u] = ld4(x, MONET_EW_IDX(u));
#pragma unroll
  for (int u = 0; u < kEwUnroll; ++u) {
    const long long i = MONET_EW_IDX(u);
    if (i >= n4) break;
    const int q = (int)(i % cq);
    const float4 m = ldc4(mean, q), sd = ldc4(invstd, q), g = ldc4(gamma, q), b = ldc4(beta, q);
    float4 o;
    o.x = bn_aff(v[u].x, m.x, sd.x, g.x, b.x);
    o.y = bn_aff(v[u].y, m.y, sd.y, g.y, b.y);
    o.z = bn_aff(v[u].z, m.z, sd.z, g.z, b.z);
    o.w = bn_aff(v[u].w, m.w, sd.w, g.w, b.w);
    st4(y, i, o);
  }
  MONET_EW_LOOP_END
}

// dx (=|+=) gamma*invstd*(dy - sum_dy/M - xhat*sum_dyxhat/M) = k*dy + cb*v + cc
// (coefficients from bn_finalize_bwd; v = x or y, see there)
__global__ void bn_bwd_apply_kernel(const float* __restrict__ s, const float* __restrict__ dy, float* dx,
                                    const float* __restrict__ gamma, const float* __restrict__ invstd,
                                    const float* __restrict__ coef_b, const float* __restrict__ coef_c,
                                    long long rows, int C, int accumulate) {
  const int cq = C / 4;
  const long long n4 = rows * cq;
  MONET_EW_LOOP_BEGIN(n4)
  float4 v[kEwUnroll], g[kEwUnroll];
#pragma unroll
  for (int u = 0; u < kEwUnroll; ++u)
    if (MONET_EW_IDX(u) < n4) {
      v[u] = ld4(s, MONET_EW_IDX(u));
      g[u] = ld4(dy, MONET_EW_IDX(u));
    }
#pragma unroll
  for (int u = 0; u < kEwUnroll; ++u) {
    const long long i = MONET_EW_IDX(u);
    if (i >= n4) break;
    const int q = (int)(i % cq);
    const float4 ga = ldc4(gamma, q), is = ldc4(invstd, q), cb = ldc4(coef_b, q), cc = ldc4(coef_c, q);
    float4 o;
    o.x = fmaf(ga.x * is.x, g[u].x, fmaf(cb.x, v[u].x, cc.x));
    o.y = fmaf(ga.y * is.y, g[u].y, fmaf(cb.y, v[u].y, cc.y));
    o.z = fmaf(ga.z * is.z, g[u].z, fmaf(cb.z, v[u].z, cc.z));
    o.w = fmaf(ga.w * is.w, g[u].w, fmaf(cb.w, v[u].w, cc.w));
    if (accumulate) {
      const float4 d = reinterpret_cast<const float4*>(dx)[i];
      o.x += d.x; o.y += d.y; o.z += d.z; o.w += d.w;
    }
    st4(dx, i, o);
  }
  MONET_EW_LOOP_END
}

// Fused BN+ReLU forward apply: z = max((x - mean) * invstd * gamma + beta, 0)
// (same expression as bn_apply, so a recompute is bit-identical and the
// backward's recomputed gate matches the forward's sign exactly).
template <bool kSix = false>
__global__ void bnrelu_apply_kernel(const float* __restrict__ x, float* z, const float* __restrict__ mean,
                                    const float* __restrict__ invstd, const float* __restrict__ gamma,
                                    const float* __restrict__ beta, long long rows, int C) {
  const int cq = C / 4;
  const long long n4 = rows * cq;
  MONET_EW_LOOP_BEGIN(n4)
  float4 v[kEwUnroll];
#pragma unroll
  for (int u = 0; u < kEwUnroll; ++u)
    if (MONET_EW_IDX(u) < n4) v[u] = ld4(x, MONET_EW_IDX(u));
#pragma unroll
  for (int u = 0; u < kEwUnroll; ++u) {
    const long long i = MONET_EW_IDX(u);
    if (i >= n4) break;
    const int q = (int)(i % cq);
    const float4 m = ldc4(mean, q), sd = ldc4(invstd, q), g = ldc4(gamma, q), b = ldc4(beta, q);
    float4 o;
    o.x = relu_val<kSix>(bn_aff(v[u].x, m.x, sd.x, g.x, b.x));
    o.y = relu_val<kSix>(bn_aff(v[u].y, m.y, sd.y, g.y, b.y));
    o.z = relu_val<kSix>(bn_aff(v[u].z, m.z, sd.z, g.z, b.z));
    o.w = relu_val<kSix>(bn_aff(v[u].w, m.w, sd.w, g.w, b.w));
    st4(z, i, o);
  }
  MONET_EW_LOOP_END
}

// Fused BN + residual add + ReLU (the last BN of a bottleneck block feeding the join):
// z = max(BN(x) + skip, 0); the BN output never exists.
__global__ void bnaddrelu_apply_kernel(const float* __restrict__ x, const float* __restrict__ skip, float* z,
                                       const float* __restrict__ mean, const float* __restrict__ invstd,
                                       const float* __restrict__ gamma, const float* __restrict__ beta, long long rows,
                                       int C) {
  const int cq = C / 4;
  const long long n4 = rows * cq;
  MONET_EW_LOOP_BEGIN(n4)
  float4 v[kEwUnroll], k[kEwUnroll];
#pragma unroll
  for (int u = 0; u < kEwUnroll; ++u)
    if (MONET_EW_IDX(u) < n4) {
      v[u] = ld4(x, MONET_EW_IDX(u));
      k[u] = ld4(skip, MONET_EW_IDX(u));
    }
#pragma unroll
  for (int u = 0; u < kEwUnroll; ++u) {
    const long long i = MONET_EW_IDX(u);
    if (i >= n4) break;
    const int q = (int)(i % cq);
    const float4 m = ldc4(mean, q), sd = ldc4(invstd, q), g = ldc4(gamma, q), b = ldc4(beta, q);
    float4 o;
    o.x = fmaxf(__fadd_rn(bn_aff(v[u].x, m.x, sd.x, g.x, b.x), k[u].x), 0.f);
    o.y = fmaxf(__fadd_rn(bn_aff(v[u].y, m.y, sd.y, g.y, b.y), k[u].y), 0.f);
    o.z = fmaxf(__fadd_rn(bn_aff(v[u].z, m.z, sd.z, g.z, b.z), k[u].z), 0.f);
    o.w = fmaxf(__fadd_rn(bn_aff(v[u].w, m.w, sd.w, g.w, b.w), k[u].w), 0.f);
    st4(z, i, o);
  }
  MONET_EW_LOOP_END
}

// its backward apply: g = dz * gate (gate_from_out: [e > 0] with e = z; else [BN(x) + e > 0] with
// e = skip); dx = k*g + cb*x + cc and dskip = g, each written or accumulated
__global__ void bnaddrelu_bwd_apply_kernel(const float* __restrict__ x, const float* __restrict__ e,
                                           int gate_from_out, const float* __restrict__ dz, float* dx, int acc_x,
                                           float* dskip, int acc_skip, const float* __restrict__ mean,
                                           const float* __restrict__ beta, const float* __restrict__ gamma,
                                           const float* __restrict__ invstd, const float* __restrict__ coef_b,
                                           const float* __restrict__ coef_c, long long rows, int C) {
  const int cq = C / 4;
  const long long n4 = rows * cq;
  MONET_EW_LOOP_BEGIN(n4)
  float4 v[kEwUnroll], ev[kEwUnroll], gz[kEwUnroll];
#pragma unroll
  for (int u = 0; u < kEwUnroll; ++u)
    if (MONET_EW_IDX(u) < n4) {
      v[u] = ld4(x, MONET_EW_IDX(u));
      ev[u] = ld4(e, MONET_EW_IDX(u));
      gz[u] = ld4(dz, MONET_EW_IDX(u));
    }
#pragma unroll
  for (int u = 0; u < kEwUnroll; ++u) {
    const long long i = MONET_EW_IDX(u);
    if (i >= n4) break;
    const int q = (int)(i % cq);
    const float4 m = ldc4(mean, q), be = ldc4(beta, q), ga = ldc4(gamma, q), is = ldc4(invstd, q);
    const float4 cb = ldc4(coef_b, q), cc = ldc4(coef_c, q);
    float4 g = gz[u];
    if (gate_from_out) {
      g.x = ev[u].x > 0.f ? g.x : 0.f;
      g.y = ev[u].y > 0.f ? g.y : 0.f;
      g.z = ev[u].z > 0.f ? g.z : 0.f;
      g.w = ev[u].w > 0.f ? g.w : 0.f;
    } else {
      g.x = (__fadd_rn(bn_aff(v[u].x, m.x, is.x, ga.x, be.x), ev[u].x) > 0.f) ? g.x : 0.f;
      g.y = (__fadd_rn(bn_aff(v[u].y, m.y, is.y, ga.y, be.y), ev[u].y) > 0.f) ? g.y : 0.f;
      g.z = (__fadd_rn(bn_aff(v[u].z, m.z, is.z, ga.z, be.z), ev[u].z) > 0.f) ? g.z : 0.f;
      g.w = (__fadd_rn(bn_aff(v[u].w, m.w, is.w, ga.w, be.w), ev[u].w) > 0.f) ? g.w : 0.f;
    }
    float4 o;
    o.x = fmaf(ga.x * is.x, g.x, fmaf(cb.x, v[u].x, cc.x));
    o.y = fmaf(ga.y * is.y, g.y, fmaf(cb.y, v[u].y, cc.y));
    o.z = fmaf(ga.z * is.z, g.z, fmaf(cb.z, v[u].z, cc.z));
    o.w = fmaf(ga.w * is.w, g.w, fmaf(cb.w, v[u].w, cc.w));
    if (acc_x) {
      const float4 d = reinterpret_cast<const float4*>(dx)[i];
      o.x += d.x; o.y += d.y; o.z += d.z; o.w += d.w;
    }
    st4(dx, i, o);
    if (acc_skip) {
      const float4 d = reinterpret_cast<const float4*>(dskip)[i];
      g.x += d.x; g.y += d.y; g.z += d.z; g.w += d.w;
    }
    st4(dskip, i, g);
  }
  MONET_EW_LOOP_END
}

// Fused BN+ReLU backward apply from x: dy = dz * [bn(x) > 0]; dx = k*dy + cb*x + cc
template <bool kSix = false>
__global__ void bnrelu_bwd_apply_kernel(const float* __restrict__ x, const float* __restrict__ dz, float* dx,
                                        const float* __restrict__ mean, const float* __restrict__ beta,
                                        const float* __restrict__ gamma, const float* __restrict__ invstd,
                                        const float* __restrict__ coef_b, const float* __restrict__ coef_c,
                                        long long rows, int C, int accumulate) {
  const int cq = C / 4;
  const long long n4 = rows * cq;
  MONET_EW_LOOP_BEGIN(n4)
  float4 v[kEwUnroll], gz[kEwUnroll];
#pragma unroll
  for (int u = 0; u < kEwUnroll; ++u)
    if (MONET_EW_IDX(u) < n4) {
      v[u] = ld4(x, MONET_EW_IDX(u));
      gz[u] = ld4(dz, MONET_EW_IDX(u));
    }
#pragma unroll
  for (int u = 0; u < kEwUnroll; ++u) {
    const long long i = MONET_EW_IDX(u);
    if (i >= n4) break;
    const int q = (int)(i % cq);
    const float4 m = ldc4(mean, q), be = ldc4(beta, q), ga = ldc4(gamma, q), is = ldc4(invstd, q);
    const float4 cb = ldc4(coef_b, q), cc = ldc4(coef_c, q);
    float4 g = gz[u];
    g.x = relu_gate<kSix>(bn_aff(v[u].x, m.x, is.x, ga.x, be.x)) ? g.x : 0.f;
    g.y = relu_gate<kSix>(bn_aff(v[u].y, m.y, is.y, ga.y, be.y)) ? g.y : 0.f;
    g.z = relu_gate<kSix>(bn_aff(v[u].z, m.z, is.z, ga.z, be.z)) ? g.z : 0.f;
    g.w = relu_gate<kSix>(bn_aff(v[u].w, m.w, is.w, ga.w, be.w)) ? g.w : 0.f;
    float4 o;
    o.x = fmaf(ga.x * is.x, g.x, fmaf(cb.x, v[u].x, cc.x));
    o.y = fmaf(ga.y * is.y, g.y, fmaf(cb.y, v[u].y, cc.y));
    o.z = fmaf(ga.z * is.z, g.z, fmaf(cb.z, v[u].z, cc.z));
    o.w = fmaf(ga.w * is.w, g.w, fmaf(cb.w, v[u].w, cc.w));
    if (accumulate) {
      const float4 d = reinterpret_cast<const float4*>(dx)[i];
      o.x += d.x; o.y += d.y; o.z += d.z; o.w += d.w;
    }
    st4(dx, i, o);
  }
  MONET_EW_LOOP_END
}

// 1/gamma with |gamma| clamped away from 0 (output-activated BN needs gamma != 0)
__global__ void bn_inv_gamma_kernel(const float* __restrict__ gamma, float* inv, int C, float min_abs) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  float g = gamma[c];
  float a = fabsf(g) < min_abs ? copysignf(min_abs, g == 0.f ? 1.f : g) : g;
  inv[c] = 1.0f / a;
}

// ------------------------------------------------------------------ pooling
// max pool, NHWC, one thread per (n, p, q, channel quad); idx8 = window index
// r*S+s of the first maximum (NaN propagates like torch).
__global__ void maxpool_fwd_kernel(const float* __restrict__ x, float* __restrict__ y, uint8_t* __restrict__ idx,
                                   int N, int H, int W, int C, int P, int Q, int R, int S, int sh, int sw, int ph,
                                   int pw) {
  const int cq = C / 4;
  const long long total = (long long)N * P * Q * cq;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    int q4 = (int)(i % cq);
    long long pix = i / cq;
    int q = (int)(pix % Q);
    int p = (int)((pix / Q) % P);
    int n = (int)(pix / ((long long)P * Q));
    float best[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
    int arg[4] = {0, 0, 0, 0};
    for (int r = 0; r < R; ++r) {
      int h = p * sh - ph + r;
      if ((unsigned)h >= (unsigned)H) continue;
      for (int s = 0; s < S; ++s) {
        int w = q * sw - pw + s;
        if ((unsigned)w >= (unsigned)W) continue;
        float4 v = *reinterpret_cast<const float4*>(x + (((long long)n * H + h) * W + w) * C + 4 * q4);
        const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (vv[c] > best[c] || isnan(vv[c])) {  // torch: later NaNs win
            best[c] = vv[c];
            arg[c] = r * S + s;
          }
        }
      }
    }
    *reinterpret_cast<float4*>(y + pix * C + 4 * q4) = make_float4(best[0], best[1], best[2], best[3]);
    if (idx) {
      uint32_t packed = arg[0] | (arg[1] << 8) | (arg[2] << 16) | (arg[3] << 24);
      *reinterpret_cast<uint32_t*>(idx + pix * C + 4 * q4) = packed;
    }
  }
}

// gather-form backward (deterministic): dx[n,h,w,c] = sum over windows (p,q)
// covering (h,w) whose argmax is (h,w) of dy[n,p,q,c].  The argmax comes from
// the saved 8-bit index, or is recomputed from x (input-activated variant).
// One thread per (n, h, w, channel quad): 16B loads of x / dy, 4B of idx.
__global__ void maxpool_bwd_kernel(const uint8_t* __restrict__ idx, const float* __restrict__ x,
                                   const float* __restrict__ dy, float* dx, int N, int H, int W, int C, int P,
                                   int Q, int R, int S, int sh, int sw, int ph, int pw, int accumulate) {
  const int cq = C / 4;
  const long long total = (long long)N * H * W * cq;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int c4 = (int)(i % cq);
    const long long pix = i / cq;
    const int w = (int)(pix % W);
    const int h = (int)((pix / W) % H);
    const int n = (int)(pix / ((long long)H * W));
    float g[4] = {0.f, 0.f, 0.f, 0.f};
    // output rows p with p*sh - ph <= h <= p*sh - ph + R - 1
    const int p_lo = max(0, (h + ph - R + sh) / sh);
    const int p_hi = min(P - 1, (h + ph) / sh);
    const int q_lo = max(0, (w + pw - S + sw) / sw);
    const int q_hi = min(Q - 1, (w + pw) / sw);
    for (int p = p_lo; p <= p_hi; ++p) {
      const int r = h - (p * sh - ph);
      if (r < 0 || r >= R) continue;
      for (int q = q_lo; q <= q_hi; ++q) {
        const int s = w - (q * sw - pw);
        if (s < 0 || s >= S) continue;
        const long long o = (((long long)n * P + p) * Q + q) * C + 4 * c4;
        int a[4];
        if (idx) {
          const uint32_t packed = *reinterpret_cast<const uint32_t*>(idx + o);
#pragma unroll
          for (int c = 0; c < 4; ++c) a[c] = (packed >> (8 * c)) & 0xFF;
        } else {
          float best[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
          a[0] = a[1] = a[2] = a[3] = 0;
          for (int rr = 0; rr < R; ++rr) {
            const int hh = p * sh - ph + rr;
            if ((unsigned)hh >= (unsigned)H) continue;
            for (int ss = 0; ss < S; ++ss) {
              const int ww = q * sw - pw + ss;
              if ((unsigned)ww >= (unsigned)W) continue;
              const float4 v4 = *reinterpret_cast<const float4*>(x + (((long long)n * H + hh) * W + ww) * C + 4 * c4);
              const float v[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
              for (int c = 0; c < 4; ++c)
                if (v[c] > best[c] || isnan(v[c])) {
                  best[c] = v[c];
                  a[c] = rr * S + ss;
                }
            }
          }
        }
        const float4 d4 = *reinterpret_cast<const float4*>(dy + o);
        const float d[4] = {d4.x, d4.y, d4.z, d4.w};
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (a[c] == r * S + s) g[c] += d[c];
      }
    }
    float* out = dx + pix * C + 4 * c4;
    if (accumulate) {
      const float4 o4 = *reinterpret_cast<const float4*>(out);
      g[0] += o4.x;
      g[1] += o4.y;
      g[2] += o4.z;
      g[3] += o4.w;
    }
    *reinterpret_cast<float4*>(out) = make_float4(g[0], g[1], g[2], g[3]);
  }
}

// Index-path backward specialised for square K x K windows at stride ST (VGG's 2x2/2,
// ResNet's 3x3/2): at most ceil(K/ST)^2 candidate windows per input pixel, fully unrolled,
// 32-bit index math (total < 2^31 checked on the host).
template <int K, int ST>
__global__ void maxpool_bwd_idx_kernel(const uint8_t* __restrict__ idx, const float* __restrict__ dy, float* dx,
                                       int H, int W, int C, int P, int Q, int pad, unsigned total, int accumulate) {
  constexpr int kWin = (K + ST - 1) / ST;
  const unsigned cq = C / 4;
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const unsigned c4 = i % cq, pix = i / cq;
    const int w = (int)(pix % W);
    const unsigned t = pix / W;
    const int h = (int)(t % H), n = (int)(t / H);
    // windows p with p*ST - pad <= h <= p*ST - pad + K - 1
    const int hp = h + pad, wp = w + pad;
    const int p_hi = hp / ST, q_hi = wp / ST;
    float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int di = 0; di < kWin; ++di) {
      const int p = p_hi - di;
      const int r = hp - p * ST;
      if (p < 0 || p >= P || r >= K) continue;
#pragma unroll
      for (int dj = 0; dj < kWin; ++dj) {
        const int q = q_hi - dj;
        const int s = wp - q * ST;
        if (q < 0 || q >= Q || s >= K) continue;
        const size_t o = (((size_t)n * P + p) * Q + q) * C + 4 * c4;
        const uint32_t packed = __ldg(reinterpret_cast<const uint32_t*>(idx + o));
        const float4 d = __ldg(reinterpret_cast<const float4*>(dy + o));
        const uint32_t me = (uint32_t)(r * K + s);
        if ((packed & 0xFF) == me) g.x += d.x;
        if (((packed >> 8) & 0xFF) == me) g.y += d.y;
        if (((packed >> 16) & 0xFF) == me) g.z += d.z;
        if ((packed >> 24) == me) g.w += d.w;
      }
    }
    float4* out = reinterpret_cast<float4*>(dx + (size_t)pix * C + 4 * c4);
    if (accumulate) {
      const float4 o4 = *out;
      g.x += o4.x;
      g.y += o4.y;
      g.z += o4.z;
      g.w += o4.w;
    }
    *out = g;
  }
}

// global average pool: y[n, c] = mean_{hw} x[n, hw, c]
__global__ void avgpool_fwd_kernel(const float* __restrict__ x, float* __restrict__ y, int N, int HW, int C) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N * C) return;
  int n = i / C, c = i % C;
  const float* base = x + (long long)n * HW * C + c;
  float s = 0.f;
  for (int j = 0; j < HW; ++j) s += base[(long long)j * C];
  y[i] = s / (float)HW;
}

// ------------------------------------------------------------------ loss
// loss = mean_n [logsumexp(z_n) - z_n[label_n]]; one block per sample row.
__global__ void xent_fwd_kernel(const float* __restrict__ z, const int* __restrict__ labels, float* row_loss,
                                int N, int K) {
  int n = blockIdx.x;
  const float* row = z + (long long)n * K;
  __shared__ float sh[32];
  float m = -INFINITY;
  for (int k = threadIdx.x; k < K; k += blockDim.x) m = fmaxf(m, row[k]);
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < blockDim.x / 32 ? sh[threadIdx.x] : -INFINITY;
    for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (threadIdx.x == 0) sh[0] = v;
  }
  __syncthreads();
  m = sh[0];
  __syncthreads();
  float s = 0.f;
  for (int k = threadIdx.x; k < K; k += blockDim.x) s += expf(row[k] - m);
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    float tot = 0.f;
    for (int j = 0; j < blockDim.x / 32; ++j) tot += sh[j];
    row_loss[n] = logf(tot) + m - row[labels[n]];
  }
}

__global__ void mean_kernel(const float* __restrict__ v, int n, float* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += v[i];
    *out = (float)(s / n);
  }
}

// Small class counts (per-pixel segmentation losses, K <= 32): one thread per row.
__global__ void xent_small_fwd_kernel(const float* __restrict__ z, const int* __restrict__ labels, float* row_loss,
                                     long long N, int K) {
  for (long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x; n < N; n += (long long)gridDim.x * blockDim.x) {
    const float* row = z + n * K;
    float m = -INFINITY;
    for (int k = 0; k < K; ++k) m = fmaxf(m, row[k]);
    float s = 0.f;
    for (int k = 0; k < K; ++k) s += expf(row[k] - m);
    row_loss[n] = logf(s) + m - row[labels[n]];
  }
}
__global__ void xent_small_bwd_kernel(const float* __restrict__ z, const int* __restrict__ labels,
                                     const float* __restrict__ dloss, float* dz, long long N, int K, int accumulate) {
  const float g = *dloss / (float)N;
  for (long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x; n < N; n += (long long)gridDim.x * blockDim.x) {
    const float* row = z + n * K;
    float m = -INFINITY;
    for (int k = 0; k < K; ++k) m = fmaxf(m, row[k]);
    float s = 0.f;
    for (int k = 0; k < K; ++k) s += expf(row[k] - m);
    const float inv = 1.f / s;
    const int lab = labels[n];
    for (int k = 0; k < K; ++k) {
      const float v = (expf(row[k] - m) * inv - (k == lab ? 1.f : 0.f)) * g;
      dz[n * K + k] = accumulate ? dz[n * K + k] + v : v;
    }
  }
}
// mean of n row losses in two fixed-order levels: 256-wide block sums (fp64), then one thread
__global__ void block_sum_kernel(const float* __restrict__ v, long long n, double* partial) {
  __shared__ double sh[256];
  const long long per = (n + gridDim.x - 1) / gridDim.x;
  const long long a = blockIdx.x * per, b = min(n, a + per);
  double s = 0.0;
  for (long long i = a + threadIdx.x; i < b; i += blockDim.x) s += v[i];
  sh[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < (int)blockDim.x; ++k) t += sh[k];
    partial[blockIdx.x] = t;
  }
}
__global__ void mean_of_partials_kernel(const double* __restrict__ partial, int nb, long long n, float* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < nb; ++i) s += partial[i];
    *out = (float)(s / (double)n);
  }
}

// dz (=|+=) dloss * (softmax(z) - onehot) / N
__global__ void xent_bwd_kernel(const float* __restrict__ z, const int* __restrict__ labels,
                                const float* __restrict__ dloss, float* dz, int N, int K, int accumulate) {
  int n = blockIdx.x;
  const float* row = z + (long long)n * K;
  __shared__ float sh[32];
  float m = -INFINITY;
  for (int k = threadIdx.x; k < K; k += blockDim.x) m = fmaxf(m, row[k]);
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < blockDim.x / 32 ? sh[threadIdx.x] : -INFINITY;
    for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (threadIdx.x == 0) sh[0] = v;
  }
  __syncthreads();
  m = sh[0];
  __syncthreads();
  float s = 0.f;
  for (int k = threadIdx.x; k < K; k += blockDim.x) s += expf(row[k] - m);
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    float tot = 0.f;
    for (int j = 0; j < blockDim.x / 32; ++j) tot += sh[j];
    sh[0] = tot;
  }
  __syncthreads();
  const float inv = 1.0f / sh[0];
  const float scale = dloss[0] / (float)N;
  const int lab = labels[n];
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    float g = (expf(row[k] - m) * inv - (k == lab ? 1.f : 0.f)) * scale;
    float* o = dz + (long long)n * K + k;
    *o = accumulate ? *o + g : g;
  }
}

// ------------------------------------------------------------------ linear helpers
__global__ void bias_fill_kernel(float* y, const float* __restrict__ b, int N, int K) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < (long long)N * K) y[i] = b[i % K];
}

// per-channel sums of the block partials bn_reduce (mode 0) left in ws: the conv
// bias gradient db[c] = sum over rows of dy[., c] (fixed order, fp64 combine)
__global__ void chan_sum_finalize_kernel(const float* __restrict__ ws, int nblocks, int C, float* db, int accumulate) {
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (c >= C) return;
  double s1, s2;
  bn_warp_sum(ws, nblocks, C, c, s1, s2);
  if ((threadIdx.x & 31) == 0) db[c] = accumulate ? db[c] + (float)s1 : (float)s1;
}

// ---------------------------------------------------------------- dropout
// Keep-mask from a counter-based hash (splitmix64 finalizer) of (step seed,
// op salt, element index in the engine's NHWC order): nothing is stored, the
// backward and every recompute regenerate the same mask.  keep <=> the top 24
// bits of the hash >= thr, thr = floor(p * 2^24).  oracle/dropout.py restates it.
MONET_DEV bool dropout_keep(unsigned long long seed, unsigned long long salt, unsigned long long i, unsigned thr) {
  unsigned long long z = seed * 0x9E3779B97F4A7C15ull + salt * 0xD1B54A32D192ED03ull + i;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return (unsigned)(z >> 40) >= thr;
}

// y = keep ? x * scale : 0   (backward: same with dy -> dx, optional accumulate)
__global__ void dropout_kernel(const float* __restrict__ x, float* y, long long n, unsigned thr, float scale,
                               const unsigned long long* __restrict__ seed_ptr, unsigned long long salt,
                               int accumulate) {
  const unsigned long long seed = *seed_ptr;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const float v = dropout_keep(seed, salt, (unsigned long long)i, thr) ? x[i] * scale : 0.f;
    y[i] = accumulate ? y[i] + v : v;
  }
}

__global__ void seed_advance_kernel(unsigned long long* seed) { *seed += 1; }

// ---------------------------------------------------------------- concat
// Channel-slice copy between NHWC tensors (the concat of GoogLeNet's inception
// branches): dst[pix, dst_off + j] (+)= src[pix, src_off + j], j < count.
// Forward puts each input into its channel range; backward takes the slices out.
__global__ void channel_copy_kernel(const float* __restrict__ src, int src_c, int src_off, float* dst, int dst_c,
                                    int dst_off, int count, long long pixels, int accumulate) {
  const int q4 = count / 4;
  const long long total = pixels * q4;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long pix = i / q4;
    const int j = (int)(i - pix * q4) * 4;
    float4 v = *reinterpret_cast<const float4*>(src + pix * src_c + src_off + j);
    float4* o = reinterpret_cast<float4*>(dst + pix * dst_c + dst_off + j);
    if (accumulate) {
      const float4 a = *o;
      v.x += a.x;
      v.y += a.y;
      v.z += a.z;
      v.w += a.w;
    }
    *o = v;
  }
}

// db[k] = sum_n dy[n, k]  (fixed order)
__global__ void col_sum_kernel(const float* __restrict__ dy, float* db, int N, int K) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  float s = 0.f;
  for (int n = 0; n < N; ++n) s += dy[(long long)n * K + k];
  db[k] = s;
}

// ------------------------------------------------------------------ optimizer
// torch.optim.SGD semantics: g' = g*grad_scale + wd*w; buf = momentum*buf + g'
// (buf = g' on the first step); w -= lr*buf
__global__ void sgd_kernel(float* w, const float* __restrict__ g, float* buf, long long n, float lr, float momentum,
                           float wd, float grad_scale, int first) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    float d = g[i] * grad_scale + wd * w[i];
    float b = first ? d : momentum * buf[i] + d;
    buf[i] = b;
    w[i] -= lr * b;
  }
}

}  // namespace monet
