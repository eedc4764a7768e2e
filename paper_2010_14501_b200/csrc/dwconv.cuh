// Depthwise convolution (groups = C, MobileNet-V2's 3x3 stride-1/2 layers) on
// NHWC fp32 tensors, weights stored [R][S][C] so that every access is a
// channel-quad float4.  R*S*C*N*P*Q MACs against one read of x and one write
// of y per pass: HBM-bound direct kernels (no tensor cores), the taps of a
// pixel reuse x through L1/L2.
//   fwd   y[n,p,q,c]  = sum_{r,s} x[n, p*sh-ph+r, q*sw-pw+s, c] * w[r,s,c]
//   dgrad dx[n,h,w,c] = sum_{r,s : (h+ph-r) % sh == 0, ...} dy[n,p,q,c] * w[r,s,c]
//   wgrad dw[r,s,c]   = sum_{n,p,q} dy[n,p,q,c] * x[n, p*sh-ph+r, q*sw-pw+s, c]
// wgrad reduces over N*P*Q rows in two fixed-order levels (per-block partials in
// the workspace, then a per-element sum over blocks): deterministic.
#pragma once
#include "gemm_tc.cuh"  // ConvGeom
#include "local_ops.cuh"

namespace monet {

constexpr int kDwMaxTaps = 9;  // 3x3 (every depthwise layer of MobileNet-V2)

MONET_DEV void fma4(float4& a, const float4& x, const float4& w) {
  a.x = fmaf(x.x, w.x, a.x);
  a.y = fmaf(x.y, w.y, a.y);
  a.z = fmaf(x.z, w.z, a.z);
  a.w = fmaf(x.w, w.w, a.w);
}

__global__ void dwconv_fwd_kernel(const float* __restrict__ x, const float* __restrict__ w, float* __restrict__ y,
                                  ConvGeom g) {
  const int c4n = g.C / 4;
  const long long total = (long long)g.N * g.P * g.Q * c4n;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int cq = (int)(i % c4n);
    long long t = i / c4n;
    const int q = (int)(t % g.Q);
    t /= g.Q;
    const int p = (int)(t % g.P);
    const int n = (int)(t / g.P);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int r = 0; r < g.R; ++r) {
      const int h = p * g.sh - g.ph + r;
      if ((unsigned)h >= (unsigned)g.H) continue;
      for (int s = 0; s < g.S; ++s) {
        const int ww = q * g.sw - g.pw + s;
        if ((unsigned)ww >= (unsigned)g.W) continue;
        const float4 xv = __ldg(reinterpret_cast<const float4*>(x + (((long long)n * g.H + h) * g.W + ww) * g.C) + cq);
        const float4 wv = __ldg(reinterpret_cast<const float4*>(w + (r * g.S + s) * g.C) + cq);
        fma4(acc, xv, wv);
      }
    }
    reinterpret_cast<float4*>(y)[i] = acc;
  }
}

__global__ void dwconv_dgrad_kernel(const float* __restrict__ dy, const float* __restrict__ w, float* dx, ConvGeom g,
                                    int accumulate) {
  const int c4n = g.C / 4;
  const long long total = (long long)g.N * g.H * g.W * c4n;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int cq = (int)(i % c4n);
    long long t = i / c4n;
    const int ww = (int)(t % g.W);
    t /= g.W;
    const int h = (int)(t % g.H);
    const int n = (int)(t / g.H);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int r = 0; r < g.R; ++r) {
      const int hp = h + g.ph - r;
      if (hp < 0 || hp % g.sh) continue;
      const int p = hp / g.sh;
      if (p >= g.P) continue;
      for (int s = 0; s < g.S; ++s) {
        const int wp = ww + g.pw - s;
        if (wp < 0 || wp % g.sw) continue;
        const int q = wp / g.sw;
        if (q >= g.Q) continue;
        const float4 gv = __ldg(reinterpret_cast<const float4*>(dy + (((long long)n * g.P + p) * g.Q + q) * g.C) + cq);
        const float4 wv = __ldg(reinterpret_cast<const float4*>(w + (r * g.S + s) * g.C) + cq);
        fma4(acc, gv, wv);
      }
    }
    float4* o = reinterpret_cast<float4*>(dx) + i;
    if (accumulate) {
      const float4 old = *o;
      acc.x += old.x;
      acc.y += old.y;
      acc.z += old.z;
      acc.w += old.w;
    }
    *o = acc;
  }
}

// Level 1: block b sums rows [b*rpb, (b+1)*rpb) of the N*P*Q output pixels.
// tpr threads cover the channel quads of a row (qpt quads each), rpi rows run
// in parallel; the rpi row-subgroups are combined in shared memory in a fixed
// order.  part[b][tap][c].
__global__ void dwconv_wgrad_partial_kernel(const float* __restrict__ x, const float* __restrict__ dy,
                                            float* __restrict__ part, ConvGeom g) {
  const int c4n = g.C / 4;
  const int tpr = c4n <= (int)blockDim.x ? c4n : (int)blockDim.x;
  const int qpt = (c4n + tpr - 1) / tpr;
  const int rpi = blockDim.x / tpr;
  const int t = threadIdx.x, rsub = t / tpr, qbase = t % tpr;
  const long long rows = (long long)g.N * g.P * g.Q;
  const long long rpb = (rows + gridDim.x - 1) / gridDim.x;
  const long long r0 = blockIdx.x * rpb, r1 = min(rows, r0 + rpb);
  const int taps = g.R * g.S;
  __shared__ float4 red[kEwThreads];
  for (int qi = 0; qi < qpt; ++qi) {
    const int cq = qbase + qi * tpr;
    float4 acc[kDwMaxTaps];
#pragma unroll
    for (int k = 0; k < kDwMaxTaps; ++k) acc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (rsub < rpi && cq < c4n) {
      for (long long row = r0 + rsub; row < r1; row += rpi) {
        const int q = (int)(row % g.Q);
        const long long tt = row / g.Q;
        const int p = (int)(tt % g.P);
        const int n = (int)(tt / g.P);
        const float4 gv = __ldg(reinterpret_cast<const float4*>(dy + row * g.C) + cq);
#pragma unroll
        for (int k = 0; k < kDwMaxTaps; ++k) {
          if (k < taps) {
            const int r = k / g.S, s = k - r * g.S;
            const int h = p * g.sh - g.ph + r, ww = q * g.sw - g.pw + s;
            if ((unsigned)h < (unsigned)g.H && (unsigned)ww < (unsigned)g.W) {
              const float4 xv =
                  __ldg(reinterpret_cast<const float4*>(x + (((long long)n * g.H + h) * g.W + ww) * g.C) + cq);
              fma4(acc[k], xv, gv);
            }
          }
        }
      }
    }
    for (int k = 0; k < taps; ++k) {
      red[t] = acc[k];
      __syncthreads();
      if (rsub == 0 && cq < c4n) {
        float4 s4 = red[qbase];
        for (int j = 1; j < rpi; ++j) {
          const float4 v = red[j * tpr + qbase];
          s4.x += v.x;
          s4.y += v.y;
          s4.z += v.z;
          s4.w += v.w;
        }
        reinterpret_cast<float4*>(part + ((long long)blockIdx.x * taps + k) * g.C)[cq] = s4;
      }
      __syncthreads();
    }
  }
}

// Level 2: dw[tap][c] = sum over blocks of part[b][tap][c] (fixed order, fp64)
__global__ void dwconv_wgrad_final_kernel(const float* __restrict__ part, int nblocks, int taps, int C, float* dw) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= taps * C) return;
  double s = 0.0;
  for (int b = 0; b < nblocks; ++b) s += part[(long long)b * taps * C + i];
  dw[i] = (float)s;
}

}  // namespace monet
