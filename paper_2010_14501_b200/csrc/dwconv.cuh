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
  const long long stride = (long long)taps * C;
  double s = 0.0;
  for (int b0 = 0; b0 < nblocks; b0 += 8) {  // 8 loads in flight, added in the same order
    float v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = b0 + u < nblocks ? part[(b0 + u) * stride + i] : 0.f;
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (b0 + u < nblocks) s += v[u];
  }
  dw[i] = (float)s;
}

}  // namespace monet

namespace monet {

// ---------------------------------------------------------------------------
// Shared-memory tiled depthwise kernels.  A CTA owns `rows` output rows of one
// image and one kDwSlab-channel slab; the source rows it needs (input rows for
// fwd / wgrad, dy rows for dgrad) are staged once into shared memory with zero
// padding, so each source pixel crosses L2 -> SM about once instead of once per
// tap.  Channel slab = 16 floats (4 quads): 64 B per pixel, two full sectors.
constexpr int kDwSlab = 16, kDwRows = 4;

// dst[i] = load(i) for i < count, blockDim-strided, 8 loads in flight per thread
template <class F>
MONET_DEV void dw_stage(float4* dst, int count, F load) {
  constexpr int kU = 8;
  for (int base = threadIdx.x; base < count; base += blockDim.x * kU) {
    float4 v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int i = base + u * (int)blockDim.x;
      v[u] = i < count ? load(i) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int i = base + u * (int)blockDim.x;
      if (i < count) dst[i] = v[u];
    }
  }
}

// fwd: out = y (P x Q), src = x (H x W); dgrad (kTrans): out = dx (H x W), src = dy (P x Q)
// flip: taps read in reverse (a stride-1 dgrad run as the forward of dy with the rotated filter)
// kStride > 0: 3x3 taps and that stride at compile time (MobileNet-V2's layers); 0: runtime geometry
template <bool kTrans, int kStride = 0>
__global__ void __launch_bounds__(256) dwconv_tile_kernel(const float* __restrict__ src, const float* __restrict__ w,
                                                          float* out, ConvGeom g, int accumulate, int rows,
                                                          int flip) {
  extern __shared__ float4 dw_smem[];
  if (kStride > 0) {
    g.sh = g.sw = kStride;
    g.R = g.S = 3;
  }
  const int OH = kTrans ? g.H : g.P, OW = kTrans ? g.W : g.Q;  // output extent
  const int SH = kTrans ? g.P : g.H, SW = kTrans ? g.Q : g.W;  // source extent
  const int c0 = blockIdx.x * kDwSlab;  // slabs fastest: a pixel's slabs share its DRAM lines in L2
  const int o0 = blockIdx.y * rows;
  const int n = blockIdx.z;
  const int orows = min(rows, OH - o0);
  // staged source window
  int s_r0, s_nr, s_c0, s_nc;
  if (!kTrans) {  // output row o reads input rows o*sh - ph + r
    s_r0 = o0 * g.sh - g.ph;
    s_nr = (orows - 1) * g.sh + g.R;
    s_c0 = -g.pw;
    s_nc = (OW - 1) * g.sw + g.S;
  } else {  // dx row h reads dy rows (h + ph - r) / sh for r with matching parity
    const int lo = o0 + g.ph - (g.R - 1), hi = o0 + orows - 1 + g.ph;
    s_r0 = lo >= 0 ? lo / g.sh : -((-lo + g.sh - 1) / g.sh);
    s_nr = hi / g.sh - s_r0 + 1;
    const int wl = g.pw - (g.S - 1), wh = OW - 1 + g.pw;
    s_c0 = wl >= 0 ? wl / g.sw : -((-wl + g.sw - 1) / g.sw);
    s_nc = wh / g.sw - s_c0 + 1;
  }
  // stage: s_nr x s_nc pixels x 4 quads of this slab (zero outside the source); 8 independent
  // loads in flight per thread before the shared-memory stores
  const int tot = s_nr * s_nc * 4;
  dw_stage(dw_smem, tot, [&](int i) {
    const int j = i & 3, pc = i >> 2;
    const int cc = pc % s_nc, rr = pc / s_nc;
    const int sr = s_r0 + rr, sc = s_c0 + cc;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if ((unsigned)sr < (unsigned)SH && (unsigned)sc < (unsigned)SW)
      v = __ldg(reinterpret_cast<const float4*>(src + (((long long)n * SH + sr) * SW + sc) * g.C + c0) + j);
    return v;
  });
  __syncthreads();
  // compute: outputs orows x OW x 4 quads; a thread's quad j is fixed (blockDim % 4 == 0),
  // so its taps' weights stay in registers
  const int outs = orows * OW * 4;
  const int jq = threadIdx.x & 3;
  float4 wreg[kDwMaxTaps];
#pragma unroll
  for (int k = 0; k < kDwMaxTaps; ++k) {
    const int tk = flip ? g.R * g.S - 1 - k : k;
    wreg[k] = k < g.R * g.S ? __ldg(reinterpret_cast<const float4*>(w + tk * g.C + c0) + jq)
                            : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  for (int i = threadIdx.x; i < outs; i += blockDim.x) {
    const int j = jq, po = i >> 2;
    const int ow = po % OW, orr = po / OW;
    const int oh = o0 + orr;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int r = 0; r < (kStride > 0 ? 3 : kDwMaxTaps); ++r) {
      if (r >= g.R) break;
      int sr;
      if (!kTrans) {
        sr = oh * g.sh - g.ph + r - s_r0;
      } else {
        const int t = oh + g.ph - r;
        if (t < 0 || t % g.sh) continue;
        sr = t / g.sh - s_r0;
        if (sr >= s_nr || t / g.sh >= SH) continue;
      }
#pragma unroll
      for (int s = 0; s < (kStride > 0 ? 3 : kDwMaxTaps); ++s) {
        if (s >= g.S) break;
        int sc;
        if (!kTrans) {
          sc = ow * g.sw - g.pw + s - s_c0;
        } else {
          const int t = ow + g.pw - s;
          if (t < 0 || t % g.sw) continue;
          sc = t / g.sw - s_c0;
          if (sc >= s_nc || t / g.sw >= SW) continue;
        }
        const float4 v = dw_smem[(sr * s_nc + sc) * 4 + j];
        fma4(acc, v, wreg[r * g.S + s]);
      }
    }
    float4* o = reinterpret_cast<float4*>(out + (((long long)n * OH + oh) * OW + ow) * g.C + c0) + j;
    if (accumulate) {
      const float4 a = *o;
      acc.x += a.x;
      acc.y += a.y;
      acc.z += a.z;
      acc.w += a.w;
    }
    *o = acc;
  }
}

// wgrad, persistent: grid (nb, C / kDwSlab); CTA b of slab z walks bands
// (n, row band) b, b + nb, ... staging the band's input rows and dy rows, and
// accumulates dw[tap][slab] for its (tap, quad) pairs over the band's pixels in
// registers (threads = 8 pixel groups x 32 (tap, quad) lanes); the groups are
// combined in shared memory once at the end -> part[b][tap][c] (fixed order).
template <int kStride = 0>
__global__ void __launch_bounds__(256) dwconv_wgrad_tile_kernel(const float* __restrict__ x,
                                                                const float* __restrict__ dy, float* __restrict__ part,
                                                                ConvGeom g, int nb) {
  extern __shared__ float4 dw_smem[];
  if (kStride > 0) {
    g.sh = g.sw = kStride;
    g.R = g.S = 3;
  }
  const int c0 = blockIdx.x * kDwSlab, wk = blockIdx.y;  // slabs fastest (walker wk of every slab together)
  const int bands_per_img = (g.P + kDwRows - 1) / kDwRows;
  const int total_bands = g.N * bands_per_img;
  const int taps = g.R * g.S;
  const int lane = threadIdx.x & 63, grp = threadIdx.x >> 6;  // 64 (tap, quad) slots x 4 pixel groups
  const int tap = lane >> 2, j = lane & 3;
  const bool active = tap < taps;
  const int r = active ? tap / g.S : 0, s = active ? tap - r * g.S : 0;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  const int x_nc = (g.Q - 1) * g.sw + g.S;
  for (int band = wk; band < total_bands; band += nb) {
    const int n = band / bands_per_img;
    const int p0 = (band - n * bands_per_img) * kDwRows;
    const int prow = min(kDwRows, g.P - p0);
    const int x_r0 = p0 * g.sh - g.ph, x_nr = (prow - 1) * g.sh + g.R;
    float4* xs = dw_smem;
    float4* ds = dw_smem + x_nr * x_nc * 4;
    __syncthreads();  // previous band's readers are done
    dw_stage(xs, x_nr * x_nc * 4, [&](int i) {
      const int jj = i & 3, pc = i >> 2;
      const int cc = pc % x_nc, rr = pc / x_nc;
      const int hr = x_r0 + rr, wc = cc - g.pw;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if ((unsigned)hr < (unsigned)g.H && (unsigned)wc < (unsigned)g.W)
        v = __ldg(reinterpret_cast<const float4*>(x + (((long long)n * g.H + hr) * g.W + wc) * g.C + c0) + jj);
      return v;
    });
    dw_stage(ds, prow * g.Q * 4, [&](int i) {
      const int jj = i & 3, pq = i >> 2;
      const int q = pq % g.Q, pr = pq / g.Q;
      return __ldg(reinterpret_cast<const float4*>(dy + (((long long)n * g.P + p0 + pr) * g.Q + q) * g.C + c0) + jj);
    });
    __syncthreads();
    if (active) {
      for (int pr = 0; pr < prow; ++pr) {
        const float4* drow = ds + pr * g.Q * 4 + j;
        const float4* xrow = xs + ((pr * g.sh + r) * x_nc + s) * 4 + j;
        for (int q = grp; q < g.Q; q += 4) fma4(acc, xrow[q * g.sw * 4], drow[q * 4]);
      }
    }
  }
  __syncthreads();
  dw_smem[threadIdx.x] = acc;
  __syncthreads();
  if (grp == 0 && active) {
    float4 t = dw_smem[lane];
    for (int k = 1; k < 4; ++k) {
      const float4 v = dw_smem[k * 64 + lane];
      t.x += v.x;
      t.y += v.y;
      t.z += v.z;
      t.w += v.w;
    }
    reinterpret_cast<float4*>(part + ((long long)wk * taps + tap) * g.C + c0)[j] = t;
  }
}

// wgrad for the 3x3 specialisations, persistent like dwconv_wgrad_tile_kernel (same grid, bands
// and part[b][tap][c] layout): thread = (kernel row r, quad j) x pixel group; a group walks a run
// of consecutive output columns of one band row and slides its three x taps along the staged row
// (stride 1: one new x load per column; stride 2: two), so a staged pixel is read about twice per
// kernel row instead of once per tap -- a third of the shared-memory reads of the per-tap walker,
// which is what bounds it.  The staged x rows get an odd pixel pitch so the three kernel rows of
// a quad fall on different banks.  Groups are combined in a fixed order at the end.
template <int kStride, bool kBatch>
__global__ void __launch_bounds__(256, kBatch ? 4 : 3) dwconv_wgrad_rows_kernel(const float* __restrict__ x,
                                                                const float* __restrict__ dy, float* __restrict__ part,
                                                                ConvGeom g, int nb, int kb) {
  extern __shared__ float4 dw_smem[];
  constexpr int kSlots = 12, kGroups = 256 / kSlots;  // 21 groups of (3 kernel rows x 4 quads)
  if constexpr (!kBatch) kb = 1;                       // the one-band-per-round variant
  const int c0 = blockIdx.x * kDwSlab, wk = blockIdx.y;  // slabs fastest (walker wk of every slab together)
  const int bands_per_img = (g.P + kDwRows - 1) / kDwRows;
  const int total_bands = g.N * bands_per_img;
  const int slot = threadIdx.x % kSlots, grp = threadIdx.x / kSlots;
  const int r = slot >> 2, j = slot & 3;
  const int x_nc = (g.Q - 1) * kStride + 3, x_pitch = x_nc | 1;
  const int x_band = ((kDwRows - 1) * kStride + 3) * x_pitch * 4, band_f4 = x_band + kDwRows * g.Q * 4;
  // runs per band row: the split of Q that fills the groups with the shortest critical path
  int nseg = 1, best = 1 << 30;
  for (int ns = 1; ns <= g.Q; ++ns) {
    const int len = (g.Q + ns - 1) / ns, nsr = (g.Q + len - 1) / len;
    const int cost = ((kb * kDwRows * nsr + kGroups - 1) / kGroups) * (len + 2);
    if (cost < best) {
      best = cost;
      nseg = nsr;
    }
  }
  const int len = (g.Q + nseg - 1) / nseg;
  float4 a0 = make_float4(0.f, 0.f, 0.f, 0.f), a1 = a0, a2 = a0;
  // rounds of kb bands (wk + (round * kb + i) * nb): all kb stagings in flight per barrier
  for (int band0 = wk; band0 < total_bands; band0 += nb * kb) {
    __syncthreads();  // previous round's readers are done
    if constexpr (kBatch) {
      // one staging pass over all kb bands (x window, then dy rows, per band): every load of the
      // round is in flight before the barrier, not one band's at a time
      dw_stage(dw_smem, kb * band_f4, [&](int e) {
        const int i = e / band_f4, o = e - i * band_f4;
        const int band = band0 + i * nb;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (band >= total_bands) return v;
        const int n = band / bands_per_img;
        const int p0 = (band - n * bands_per_img) * kDwRows;
        const int jj = o & 3;
        if (o < x_band) {
          const int pc = o >> 2, cc = pc % x_pitch, rr = pc / x_pitch;
          const int hr = p0 * kStride - g.ph + rr, wc = cc - g.pw;
          if (rr < (min(kDwRows, g.P - p0) - 1) * kStride + 3 && (unsigned)hr < (unsigned)g.H &&
              (unsigned)wc < (unsigned)g.W)
            v = __ldg(reinterpret_cast<const float4*>(x + (((long long)n * g.H + hr) * g.W + wc) * g.C + c0) + jj);
        } else {
          const int pq = (o - x_band) >> 2, q = pq % g.Q, pr = pq / g.Q;
          if (p0 + pr < g.P)
            v = __ldg(reinterpret_cast<const float4*>(dy + (((long long)n * g.P + p0 + pr) * g.Q + q) * g.C + c0) + jj);
        }
        return v;
      });
    } else {  // one band per round (kb == 1): the two plain staging loops keep the registers down
      const int n = band0 / bands_per_img;
      const int p0 = (band0 - n * bands_per_img) * kDwRows;
      const int prow = min(kDwRows, g.P - p0);
      const int x_r0 = p0 * kStride - g.ph, x_nr = (prow - 1) * kStride + 3;
      dw_stage(dw_smem, x_nr * x_pitch * 4, [&](int e) {
        const int jj = e & 3, pc = e >> 2;
        const int cc = pc % x_pitch, rr = pc / x_pitch;
        const int hr = x_r0 + rr, wc = cc - g.pw;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if ((unsigned)hr < (unsigned)g.H && (unsigned)wc < (unsigned)g.W)
          v = __ldg(reinterpret_cast<const float4*>(x + (((long long)n * g.H + hr) * g.W + wc) * g.C + c0) + jj);
        return v;
      });
      dw_stage(dw_smem + x_band, prow * g.Q * 4, [&](int e) {
        const int jj = e & 3, pq = e >> 2;
        const int q = pq % g.Q, pr = pq / g.Q;
        return __ldg(reinterpret_cast<const float4*>(dy + (((long long)n * g.P + p0 + pr) * g.Q + q) * g.C + c0) +
                     jj);
      });
    }
    __syncthreads();
    if (grp < kGroups) {
      for (int it = grp; it < kb * kDwRows * nseg; it += kGroups) {
        const int i = it / (kDwRows * nseg), rem = it - i * (kDwRows * nseg);
        const int pr = rem / nseg, q0 = (rem - pr * nseg) * len, q1 = min(q0 + len, g.Q);
        const int band = band0 + i * nb;
        if (band >= total_bands || (band % bands_per_img) * kDwRows + pr >= g.P) continue;
        const float4* xr = dw_smem + i * band_f4 + (pr * kStride + r) * x_pitch * 4 + j;
        const float4* dr = dw_smem + i * band_f4 + x_band + pr * g.Q * 4 + j;
        float4 u0 = xr[q0 * kStride * 4];
        float4 u1 = kStride == 1 ? xr[(q0 + 1) * 4] : u0;
        for (int q = q0; q < q1; ++q) {
          const float4 d = dr[q * 4];
          if (kStride != 1) u1 = xr[(q * kStride + 1) * 4];
          const float4 u2 = xr[(q * kStride + 2) * 4];
          fma4(a0, u0, d);
          fma4(a1, u1, d);
          fma4(a2, u2, d);
          if (kStride == 1) {
            u0 = u1;
            u1 = u2;
          } else {
            u0 = u2;
          }
        }
      }
    }
  }
  __syncthreads();
  if (grp < kGroups) {
    float4* red = dw_smem + (grp * kSlots + slot) * 3;
    red[0] = a0;
    red[1] = a1;
    red[2] = a2;
  }
  __syncthreads();
  if (threadIdx.x < 36) {  // (tap, quad): fixed-order sum over the groups
    const int tap = threadIdx.x >> 2, jj = threadIdx.x & 3;
    const int sl = (tap / 3) * 4 + jj, s = tap % 3;
    float4 t = dw_smem[sl * 3 + s];
    for (int k = 1; k < kGroups; ++k) {
      const float4 v = dw_smem[(k * kSlots + sl) * 3 + s];
      t.x += v.x;
      t.y += v.y;
      t.z += v.z;
      t.w += v.w;
    }
    reinterpret_cast<float4*>(part + ((long long)wk * 9 + tap) * g.C + c0)[jj] = t;
  }
}

}  // namespace monet
