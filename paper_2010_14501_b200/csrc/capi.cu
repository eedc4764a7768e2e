// extern "C" boundary of libmonet_b200.so (declared in include/monet_b200.h).
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "../../include/monet_b200.h"
#include "gemm_bf16x3.cuh"
#include "gemm_tc.cuh"
#include "local_ops.cuh"
#include "dwconv.cuh"

using namespace monet;

namespace {

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline int last_error() {
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : -static_cast<int>(e);
}

inline int ew_blocks(long long work_items) {
  long long b = (work_items + kEwThreads - 1) / kEwThreads;
  return (int)std::max(1LL, std::min(b, (long long)kNumSMs * 8));
}

// ----------------------------------------------------------------- GEMM setup
// Split-K factor of the "splitk" variant.  The persistent kernel walks tiles x splits
// units in rounds of kNumSMs; a round's time is set by its longest unit (kb_per_split
// k-blocks, rounded up to whole bf16x3 stages).  Up to the old target of ~2 units per SM,
// pick the split count with the least modeled time rounds * kb_per_split (ties: fewer
// splits, i.e. less partial-sum traffic): e.g. 36 tiles -> 8 splits (288 units, 2 full
// rounds) instead of 9 (324 units, a third round for 28 of them).  Never more splits than
// the old rule, so the workspace never grows.
int choose_splits(int variant, int M, int N, int Kd, int n_pitch = BN) {
  const int tiles = ((M + BM - 1) / BM) * ((N + n_pitch - 1) / n_pitch);
  const int kblocks = (Kd + BK - 1) / BK;
  if (variant != MONET_CONV_SPLITK) return 1;
  if (tiles >= kNumSMs) return 1;
  const int want = (2 * kNumSMs + tiles - 1) / tiles;
  const int hi = std::max(1, std::min(want, std::max(1, kblocks / 4)));
  int best = 1;
  long long best_cost = -1;
  for (int s = 1; s <= hi; ++s) {
    int kbps = (kblocks + s - 1) / s;
    kbps = (kbps + 1) & ~1;
    const int splits = (kblocks + kbps - 1) / kbps;
    const long long rounds = (tiles * (long long)splits + kNumSMs - 1) / kNumSMs;
    const long long cost = rounds * kbps;
    if (best_cost < 0 || cost < best_cost) {
      best_cost = cost;
      best = s;
    }
  }
  return best;
}

size_t gemm_ws(int variant, int M, int N, int Kd, int n_pitch = BN) {
  int s = choose_splits(variant, M, N, Kd, n_pitch);
  return s > 1 ? (size_t)s * M * N * sizeof(float) : 0;
}

// One instantiation per (A mode, B mode) pair used by conv / linear / gemm.
// kBx3 selects the bf16x3 A-in-TMEM kernel (gemm_bf16x3.cuh, the product
// path); otherwise the 3xTF32 / TF32 all-smem kernel (gemm_tc.cuh).
template <bool kBx3, bool kPair, int AM, int BMODE, int NB = BN, bool ST = false>
int launch_inst(const GemmParams& p, int grid, cudaStream_t st) {
  static bool attr = false;
  if constexpr (kBx3) {
    auto kern = bx3::gemm_bf16x3_kernel<AM, BMODE, kPair, NB, ST>;
    if (!attr) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bx3::Cfg<BMODE, NB>::kSmemBytes);
      attr = true;
    }
    if constexpr (kPair) {  // CTA pairs: clusters of 2 (the two SMs of a TPC)
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(grid);
      cfg.blockDim = dim3(bx3::kThreads);
      cfg.dynamicSmemBytes = bx3::Cfg<BMODE, NB>::kSmemBytes;
      cfg.stream = st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 2;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaError_t e = cudaLaunchKernelEx(&cfg, kern, p);
      return e == cudaSuccess ? 0 : -(int)e;
    } else {
      kern<<<grid, bx3::kThreads, bx3::Cfg<BMODE, NB>::kSmemBytes, st>>>(p);
    }
  } else {
    if (!attr) {
      cudaFuncSetAttribute(gemm_tf32_kernel<AM, BMODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
      attr = true;
    }
    gemm_tf32_kernel<AM, BMODE><<<grid, kThreads, kSmemBytes, st>>>(p);
  }
  return 0;
}

template <bool kBx3, bool kPair, int NB = BN>
int dispatch_modes(const GemmParams& p, int grid, cudaStream_t st) {
  const int a = p.a.mode, b = p.b.mode;
  if (a == OP_IM2COL_FPROP && b == OP_KMAJOR) return launch_inst<kBx3, kPair, OP_IM2COL_FPROP, OP_KMAJOR, NB>(p, grid, st);
  if (a == OP_KMAJOR && b == OP_KMAJOR) return launch_inst<kBx3, kPair, OP_KMAJOR, OP_KMAJOR, NB>(p, grid, st);
  if (a == OP_IM2COL_DGRAD && b == OP_MNMAJOR) return launch_inst<kBx3, kPair, OP_IM2COL_DGRAD, OP_MNMAJOR, NB>(p, grid, st);
  if (a == OP_KMAJOR && b == OP_MNMAJOR) return launch_inst<kBx3, kPair, OP_KMAJOR, OP_MNMAJOR, NB>(p, grid, st);
  if (a == OP_MNMAJOR && b == OP_IM2COL_WGRAD) return launch_inst<kBx3, kPair, OP_MNMAJOR, OP_IM2COL_WGRAD, NB>(p, grid, st);
  if (a == OP_MNMAJOR && b == OP_MNMAJOR) return launch_inst<kBx3, kPair, OP_MNMAJOR, OP_MNMAJOR, NB>(p, grid, st);
  if (a == OP_MNMAJOR && b == OP_KMAJOR) return launch_inst<kBx3, kPair, OP_MNMAJOR, OP_KMAJOR, NB>(p, grid, st);
  if constexpr (kBx3) {  // swapped wgrad of narrow convs: A = im2col(x)^T, B = dy^T
    if (a == OP_IM2COL_WGRAD && b == OP_MNMAJOR)
      return launch_inst<kBx3, kPair, OP_IM2COL_WGRAD, OP_MNMAJOR, NB>(p, grid, st);
    if constexpr (!kPair) {  // pre-split bf16 weights (fprop B = w, dgrad B = w^T)
      if (a == OP_IM2COL_FPROP && b == OP_W16_KMAJOR)
        return p.stats ? launch_inst<kBx3, kPair, OP_IM2COL_FPROP, OP_W16_KMAJOR, NB, true>(p, grid, st)
                       : launch_inst<kBx3, kPair, OP_IM2COL_FPROP, OP_W16_KMAJOR, NB>(p, grid, st);
      if (a == OP_KMAJOR && b == OP_W16_KMAJOR)
        return p.stats ? launch_inst<kBx3, kPair, OP_KMAJOR, OP_W16_KMAJOR, NB, true>(p, grid, st)
                       : launch_inst<kBx3, kPair, OP_KMAJOR, OP_W16_KMAJOR, NB>(p, grid, st);
      if (a == OP_IM2COL_DGRAD && b == OP_W16_MNMAJOR)
        return launch_inst<kBx3, kPair, OP_IM2COL_DGRAD, OP_W16_MNMAJOR, NB>(p, grid, st);
      if (a == OP_KMAJOR && b == OP_W16_MNMAJOR) return launch_inst<kBx3, kPair, OP_KMAJOR, OP_W16_MNMAJOR, NB>(p, grid, st);
    }
  }
  return -(int)cudaErrorInvalidValue;
}

bool uses_bx3(int variant) {
  return variant == MONET_CONV_IMPLICIT || variant == MONET_CONV_SPLITK || variant == MONET_CONV_PAIR;
}

// ----------------------------------------------------------------- TMA maps
// The driver's tensor-map encoders, resolved through the runtime (no -lcuda).
PFN_cuTensorMapEncodeTiled_v12000 g_enc_tiled = nullptr;
PFN_cuTensorMapEncodeIm2col_v12000 g_enc_im2col = nullptr;

bool tma_available() {
  static int state = 0;
  if (state == 0) {
    cudaDriverEntryPointQueryResult q1, q2;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&g_enc_tiled), cudaEnableDefault, &q1);
    cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", reinterpret_cast<void**>(&g_enc_im2col), cudaEnableDefault,
                            &q2);
    state = (g_enc_tiled && g_enc_im2col) ? 1 : -1;
    cudaGetLastError();
  }
  return state == 1;
}

int tiled_map(CUtensorMap* m, const float* ptr, int rank, const cuuint64_t* dims, const cuuint64_t* strides,
              const cuuint32_t* box, CUtensorMapSwizzle sw) {
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = g_enc_tiled(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, const_cast<float*>(ptr), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 1 : 0;
}

// bf16 planes (pre-split weights): SWIZZLE_128B boxes of 64 bf16 = 128 B rows, the
// MMA's stage-tile layout as loaded
int tiled_map_bf16(CUtensorMap* m, const void* ptr, int rank, const cuuint64_t* dims, const cuuint64_t* strides,
                   const cuuint32_t* box) {
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult r = g_enc_tiled(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(ptr), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 1 : 0;
}

// im2col map over an NHWC tensor [n][h][w][c]; corners / offsets index 0 = W, 1 = H
// (pinned on the B200 by tools/tma_probe.cu)
int im2col_map(CUtensorMap* m, const float* ptr, int n, int h, int w, int c, int lo_w, int lo_h, int up_w, int up_h,
               int es_w, int es_h, int channels, int pixels, CUtensorMapSwizzle sw) {
  const int corners[4] = {lo_w, lo_h, up_w, up_h};
  for (int v : corners)
    if (v < -128 || v > 127) return 0;
  cuuint64_t dims[4] = {(cuuint64_t)c, (cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)n};
  cuuint64_t strides[3] = {(cuuint64_t)c * 4, (cuuint64_t)w * c * 4, (cuuint64_t)h * w * c * 4};
  int lo[2] = {lo_w, lo_h}, up[2] = {up_w, up_h};
  cuuint32_t es[4] = {1, (cuuint32_t)es_w, (cuuint32_t)es_h, 1};
  CUresult r = g_enc_im2col(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(ptr), dims, strides, lo, up,
                            channels, pixels, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 2 : 0;
}

// TMA descriptor for one bf16x3 operand; returns Operand::tma (0 = use the
// 16B cp.async fallback).  Raw layouts: K-major boxes are 32 fp32 x 128 rows
// with SWIZZLE_128B, MN-major boxes 128 (or p.mn_seg) rows x 32 k, unswizzled.
int make_tma(GemmParams& p, Operand& op, CUtensorMap* m) {
  if (!tma_available() || (reinterpret_cast<uintptr_t>(op.ptr) & 15) != 0) return 0;
  const ConvGeom& g = p.g;
  if (p.wv_q) {  // wgrad tap view (k = (n, p, q < wv_q)); out-of-range q / r load as zeros
    if (op.mode == OP_MNMAJOR) {  // dy[n][p][q][kout] as {kout, q, n*p}
      cuuint64_t dims[3] = {(cuuint64_t)g.K, (cuuint64_t)g.Q, (cuuint64_t)g.N * g.P};
      cuuint64_t strides[2] = {(cuuint64_t)g.K * 4, (cuuint64_t)g.Q * g.K * 4};
      cuuint32_t box[3] = {(cuuint32_t)op.rows_box, 32, 1};
      return tiled_map(m, op.ptr, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_NONE) ? 4 : 0;
    }
    // zero-padded input xp[n][Hp][Wp][c]: element (s*C + c, q, r, p, n) = xp[n][p*sh + r][q*sw + s][c];
    // the q stride (sw*C floats) is below the s*C extent -- overlapping rows, accepted by the
    // encoder and pinned on the B200 by tools/tma_overlap_probe.cu
    const long long Wp = (long long)(g.Q - 1) * g.sw + g.S, Hp = (long long)(g.P - 1) * g.sh + g.R;
    cuuint64_t dims[5] = {(cuuint64_t)g.S * g.C, (cuuint64_t)g.Q, (cuuint64_t)g.R, (cuuint64_t)g.P,
                          (cuuint64_t)g.N};
    cuuint64_t strides[4] = {(cuuint64_t)g.sw * g.C * 4, (cuuint64_t)Wp * g.C * 4, (cuuint64_t)g.sh * Wp * g.C * 4,
                             (cuuint64_t)Hp * Wp * g.C * 4};
    cuuint32_t box[5] = {(cuuint32_t)g.S * g.C, 32, (cuuint32_t)(op.rows_box / (g.S * g.C)), 1, 1};
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    CUresult r = g_enc_tiled(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<float*>(op.ptr), dims, strides, box,
                             es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 4 : 0;
  }
  if (p.fv_q && op.mode == OP_IM2COL_FPROP) {
    // fprop tap view over the zero-padded input xp[n][Hp][Wp][c]: element (j, q, r, p, n) =
    // xp[n][p*sh + r][q*sw][j] for j < 32 -- the filter row's S*C taps x channels (S*C <= 32;
    // j >= S*C reads the next pixels, multiplied by the zero-padded weights) -- with the q
    // stride sw*C below the 32-float row: overlapping rows, as in the wgrad tap view
    const long long Wp = (long long)(g.Q - 1) * g.sw + g.S, Hp = (long long)(g.P - 1) * g.sh + g.R;
    cuuint64_t dims[5] = {32, (cuuint64_t)p.fv_q, (cuuint64_t)g.R, (cuuint64_t)g.P, (cuuint64_t)g.N};
    cuuint64_t strides[4] = {(cuuint64_t)g.sw * g.C * 4, (cuuint64_t)Wp * g.C * 4, (cuuint64_t)g.sh * Wp * g.C * 4,
                             (cuuint64_t)Hp * Wp * g.C * 4};
    cuuint32_t box[5] = {32, (cuuint32_t)p.fv_q, 1, 1, 1};
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    CUresult r = g_enc_tiled(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<float*>(op.ptr), dims, strides, box,
                             es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 5 : 0;
  }
  switch (op.mode) {
    case OP_W16_KMAJOR: {  // hi / lo planes [rows][ld]: {k, row, plane}, one 64 x rows_box box per plane
      if (op.ld % 8 || op.plane <= 0 || op.plane % 16) return 0;
      cuuint64_t dims[3] = {(cuuint64_t)p.Kd, (cuuint64_t)op.rows, 2};
      cuuint64_t strides[2] = {(cuuint64_t)op.ld * 2, (cuuint64_t)op.plane};
      cuuint32_t box[3] = {64, (cuuint32_t)op.rows_box, 1};
      return tiled_map_bf16(m, op.ptr, 3, dims, strides, box);
    }
    case OP_W16_MNMAJOR: {  // w^T: {row (= c), tap, kout, plane}, boxes of 64 channels x 32 kout
      if (op.kdiv % 32 || op.ld % 8 || op.ks1 % 8 || op.plane <= 0 || op.plane % 16) return 0;
      if (!p.ph.on && p.Kd % op.kdiv) return 0;
      const int ntaps = p.ph.on ? g.R * g.S : p.Kd / op.kdiv;
      cuuint64_t dims[4] = {(cuuint64_t)op.rows, (cuuint64_t)ntaps, (cuuint64_t)op.kdiv, 2};
      cuuint64_t strides[3] = {(cuuint64_t)op.ks1 * 2, (cuuint64_t)op.ld * 2, (cuuint64_t)op.plane};
      cuuint32_t box[4] = {64, 1, 32, 1};
      return tiled_map_bf16(m, op.ptr, 4, dims, strides, box);
    }
    case OP_KMAJOR: {
      if (op.ld % 4) return 0;
      cuuint64_t dims[2] = {(cuuint64_t)p.Kd, (cuuint64_t)op.rows};
      cuuint64_t strides[1] = {(cuuint64_t)op.ld * 4};
      cuuint32_t box[2] = {32, (cuuint32_t)op.rows_box};
      return tiled_map(m, op.ptr, 2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
    }
    case OP_MNMAJOR: {
      if (op.ld % 4) return 0;
      if (op.kdiv >= p.Kd && !p.ph.on) {
        cuuint64_t dims[2] = {(cuuint64_t)op.rows, (cuuint64_t)p.Kd};
        cuuint64_t strides[1] = {(cuuint64_t)op.ld * 4};
        cuuint32_t box[2] = {(cuuint32_t)op.rows_box, 32};
        return tiled_map(m, op.ptr, 2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_NONE);
      }
      if (op.kdiv % 32 || op.ks1 % 4 || p.Kd % op.kdiv) return 0;
      // taps dimension: every filter tap (a stride phase addresses a subset by tap id)
      const int ntaps = p.ph.on ? g.R * g.S : p.Kd / op.kdiv;
      cuuint64_t dims[3] = {(cuuint64_t)op.rows, (cuuint64_t)ntaps, (cuuint64_t)op.kdiv};
      cuuint64_t strides[2] = {(cuuint64_t)op.ks1 * 4, (cuuint64_t)op.ld * 4};
      cuuint32_t box[3] = {(cuuint32_t)op.rows_box, 1, 32};
      return tiled_map(m, op.ptr, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_NONE);
    }
    case OP_IM2COL_FPROP:
      if (g.C == 4 || g.C == 8 || g.C == 16)  // one box of C channels per filter tap
        return im2col_map(m, op.ptr, g.N, g.H, g.W, g.C, -g.pw, -g.ph, g.pw - (g.S - 1), g.ph - (g.R - 1), g.sw,
                          g.sh, g.C, 128, CU_TENSOR_MAP_SWIZZLE_NONE)
                   ? 3
                   : 0;
      if (g.C % 32) return 0;
      return im2col_map(m, op.ptr, g.N, g.H, g.W, g.C, -g.pw, -g.ph, g.pw - (g.S - 1), g.ph - (g.R - 1), g.sw, g.sh,
                        32, 128, CU_TENSOR_MAP_SWIZZLE_128B);
    case OP_IM2COL_DGRAD:  // forward conv over dy with flipped taps; stride 1, or one stride phase
      if (g.K % 32) return 0;
      if (p.ph.on)
        return im2col_map(m, op.ptr, g.N, g.P, g.Q, g.K, p.ph.lo_w, p.ph.lo_h, p.ph.Wp - g.Q + p.ph.lo_w,
                          p.ph.Hp - g.P + p.ph.lo_h, 1, 1, 32, 128, CU_TENSOR_MAP_SWIZZLE_128B);
      if (g.sh != 1 || g.sw != 1) return 0;
      return im2col_map(m, op.ptr, g.N, g.P, g.Q, g.K, -(g.S - 1 - g.pw), -(g.R - 1 - g.ph), -g.pw, -g.ph, 1, 1, 32,
                        128, CU_TENSOR_MAP_SWIZZLE_128B);
    case OP_IM2COL_WGRAD: {
      // segments of C (< 128) or 128 channels; below 32 channels (the stem) the
      // 32-TMA-per-k-block segment loop loses to the 16B cp.async fallback
      const int rb = op.rows_box;
      if (g.C < rb ? rb % g.C || g.C < 32 : g.C % rb) return 0;
      const int seg = std::min(g.C, rb);
      const int r = im2col_map(m, op.ptr, g.N, g.H, g.W, g.C, -g.pw, -g.ph, g.pw - (g.S - 1), g.ph - (g.R - 1),
                               g.sw, g.sh, seg, 32, CU_TENSOR_MAP_SWIZZLE_NONE);
      if (r) op.seg = seg;
      return r;
    }
  }
  return 0;
}

float* g_dbg_a = nullptr;
float* g_dbg_b = nullptr;
unsigned long long* g_dbg_t = nullptr;

bool al16(const void* p);

int launch_gemm(GemmParams p, int variant, int accumulate, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (p.M <= 0 || p.N <= 0) return 0;
  p.dbg_a = g_dbg_a;
  p.dbg_b = g_dbg_b;
  p.dbg_t = g_dbg_t;
#ifdef MONET_DEBUG
  static const int dbg_mode = getenv("MONET_DBG_MODE") ? atoi(getenv("MONET_DBG_MODE")) : 0;
  p.dbg_mode = dbg_mode;
#endif
  const bool bx = uses_bx3(variant);
  // variant "pair" (cta_group::2, 256-row tiles) is retired: 15-25 % slower than one CTA per
  // tile on every ResNet-50 shape, and one wrong-tile result seen in round-2 GPU testing that
  // 360 stress repetitions did not reproduce
  if (variant == MONET_CONV_PAIR) return -(int)cudaErrorNotSupported;
  const bool pair = false;
  // 64-wide N tiles when the whole problem is at most 64 columns wide (64-channel convs)
  const bool narrow = bx && !pair && !p.wv_q && p.N <= 64;
  if (p.n_pitch == 0) p.n_pitch = narrow ? 64 : BN;
  p.a.rows_box = BM;
  p.b.rows_box = pair ? BN / 2 : (p.wv_q || narrow ? p.n_pitch : BN);
  if (bx) {
    // MONET_TMA_MASK (debug): bit 0 enables TMA for A, bit 1 for B (default 3)
    static const int mask = getenv("MONET_TMA_MASK") ? atoi(getenv("MONET_TMA_MASK")) : 3;
    p.a.seg = p.a.rows_box;
    p.b.seg = p.wv_q ? p.g.S * p.g.C : p.b.rows_box;
    // MMA stages (64 k each) per TMEM accumulation chain before a flush to fp32 memory: 16
    // (K = 1024).  The tensor core's fp32 accumulation does not round to nearest, so a chain's
    // error is biased and grows with its length (tools/chunk_accuracy.py: 5.7e-6 at 16 stages,
    // 6-9e-6 at 36, 1.8e-5 at 72); a bias in dz survives the 577k-row sums of the BN weight
    // gradients, which at 36 stages missed the headline parity test's 1e-3 bar by 30x.
    // MONET_CHUNK (debug) overrides it.
    static const int chunk = getenv("MONET_CHUNK") ? atoi(getenv("MONET_CHUNK")) : 16;
    p.chunk_stages = chunk > 0 ? chunk : 16;
    p.a.tma = (mask & 1) ? make_tma(p, p.a, &p.tma_a) : 0;
    p.b.tma = (mask & 2) ? make_tma(p, p.b, &p.tma_b) : 0;
    // the tap views' layouts exist only as tensor maps: no cp.async fallback
    if (p.wv_q && (p.a.tma != 4 || p.b.tma != 4)) return -(int)cudaErrorNotSupported;
    if (p.fv_q && p.a.tma != 5) return -(int)cudaErrorNotSupported;
    // pre-split weights load only by TMA; the caller then takes the fp32 path
    if (mode_is_w16(p.b.mode) && !p.b.tma) return -(int)cudaErrorNotSupported;
  }
  p.split_tf32 = variant == MONET_CONV_TF32 ? 0 : 1;
  p.c_tma = 0;
  p.m_tiles = (p.M + (pair ? 2 * BM : BM) - 1) / (pair ? 2 * BM : BM);
  p.n_tiles = (p.N + p.n_pitch - 1) / p.n_pitch;
  const int kblocks = std::max(1, (p.Kd + BK - 1) / BK);
  int splits = p.ph.on ? 1 : choose_splits(variant, p.M, p.N, p.Kd, p.n_pitch);  // phase rows scatter: no split-K
  size_t need = splits > 1 ? (size_t)splits * p.M * p.N * sizeof(float) : 0;
  if (need > ws_bytes || (need && ws == nullptr)) {
    splits = 1;  // never write outside the caller's workspace
    need = 0;
  }
  p.kb_per_split = (kblocks + splits - 1) / splits;
  if (bx) p.kb_per_split = (p.kb_per_split + 1) & ~1;  // bf16x3 stages hold two raw k-blocks
  p.splits = (kblocks + p.kb_per_split - 1) / p.kb_per_split;
  p.ws = static_cast<float*>(ws);
  p.epi = p.splits > 1 ? EPI_PARTIAL : (accumulate ? EPI_ACCUM : EPI_STORE);
  // pre-split-B kernels: output blocks through smem + TMA store when the output rows are plain
  // (no phase scatter, tap-view padding rows or transposed store) and 16-B aligned
  if (bx && mode_is_w16(p.b.mode) && !p.ph.on && !p.fv_q && !p.c_trans && p.n_pitch % 32 == 0) {
    float* out = p.epi == EPI_PARTIAL ? p.ws : p.c;
    const long long ld = p.epi == EPI_PARTIAL ? p.N : p.ldc;
    if (al16(out) && ld % 4 == 0) {
      cuuint64_t dims[3] = {(cuuint64_t)p.N, (cuuint64_t)p.M, (cuuint64_t)(p.epi == EPI_PARTIAL ? p.splits : 1)};
      cuuint64_t strides[2] = {(cuuint64_t)ld * 4, (cuuint64_t)p.M * ld * 4};
      cuuint32_t box[3] = {32, 32, 1};
      p.c_tma = tiled_map(&p.tma_c, out, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
    }
  }
  // BN statistics from the epilogue: only where every output element is final in one TMEM
  // chain (no split-K, no chunk flushes), the TMA-store epilogue runs, and the reduction is long
  // enough (K >= 512) to hide the column walk behind the MMAs -- output-heavy short-K convs
  // (1x1 64 -> 256: +300 us in the epilogue vs ~90 us for one pass over y) take the pass instead
  if (p.stats && !(p.c_tma && p.epi == EPI_STORE && p.splits == 1 && p.Kd >= 512 &&
                   (p.kb_per_split + 1) / 2 <= p.chunk_stages))
    p.stats = nullptr;
  if (p.stats_done) *p.stats_done = p.stats != nullptr;
  const int tiles = p.m_tiles * p.n_tiles * p.splits;
  const int grid = pair ? 2 * std::min(tiles, kNumSMs / 2) : std::min(tiles, kNumSMs);
  const int e = !bx     ? dispatch_modes<false, false>(p, grid, st)
                : narrow ? dispatch_modes<true, false, 64>(p, grid, st)
                         : dispatch_modes<true, false>(p, grid, st);
  if (e) return e;
  if (p.splits > 1) {
    long long total = (long long)p.M * p.N;
    splitk_reduce_kernel<<<ew_blocks(total), kEwThreads, 0, st>>>(p.ws, p.c, p.M, p.N, p.ldc, p.splits, accumulate,
                                                                  p.bias, p.c_trans);
  }
  return last_error();
}

bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// Launch with the weight operand B taken from its pre-split bf16 planes (hi, lo: the
// same element offsets as the fp32 weights at p.b.ptr) when the shape allows it, else
// (or without planes) from the fp32 weights: the two give bit-identical results, the
// split being the one the B-split warps would do (split_pair).
int launch_gemm_w16(const GemmParams& p, const uint16_t* hi, const uint16_t* lo, int variant, int accumulate,
                    void* ws, size_t ws_bytes, cudaStream_t st) {
  if (hi != nullptr && lo != nullptr && lo > hi && uses_bx3(variant) && al16(hi) &&
      (p.b.mode == OP_KMAJOR || p.b.mode == OP_MNMAJOR)) {
    GemmParams q = p;
    q.b.mode = p.b.mode == OP_KMAJOR ? OP_W16_KMAJOR : OP_W16_MNMAJOR;
    q.b.ptr = reinterpret_cast<const float*>(hi);
    q.b.plane = reinterpret_cast<const char*>(lo) - reinterpret_cast<const char*>(hi);
    const int e = launch_gemm(q, variant, accumulate, ws, ws_bytes, st);
    if (e != -(int)cudaErrorNotSupported) return e;
  }
  return launch_gemm(p, variant, accumulate, ws, ws_bytes, st);
}

// hi = bf16(x), lo = bf16(x - hi), round to nearest even: the B split's own rounding
__device__ __forceinline__ void split_one(float x, uint16_t& h, uint16_t& l) {
  uint32_t h2, l2;
  bx3::split_pair(x, 0.f, h2, l2);  // element x in the low halves
  h = (uint16_t)(h2 & 0xFFFFu);
  l = (uint16_t)(l2 & 0xFFFFu);
}

__global__ void split_bf16_kernel(const float* __restrict__ src, uint16_t* hi, uint16_t* lo, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    split_one(src[i], hi[i], lo[i]);
}

// segments {src_off, dst_off, count} (elements), one grid row per segment
__global__ void split_bf16_segments_kernel(const float* __restrict__ src, uint16_t* hi, uint16_t* lo,
                                           const long long* __restrict__ table) {
  const long long s0 = table[3 * blockIdx.y], d0 = table[3 * blockIdx.y + 1], n = table[3 * blockIdx.y + 2];
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    split_one(src[s0 + i], hi[d0 + i], lo[d0 + i]);
}

Operand op_kmajor(const float* ptr, int rows, long long ld, int kd) {
  return Operand{OP_KMAJOR, rows, ptr, ld, 1 << 30, 0, (al16(ptr) && ld % 4 == 0 && kd % 4 == 0) ? 1 : 0};
}
Operand op_mnmajor(const float* ptr, int rows, long long ld) {
  return Operand{OP_MNMAJOR, rows, ptr, ld, 1 << 30, 0, (al16(ptr) && ld % 4 == 0 && rows % 4 == 0) ? 1 : 0};
}
Operand op_gather(int mode, const float* ptr, int rows) {
  return Operand{mode, rows, ptr, 0, 1 << 30, 0, 1};  // conv gathers: C, K % 4 == 0 checked by check_desc
}

ConvGeom geom(const monet_conv_desc* d) {
  return ConvGeom{d->n, d->h, d->w, d->c, d->k, d->r, d->s, d->p, d->q, d->stride_h, d->stride_w, d->pad_h, d->pad_w};
}

bool is_pointwise(const monet_conv_desc* d) {
  return d->r == 1 && d->s == 1 && d->stride_h == 1 && d->stride_w == 1 && d->pad_h == 0 && d->pad_w == 0;
}

GemmParams conv_params(int pass, const monet_conv_desc* d, const float* in0, const float* in1, float* out) {
  GemmParams p{};
  p.g = geom(d);
  const int rsc = d->r * d->s * d->c;
  if (pass == MONET_PASS_FWD) {  // in0 = x, in1 = w
    p.M = d->n * d->p * d->q;
    p.N = d->k;
    p.Kd = rsc;
    p.a = is_pointwise(d) ? op_kmajor(in0, p.M, d->c, p.Kd) : op_gather(OP_IM2COL_FPROP, in0, p.M);
    p.b = op_kmajor(in1, d->k, rsc, p.Kd);
    p.c = out;
    p.ldc = d->k;
  } else if (pass == MONET_PASS_DGRAD) {  // in0 = dy, in1 = w
    p.M = d->n * d->h * d->w;
    p.N = d->c;
    p.Kd = d->r * d->s * d->k;
    p.a = is_pointwise(d) ? op_kmajor(in0, p.M, d->k, p.Kd) : op_gather(OP_IM2COL_DGRAD, in0, p.M);
    // B[c, (tap, kout)] = w[kout, tap, c]
    p.b = Operand{OP_MNMAJOR, d->c, in1, (long long)rsc, d->k, (long long)d->c, al16(in1) ? 1 : 0};
    p.c = out;
    p.ldc = d->c;
  } else {  // wgrad: in0 = x, in1 = dy
    p.M = d->k;
    p.N = rsc;
    p.Kd = d->n * d->p * d->q;
    p.a = op_mnmajor(in1, d->k, d->k);  // A[kout, pix] = dy[pix, kout]
    p.b = is_pointwise(d) ? op_mnmajor(in0, d->c, d->c) : op_gather(OP_IM2COL_WGRAD, in0, rsc);
    p.c = out;
    p.ldc = rsc;
  }
  return p;
}

// Sub-pixel phases of a strided dgrad (bf16x3 path).  Returns false for an
// empty phase grid; ntap == 0 means the phase's dx pixels receive no gradient.
bool make_phase(const monet_conv_desc* d, int a, int b, PhaseInfo& ph) {
  ph = PhaseInfo{};
  ph.on = 1;
  ph.a = a;
  ph.b = b;
  ph.Hp = (d->h - a + d->stride_h - 1) / d->stride_h;
  ph.Wp = (d->w - b + d->stride_w - 1) / d->stride_w;
  if (ph.Hp <= 0 || ph.Wp <= 0) return false;
  ph.lo_h = ph.lo_w = 1 << 20;
  for (int r = 0; r < d->r; ++r) {
    const int nr = a + d->pad_h - r;
    if (((nr % d->stride_h) + d->stride_h) % d->stride_h) continue;
    for (int s = 0; s < d->s; ++s) {
      const int ns = b + d->pad_w - s;
      if (((ns % d->stride_w) + d->stride_w) % d->stride_w) continue;
      const int dr = nr >= 0 ? nr / d->stride_h : -((-nr) / d->stride_h);
      const int ds = ns >= 0 ? ns / d->stride_w : -((-ns) / d->stride_w);
      ph.dr[ph.ntap] = (signed char)dr;
      ph.ds[ph.ntap] = (signed char)ds;
      ph.tap[ph.ntap] = (signed char)(r * d->s + s);
      ph.lo_h = std::min(ph.lo_h, dr);
      ph.lo_w = std::min(ph.lo_w, ds);
      ++ph.ntap;
    }
  }
  if (ph.ntap == 0) ph.lo_h = ph.lo_w = 0;
  return true;
}

// stride >= 2 and R, S <= 8 keep every phase at <= 16 taps (PhaseInfo tables)
bool use_phases(int variant, const monet_conv_desc* d) {
  return uses_bx3(variant) && (d->stride_h > 1 || d->stride_w > 1) && d->r <= 8 && d->s <= 8;
}

// Wgrad "tap view" for inputs with C < 32 (the 7x7/2 stem): the reduction runs
// over k = (n, p, q padded to a multiple of 32) so that every 32-deep k-block is
// one TMA box per operand -- dy {kout, 32 q, 1} and, over a zero-padded copy of
// the input in the workspace, {S*C, 32 q, R-segments} with overlapping q / s
// strides.  An n-tile covers floor(128 / (S*C)) filter rows (112 columns for the
// stem).  Replaces the 16B cp.async gather (per-group divisions) for these layers
// when the reduction is long (>= 32K output pixels).
struct WView {
  bool on;
  int qpad, n_pitch;
  long long kd;
  size_t pad_bytes;
};

WView wgrad_view(int variant, const monet_conv_desc* d) {
  WView v{};
  if (!uses_bx3(variant) || variant == MONET_CONV_PAIR || is_pointwise(d) || d->c >= 32 || d->s * d->c > 128)
    return v;
  // below 32K output pixels the gather is cheap and the padded copy is not worth its workspace
  if ((long long)d->n * d->p * d->q < (1 << 15)) return v;
  v.on = true;
  v.qpad = (d->q + 31) / 32 * 32;
  v.n_pitch = (128 / (d->s * d->c)) * d->s * d->c;
  v.kd = (long long)d->n * d->p * v.qpad;
  const long long hp = (long long)(d->p - 1) * d->stride_h + d->r, wp = (long long)(d->q - 1) * d->stride_w + d->s;
  v.pad_bytes = (size_t)d->n * hp * wp * d->c * sizeof(float);
  return v;
}

size_t align256(size_t b) { return (b + 255) / 256 * 256; }

// Fprop "tap view" for narrow-channel inputs (the 7x7/2 stem, C = 4): the 4-channel im2col
// boxes (16 B per pixel row, one TMA per filter tap) cap the stem forward at ~55 TF/s.
// Instead the GEMM rows are (n, p, q padded to 128) -- one output row per M tile -- and the
// reduction runs over k = (r, s*C + c padded to 32): every k-block is ONE tiled TMA box of
// 128 x 32 floats over a zero-padded copy of the input (overlapping q rows), and the
// weights are repacked to [K][R][32] with zeros for the padding.  Workspace = the padded
// copy + the repacked weights, so it is the "splitk" (workspace) forward variant.
struct FView {
  bool on;
  size_t pad_bytes, w_bytes;
};

FView fprop_view(int variant, const monet_conv_desc* d) {
  FView v{};
  if (variant != MONET_CONV_SPLITK || is_pointwise(d) || d->s * d->c > 32 || d->q > BM || d->c % 4) return v;
  if ((long long)d->n * d->p * d->q < (1 << 15)) return v;  // small problems: the gather is fine
  v.on = true;
  const long long hp = (long long)(d->p - 1) * d->stride_h + d->r, wp = (long long)(d->q - 1) * d->stride_w + d->s;
  // + slack: the last row's padded q (and j >= S*C) read up to one output row past the copy
  v.pad_bytes = align256((size_t)d->n * hp * wp * d->c * sizeof(float) + (size_t)BM * d->stride_w * d->c * 4 + 4096);
  v.w_bytes = align256((size_t)d->k * d->r * 32 * sizeof(float));
  return v;
}

// w'[k][r][j] = w[k][r][s][c] for j = s*C + c < S*C, else 0
__global__ void fview_weight_kernel(const float* __restrict__ w, float* __restrict__ wp, int K, int R, int S, int C) {
  const int total = K * R * 32;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int j = i % 32, t = i / 32, r = t % R, k = t / R;
    wp[i] = j < S * C ? w[((k * R + r) * S) * C + j] : 0.f;
  }
}

// Wgrad of a narrow conv (K_out < 128 output channels, e.g. ResNet-50's 64-channel layer1):
// the natural mapping M = K_out fills only half of every 128-row MMA.  Swapped, the GEMM
// rows are the filter taps x input channels (M = R*S*C) and the columns the output
// channels on a 64-wide N tile; the epilogue stores the result transposed into the KRSC
// weight gradient.  Same tile count and split-K workspace as the natural mapping.
bool wgrad_swapped(int variant, const monet_conv_desc* d) {
  return uses_bx3(variant) && d->k < BM && (long long)d->r * d->s * d->c > d->k;
}

GemmParams wgrad_swapped_params(const monet_conv_desc* d, const float* x, const float* dy, float* dw) {
  GemmParams p{};
  p.g = geom(d);
  const int rsc = d->r * d->s * d->c;
  p.M = rsc;
  p.N = d->k;
  p.Kd = d->n * d->p * d->q;
  p.a = is_pointwise(d) ? op_mnmajor(x, d->c, d->c) : op_gather(OP_IM2COL_WGRAD, x, rsc);  // A[(tap, c), pix]
  p.b = op_mnmajor(dy, d->k, d->k);                                                          // B[kout, pix]
  p.c = dw;
  p.ldc = rsc;
  p.c_trans = 1;
  return p;
}

// xp[n][hp][wp][c] = x[n][hp - pad_h][wp - pad_w][c], zero outside
__global__ void wgrad_pad_kernel(const float* __restrict__ x, float* __restrict__ xp, int n, int h, int w, int c,
                                 int hp, int wp, int pad_h, int pad_w) {
  const int c4 = c / 4;
  const long long total = (long long)n * hp * wp * c4;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int cc = (int)(i % c4);
    long long t = i / c4;
    const int j = (int)(t % wp);
    t /= wp;
    const int ii = (int)(t % hp);
    const int nn = (int)(t / hp);
    const int hh = ii - pad_h, ww = j - pad_w;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if ((unsigned)hh < (unsigned)h && (unsigned)ww < (unsigned)w)
      v = __ldg(reinterpret_cast<const float4*>(x + (((long long)nn * h + hh) * w + ww) * c) + cc);
    reinterpret_cast<float4*>(xp)[i] = v;
  }
}

GemmParams phase_params(const monet_conv_desc* d, const PhaseInfo& ph, const float* dy, const float* w, float* dx) {
  GemmParams p{};
  p.g = geom(d);
  p.ph = ph;
  p.M = d->n * ph.Hp * ph.Wp;
  p.N = d->c;
  p.Kd = ph.ntap * d->k;
  p.a = op_gather(OP_IM2COL_DGRAD, dy, p.M);
  // B[c, (t, kout)] = w[kout][tap[t]][c]
  p.b = Operand{OP_MNMAJOR, d->c, w, (long long)d->r * d->s * d->c, d->k, (long long)d->c, al16(w) ? 1 : 0, 0};
  p.c = dx;
  p.ldc = d->c;
  return p;
}

__global__ void dgrad_phase_zero_kernel(float* dx, int n, int h, int w, int c, int a, int b, int sh, int sw) {
  const int hp = (h - a + sh - 1) / sh, wp = (w - b + sw - 1) / sw;
  const long long total = (long long)n * hp * wp * (c / 4);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int c4 = (int)(i % (c / 4));
    long long t = i / (c / 4);
    const int j = (int)(t % wp);
    t /= wp;
    const int ii = (int)(t % hp);
    const int nn = (int)(t / hp);
    float* dst = dx + (((long long)nn * h + ii * sh + a) * w + j * sw + b) * c + 4 * c4;
    *reinterpret_cast<float4*>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

int check_desc(const monet_conv_desc* d) {
  if (!d || d->c % 4 || d->k % 4 || d->n <= 0) return -(int)cudaErrorInvalidValue;
  return 0;
}

}  // namespace

extern "C" {

const char* monet_version(void) { return "monet_b200 0.1.0 sm_100a"; }

int monet_device_check(void) {
  int dev = 0, major = 0, minor = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  return (major == 10 && minor == 0) ? 0 : -2;
}

#ifdef MONET_DEBUG
// debug build only (libmonet_b200_dbg.so; not in include/monet_b200.h): the bf16x3 splitters
// dump the raw operands they consume ([rows][K padded to 64]); per-role wait counters
void monet_debug_dump(float* a_dump, float* b_dump) {
  g_dbg_a = a_dump;
  g_dbg_b = b_dump;
}

void monet_debug_timers(unsigned long long* counters) { g_dbg_t = counters; }
#endif

int monet_copy_async(void* dst, const void* src, size_t bytes, void* stream) {
  if (bytes == 0) return 0;
  cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, S(stream));
  return e == cudaSuccess ? 0 : -static_cast<int>(e);
}

// ------------------------------------------------------------------- conv
size_t monet_conv_ws_bytes(int variant, int pass, const monet_conv_desc* d) {
  if (check_desc(d)) return 0;
  if (pass == MONET_PASS_FWD) {
    const FView f = fprop_view(variant, d);
    if (f.on) return f.pad_bytes + f.w_bytes;
  }
  if (pass == MONET_PASS_BWD)
    return std::max(monet_conv_ws_bytes(variant, MONET_PASS_DGRAD, d), monet_conv_ws_bytes(variant, MONET_PASS_WGRAD, d));
  if (pass == MONET_PASS_DGRAD && use_phases(variant, d)) return 0;  // phase GEMMs never split K
  GemmParams p = conv_params(pass, d, nullptr, nullptr, nullptr);
  if (pass == MONET_PASS_WGRAD) {
    const WView v = wgrad_view(variant, d);
    if (v.on) return align256(gemm_ws(variant, p.M, p.N, (int)v.kd, v.n_pitch)) + v.pad_bytes;
  }
  return gemm_ws(variant, p.M, p.N, p.Kd);
}

static int conv_fwd_impl(int variant, const monet_conv_desc* d, const float* x, const float* w, const uint16_t* w_hi,
                         const uint16_t* w_lo, float* y, void* ws, size_t ws_bytes, void* stream,
                         float* stats = nullptr, int* stats_done = nullptr) {
  if (stats_done) *stats_done = 0;
  if (int e = check_desc(d)) return e;
  const FView f = fprop_view(variant, d);
  if (f.on && ws != nullptr && ws_bytes >= f.pad_bytes + f.w_bytes && tma_available()) {
    float* xp = static_cast<float*>(ws);
    float* wp = reinterpret_cast<float*>(static_cast<char*>(ws) + f.pad_bytes);
    const int hp = (d->p - 1) * d->stride_h + d->r, wpx = (d->q - 1) * d->stride_w + d->s;
    wgrad_pad_kernel<<<ew_blocks((long long)d->n * hp * wpx * (d->c / 4)), kEwThreads, 0, S(stream)>>>(
        x, xp, d->n, d->h, d->w, d->c, hp, wpx, d->pad_h, d->pad_w);
    fview_weight_kernel<<<(d->k * d->r * 32 + 255) / 256, 256, 0, S(stream)>>>(w, wp, d->k, d->r, d->s, d->c);
    GemmParams p{};
    p.g = geom(d);
    p.fv_q = BM;
    p.M = d->n * d->p * BM;
    p.N = d->k;
    p.Kd = d->r * 32;
    p.a = op_gather(OP_IM2COL_FPROP, xp, p.M);
    p.b = op_kmajor(wp, d->k, p.Kd, p.Kd);
    p.c = y;
    p.ldc = d->k;
    return launch_gemm(p, MONET_CONV_IMPLICIT, 0, nullptr, 0, S(stream));
  }
  GemmParams p = conv_params(MONET_PASS_FWD, d, x, w, y);
  p.stats = stats;
  p.stats_done = stats_done;
  return launch_gemm_w16(p, w_hi, w_lo, variant, 0, ws, ws_bytes, S(stream));
}

int monet_conv_fwd(int variant, const monet_conv_desc* d, const float* x, const float* w, float* y, void* ws,
                   size_t ws_bytes, void* stream) {
  return conv_fwd_impl(variant, d, x, w, nullptr, nullptr, y, ws, ws_bytes, stream);
}

static int bn_blocks(int64_t rows);

static int conv_fwd_bias_impl(int variant, const monet_conv_desc* d, const float* x, const float* w,
                              const uint16_t* w_hi, const uint16_t* w_lo, const float* bias, float* y, void* ws,
                              size_t ws_bytes, void* stream, float* stats = nullptr, int* stats_done = nullptr) {
  if (stats_done) *stats_done = 0;
  if (int e = check_desc(d)) return e;
  GemmParams p = conv_params(MONET_PASS_FWD, d, x, w, y);
  if (uses_bx3(variant)) {  // bias added in the epilogue (or the split-K reduce)
    p.bias = bias;
    p.stats = stats;
    p.stats_done = stats_done;
    return launch_gemm_w16(p, w_hi, w_lo, variant, 0, ws, ws_bytes, S(stream));
  }
  const long long tot = (long long)p.M * p.N;
  bias_fill_kernel<<<(int)((tot + 255) / 256), 256, 0, S(stream)>>>(y, bias, p.M, p.N);
  return launch_gemm(p, variant, 1, ws, ws_bytes, S(stream));
}

int monet_conv_fwd_bias(int variant, const monet_conv_desc* d, const float* x, const float* w, const float* bias,
                        float* y, void* ws, size_t ws_bytes, void* stream) {
  return conv_fwd_bias_impl(variant, d, x, w, nullptr, nullptr, bias, y, ws, ws_bytes, stream);
}

int monet_conv_fwd_w16(int variant, const monet_conv_desc* d, const float* x, const float* w, const uint16_t* w_hi,
                       const uint16_t* w_lo, const float* bias, float* y, void* ws, size_t ws_bytes, void* stream) {
  if (bias != nullptr) return conv_fwd_bias_impl(variant, d, x, w, w_hi, w_lo, bias, y, ws, ws_bytes, stream);
  return conv_fwd_impl(variant, d, x, w, w_hi, w_lo, y, ws, ws_bytes, stream);
}

// ------------------------------------------------------- conv -> BN statistics
// Per-tile (128-row) BN statistics of a conv output [M][K]: (mean, M2) per channel
// ([T][2][K], T = ceil(M / 128)), computed in the GEMM epilogue when the tile is final in
// one chain, else by tile_stats_kernel over y (pivot = the tile's first row).  The BN
// forward then merges the tiles (bn_tile_merge -> bn_finalize_tiles, Chan's formula in fp64,
// fixed order) instead of re-reading the conv output.
static long long conv_rows(const monet_conv_desc* d) { return (long long)d->n * d->p * d->q; }
static long long stat_tiles(long long rows) { return (rows + 127) / 128; }

// one 128-row tile per block: thread t takes channel quad t % (C/4) (BnLayout) and every rpi-th
// row, four rows in flight; sums around the tile's first row (a common pivot), combined in smem
// 128-row tiles, a grid-stride loop of blocks over them: thread t takes channel quad t % (C/4)
// (BnLayout) and every rpi-th row, four rows in flight; sums around the tile's first row (a
// common pivot), combined in smem
__global__ void tile_stats_kernel(const float* __restrict__ y, long long M, int N, float* stats) {
  const BnLayout L = bn_layout(N);
  const long long T = (M + 127) / 128;
  const int rsub = threadIdx.x / L.tpr, qb = threadIdx.x % L.tpr;
  __shared__ float red[2][kEwThreads * 4];
  for (long long tile = blockIdx.x; tile < T; tile += gridDim.x) {
    const long long r0 = tile * 128;
    const int cnt = (int)min(128LL, M - r0);
    for (int qi = 0; qi < L.qpt; ++qi) {
      const int q = qb + qi * L.tpr;
      float s1[4] = {0.f, 0.f, 0.f, 0.f}, s2[4] = {0.f, 0.f, 0.f, 0.f};
      float4 piv = make_float4(0.f, 0.f, 0.f, 0.f);
      if (q < N / 4) piv = *reinterpret_cast<const float4*>(y + r0 * N + 4 * q);
      if (rsub < L.rpi && q < N / 4) {
        auto acc = [&](const float4& v) {
          const float d0 = v.x - piv.x, d1 = v.y - piv.y, d2 = v.z - piv.z, d3 = v.w - piv.w;
          s1[0] += d0; s1[1] += d1; s1[2] += d2; s1[3] += d3;
          s2[0] += d0 * d0; s2[1] += d1 * d1; s2[2] += d2 * d2; s2[3] += d3 * d3;
        };
        int r = rsub;
        for (; r + 7 * L.rpi < cnt; r += 8 * L.rpi) {
          float4 v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) v[u] = *reinterpret_cast<const float4*>(y + (r0 + r + u * L.rpi) * N + 4 * q);
#pragma unroll
          for (int u = 0; u < 8; ++u) acc(v[u]);
        }
        for (; r < cnt; r += L.rpi) acc(*reinterpret_cast<const float4*>(y + (r0 + r) * N + 4 * q));
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        red[0][threadIdx.x * 4 + j] = s1[j];
        red[1][threadIdx.x * 4 + j] = s2[j];
      }
      __syncthreads();
      if (rsub == 0 && q < N / 4) {
        const float pv[4] = {piv.x, piv.y, piv.z, piv.w};
        for (int j = 0; j < 4; ++j) {
          float a1 = 0.f, a2 = 0.f;
          for (int k = 0; k < L.rpi; ++k) {
            a1 += red[0][(k * L.tpr + qb) * 4 + j];
            a2 += red[1][(k * L.tpr + qb) * 4 + j];
          }
          stats[(tile * 2) * N + 4 * q + j] = pv[j] + a1 / cnt;
          stats[(tile * 2 + 1) * N + 4 * q + j] = fmaxf(a2 - a1 * a1 / cnt, 0.f);
        }
      }
      __syncthreads();
    }
  }
}

struct Welford {
  double n, mean, m2;
};
__device__ __forceinline__ Welford chan_merge(Welford a, Welford b) {
  if (b.n == 0.0) return a;
  if (a.n == 0.0) return b;
  const double n = a.n + b.n, delta = b.mean - a.mean;
  return Welford{n, a.mean + delta * (b.n / n), a.m2 + b.m2 + delta * delta * (a.n * b.n / n)};
}

// groups of 32 tiles x 32 channels per block: warp w merges tiles 4w..4w+3 (lane = channel,
// coalesced), warp 0 merges the 8 warps in order -> part[g] = (n, mean, M2) in fp64
__global__ void bn_tile_merge_kernel(const float* __restrict__ stats, long long T, long long M, int C,
                                     double* part) {
  __shared__ double sm[8][3][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.y * 32 + lane;
  Welford acc{0.0, 0.0, 0.0};
  if (c < C) {
    for (int i = 0; i < 4; ++i) {
      const long long t = (long long)blockIdx.x * 32 + warp * 4 + i;
      if (t >= T) break;
      const double cnt = (double)min(128LL, M - t * 128);
      acc = chan_merge(acc, Welford{cnt, (double)stats[(t * 2) * C + c], (double)stats[(t * 2 + 1) * C + c]});
    }
  }
  sm[warp][0][lane] = acc.n;
  sm[warp][1][lane] = acc.mean;
  sm[warp][2][lane] = acc.m2;
  __syncthreads();
  if (warp == 0 && c < C) {
    Welford a{0.0, 0.0, 0.0};
    for (int w = 0; w < 8; ++w) a = chan_merge(a, Welford{sm[w][0][lane], sm[w][1][lane], sm[w][2][lane]});
    part[((long long)blockIdx.x * 3) * C + c] = a.n;
    part[((long long)blockIdx.x * 3 + 1) * C + c] = a.mean;
    part[((long long)blockIdx.x * 3 + 2) * C + c] = a.m2;
  }
}

// one warp per channel: lanes merge groups lane, lane+32, ... then a fixed xor tree (lower lane
// first) -> mean, invstd, running statistics
__global__ void bn_finalize_tiles_kernel(const double* __restrict__ part, long long G, long long rows, int C,
                                         float eps, float momentum, int update_running, float* mean_out,
                                         float* invstd_out, float* running_mean, float* running_var) {
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (c >= C) return;
  Welford a{0.0, 0.0, 0.0};
  for (long long g = lane; g < G; g += 32)
    a = chan_merge(a, Welford{part[(g * 3) * C + c], part[(g * 3 + 1) * C + c], part[(g * 3 + 2) * C + c]});
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const Welford b{__shfl_xor_sync(0xffffffffu, a.n, o), __shfl_xor_sync(0xffffffffu, a.mean, o),
                    __shfl_xor_sync(0xffffffffu, a.m2, o)};
    a = (lane & o) ? chan_merge(b, a) : chan_merge(a, b);
  }
  if (lane != 0) return;
  double var = a.m2 / (double)rows;
  if (var < 0.0) var = 0.0;
  mean_out[c] = (float)a.mean;
  invstd_out[c] = (float)(1.0 / sqrt(var + (double)eps));
  if (update_running) {
    const double unbiased = rows > 1 ? a.m2 / (double)(rows - 1) : var;
    running_mean[c] = (float)((1.0 - momentum) * running_mean[c] + momentum * a.mean);
    running_var[c] = (float)((1.0 - momentum) * running_var[c] + momentum * unbiased);
  }
}

size_t monet_conv_stats_bytes(const monet_conv_desc* d) {
  if (!d) return 0;
  const long long T = stat_tiles(conv_rows(d)), G = (T + 31) / 32;
  return align256((size_t)T * 2 * d->k * sizeof(float)) + align256((size_t)G * 3 * d->k * sizeof(double));
}

int monet_conv_fwd_w16_stats(int variant, const monet_conv_desc* d, const float* x, const float* w,
                             const uint16_t* w_hi, const uint16_t* w_lo, const float* bias, float* y, void* stats,
                             void* ws, size_t ws_bytes, void* stream) {
  if (!stats) return -(int)cudaErrorInvalidValue;
  float* st = static_cast<float*>(stats);
  int fused = 0;
  const int e = bias != nullptr
                    ? conv_fwd_bias_impl(variant, d, x, w, w_hi, w_lo, bias, y, ws, ws_bytes, stream, st, &fused)
                    : conv_fwd_impl(variant, d, x, w, w_hi, w_lo, y, ws, ws_bytes, stream, st, &fused);
  if (e) return e;
  if (!fused)  // split-K, chunked chains or the fp32-weight path: one pass over y
    tile_stats_kernel<<<(int)std::min<long long>(stat_tiles(conv_rows(d)), 8LL * kNumSMs), kEwThreads, 0, S(stream)>>>(
        y, conv_rows(d), d->k, st);
  return last_error();
}

int monet_bn_stats_finalize(const void* stats, int64_t rows, int c, float eps, float momentum, int update_running,
                            float* mean, float* invstd, float* running_mean, float* running_var, void* stream) {
  if (!stats || rows <= 0 || c <= 0) return -(int)cudaErrorInvalidValue;
  const long long T = stat_tiles(rows), G = (T + 31) / 32;
  const float* st = static_cast<const float*>(stats);
  double* part = reinterpret_cast<double*>(static_cast<char*>(const_cast<void*>(stats)) +
                                           align256((size_t)T * 2 * c * sizeof(float)));
  bn_tile_merge_kernel<<<dim3((unsigned)G, (c + 31) / 32), 256, 0, S(stream)>>>(st, T, rows, c, part);
  bn_finalize_tiles_kernel<<<(c + 7) / 8, 256, 0, S(stream)>>>(part, G, rows, c, eps, momentum, update_running, mean,
                                                               invstd, running_mean, running_var);
  return last_error();
}

int monet_split_bf16(const float* src, uint16_t* hi, uint16_t* lo, int64_t n, void* stream) {
  if (n < 0) return -(int)cudaErrorInvalidValue;
  if (n == 0) return 0;
  split_bf16_kernel<<<ew_blocks(n), kEwThreads, 0, S(stream)>>>(src, hi, lo, n);
  return last_error();
}

int monet_split_bf16_segments(const float* src, uint16_t* hi, uint16_t* lo, const int64_t* table, int nseg,
                              int64_t max_count, void* stream) {
  if (nseg < 0 || nseg > 65535 || max_count < 0) return -(int)cudaErrorInvalidValue;
  if (nseg == 0 || max_count == 0) return 0;
  const int bx = (int)std::min<int64_t>((max_count + kEwThreads - 1) / kEwThreads, 8 * kNumSMs / std::max(1, nseg / 8 + 1));
  split_bf16_segments_kernel<<<dim3(std::max(bx, 1), nseg), kEwThreads, 0, S(stream)>>>(
      src, hi, lo, reinterpret_cast<const long long*>(table));
  return last_error();
}

int monet_bias_grad(const float* dy, float* db, int64_t rows, int c, int accumulate, void* scratch, void* stream) {
  if (c % 4 || rows <= 0) return -(int)cudaErrorInvalidValue;
  cudaStream_t st = S(stream);
  float* ws = static_cast<float*>(scratch);
  const int nb = bn_blocks(rows);
  bn_reduce_kernel<<<nb, kEwThreads, 0, st>>>(0, dy, nullptr, nullptr, nullptr, rows, c, ws);
  chan_sum_finalize_kernel<<<(c + 7) / 8, 256, 0, st>>>(ws, nb, c, db, accumulate);
  return last_error();
}

// thr = floor(p * 2^24); p in [0, 1)
static unsigned dropout_thr(float p) { return (unsigned)((double)p * 16777216.0); }

int monet_dropout_fwd(const float* x, float* y, int64_t n, float p, const unsigned long long* seed, uint64_t salt,
                      void* stream) {
  if (!(p >= 0.f && p < 1.f) || n < 0) return -(int)cudaErrorInvalidValue;
  if (n == 0) return 0;
  dropout_kernel<<<ew_blocks(n), kEwThreads, 0, S(stream)>>>(x, y, n, dropout_thr(p), (float)(1.0 / (1.0 - p)),
                                                              seed, salt, 0);
  return last_error();
}

int monet_dropout_bwd(const float* dy, float* dx, int64_t n, float p, const unsigned long long* seed, uint64_t salt,
                      int accumulate, void* stream) {
  if (!(p >= 0.f && p < 1.f) || n < 0) return -(int)cudaErrorInvalidValue;
  if (n == 0) return 0;
  dropout_kernel<<<ew_blocks(n), kEwThreads, 0, S(stream)>>>(dy, dx, n, dropout_thr(p), (float)(1.0 / (1.0 - p)),
                                                              seed, salt, accumulate);
  return last_error();
}

int monet_seed_advance(unsigned long long* seed, void* stream) {
  seed_advance_kernel<<<1, 1, 0, S(stream)>>>(seed);
  return last_error();
}

static int conv_dgrad_impl(int variant, const monet_conv_desc* d, const float* dy, const float* w,
                           const uint16_t* w_hi, const uint16_t* w_lo, float* dx, int accumulate, void* ws,
                           size_t ws_bytes, void* stream) {
  if (int e = check_desc(d)) return e;
  if (use_phases(variant, d)) {  // stride > 1: one stride-1 GEMM per output parity class
    for (int a = 0; a < d->stride_h; ++a)
      for (int b = 0; b < d->stride_w; ++b) {
        PhaseInfo ph;
        if (!make_phase(d, a, b, ph)) continue;  // no dx pixels of this parity
        if (ph.ntap == 0) {                      // pixels no tap reaches: zero gradient
          if (!accumulate)
            dgrad_phase_zero_kernel<<<ew_blocks((long long)d->n * ph.Hp * ph.Wp * d->c / 4), kEwThreads, 0,
                                      S(stream)>>>(dx, d->n, d->h, d->w, d->c, a, b, d->stride_h, d->stride_w);
          continue;
        }
        if (int e = launch_gemm_w16(phase_params(d, ph, dy, w, dx), w_hi, w_lo, variant, accumulate, ws, ws_bytes,
                                    S(stream)))
          return e;
      }
    return last_error();
  }
  return launch_gemm_w16(conv_params(MONET_PASS_DGRAD, d, dy, w, dx), w_hi, w_lo, variant, accumulate, ws, ws_bytes,
                         S(stream));
}

int monet_conv_dgrad(int variant, const monet_conv_desc* d, const float* dy, const float* w, float* dx,
                     int accumulate, void* ws, size_t ws_bytes, void* stream) {
  return conv_dgrad_impl(variant, d, dy, w, nullptr, nullptr, dx, accumulate, ws, ws_bytes, stream);
}

int monet_conv_dgrad_w16(int variant, const monet_conv_desc* d, const float* dy, const float* w, const uint16_t* w_hi,
                         const uint16_t* w_lo, float* dx, int accumulate, void* ws, size_t ws_bytes, void* stream) {
  return conv_dgrad_impl(variant, d, dy, w, w_hi, w_lo, dx, accumulate, ws, ws_bytes, stream);
}

int monet_conv_wgrad(int variant, const monet_conv_desc* d, const float* x, const float* dy, float* dw,
                     int accumulate, void* ws, size_t ws_bytes, void* stream) {
  if (int e = check_desc(d)) return e;
  const WView v = wgrad_view(variant, d);
  if (!v.on && wgrad_swapped(variant, d))
    return launch_gemm(wgrad_swapped_params(d, x, dy, dw), variant, accumulate, ws, ws_bytes, S(stream));
  GemmParams p = conv_params(MONET_PASS_WGRAD, d, x, dy, dw);
  if (v.on) {
    const size_t part = align256(gemm_ws(variant, p.M, p.N, (int)v.kd, v.n_pitch));
    // a workspace without room for the padded input (callers sizing it by hand) takes the gather path
    if (ws != nullptr && ws_bytes >= part + v.pad_bytes && tma_available()) {
      float* xp = reinterpret_cast<float*>(static_cast<char*>(ws) + part);
      const int hp = (d->p - 1) * d->stride_h + d->r, wp = (d->q - 1) * d->stride_w + d->s;
      wgrad_pad_kernel<<<ew_blocks((long long)d->n * hp * wp * (d->c / 4)), kEwThreads, 0, S(stream)>>>(
          x, xp, d->n, d->h, d->w, d->c, hp, wp, d->pad_h, d->pad_w);
      p.Kd = (int)v.kd;
      p.b.ptr = xp;
      p.wv_q = v.qpad;
      p.n_pitch = v.n_pitch;
      return launch_gemm(p, variant, accumulate, ws, part, S(stream));
    }
  }
  return launch_gemm(p, variant, accumulate, ws, ws_bytes, S(stream));
}

// ------------------------------------------------------------------- linear
size_t monet_linear_ws_bytes(int variant, int pass, int n, int in_f, int out_f) {
  if (pass == MONET_PASS_FWD) return gemm_ws(variant, n, out_f, in_f);
  return std::max(gemm_ws(variant, n, in_f, out_f), gemm_ws(variant, out_f, in_f, n));
}

int monet_linear_fwd(int variant, const float* x, const float* w, const float* b, float* y, int n, int in_f,
                     int out_f, void* ws, size_t ws_bytes, void* stream) {
  cudaStream_t st = S(stream);
  long long tot = (long long)n * out_f;
  bias_fill_kernel<<<(int)((tot + 255) / 256), 256, 0, st>>>(y, b, n, out_f);
  GemmParams p{};
  p.M = n;
  p.N = out_f;
  p.Kd = in_f;
  p.a = op_kmajor(x, n, in_f, in_f);
  p.b = op_kmajor(w, out_f, in_f, in_f);
  p.c = y;
  p.ldc = out_f;
  return launch_gemm(p, variant, 1, ws, ws_bytes, st);
}

int monet_linear_bwd(int variant, const float* x, const float* w, const float* dy, float* dx, int dx_accumulate,
                     float* dw, float* db, int n, int in_f, int out_f, void* ws, size_t ws_bytes, void* stream) {
  cudaStream_t st = S(stream);
  if (dx) {
    GemmParams p{};
    p.M = n;
    p.N = in_f;
    p.Kd = out_f;
    p.a = op_kmajor(dy, n, out_f, out_f);
    p.b = op_mnmajor(w, in_f, in_f);  // B[i, o] = W[o, i]
    p.c = dx;
    p.ldc = in_f;
    if (int e = launch_gemm(p, variant, dx_accumulate, ws, ws_bytes, st)) return e;
  }
  GemmParams q{};
  q.M = out_f;
  q.N = in_f;
  q.Kd = n;
  q.a = op_mnmajor(dy, out_f, out_f);  // A[o, n] = dy[n, o]
  q.b = op_mnmajor(x, in_f, in_f);     // B[i, n] = x[n, i]
  q.c = dw;
  q.ldc = in_f;
  if (int e = launch_gemm(q, variant, 0, ws, ws_bytes, st)) return e;
  col_sum_kernel<<<(out_f + 255) / 256, 256, 0, st>>>(dy, db, n, out_f);
  return last_error();
}

// ------------------------------------------------------------------- generic GEMM
size_t monet_gemm_ws_bytes(int variant, int m, int n, int k) { return gemm_ws(variant, m, n, k); }

int monet_gemm(int variant, const float* a, int a_mn, int64_t lda, const float* b, int b_mn, int64_t ldb, float* c,
               int64_t ldc, int m, int n, int k, int accumulate, void* ws, size_t ws_bytes, void* stream) {
  GemmParams p{};
  p.M = m;
  p.N = n;
  p.Kd = k;
  p.a = a_mn ? op_mnmajor(a, m, lda) : op_kmajor(a, m, lda, k);
  p.b = b_mn ? op_mnmajor(b, n, ldb) : op_kmajor(b, n, ldb, k);
  p.c = c;
  p.ldc = ldc;
  return launch_gemm(p, variant, accumulate, ws, ws_bytes, S(stream));
}

// ------------------------------------------------------------------- ReLU
int monet_relu_fwd(const float* x, float* y, uint32_t* mask, int64_t n, void* stream) {
  relu_fwd_kernel<false><<<ew_blocks((n + 7) / 8), kEwThreads, 0, S(stream)>>>(x, y, mask, n);
  return last_error();
}
int monet_relu_bwd_mask(const uint32_t* mask, const float* dy, float* dx, int64_t n, int accumulate, void* stream) {
  relu_bwd_mask_kernel<<<ew_blocks((n + 7) / 8), kEwThreads, 0, S(stream)>>>(mask, dy, dx, n, accumulate);
  return last_error();
}
int monet_relu_bwd_out(const float* y, const float* dy, float* dx, int64_t n, int accumulate, void* stream) {
  relu_bwd_sign_kernel<false><<<ew_blocks(n / 4 + 1), kEwThreads, 0, S(stream)>>>(y, dy, dx, n, accumulate);
  return last_error();
}
int monet_relu_bwd_in(const float* x, const float* dy, float* dx, int64_t n, int accumulate, void* stream) {
  return monet_relu_bwd_out(x, dy, dx, n, accumulate, stream);
}

// ReLU6 (hardtanh(0, 6)): the mask bit is the gradient gate 0 < x < 6, so the
// backward from the mask is monet_relu_bwd_mask; from the output or the input
// the gate is the same test.
int monet_relu6_fwd(const float* x, float* y, uint32_t* mask, int64_t n, void* stream) {
  relu_fwd_kernel<true><<<ew_blocks((n + 7) / 8), kEwThreads, 0, S(stream)>>>(x, y, mask, n);
  return last_error();
}
int monet_relu6_bwd_out(const float* y, const float* dy, float* dx, int64_t n, int accumulate, void* stream) {
  relu_bwd_sign_kernel<true><<<ew_blocks(n / 4 + 1), kEwThreads, 0, S(stream)>>>(y, dy, dx, n, accumulate);
  return last_error();
}
int monet_relu6_bwd_in(const float* x, const float* dy, float* dx, int64_t n, int accumulate, void* stream) {
  return monet_relu6_bwd_out(x, dy, dx, n, accumulate, stream);
}

// ------------------------------------------------------------ concat slices
int monet_channel_copy(const float* src, int src_c, int src_off, float* dst, int dst_c, int dst_off, int count,
                       int64_t pixels, int accumulate, void* stream) {
  if (count % 4 || src_c % 4 || dst_c % 4 || src_off % 4 || dst_off % 4 || src_off + count > src_c ||
      dst_off + count > dst_c)
    return -(int)cudaErrorInvalidValue;
  if (pixels == 0 || count == 0) return 0;
  channel_copy_kernel<<<ew_blocks(pixels * (count / 4)), kEwThreads, 0, S(stream)>>>(src, src_c, src_off, dst, dst_c,
                                                                                      dst_off, count, pixels,
                                                                                      accumulate);
  return last_error();
}

// ------------------------------------------------------------ depthwise conv
static int dw_check(const monet_conv_desc* d) {
  if (!d || d->c % 4 || d->k != d->c || d->r * d->s > kDwMaxTaps || d->n <= 0) return -(int)cudaErrorInvalidValue;
  return 0;
}
static int dw_blocks(const monet_conv_desc* d) {
  const long long rows = (long long)d->n * d->p * d->q;
  return (int)std::max(1LL, std::min((rows + 63) / 64, (long long)kNumSMs * 4));
}
// shared-memory tiled kernels (csrc/dwconv.cuh): channel slabs of 16, staged window <= 200 KB
constexpr size_t kDwSmemMax = 200 * 1024;
static size_t dw_fwd_smem(const monet_conv_desc* d, int rows = kDwRows) {
  const int nr = (rows - 1) * d->stride_h + d->r, nc = (d->q - 1) * d->stride_w + d->s;
  return (size_t)nr * nc * kDwSlab * sizeof(float);
}
static size_t dw_dgrad_smem(const monet_conv_desc* d, int rows = kDwRows) {
  const int nr = (rows + d->r - 1) / d->stride_h + 2, nc = (d->w + d->s - 1) / d->stride_w + 2;
  return (size_t)nr * nc * kDwSlab * sizeof(float);
}
static size_t dw_wgrad_band_bytes(const monet_conv_desc* d) {  // one staged band (odd x pitch)
  const int nr = (kDwRows - 1) * d->stride_h + d->r, nc = ((d->q - 1) * d->stride_w + d->s) | 1;
  return (size_t)(nr * nc + kDwRows * d->q) * kDwSlab * sizeof(float);
}
// bands staged per barrier round by the 3x3 row walker (up to 32 KB of staging per round)
static int dw_wgrad_kb(const monet_conv_desc* d) {
  return (int)std::max<size_t>(1, std::min<size_t>(8, (32 << 10) / dw_wgrad_band_bytes(d)));
}
static size_t dw_wgrad_smem(const monet_conv_desc* d) {  // staged bands, or the final reduction
  return std::max(dw_wgrad_band_bytes(d) * dw_wgrad_kb(d), (size_t)256 * 3 * sizeof(float4));
}
static bool dw_tiled(const monet_conv_desc* d) {
  return d->c % kDwSlab == 0 && dw_fwd_smem(d) <= kDwSmemMax && dw_dgrad_smem(d) <= kDwSmemMax &&
         dw_wgrad_smem(d) <= kDwSmemMax;
}
// output rows per fwd / dgrad CTA: about `pix` output pixels (whole images for the 7x7 and 14x14
// layers, whose 4-row CTAs were launch- and halo-bound), at least kDwRows, with the staged window
// under `cap` bytes so 5+ CTAs stay resident (measured per MobileNet-V2 shape: tools/dw_bench.py)
static int dw_rows(const monet_conv_desc* d, bool trans) {
  const int oh = trans ? d->h : d->p, ow = trans ? d->w : d->q;
  const int pix = trans ? 1024 : 448;
  const size_t cap = trans ? 40 << 10 : 32 << 10;
  int rows = std::min(oh, std::max(kDwRows, (pix + ow - 1) / ow));
  while (rows > kDwRows && (trans ? dw_dgrad_smem(d, rows) : dw_fwd_smem(d, rows)) > cap) --rows;
  return std::max(1, std::min(oh, rows));
}
// 1 / 2: the 3x3 stride-1 / stride-2 specialisations; 0: runtime geometry
static int dw_kind(const monet_conv_desc* d) {
  if (d->r != 3 || d->s != 3 || d->stride_h != d->stride_w) return 0;
  return (d->stride_h == 1 || d->stride_h == 2) ? d->stride_h : 0;
}
}  // extern "C"
namespace {
template <bool kTrans>
void dw_launch(const monet_conv_desc* d, dim3 grid, size_t smem, const float* src, const float* w, float* out,
               int accumulate, cudaStream_t st, int flip = 0) {
  static bool attr = false;  // the three specialisations share a signature: set all of them once
  if (!attr) {
    for (auto kern : {dwconv_tile_kernel<kTrans, 0>, dwconv_tile_kernel<kTrans, 1>, dwconv_tile_kernel<kTrans, 2>})
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDwSmemMax);
    attr = true;
  }
  const int rows = dw_rows(d, kTrans);
  auto run = [&](auto kern) { kern<<<grid, 256, smem, st>>>(src, w, out, geom(d), accumulate, rows, flip); };
  const int k = dw_kind(d);
  if (k == 1)
    run(dwconv_tile_kernel<kTrans, 1>);
  else if (k == 2)
    run(dwconv_tile_kernel<kTrans, 2>);
  else
    run(dwconv_tile_kernel<kTrans, 0>);
}
}  // namespace
extern "C" {
static int dw_tile_nb(const monet_conv_desc* d) {  // band walkers per channel slab (wgrad)
  const int bands = d->n * ((d->p + kDwRows - 1) / kDwRows);
  return std::max(1, std::min(bands, kNumSMs * 4 / std::max(1, d->c / kDwSlab)));
}
size_t monet_dwconv_ws_bytes(const monet_conv_desc* d) {
  if (dw_check(d)) return 0;
  const int nb = dw_tiled(d) ? dw_tile_nb(d) : dw_blocks(d);
  return (size_t)nb * d->r * d->s * d->c * sizeof(float);
}
int monet_dwconv_fwd(const monet_conv_desc* d, const float* x, const float* w, float* y, void* stream) {
  if (int e = dw_check(d)) return e;
  if (dw_tiled(d)) {
    const int rows = dw_rows(d, false);
    dim3 grid(d->c / kDwSlab, (d->p + rows - 1) / rows, d->n);
    dw_launch<false>(d, grid, dw_fwd_smem(d, rows), x, w, y, 0, S(stream));
    return last_error();
  }
  const long long total = (long long)d->n * d->p * d->q * (d->c / 4);
  dwconv_fwd_kernel<<<ew_blocks(total), kEwThreads, 0, S(stream)>>>(x, w, y, geom(d));
  return last_error();
}
int monet_dwconv_dgrad(const monet_conv_desc* d, const float* dy, const float* w, float* dx, int accumulate,
                       void* stream) {
  if (int e = dw_check(d)) return e;
  if (dw_tiled(d) && dw_kind(d) == 1) {
    // stride 1: dx is the forward conv of dy with the rotated filter and padding R-1-pad, which runs on
    // the forward kernel's tighter staging (tools/dw_bench.py: 56x56 404 -> ~330 us)
    monet_conv_desc e = *d;
    e.h = d->p, e.w = d->q, e.p = d->h, e.q = d->w;
    e.pad_h = d->r - 1 - d->pad_h, e.pad_w = d->s - 1 - d->pad_w;
    if (dw_tiled(&e) && dw_kind(&e) == 1) {
      const int rows = dw_rows(&e, false);
      dim3 grid(e.c / kDwSlab, (e.p + rows - 1) / rows, e.n);
      dw_launch<false>(&e, grid, dw_fwd_smem(&e, rows), dy, w, dx, accumulate, S(stream), 1);
      return last_error();
    }
  }
  if (dw_tiled(d)) {
    const int rows = dw_rows(d, true);
    dim3 grid(d->c / kDwSlab, (d->h + rows - 1) / rows, d->n);
    dw_launch<true>(d, grid, dw_dgrad_smem(d, rows), dy, w, dx, accumulate, S(stream));
    return last_error();
  }
  const long long total = (long long)d->n * d->h * d->w * (d->c / 4);
  dwconv_dgrad_kernel<<<ew_blocks(total), kEwThreads, 0, S(stream)>>>(dy, w, dx, geom(d), accumulate);
  return last_error();
}
int monet_dwconv_wgrad(const monet_conv_desc* d, const float* x, const float* dy, float* dw, void* ws,
                       size_t ws_bytes, void* stream) {
  if (int e = dw_check(d)) return e;
  if (ws == nullptr || ws_bytes < monet_dwconv_ws_bytes(d)) return -(int)cudaErrorInvalidValue;
  const int taps = d->r * d->s;
  float* part = static_cast<float*>(ws);
  int nb;
  if (dw_tiled(d)) {
    nb = dw_tile_nb(d);
    const dim3 grid(d->c / kDwSlab, nb);
    const int k = dw_kind(d);
    static bool attr = false;  // all three specialisations at once (shared signature)
    if (!attr) {
      for (auto kern : {dwconv_wgrad_tile_kernel<0>, dwconv_wgrad_tile_kernel<1>, dwconv_wgrad_tile_kernel<2>})
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDwSmemMax);
      for (auto kern : {dwconv_wgrad_rows_kernel<1, false>, dwconv_wgrad_rows_kernel<2, false>,
                        dwconv_wgrad_rows_kernel<1, true>, dwconv_wgrad_rows_kernel<2, true>})
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDwSmemMax);
      attr = true;
    }
    const size_t smem = dw_wgrad_smem(d);
    // row walker for rows >= 56 wide (it reads a third of the shared memory, which bounds those);
    // the per-tap walker below that, where the band staging latency dominates (tools/dw_bench.py)
    // per row width (tools/dw_bench.py, MobileNet-V2 b272): input rows <= 14 wide -> row walker staging
    // kb bands per barrier at 4 CTAs / SM (latency-bound: ~60 bands per walker); outputs up to 55 wide
    // -> the per-tap walker; >= 56 -> row walker, one band per round (shared-memory-read bound)
    const bool narrow = d->q * d->stride_w <= 14;  // 7x7 / 14x14 outputs of stride 1, 7x7 of stride 2
    const int kb = narrow ? dw_wgrad_kb(d) : 1;
    const auto args = [&](auto kern) { kern<<<grid, 256, smem, S(stream)>>>(x, dy, part, geom(d), nb, kb); };
    if (k == 1 && narrow)
      args(dwconv_wgrad_rows_kernel<1, true>);
    else if (k == 2 && narrow)
      args(dwconv_wgrad_rows_kernel<2, true>);
    else if (k == 1 && d->q < 56)
      dwconv_wgrad_tile_kernel<1><<<grid, 256, smem, S(stream)>>>(x, dy, part, geom(d), nb);
    else if (k == 2 && d->q < 56)
      dwconv_wgrad_tile_kernel<2><<<grid, 256, smem, S(stream)>>>(x, dy, part, geom(d), nb);
    else if (k == 1)
      args(dwconv_wgrad_rows_kernel<1, false>);
    else if (k == 2)
      args(dwconv_wgrad_rows_kernel<2, false>);
    else
      dwconv_wgrad_tile_kernel<0><<<grid, 256, smem, S(stream)>>>(x, dy, part, geom(d), nb);
  } else {
    nb = dw_blocks(d);
    dwconv_wgrad_partial_kernel<<<nb, kEwThreads, 0, S(stream)>>>(x, dy, part, geom(d));
  }
  dwconv_wgrad_final_kernel<<<(taps * d->c + 255) / 256, 256, 0, S(stream)>>>(part, nb, taps, d->c, dw);
  return last_error();
}

// ------------------------------------------------------------------- BatchNorm
static int bn_blocks(int64_t rows) {
  long long b = (rows + 255) / 256;
  return (int)std::max(1LL, std::min(b, (long long)kNumSMs * 4));
}

size_t monet_bn_scratch_bytes(int64_t rows, int c) {
  // partials [blocks][2][c] + coef_b[c] + coef_c[c] + inv_gamma[c] (bn_bwd_common)
  return ((size_t)bn_blocks(rows) * 2 * c + 3 * (size_t)c) * sizeof(float);
}

int monet_bn_fwd_train(const float* x, float* y, const float* gamma, const float* beta, float* saved_mean,
                       float* saved_invstd, float* running_mean, float* running_var, int64_t rows, int c, float eps,
                       float momentum, int update_running, void* scratch, void* stream) {
  if (c % 4) return -(int)cudaErrorInvalidValue;
  cudaStream_t st = S(stream);
  float* ws = static_cast<float*>(scratch);
  int nb = bn_blocks(rows);
  bn_reduce_kernel<<<nb, kEwThreads, 0, st>>>(7, x, nullptr, nullptr, nullptr, rows, c, ws);
  bn_finalize_fwd_kernel<<<(c + 7) / 8, 256, 0, st>>>(ws, nb, rows, c, eps, momentum, update_running, saved_mean,
                                                          saved_invstd, running_mean, running_var, x);
  bn_apply_kernel<<<ew_blocks(rows * c / 4), kEwThreads, 0, st>>>(x, y, saved_mean, saved_invstd, gamma, beta, rows,
                                                                  c);
  return last_error();
}

int monet_bn_fwd_replay(const float* x, float* y, const float* gamma, const float* beta, const float* saved_mean,
                        const float* saved_invstd, int64_t rows, int c, void* stream) {
  if (c % 4) return -(int)cudaErrorInvalidValue;
  bn_apply_kernel<<<ew_blocks(rows * c / 4), kEwThreads, 0, S(stream)>>>(x, y, saved_mean, saved_invstd, gamma, beta,
                                                                         rows, c);
  return last_error();
}

static int bn_bwd_common(const float* src, const float* dy, float* dx, int accumulate, const float* gamma,
                         const float* p0, const float* p1, const float* invstd, float* dgamma, float* dbeta,
                         int64_t rows, int c, int mode, float* ws, cudaStream_t st) {
  int nb = bn_blocks(rows);
  float* coef_b = ws + (size_t)nb * 2 * c;  // scratch layout: partials, coef_b[c], coef_c[c], inv_gamma[c]
  float* coef_c = coef_b + c;
  bn_reduce_kernel<<<nb, kEwThreads, 0, st>>>(mode, src, dy, p0, p1, rows, c, ws);
  bn_finalize_bwd_kernel<<<(c + 7) / 8, 256, 0, st>>>(ws, nb, c, rows, p0, p1, gamma, invstd, coef_b, coef_c, dgamma,
                                                      dbeta);
  bn_bwd_apply_kernel<<<ew_blocks(rows * c / 4), kEwThreads, 0, st>>>(src, dy, dx, gamma, invstd, coef_b, coef_c,
                                                                      rows, c, accumulate);
  return last_error();
}

int monet_bn_bwd_in(const float* x, const float* dy, float* dx, int accumulate, const float* gamma,
                    const float* saved_mean, const float* saved_invstd, float* dgamma, float* dbeta, int64_t rows,
                    int c, void* scratch, void* stream) {
  if (c % 4) return -(int)cudaErrorInvalidValue;
  return bn_bwd_common(x, dy, dx, accumulate, gamma, saved_mean, saved_invstd, saved_invstd, dgamma, dbeta, rows, c,
                       1, static_cast<float*>(scratch), S(stream));
}

int monet_bn_bwd_out(const float* y, const float* dy, float* dx, int accumulate, const float* gamma,
                     const float* beta, const float* saved_invstd, float* dgamma, float* dbeta, int64_t rows, int c,
                     void* scratch, void* stream) {
  if (c % 4) return -(int)cudaErrorInvalidValue;
  cudaStream_t st = S(stream);
  float* ws = static_cast<float*>(scratch);
  float* inv_gamma = ws + (size_t)bn_blocks(rows) * 2 * c + 2 * (size_t)c;
  bn_inv_gamma_kernel<<<(c + 255) / 256, 256, 0, st>>>(gamma, inv_gamma, c, 1e-12f);
  return bn_bwd_common(y, dy, dx, accumulate, gamma, beta, inv_gamma, saved_invstd, dgamma, dbeta, rows, c, 2, ws, st);
}

// ------------------------------------------------------------------- fused BN+ReLU (K9 / K10)
}  // extern "C"

namespace {
template <bool kSix>
int bnrelu_fwd_train(const float* x, float* z, const float* gamma, const float* beta, float* saved_mean,
                            float* saved_invstd, float* running_mean, float* running_var, int64_t rows, int c,
                            float eps, float momentum, int update_running, void* scratch, void* stream) {
  if (c % 4) return -(int)cudaErrorInvalidValue;
  cudaStream_t st = S(stream);
  float* ws = static_cast<float*>(scratch);
  int nb = bn_blocks(rows);
  bn_reduce_kernel<<<nb, kEwThreads, 0, st>>>(7, x, nullptr, nullptr, nullptr, rows, c, ws);
  bn_finalize_fwd_kernel<<<(c + 7) / 8, 256, 0, st>>>(ws, nb, rows, c, eps, momentum, update_running, saved_mean,
                                                      saved_invstd, running_mean, running_var, x);
  bnrelu_apply_kernel<kSix><<<ew_blocks(rows * c / 4), kEwThreads, 0, st>>>(x, z, saved_mean, saved_invstd, gamma,
                                                                            beta, rows, c);
  return last_error();
}

template <bool kSix>
int bnrelu_fwd_replay(const float* x, float* z, const float* gamma, const float* beta,
                             const float* saved_mean, const float* saved_invstd, int64_t rows, int c, void* stream) {
  if (c % 4) return -(int)cudaErrorInvalidValue;
  bnrelu_apply_kernel<kSix><<<ew_blocks(rows * c / 4), kEwThreads, 0, S(stream)>>>(x, z, saved_mean, saved_invstd,
                                                                                   gamma, beta, rows, c);
  return last_error();
}

template <bool kSix>
int bnrelu_bwd(const float* x, const float* dz, float* dx, int accumulate, const float* gamma,
                      const float* beta, const float* saved_mean, const float* saved_invstd, float* dgamma,
                      float* dbeta, int64_t rows, int c, void* scratch, void* stream) {
  if (c % 4) return -(int)cudaErrorInvalidValue;
  cudaStream_t st = S(stream);
  float* ws = static_cast<float*>(scratch);
  int nb = bn_blocks(rows);
  float* coef_b = ws + (size_t)nb * 2 * c;
  float* coef_c = coef_b + c;
  bn_reduce_kernel<<<nb, kEwThreads, 0, st>>>(kSix ? 4 : 3, x, dz, saved_mean, saved_invstd, rows, c, ws, gamma,
                                              beta);
  bn_finalize_bwd_kernel<<<(c + 7) / 8, 256, 0, st>>>(ws, nb, c, rows, saved_mean, saved_invstd, gamma,
                                                      saved_invstd, coef_b, coef_c, dgamma, dbeta);
  bnrelu_bwd_apply_kernel<kSix><<<ew_blocks(rows * c / 4), kEwThreads, 0, st>>>(
      x, dz, dx, saved_mean, beta, gamma, saved_invstd, coef_b, coef_c, rows, c, accumulate);
  return last_error();
}
}  // namespace

extern "C" {

int monet_bnrelu_fwd_train(const float* x, float* z, const float* gamma, const float* beta, float* saved_mean,
                           float* saved_invstd, float* running_mean, float* running_var, int64_t rows, int c,
                           float eps, float momentum, int update_running, void* scratch, void* stream) {
  return bnrelu_fwd_train<false>(x, z, gamma, beta, saved_mean, saved_invstd, running_mean, running_var, rows, c, eps,
                                 momentum, update_running, scratch, stream);
}
int monet_bnrelu_fwd_replay(const float* x, float* z, const float* gamma, const float* beta, const float* saved_mean,
                            const float* saved_invstd, int64_t rows, int c, void* stream) {
  return bnrelu_fwd_replay<false>(x, z, gamma, beta, saved_mean, saved_invstd, rows, c, stream);
}
int monet_bnrelu_bwd(const float* x, const float* dz, float* dx, int accumulate, const float* gamma,
                     const float* beta, const float* saved_mean, const float* saved_invstd, float* dgamma,
                     float* dbeta, int64_t rows, int c, void* scratch, void* stream) {
  return bnrelu_bwd<false>(x, dz, dx, accumulate, gamma, beta, saved_mean, saved_invstd, dgamma, dbeta, rows, c,
                           scratch, stream);
}

// fused BN+ReLU6 (MobileNet-V2): z = min(max(BN(x), 0), 6), backward gated by 0 < BN(x) < 6
int monet_bnrelu6_fwd_train(const float* x, float* z, const float* gamma, const float* beta, float* saved_mean,
                            float* saved_invstd, float* running_mean, float* running_var, int64_t rows, int c,
                            float eps, float momentum, int update_running, void* scratch, void* stream) {
  return bnrelu_fwd_train<true>(x, z, gamma, beta, saved_mean, saved_invstd, running_mean, running_var, rows, c, eps,
                                momentum, update_running, scratch, stream);
}
int monet_bnrelu6_fwd_replay(const float* x, float* z, const float* gamma, const float* beta,
                             const float* saved_mean, const float* saved_invstd, int64_t rows, int c, void* stream) {
  return bnrelu_fwd_replay<true>(x, z, gamma, beta, saved_mean, saved_invstd, rows, c, stream);
}
int monet_bnrelu6_bwd(const float* x, const float* dz, float* dx, int accumulate, const float* gamma,
                      const float* beta, const float* saved_mean, const float* saved_invstd, float* dgamma,
                      float* dbeta, int64_t rows, int c, void* scratch, void* stream) {
  return bnrelu_bwd<true>(x, dz, dx, accumulate, gamma, beta, saved_mean, saved_invstd, dgamma, dbeta, rows, c,
                          scratch, stream);
}

// fused BN + residual add + ReLU: z = max(BN(x) + skip, 0)
int monet_bnaddrelu_fwd_train(const float* x, const float* skip, float* z, const float* gamma, const float* beta,
                              float* saved_mean, float* saved_invstd, float* running_mean, float* running_var,
                              int64_t rows, int c, float eps, float momentum, int update_running, void* scratch,
                              void* stream) {
  if (c % 4) return -(int)cudaErrorInvalidValue;
  cudaStream_t st = S(stream);
  float* ws = static_cast<float*>(scratch);
  int nb = bn_blocks(rows);
  bn_reduce_kernel<<<nb, kEwThreads, 0, st>>>(7, x, nullptr, nullptr, nullptr, rows, c, ws);
  bn_finalize_fwd_kernel<<<(c + 7) / 8, 256, 0, st>>>(ws, nb, rows, c, eps, momentum, update_running, saved_mean,
                                                      saved_invstd, running_mean, running_var, x);
  bnaddrelu_apply_kernel<<<ew_blocks(rows * c / 4), kEwThreads, 0, st>>>(x, skip, z, saved_mean, saved_invstd, gamma,
                                                                         beta, rows, c);
  return last_error();
}
int monet_bnaddrelu_fwd_replay(const float* x, const float* skip, float* z, const float* gamma, const float* beta,
                               const float* saved_mean, const float* saved_invstd, int64_t rows, int c, void* stream) {
  if (c % 4) return -(int)cudaErrorInvalidValue;
  bnaddrelu_apply_kernel<<<ew_blocks(rows * c / 4), kEwThreads, 0, S(stream)>>>(x, skip, z, saved_mean, saved_invstd,
                                                                                gamma, beta, rows, c);
  return last_error();
}
// gate_src = z (gate_from_out = 1, output-activated) or skip (0, input-activated)
int monet_bnaddrelu_bwd(const float* x, const float* gate_src, int gate_from_out, const float* dz, float* dx,
                        int acc_x, float* dskip, int acc_skip, const float* gamma, const float* beta,
                        const float* saved_mean, const float* saved_invstd, float* dgamma, float* dbeta, int64_t rows,
                        int c, void* scratch, void* stream) {
  if (c % 4) return -(int)cudaErrorInvalidValue;
  cudaStream_t st = S(stream);
  float* ws = static_cast<float*>(scratch);
  int nb = bn_blocks(rows);
  float* coef_b = ws + (size_t)nb * 2 * c;
  float* coef_c = coef_b + c;
  bn_reduce_kernel<<<nb, kEwThreads, 0, st>>>(gate_from_out ? 5 : 6, x, dz, saved_mean, saved_invstd, rows, c, ws,
                                              gamma, beta, gate_src);
  bn_finalize_bwd_kernel<<<(c + 7) / 8, 256, 0, st>>>(ws, nb, c, rows, saved_mean, saved_invstd, gamma,
                                                      saved_invstd, coef_b, coef_c, dgamma, dbeta);
  bnaddrelu_bwd_apply_kernel<<<ew_blocks(rows * c / 4), kEwThreads, 0, st>>>(
      x, gate_src, gate_from_out, dz, dx, acc_x, dskip, acc_skip, saved_mean, beta, gamma, saved_invstd, coef_b,
      coef_c, rows, c);
  return last_error();
}

// ------------------------------------------------------------------- add / pass
int monet_add_fwd(const float* a, const float* b, float* y, int64_t n, void* stream) {
  add_kernel<<<ew_blocks(n / 4 + 1), kEwThreads, 0, S(stream)>>>(a, b, y, n);
  return last_error();
}
int monet_addrelu_fwd(const float* a, const float* b, float* z, int64_t n, void* stream) {
  addrelu_kernel<<<ew_blocks(n / 4 + 1), kEwThreads, 0, S(stream)>>>(a, b, z, n);
  return last_error();
}
int monet_addrelu_bwd_out(const float* z, const float* dz, float* da, int acc_a, float* db, int acc_b, int64_t n,
                          void* stream) {
  addrelu_bwd_kernel<<<ew_blocks(n / 4 + 1), kEwThreads, 0, S(stream)>>>(z, nullptr, dz, da, acc_a, db, acc_b, n);
  return last_error();
}
int monet_addrelu_bwd_in(const float* a, const float* b, const float* dz, float* da, int acc_a, float* db, int acc_b,
                         int64_t n, void* stream) {
  addrelu_bwd_kernel<<<ew_blocks(n / 4 + 1), kEwThreads, 0, S(stream)>>>(a, b, dz, da, acc_a, db, acc_b, n);
  return last_error();
}
int monet_grad_pass(const float* dy, float* dx, int64_t n, float scale, int accumulate, void* stream) {
  scale_acc_kernel<<<ew_blocks(n / 4 + 1), kEwThreads, 0, S(stream)>>>(dy, dx, n, scale, accumulate);
  return last_error();
}

// ------------------------------------------------------------------- pooling
int monet_maxpool_fwd(const monet_conv_desc* d, const float* x, float* y, uint8_t* idx8, void* stream) {
  if (d->c % 4) return -(int)cudaErrorInvalidValue;
  long long total = (long long)d->n * d->p * d->q * (d->c / 4);
  maxpool_fwd_kernel<<<ew_blocks(total), kEwThreads, 0, S(stream)>>>(x, y, idx8, d->n, d->h, d->w, d->c, d->p, d->q,
                                                                     d->r, d->s, d->stride_h, d->stride_w, d->pad_h,
                                                                     d->pad_w);
  return last_error();
}
int monet_maxpool_bwd(const monet_conv_desc* d, const uint8_t* idx8, const float* x, const float* dy, float* dx,
                      int accumulate, void* stream) {
  if (d->c % 4) return -(int)cudaErrorInvalidValue;
  long long total = (long long)d->n * d->h * d->w * (d->c / 4);
  const bool sq = idx8 && d->r == d->s && d->stride_h == d->stride_w && d->pad_h == d->pad_w &&
                  total < (1LL << 31) && ((long long)d->n * d->p * d->q * d->c) < (1LL << 40);
  if (sq && d->r == 2 && d->stride_h == 2) {
    maxpool_bwd_idx_kernel<2, 2><<<ew_blocks(total), kEwThreads, 0, S(stream)>>>(
        idx8, dy, dx, d->h, d->w, d->c, d->p, d->q, d->pad_h, (unsigned)total, accumulate);
    return last_error();
  }
  if (sq && d->r == 3 && d->stride_h == 2) {
    maxpool_bwd_idx_kernel<3, 2><<<ew_blocks(total), kEwThreads, 0, S(stream)>>>(
        idx8, dy, dx, d->h, d->w, d->c, d->p, d->q, d->pad_h, (unsigned)total, accumulate);
    return last_error();
  }
  maxpool_bwd_kernel<<<ew_blocks(total), kEwThreads, 0, S(stream)>>>(idx8, x, dy, dx, d->n, d->h, d->w, d->c, d->p,
                                                                     d->q, d->r, d->s, d->stride_h, d->stride_w,
                                                                     d->pad_h, d->pad_w, accumulate);
  return last_error();
}
int monet_avgpool_fwd(const float* x, float* y, int n, int hw, int c, void* stream) {
  avgpool_fwd_kernel<<<(n * c + 255) / 256, 256, 0, S(stream)>>>(x, y, n, hw, c);
  return last_error();
}
__global__ void avgpool_bwd_kernel(const float* __restrict__ dy, float* dx, int n, int hw, int c, int accumulate) {
  long long total = (long long)n * hw * c;
  float inv = 1.0f / (float)hw;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    long long ci = i % c, ni = i / ((long long)hw * c);
    float v = dy[ni * c + ci] * inv;
    dx[i] = accumulate ? dx[i] + v : v;
  }
}
int monet_avgpool_bwd(const float* dy, float* dx, int n, int hw, int c, int accumulate, void* stream) {
  avgpool_bwd_kernel<<<ew_blocks((long long)n * hw * c), kEwThreads, 0, S(stream)>>>(dy, dx, n, hw, c, accumulate);
  return last_error();
}

// ------------------------------------------------------------------- loss / SGD
// rows (n) x classes logits; per-pixel segmentation losses are rows = N*H*W of an NHWC tensor
constexpr int kXentSmallK = 32, kXentPartials = 1024;
size_t monet_xent_scratch_bytes(int n) {
  return ((size_t)n * sizeof(float) + 15) / 16 * 16 + (size_t)kXentPartials * sizeof(double);
}

int monet_xent_fwd(const float* logits, const int32_t* labels, float* loss, int n, int classes, void* scratch,
                   void* stream) {
  cudaStream_t st = S(stream);
  float* rows = static_cast<float*>(scratch);
  if (classes <= kXentSmallK) {
    double* part = reinterpret_cast<double*>(static_cast<char*>(scratch) + ((size_t)n * sizeof(float) + 15) / 16 * 16);
    xent_small_fwd_kernel<<<ew_blocks(n), kEwThreads, 0, st>>>(logits, labels, rows, n, classes);
    const int nb = (int)std::min<long long>(kXentPartials, std::max(1, (n + 4095) / 4096));
    block_sum_kernel<<<nb, 256, 0, st>>>(rows, n, part);
    mean_of_partials_kernel<<<1, 32, 0, st>>>(part, nb, n, loss);
    return last_error();
  }
  xent_fwd_kernel<<<n, 256, 0, st>>>(logits, labels, rows, n, classes);
  mean_kernel<<<1, 32, 0, st>>>(rows, n, loss);
  return last_error();
}

int monet_xent_bwd(const float* logits, const int32_t* labels, const float* dloss, float* dlogits, int n,
                   int classes, int accumulate, void* stream) {
  if (classes <= kXentSmallK) {
    xent_small_bwd_kernel<<<ew_blocks(n), kEwThreads, 0, S(stream)>>>(logits, labels, dloss, dlogits, n, classes,
                                                                       accumulate);
    return last_error();
  }
  xent_bwd_kernel<<<n, 256, 0, S(stream)>>>(logits, labels, dloss, dlogits, n, classes, accumulate);
  return last_error();
}

// ---------------------------------------------------------------- transposed conv
// ConvTranspose2d (UNet's up-sampling) as the adjoint of the conv described by d:
// d's input is the transposed conv's OUTPUT y [n][h][w][c], d's output is its INPUT
// x [n][p][q][k], weights KRSC = torch [in][out][R][S] permuted (in = k, out = c).
//   forward: y = dgrad(dy := x) (+ bias);  dx = fwd conv of dy_T;  dw = wgrad(x := dy_T, dy := x)
size_t monet_convT_ws_bytes(int variant, int pass, const monet_conv_desc* d) {
  if (pass == MONET_PASS_FWD) return monet_conv_ws_bytes(variant, MONET_PASS_DGRAD, d);
  return std::max(monet_conv_ws_bytes(variant, MONET_PASS_FWD, d), monet_conv_ws_bytes(variant, MONET_PASS_WGRAD, d));
}
int monet_convT_fwd(int variant, const monet_conv_desc* d, const float* x, const float* w, const float* bias, float* y,
                    void* ws, size_t ws_bytes, void* stream) {
  if (int e = check_desc(d)) return e;
  if (bias) {
    const long long tot = (long long)d->n * d->h * d->w * d->c;
    bias_fill_kernel<<<(int)((tot + 255) / 256), 256, 0, S(stream)>>>(y, bias, (int)(tot / d->c), d->c);
  }
  return monet_conv_dgrad(variant, d, x, w, y, bias ? 1 : 0, ws, ws_bytes, stream);
}
int monet_convT_bwd(int variant, const monet_conv_desc* d, const float* x, const float* w, const float* dy, float* dx,
                    int dx_accumulate, float* dw, void* ws, size_t ws_bytes, void* stream) {
  if (int e = check_desc(d)) return e;
  if (dx) {
    GemmParams p = conv_params(MONET_PASS_FWD, d, dy, w, dx);
    if (int e = launch_gemm(p, variant, dx_accumulate, ws, ws_bytes, S(stream))) return e;
  }
  return monet_conv_wgrad(variant, d, dy, x, dw, 0, ws, ws_bytes, stream);
}

int monet_sgd_step(float* w, const float* g, float* momentum_buf, int64_t n, float lr, float momentum,
                   float weight_decay, float grad_scale, int first_step, void* stream) {
  sgd_kernel<<<ew_blocks(n), kEwThreads, 0, S(stream)>>>(w, g, momentum_buf, n, lr, momentum, weight_decay, grad_scale,
                                                         first_step);
  return last_error();
}

}  // extern "C"
