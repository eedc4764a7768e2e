// tcgen05 (kind::tf32, 3xTF32-split) persistent GEMM with implicit-GEMM
// convolution operand loaders.  One CTA per SM, warp-specialised:
//
//   warps 0-3  producers: gather 16B operand groups from HBM/L2 (im2col
//              addressing computed in registers), split each fp32 into
//              tf32 hi + lo, store both into SWIZZLE_128B smem tiles
//   warps 4-7  epilogue: tcgen05.ld the 128x128 fp32 accumulator from TMEM,
//              store / accumulate / write split-K partials
//   warp  8    MMA issuer (one lane) + TMEM owner
//
// C[m, n] = sum_k A[m, k] * B[n, k]; per 8-wide k step the issuer runs
// A_hi*B_hi + A_hi*B_lo + A_lo*B_hi into the same TMEM accumulator, which
// restores ~fp32 accuracy (SURVEY.md §7 hard part 1).
#pragma once
#include "common.cuh"

namespace monet {

// Operand fetch modes (each fetch is a 16B group of 4 consecutive elements
// along the operand's contiguous dimension).
enum OperandMode : int {
  OP_KMAJOR = 0,       // element(row,k) = ptr[row*ld + k]                      (k contiguous)
  OP_MNMAJOR = 1,      // element(row,k) = ptr[(k/kdiv)*ks1 + (k%kdiv)*ld + row] (row contiguous)
  OP_IM2COL_FPROP = 2, // rows = output pixels (n,p,q), k = (r,s,c)             (K-major)
  OP_IM2COL_DGRAD = 3, // rows = input pixels (n,h,w), k = (r,s,kout) over dy   (K-major)
  OP_IM2COL_WGRAD = 4, // rows = (r,s,c), k = output pixel (n,p,q) over x       (MN-major)
};

struct ConvGeom {
  int N, H, W, C, K, R, S, P, Q, sh, sw, ph, pw;
};

struct Operand {
  int mode;
  int rows;  // extent of the operand's M (or N) dimension
  const float* ptr;
  long long ld;
  int kdiv;
  long long ks1;
  int aligned;  // 16B groups are aligned and never straddle an edge (host-checked)
};

// Scalar fallback for operands whose 16B groups are misaligned or ragged:
// element e of the group sits at base + e*step and exists iff e < count.
MONET_DEV float4 load4_scalar(const float* base, long long step, int count) {
  float v[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) v[e] = e < count ? __ldg(base + e * step) : 0.f;
  return make_float4(v[0], v[1], v[2], v[3]);
}

enum EpiMode : int { EPI_STORE = 0, EPI_ACCUM = 1, EPI_PARTIAL = 2 };

struct GemmParams {
  int M, N, Kd;
  Operand a, b;
  ConvGeom g;
  float* c;
  long long ldc;
  int epi;
  float* ws;        // split-K partials [splits][M][N]
  int splits;
  int kb_per_split;
  int m_tiles, n_tiles;
  int split_tf32;   // 1: 3xTF32 (hi/lo), 0: plain tf32
};

constexpr int BM = 128, BN = 128, BK = 32;
constexpr int kStages = 3;
constexpr int kTileBytes = BM * BK * 4;  // 16 KB, BM == BN
constexpr int kStageBytes = 4 * kTileBytes;  // A_hi, A_lo, B_hi, B_lo
constexpr int kProducerWarps = 4, kEpilogueWarps = 4;
constexpr int kThreads = (kProducerWarps + kEpilogueWarps + 1) * 32;
constexpr int kAccStages = 2;
// TMEM accumulation is flushed to the fp32 output every kChunk k-blocks: the
// tensor core's accumulator does not round-to-nearest, so very long single
// accumulation chains (wgrad reduces over up to 577k pixels) drift; chunk
// partial sums are combined in the epilogue with ordinary fp32 adds.
constexpr int kChunk = 16;
constexpr int kTmemCols = kAccStages * BN;  // 256
constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;

// --------------------------------------------------------------------------
// Producer side: per-tile row decode and per-stage 16B fetches

struct KRowState {  // K-major operand: this thread's 8 rows of the tile
  long long base[8];  // element offset of the row's origin (mode dependent)
  int hb[8], wb[8];   // spatial origin (im2col modes)
  int valid;          // bitmask of in-range rows
};

MONET_DEV void decode_kmajor_rows(const GemmParams& p, const Operand& op, int tile_row0, int t,
                                  KRowState& st) {
  st.valid = 0;
  const ConvGeom& g = p.g;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    int row = tile_row0 + (t >> 3) + 16 * i;
    st.base[i] = 0;
    st.hb[i] = 0;
    st.wb[i] = 0;
    if (row >= op.rows) continue;
    st.valid |= 1 << i;
    if (op.mode == OP_KMAJOR) {
      st.base[i] = (long long)row * op.ld;
    } else if (op.mode == OP_IM2COL_FPROP) {
      int q = row % g.Q;
      int tmp = row / g.Q;
      int pp = tmp % g.P;
      int n = tmp / g.P;
      st.base[i] = (long long)n * g.H * g.W * g.C;
      st.hb[i] = pp * g.sh - g.ph;
      st.wb[i] = q * g.sw - g.pw;
    } else {  // OP_IM2COL_DGRAD: rows are dx pixels
      int w = row % g.W;
      int tmp = row / g.W;
      int h = tmp % g.H;
      int n = tmp / g.H;
      st.base[i] = (long long)n * g.P * g.Q * g.K;
      st.hb[i] = h + g.ph;
      st.wb[i] = w + g.pw;
    }
  }
}

// Fetch the 16B group (row i of this thread, chunk j) at reduction index k.
MONET_DEV float4 fetch_kmajor(const GemmParams& p, const Operand& op, const KRowState& st, int i, int k,
                              int tap_r, int tap_s, int kin) {
  float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
  if (!((st.valid >> i) & 1) || k >= p.Kd) return z;
  const ConvGeom& g = p.g;
  if (op.mode == OP_KMAJOR) {
    if (!op.aligned) return load4_scalar(op.ptr + st.base[i] + k, 1, min(4, p.Kd - k));
    return __ldg(reinterpret_cast<const float4*>(op.ptr + st.base[i] + k));
  } else if (op.mode == OP_IM2COL_FPROP) {
    int h = st.hb[i] + tap_r, w = st.wb[i] + tap_s;
    if ((unsigned)h >= (unsigned)g.H || (unsigned)w >= (unsigned)g.W) return z;
    return __ldg(reinterpret_cast<const float4*>(op.ptr + st.base[i] + ((long long)h * g.W + w) * g.C + kin));
  } else {
    int hp = st.hb[i] - tap_r, wp = st.wb[i] - tap_s;
    if (hp < 0 || wp < 0) return z;
    int pp = hp / g.sh, q = wp / g.sw;
    if (pp * g.sh != hp || q * g.sw != wp || pp >= g.P || q >= g.Q) return z;
    return __ldg(reinterpret_cast<const float4*>(op.ptr + st.base[i] + ((long long)pp * g.Q + q) * g.K + kin));
  }
}

struct MRowState {  // MN-major operand: this thread's 4-element group along MN and 8 k-rows
  long long gbase;   // OP_MNMAJOR: row offset; OP_IM2COL_WGRAD: channel offset c
  int tap_r, tap_s;  // OP_IM2COL_WGRAD
  bool gvalid;
  int kq[8], kp[8], kn[8];  // OP_IM2COL_WGRAD: pixel counters of the 8 k-rows
};

MONET_DEV void decode_mnmajor_group(const GemmParams& p, const Operand& op, int tile_row0, int t,
                                    MRowState& st) {
  int row = tile_row0 + 4 * (t & 31);
  st.gvalid = row < op.rows;
  st.gbase = row;
  st.tap_r = st.tap_s = 0;
  if (op.mode == OP_IM2COL_WGRAD && st.gvalid) {
    const ConvGeom& g = p.g;
    int tap = row / g.C;
    st.gbase = row - tap * g.C;
    st.tap_r = tap / g.S;
    st.tap_s = tap - st.tap_r * g.S;
  }
}

MONET_DEV void init_pixel_counters(const GemmParams& p, int k0, int t, MRowState& st) {
  const ConvGeom& g = p.g;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    int k = k0 + (t >> 5) + 4 * i;
    st.kq[i] = k % g.Q;
    int tmp = k / g.Q;
    st.kp[i] = tmp % g.P;
    st.kn[i] = tmp / g.P;
  }
}

MONET_DEV void advance_pixel_counters(const GemmParams& p, MRowState& st) {
  const ConvGeom& g = p.g;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    st.kq[i] += BK;
    while (st.kq[i] >= g.Q) {
      st.kq[i] -= g.Q;
      if (++st.kp[i] == g.P) {
        st.kp[i] = 0;
        ++st.kn[i];
      }
    }
  }
}

MONET_DEV float4 fetch_mnmajor(const GemmParams& p, const Operand& op, const MRowState& st, int i, int k) {
  float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
  if (!st.gvalid || k >= p.Kd) return z;
  if (op.mode == OP_MNMAJOR) {
    int kh = k / op.kdiv, kl = k - kh * op.kdiv;
    const float* src = op.ptr + kh * op.ks1 + (long long)kl * op.ld + st.gbase;
    if (!op.aligned) return load4_scalar(src, 1, min(4, op.rows - (int)st.gbase));
    return __ldg(reinterpret_cast<const float4*>(src));
  }
  const ConvGeom& g = p.g;
  int h = st.kp[i] * g.sh - g.ph + st.tap_r;
  int w = st.kq[i] * g.sw - g.pw + st.tap_s;
  if ((unsigned)h >= (unsigned)g.H || (unsigned)w >= (unsigned)g.W) return z;
  return __ldg(reinterpret_cast<const float4*>(op.ptr + (((long long)st.kn[i] * g.H + h) * g.W + w) * g.C + st.gbase));
}

MONET_DEV void store_split(uint8_t* hi_tile, uint8_t* lo_tile, uint32_t off, float4 v, int split) {
  if (split) {
    float4 h, l;
    split_tf32(v.x, h.x, l.x);
    split_tf32(v.y, h.y, l.y);
    split_tf32(v.z, h.z, l.z);
    split_tf32(v.w, h.w, l.w);
    *reinterpret_cast<float4*>(hi_tile + off) = h;
    *reinterpret_cast<float4*>(lo_tile + off) = l;
  } else {
    *reinterpret_cast<float4*>(hi_tile + off) = v;
  }
}

// One operand tile (128 rows x 32 k) for k-block kb.
template <bool kIsA>
MONET_DEV void produce_operand(const GemmParams& p, const Operand& op, int kb, int t, const KRowState& ks,
                               MRowState& ms, uint8_t* hi_tile, uint8_t* lo_tile) {
  const int k0 = kb * BK;
  if (op.mode == OP_MNMAJOR || op.mode == OP_IM2COL_WGRAD) {
    // 32 k-rows x 32 groups; thread: group (t&31), k-rows (t>>5)+4i
    const int grp = t & 31;
    const int chunk_region = grp >> 3;  // which 32-element MN chunk (4 KB region)
    const int chunk = grp & 7;
    float4 v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = fetch_mnmajor(p, op, ms, i, k0 + (t >> 5) + 4 * i);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      int kr = (t >> 5) + 4 * i;
      uint32_t off = chunk_region * 4096 + sw128b32_offset(kr, chunk);
      store_split(hi_tile, lo_tile, off, v[i], p.split_tf32);
    }
    if (op.mode == OP_IM2COL_WGRAD) advance_pixel_counters(p, ms);
  } else {
    // 128 rows x 8 chunks; thread: chunk (t&7), rows (t>>3)+16i
    const int j = t & 7;
    const int k = k0 + 4 * j;
    int tap_r = 0, tap_s = 0, kin = 0;
    if (op.mode == OP_IM2COL_FPROP) {
      int tap = k / p.g.C;
      kin = k - tap * p.g.C;
      tap_r = tap / p.g.S;
      tap_s = tap - tap_r * p.g.S;
    } else if (op.mode == OP_IM2COL_DGRAD) {
      int tap = k / p.g.K;
      kin = k - tap * p.g.K;
      tap_r = tap / p.g.S;
      tap_s = tap - tap_r * p.g.S;
    }
    float4 v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = fetch_kmajor(p, op, ks, i, k, tap_r, tap_s, kin);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      int row = (t >> 3) + 16 * i;
      store_split(hi_tile, lo_tile, sw128_offset(row, j), v[i], p.split_tf32);
    }
  }
}

MONET_DEV void tile_coords(const GemmParams& p, int tile, int& mt, int& nt, int& sp) {
  int per_split = p.m_tiles * p.n_tiles;
  sp = tile / per_split;
  int r = tile - sp * per_split;
  mt = r / p.n_tiles;
  nt = r - mt * p.n_tiles;
}

MONET_DEV void kb_range(const GemmParams& p, int sp, int& kb0, int& kb1) {
  int total = (p.Kd + BK - 1) / BK;
  kb0 = sp * p.kb_per_split;
  kb1 = min(total, kb0 + p.kb_per_split);
}

// Descriptor of the 8-wide k slice `kk` (0..3) of a tile.
MONET_DEV uint64_t operand_desc(uint32_t tile_addr, bool mn_major, int kk) {
  if (mn_major) {
    // canonical MN-major SW128_BASE32B: ((T,8,m),(4,k)) with 32-element MN
    // chunks every 4096 B (LBO) and 4-row k groups every 512 B (SBO); one
    // k step = 8 rows = 1024 B
    return smem_desc(tile_addr + kk * 1024, 4096, 512, 1);
  }
  // canonical K-major SW128: 8-row groups every 1024 B (SBO); k step = 32 B
  return smem_desc(tile_addr + kk * 32, 16, 1024, 2);
}

__global__ void __launch_bounds__(kThreads, 1) gemm_tf32_kernel(const GemmParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty_bar = full_bar + kStages;
  uint64_t* tfull_bar = empty_bar + kStages;
  uint64_t* tempty_bar = tfull_bar + kAccStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + kAccStages);

  const int warp = warp_id();
  const int lane = lane_id();
  const int n_tiles_total = p.m_tiles * p.n_tiles * p.splits;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], kProducerWarps * 32);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < kAccStages; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], kEpilogueWarps * 32);
    }
    mbar_fence_init();
  }
  if (warp == kProducerWarps + kEpilogueWarps) tmem_alloc(tmem_slot, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const bool a_mn = (p.a.mode == OP_MNMAJOR || p.a.mode == OP_IM2COL_WGRAD);
  const bool b_mn = (p.b.mode == OP_MNMAJOR || p.b.mode == OP_IM2COL_WGRAD);

  if (warp < kProducerWarps) {
    // ------------------------------------------------------------ producers
    const int t = threadIdx.x;
    int stage = 0;
    uint32_t phase = 0;
    for (int tile = blockIdx.x; tile < n_tiles_total; tile += gridDim.x) {
      int mt, nt, sp, kb0, kb1;
      tile_coords(p, tile, mt, nt, sp);
      kb_range(p, sp, kb0, kb1);
      KRowState ka, kbst;
      MRowState ma, mb;
      if (a_mn) {
        decode_mnmajor_group(p, p.a, mt * BM, t, ma);
        if (p.a.mode == OP_IM2COL_WGRAD) init_pixel_counters(p, kb0 * BK, t, ma);
      } else {
        decode_kmajor_rows(p, p.a, mt * BM, t, ka);
      }
      if (b_mn) {
        decode_mnmajor_group(p, p.b, nt * BN, t, mb);
        if (p.b.mode == OP_IM2COL_WGRAD) init_pixel_counters(p, kb0 * BK, t, mb);
      } else {
        decode_kmajor_rows(p, p.b, nt * BN, t, kbst);
      }
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&empty_bar[stage], phase ^ 1);
        uint8_t* st_base = smem + stage * kStageBytes;
        produce_operand<true>(p, p.a, kb, t, ka, ma, st_base, st_base + kTileBytes);
        produce_operand<false>(p, p.b, kb, t, kbst, mb, st_base + 2 * kTileBytes, st_base + 3 * kTileBytes);
        fence_proxy_async_smem();
        mbar_arrive(&full_bar[stage]);
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp < kProducerWarps + kEpilogueWarps) {
    // ------------------------------------------------------------ epilogue
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < n_tiles_total; tile += gridDim.x) {
      int mt, nt, sp, kb0, kb1;
      tile_coords(p, tile, mt, nt, sp);
      kb_range(p, sp, kb0, kb1);
      const int nchunks = (kb1 - kb0 + kChunk - 1) / kChunk;
      for (int chunk = 0; chunk < nchunks; ++chunk) {
      const bool add_old = chunk > 0 || p.epi == EPI_ACCUM;
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const int m = mt * BM + quarter * 32 + lane;
      for (int cc = 0; cc < BN / 32; ++cc) {
        float v[32];
        tmem_ld32(tmem_base + acc * BN + cc * 32 + ((uint32_t)(quarter * 32) << 16), v);
        const int n0 = nt * BN + cc * 32;
        if (m < p.M && n0 < p.N) {
          float* dst;
          long long ld;
          if (p.epi == EPI_PARTIAL) {
            dst = p.ws + (long long)sp * p.M * p.N + (long long)m * p.N + n0;
            ld = p.N;
          } else {
            dst = p.c + (long long)m * p.ldc + n0;
            ld = p.ldc;
          }
          const int ncols = min(32, p.N - n0);
          const bool vec = (ncols == 32) && ((ld & 3) == 0) && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0);
          if (vec) {
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
              float4 o = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
              if (add_old) {
                float4 c = *reinterpret_cast<const float4*>(dst + j);
                o.x += c.x;
                o.y += c.y;
                o.z += c.z;
                o.w += c.w;
              }
              *reinterpret_cast<float4*>(dst + j) = o;
            }
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              if (j < ncols) {
                float o = v[j];
                if (add_old) o += dst[j];
                dst[j] = o;
              }
            }
          }
        }
        __syncwarp();
      }
      tc_fence_before();
      mbar_arrive(&tempty_bar[acc]);
      if (++acc == kAccStages) {
        acc = 0;
        acc_phase ^= 1;
      }
      }  // chunk
    }
  } else {
    // ------------------------------------------------------------ MMA issuer
    const uint32_t idesc = idesc_tf32(BM, BN, a_mn ? 1 : 0, b_mn ? 1 : 0);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < n_tiles_total; tile += gridDim.x) {
      int mt, nt, sp, kb0, kb1;
      tile_coords(p, tile, mt, nt, sp);
      kb_range(p, sp, kb0, kb1);
      for (int c0 = kb0; c0 < kb1; c0 += kChunk) {
      const int c1 = min(kb1, c0 + kChunk);
      mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      for (int kb = c0; kb < c1; ++kb) {
        mbar_wait(&full_bar[stage], phase);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t base = smem_u32(smem + stage * kStageBytes);
          const uint32_t a_hi = base, a_lo = base + kTileBytes;
          const uint32_t b_hi = base + 2 * kTileBytes, b_lo = base + 3 * kTileBytes;
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk) {
            const uint32_t first = (kb == c0 && kk == 0) ? 0u : 1u;
            if (p.split_tf32) {
              mma_tf32(d_tmem, operand_desc(a_lo, a_mn, kk), operand_desc(b_hi, b_mn, kk), idesc, first);
              mma_tf32(d_tmem, operand_desc(a_hi, a_mn, kk), operand_desc(b_lo, b_mn, kk), idesc, 1u);
              mma_tf32(d_tmem, operand_desc(a_hi, a_mn, kk), operand_desc(b_hi, b_mn, kk), idesc, 1u);
            } else {
              mma_tf32(d_tmem, operand_desc(a_hi, a_mn, kk), operand_desc(b_hi, b_mn, kk), idesc, first);
            }
          }
          mma_commit(&empty_bar[stage]);
          if (kb == c1 - 1) mma_commit(&tfull_bar[acc]);
        }
        __syncwarp();
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (++acc == kAccStages) {
        acc = 0;
        acc_phase ^= 1;
      }
      }  // chunk
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == kProducerWarps + kEpilogueWarps) {
    tc_fence_after();
    tmem_dealloc(tmem_base, kTmemCols);
  }
}

// Deterministic split-K reduction: out[m, n] (=|+=) sum_{s=0..S-1} ws[s, m, n].
__global__ void splitk_reduce_kernel(const float* __restrict__ ws, float* __restrict__ out, int M, int N,
                                     long long ldc, int splits, int accumulate) {
  long long total = (long long)M * N;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int k = 0; k < splits; ++k) s += ws[(long long)k * total + i];
    long long m = i / N, n = i - m * N;
    float* o = out + m * ldc + n;
    *o = accumulate ? (*o + s) : s;
  }
}

}  // namespace monet
