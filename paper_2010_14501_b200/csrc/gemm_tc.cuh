// tcgen05 (kind::tf32, 3xTF32-split) persistent GEMM with implicit-GEMM
// convolution operand loaders.  One CTA per SM, warp-specialised:
//
//   warps 0-7   producers: cp.async 16B operand chunks straight from HBM/L2
//               into raw fp32 staging (im2col addressing computed in
//               registers, zero-fill for padding), three k-blocks in flight;
//               then each thread splits the chunks it loaded itself into
//               tf32 hi + lo SWIZZLE_128B tiles (no register round trip for
//               the loads, no barrier on the staging buffers)
//   warps 8-11  epilogue: tcgen05.ld the 128x128 fp32 accumulator from TMEM,
//               store / accumulate / write split-K partials
//   warp  12    MMA issuer (one lane) + TMEM owner
//
// C[m, n] = sum_k A[m, k] * B[n, k]; per 8-wide k step the issuer runs
// A_lo*B_hi + A_hi*B_lo + A_hi*B_hi into the same TMEM accumulator, which
// restores ~fp32 accuracy (SURVEY.md §7 hard part 1).  Operand addressing
// modes are template parameters so every instantiation is branch-free in its
// producer loop.
#pragma once
#include <cuda.h>

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
  // bf16x3 kernel only: the operand is already split into bf16 hi / lo planes in global
  // memory (conv weights, split once per step); TMA loads them straight into the MMA's
  // SWIZZLE_128B stage tiles -- no fp32 staging, no split warps
  OP_W16_KMAJOR = 5,   // element(row,k) = plane[row*ld + k]                    (fprop B = w)
  OP_W16_MNMAJOR = 6,  // element(row,k) = plane[(k/kdiv)*ks1 + (k%kdiv)*ld + row] (dgrad B = w^T)
};

__host__ __device__ constexpr bool mode_is_mn(int m) {
  return m == OP_MNMAJOR || m == OP_IM2COL_WGRAD || m == OP_W16_MNMAJOR;
}
__host__ __device__ constexpr bool mode_is_w16(int m) { return m == OP_W16_KMAJOR || m == OP_W16_MNMAJOR; }

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
  int tma;      // bf16x3 kernel: 0 = 16B cp.async groups, 1 = TMA tiled map, 2 = TMA im2col map,
                //   3 = TMA im2col with C < 32: one box per filter tap, chunk-major raw layout,
                //   4 = wgrad tap view (C < 32): tiled maps over k = (n, p, q padded to wv_q) --
                //       A = dy as {kout, q, n*p}, B = the zero-padded input as {s*c, q, r, p, n}
  int rows_box; // bf16x3 kernel: rows of this operand one CTA loads per tile (128, or 64 for a
                //   64-wide N tile)
  int seg;      // bf16x3 kernel, MN-major operands: rows per segment of the raw smem layout
                //   (rows_box, or C when a wgrad im2col tile spans several filter taps)
  long long plane;  // OP_W16_*: bytes from the hi plane (ptr) to the lo plane
};

enum EpiMode : int { EPI_STORE = 0, EPI_ACCUM = 1, EPI_PARTIAL = 2 };

// Strided-conv dgrad as sub-pixel phases (bf16x3 kernel): output pixels with
// (h % sh, w % sw) == (a, b) form a stride-1 problem over dy that uses only the
// filter taps of matching parity.  GEMM row m = (n, i, j) of the Hp x Wp phase
// grid writes dx[n][i*sh + a][j*sw + b]; phase tap t reads dy[n][i + dr[t]][j + ds[t]]
// and filter tap tap[t] = r*S + s.
struct PhaseInfo {
  int on;
  int a, b, Hp, Wp, ntap, lo_h, lo_w;
  signed char dr[16], ds[16], tap[16];
};

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
  int c_trans;      // bf16x3: element (m, n) of the result is stored at c[n * ldc + m] (the swapped
                    //   wgrad of narrow convs: rows = (tap, c), columns = output channels, dw is KRSC)
  PhaseInfo ph;     // bf16x3: strided dgrad phase (ph.on == 0 otherwise)
  int chunk_stages; // bf16x3: MMA stages accumulated in TMEM before a flush to fp32 memory
  int n_pitch;      // output columns per n-tile (BN, or R-segments x S*C for the wgrad tap view)
  int wv_q;         // wgrad tap view: output-row length padded to a multiple of 32 (0 = off)
  int fv_q;         // fprop tap view: GEMM rows per output row (= BM; rows q >= Q are padding, 0 = off)
  const float* bias;  // bf16x3 EPI_STORE / split-K reduce: per-column bias added to the output (nullptr = none)
  int dbg_mode;     // debug build only: skip pipeline work to find the limiter (1 A split, 2 B split, 4 MMA, 8 stores)
  unsigned long long* dbg_t;  // debug: per-CTA wait-time counters of the bf16x3 pipeline roles (nullptr = off)
  float* dbg_a;     // debug: bf16x3 A-split dumps the raw A operand [M][Kpad] here (nullptr = off)
  float* dbg_b;     // debug: bf16x3 B-split dumps the raw B operand [N][Kpad]
  float* stats;     // bf16x3 pre-split-B kernels, single-chain EPI_STORE tiles: per-tile BN statistics of the
                    //   output, [m_tiles][2][N] = (mean, M2) over the tile's rows (nullptr = off)
  int* stats_done;  // host: set to 1 when the launch computes `stats` (else the caller reduces the output)
  int c_tma;        // bf16x3 pre-split-B kernels: the epilogue stages 32x32 blocks in smem and
                    //   stores (or reduce-adds) them with TMA through tma_c (0 = per-thread stores)
  CUtensorMap tma_a, tma_b;  // bf16x3: TMA descriptors (valid when Operand::tma != 0)
  CUtensorMap tma_c;         // output [rows][N] (EPI_PARTIAL: the split-K workspace [splits*M][N])
};

constexpr int BM = 128, BN = 128, BK = 32;
constexpr int kTileBytes = BM * BK * 4;  // 16 KB, BM == BN
constexpr int kRawStages = 3;
constexpr int kRawBytes = 2 * kTileBytes;      // A, B (fp32 as loaded)
constexpr int kStages = 2;                     // MMA-ready stages
constexpr int kStageBytes = 4 * kTileBytes;    // A_hi, A_lo, B_hi, B_lo
constexpr int kProducerWarps = 8, kEpilogueWarps = 4;
constexpr int kProducerThreads = kProducerWarps * 32;
constexpr int kPerThread = (BM * BK / 4) / kProducerThreads;  // 16B chunks per operand per thread = 4
constexpr int kThreads = (kProducerWarps + kEpilogueWarps + 1) * 32;
constexpr int kMmaWarp = kProducerWarps + kEpilogueWarps;
constexpr int kAccStages = 2;
// TMEM accumulation is flushed to the fp32 output every kChunk k-blocks: the
// tensor core's accumulator does not round-to-nearest, so very long single
// accumulation chains (wgrad reduces over up to 577k pixels) drift; chunk
// partial sums are combined in the epilogue with ordinary fp32 adds.
constexpr int kChunk = 16;
constexpr int kTmemCols = kAccStages * BN;  // 256
constexpr int kSmemBytes = kRawStages * kRawBytes + kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
static_assert(kPerThread == 4, "chunk ownership below assumes 256 producer threads");

// --------------------------------------------------------------------------
// chunk ownership: K-major tile = 128 rows x 8 chunks, thread t owns chunk
// (t & 7) of rows (t >> 3) + 32 i; MN-major tile = 32 k-rows x 32 groups,
// thread t owns group (t & 31) of k-rows (t >> 5) + 8 i.  Raw and ready
// tiles share the layout, so the split pass works in place per thread.
template <bool kMN>
MONET_DEV uint32_t chunk_offset(int t, int i) {
  if constexpr (kMN) {
    const int grp = t & 31;
    return (grp >> 3) * 4096 + sw128b32_offset((t >> 5) + 8 * i, grp & 7);
  } else {
    return sw128_offset((t >> 3) + 32 * i, t & 7);
  }
}

// Per-tile producer state of one operand.
template <int MODE>
struct OpState {
  // K-major modes: 4 rows per thread
  long long base[kPerThread];
  int hb[kPerThread], wb[kPerThread];
  int valid;
  // MN-major modes: one 4-element group, 4 k-rows (pixel counters for wgrad)
  long long gbase;
  int tap_r, tap_s;
  int kq[kPerThread], kp[kPerThread], kn[kPerThread];

  MONET_DEV void decode(const GemmParams& p, const Operand& op, int row0, int t, int k0) {
    const ConvGeom& g = p.g;
    if constexpr (mode_is_mn(MODE)) {
      const int row = row0 + 4 * (t & 31);
      valid = row < op.rows;
      gbase = row;
      tap_r = tap_s = 0;
      if constexpr (MODE == OP_IM2COL_WGRAD) {
        if (valid) {
          const int tap = row / g.C;
          gbase = row - tap * g.C;
          tap_r = tap / g.S;
          tap_s = tap - tap_r * g.S;
        }
#pragma unroll
        for (int i = 0; i < kPerThread; ++i) {
          const int k = k0 + (t >> 5) + 8 * i;
          kq[i] = k % g.Q;
          const int tmp = k / g.Q;
          kp[i] = tmp % g.P;
          kn[i] = tmp / g.P;
        }
      }
    } else {
      valid = 0;
#pragma unroll
      for (int i = 0; i < kPerThread; ++i) {
        const int row = row0 + (t >> 3) + 32 * i;
        base[i] = 0;
        hb[i] = wb[i] = 0;
        if (row >= op.rows) continue;
        valid |= 1 << i;
        if constexpr (MODE == OP_KMAJOR) {
          base[i] = (long long)row * op.ld;
        } else if constexpr (MODE == OP_IM2COL_FPROP) {
          const int q = row % g.Q;
          const int tmp = row / g.Q;
          const int pp = tmp % g.P;
          base[i] = (long long)(tmp / g.P) * g.H * g.W * g.C;
          hb[i] = pp * g.sh - g.ph;
          wb[i] = q * g.sw - g.pw;
        } else {  // OP_IM2COL_DGRAD: rows are dx pixels
          const int w = row % g.W;
          const int tmp = row / g.W;
          base[i] = (long long)(tmp / g.H) * g.P * g.Q * g.K;
          hb[i] = tmp % g.H + g.ph;
          wb[i] = w + g.pw;
        }
      }
    }
  }

  MONET_DEV void advance(const GemmParams& p) {
    if constexpr (MODE == OP_IM2COL_WGRAD) {
      const ConvGeom& g = p.g;
#pragma unroll
      for (int i = 0; i < kPerThread; ++i) {
        kq[i] += BK;
        while (kq[i] >= g.Q) {
          kq[i] -= g.Q;
          if (++kp[i] == g.P) {
            kp[i] = 0;
            ++kn[i];
          }
        }
      }
    }
  }
};

MONET_DEV void cp_async16(uint32_t dst, const float* src, const float* dummy) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src ? src : dummy),
               "r"(src ? 16 : 0)
               : "memory");
}
MONET_DEV void cp_async4(uint32_t dst, const float* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(valid ? 4 : 0) : "memory");
}
MONET_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
MONET_DEV void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Issue the cp.async loads of this thread's chunks of one operand tile.
template <int MODE>
MONET_DEV void issue_operand(const GemmParams& p, const Operand& op, int kb, int t, OpState<MODE>& st,
                             uint32_t raw_tile) {
  const int k0 = kb * BK;
  const ConvGeom& g = p.g;
  if constexpr (mode_is_mn(MODE)) {
#pragma unroll
    for (int i = 0; i < kPerThread; ++i) {
      const int k = k0 + (t >> 5) + 8 * i;
      const uint32_t dst = raw_tile + chunk_offset<true>(t, i);
      const float* src = nullptr;
      if (st.valid && k < p.Kd) {
        if constexpr (MODE == OP_MNMAJOR) {
          const int kh = k / op.kdiv, kl = k - kh * op.kdiv;
          src = op.ptr + kh * op.ks1 + (long long)kl * op.ld + st.gbase;
        } else {
          const int h = st.kp[i] * g.sh - g.ph + st.tap_r;
          const int w = st.kq[i] * g.sw - g.pw + st.tap_s;
          if ((unsigned)h < (unsigned)g.H && (unsigned)w < (unsigned)g.W)
            src = op.ptr + (((long long)st.kn[i] * g.H + h) * g.W + w) * g.C + st.gbase;
        }
      }
      if (MODE != OP_MNMAJOR || op.aligned || src == nullptr) {
        cp_async16(dst, src, op.ptr);
      } else {
        const int cnt = op.rows - (int)st.gbase;
#pragma unroll
        for (int e = 0; e < 4; ++e) cp_async4(dst + 4 * e, e < cnt ? src + e : op.ptr, e < cnt);
      }
    }
    st.advance(p);
  } else {
    const int k = k0 + 4 * (t & 7);
    int tap_r = 0, tap_s = 0, kin = 0;
    if constexpr (MODE == OP_IM2COL_FPROP) {
      const int tap = k / g.C;
      kin = k - tap * g.C;
      tap_r = tap / g.S;
      tap_s = tap - tap_r * g.S;
    } else if constexpr (MODE == OP_IM2COL_DGRAD) {
      const int tap = k / g.K;
      kin = k - tap * g.K;
      tap_r = tap / g.S;
      tap_s = tap - tap_r * g.S;
    }
    const bool kin_range = k < p.Kd;
#pragma unroll
    for (int i = 0; i < kPerThread; ++i) {
      const uint32_t dst = raw_tile + chunk_offset<false>(t, i);
      const float* src = nullptr;
      if (((st.valid >> i) & 1) && kin_range) {
        if constexpr (MODE == OP_KMAJOR) {
          src = op.ptr + st.base[i] + k;
        } else if constexpr (MODE == OP_IM2COL_FPROP) {
          const int h = st.hb[i] + tap_r, w = st.wb[i] + tap_s;
          if ((unsigned)h < (unsigned)g.H && (unsigned)w < (unsigned)g.W)
            src = op.ptr + st.base[i] + ((long long)h * g.W + w) * g.C + kin;
        } else {
          const int hp = st.hb[i] - tap_r, wp = st.wb[i] - tap_s;
          if (hp >= 0 && wp >= 0) {
            const int pp = hp / g.sh, q = wp / g.sw;
            if (pp * g.sh == hp && q * g.sw == wp && pp < g.P && q < g.Q)
              src = op.ptr + st.base[i] + ((long long)pp * g.Q + q) * g.K + kin;
          }
        }
      }
      if (MODE != OP_KMAJOR || op.aligned || src == nullptr) {
        cp_async16(dst, src, op.ptr);
      } else {
        const int cnt = min(4, p.Kd - k);
#pragma unroll
        for (int e = 0; e < 4; ++e) cp_async4(dst + 4 * e, e < cnt ? src + e : op.ptr, e < cnt);
      }
    }
  }
}

// Split this thread's landed chunks of one operand: raw fp32 -> tf32 hi + lo.
template <bool kMN>
MONET_DEV void split_operand(int t, const uint8_t* raw_tile, uint8_t* hi_tile, uint8_t* lo_tile, int split) {
#pragma unroll
  for (int i = 0; i < kPerThread; ++i) {
    const uint32_t off = chunk_offset<kMN>(t, i);
    float4 v = *reinterpret_cast<const float4*>(raw_tile + off);
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
}

MONET_DEV void tile_coords(const GemmParams& p, int tile, int& mt, int& nt, int& sp) {
  const int per_split = p.m_tiles * p.n_tiles;
  sp = tile / per_split;
  const int r = tile - sp * per_split;
  mt = r / p.n_tiles;
  nt = r - mt * p.n_tiles;
}

MONET_DEV void kb_range(const GemmParams& p, int sp, int& kb0, int& kb1) {
  const int total = (p.Kd + BK - 1) / BK;
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

template <int AM, int BMODE>
__global__ void __launch_bounds__(kThreads, 1) gemm_tf32_kernel(const GemmParams p) {
  constexpr bool a_mn = mode_is_mn(AM), b_mn = mode_is_mn(BMODE);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* raw = smem;                                  // kRawStages x (A, B) fp32
  uint8_t* ready = smem + kRawStages * kRawBytes;       // kStages x (A_hi, A_lo, B_hi, B_lo)
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(ready + kStages * kStageBytes);
  uint64_t* empty_bar = full_bar + kStages;
  uint64_t* tfull_bar = empty_bar + kStages;
  uint64_t* tempty_bar = tfull_bar + kAccStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + kAccStages);

  const int warp = warp_id();
  const int lane = lane_id();
  const int n_tiles_total = p.m_tiles * p.n_tiles * p.splits;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], kProducerThreads);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < kAccStages; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], kEpilogueWarps * 32);
    }
    mbar_fence_init();
  }
  if (warp == kMmaWarp) tmem_alloc(tmem_slot, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp < kProducerWarps) {
    // ------------------------------------------------------------ producers
    // Item j = j-th k-block of this CTA's tile sequence.  Loads of items
    // j+1..j+kRawStages-1 are in flight while item j is split into the
    // MMA-ready stage; a thread only reads back chunks it loaded itself.
    const int t = threadIdx.x;
    int n_items = 0;
    for (int tile = blockIdx.x; tile < n_tiles_total; tile += gridDim.x) {
      int mt, nt, sp, kb0, kb1;
      tile_coords(p, tile, mt, nt, sp);
      kb_range(p, sp, kb0, kb1);
      n_items += kb1 - kb0;
    }
    int it_tile = (int)blockIdx.x - (int)gridDim.x, it_kb = 0, it_kb1 = 0;
    OpState<AM> sa;
    OpState<BMODE> sb;
    auto issue_next = [&](int slot) {
      if (it_kb >= it_kb1) {
        it_tile += gridDim.x;
        int mt, nt, sp;
        tile_coords(p, it_tile, mt, nt, sp);
        kb_range(p, sp, it_kb, it_kb1);
        sa.decode(p, p.a, mt * BM, t, it_kb * BK);
        sb.decode(p, p.b, nt * BN, t, it_kb * BK);
      }
      const uint32_t base = smem_u32(raw + slot * kRawBytes);
      issue_operand<AM>(p, p.a, it_kb, t, sa, base);
      issue_operand<BMODE>(p, p.b, it_kb, t, sb, base + kTileBytes);
      ++it_kb;
    };
#pragma unroll 1
    for (int r = 0; r < kRawStages; ++r) {
      if (r < n_items) issue_next(r);
      cp_async_commit();
    }
    int stage = 0;
    uint32_t phase = 0;
#pragma unroll 1
    for (int j = 0; j < n_items; ++j) {
      const int slot = j % kRawStages;
      cp_async_wait<kRawStages - 1>();  // item j has landed (groups retire in order)
      mbar_wait(&empty_bar[stage], phase ^ 1);
      const uint8_t* rs = raw + slot * kRawBytes;
      uint8_t* st_base = ready + stage * kStageBytes;
      split_operand<a_mn>(t, rs, st_base, st_base + kTileBytes, p.split_tf32);
      split_operand<b_mn>(t, rs + kTileBytes, st_base + 2 * kTileBytes, st_base + 3 * kTileBytes, p.split_tf32);
      fence_proxy_async_smem();
      mbar_arrive(&full_bar[stage]);
      if (j + kRawStages < n_items) issue_next(slot);
      cp_async_commit();
      if (++stage == kStages) {
        stage = 0;
        phase ^= 1;
      }
    }
    cp_async_wait<0>();
  } else if (warp < kMmaWarp) {
    // ------------------------------------------------------------ epilogue
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < n_tiles_total; tile += gridDim.x) {
      int mt, nt, sp, kb0, kb1;
      tile_coords(p, tile, mt, nt, sp);
      kb_range(p, sp, kb0, kb1);
      const int nchunks = (kb1 - kb0 + kChunk - 1) / kChunk;
      const int m = mt * BM + quarter * 32 + lane;
      for (int chunk = 0; chunk < nchunks; ++chunk) {
        const bool add_old = chunk > 0 || p.epi == EPI_ACCUM;
        mbar_wait(&tfull_bar[acc], acc_phase);
        tc_fence_after();
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
                  const float4 c = *reinterpret_cast<const float4*>(dst + j);
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
      }
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
            const uint32_t base = smem_u32(ready + stage * kStageBytes);
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
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    tmem_dealloc(tmem_base, kTmemCols);
  }
}

// Deterministic split-K reduction: out[m, n] (=|+=) sum_{s=0..S-1} ws[s, m, n].
__global__ void splitk_reduce_kernel(const float* __restrict__ ws, float* __restrict__ out, int M, int N,
                                     long long ldc, int splits, int accumulate, const float* __restrict__ bias,
                                     int trans) {
  const long long total = (long long)M * N;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    long long m, n;
    if (trans) {  // out[n][m]: walk m fastest so the stores coalesce
      n = i / M;
      m = i - n * M;
    } else {
      m = i / N;
      n = i - m * N;
    }
    const long long e = m * N + n;
    float s = 0.f;
    for (int k = 0; k < splits; ++k) s += ws[(long long)k * total + e];
    if (bias) s += bias[n];
    float* o = trans ? out + n * ldc + m : out + m * ldc + n;
    *o = accumulate ? (*o + s) : s;
  }
}

}  // namespace monet
