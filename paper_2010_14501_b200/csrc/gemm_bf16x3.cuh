// bf16x3 tcgen05 persistent GEMM with the A operand staged in TMEM.
//
// Why this shape (profiles/ncu_gemm_r1.md): the 3xTF32 kernel (gemm_tc.cuh)
// is shared-memory-bandwidth bound -- every operand element crosses the
// 128 B/clk smem port five times (cp.async in, read back, hi + lo written,
// read three times by the MMAs) and the tensor pipe idles at ~25%.  Here:
//
//   * fp32 x = b0 + b1 with b0 = bf16(x), b1 = bf16(x - b0); the product
//     x*y ~= a0*b0 + a0*b1 + a1*b0 drops only terms of relative size 2^-18,
//     so three kind::f16 (bf16) MMAs -- at twice the TF32 rate -- give ~1e-5
//     relative accuracy, inside the rel 1e-4 parity bar;
//   * the A tile never goes back to shared memory: four "A-split" warps read
//     their own row of the raw fp32 tile, split it in registers and write
//     a_hi / a_lo straight into TMEM with tcgen05.st; the MMAs read A from
//     TMEM and only B (bf16 hi / lo, half the bytes of fp32) from smem.
//
// Warp roles (800 threads, one CTA per SM, persistent over output tiles):
//   warps 0-3   loaders (threads 0-63 A, 64-127 B): the raw fp32 k-block
//               (BK = 32) of each operand arrives by TMA -- tiled 2D / 3D maps
//               for plain operands, im2col maps (zero fill for padding) for
//               the fprop / stride-1 / phase dgrad / wgrad gathers -- issued
//               by one thread and completing on the slot's mbarrier
//               (expect_tx); shapes TMA cannot express fall back to 16B
//               cp.async groups from 64 threads (cp.async.mbarrier.arrive.noinc)
//   warps 4-11  A-split: lane quarter (warp & 3) x raw k-block of the stage;
//               LDS the row, split, tcgen05.st into the TMEM A stage
//   warps 12-19 B-split: raw fp32 -> bf16 hi / lo SWIZZLE_128B tiles
//   warps 20-23 epilogue: tcgen05.ld the 128x128 fp32 accumulator, store or
//               red.global.add (chunk flushes / accumulate)
//   warp  24    MMA issuer (one lane) and TMEM owner
//
// Measured limits (tools/gemm_waits.py, profiles/ncu_r1.md): with fp32
// operands a 128x128 tile moves 32 KB per 32-deep k-block from L2; the TMA
// issue path saturates near 6.6 TB/s chip-wide, which caps this shape at
// ~230 TF/s of useful work -- the next step is 256-wide tiles (cta_group::2).
#pragma once
#include "gemm_tc.cuh"

namespace monet {
namespace bx3 {

constexpr int BM = 128, BN = 128;
constexpr int BKR = 32;              // raw k-block (fp32, 128B rows)
constexpr int BKS = 64;              // MMA stage (bf16, 128B rows) = 2 raw k-blocks
constexpr int kRawTile = BM * BKR * 4;          // 16 KB (A or B raw, fp32)
constexpr int kAStages = 3;                      // MMA stages of A (TMEM)
constexpr int kLoaderWarps = 4, kASplitWarps = 8, kBSplitWarps = 8, kEpiWarps = 4;
constexpr int kLoaderThreads = kLoaderWarps * 32;
constexpr int kWarpASplit = kLoaderWarps;                       // 4
constexpr int kWarpBSplit = kWarpASplit + kASplitWarps;         // 12 (A split: 4 lane quarters x 2 halves)
constexpr int kWarpEpi = kWarpBSplit + kBSplitWarps;            // 16
constexpr int kWarpMma = kWarpEpi + kEpiWarps;                  // 20
constexpr int kThreads = (kWarpMma + 1) * 32;                   // 672
constexpr int kAccStages = 2;
constexpr int kTmemCols = 512;
constexpr int kTmemA = kAccStages * BN;          // A stages start at column 256
constexpr int kAStageCols = 64;                  // 32 cols hi + 32 cols lo (bf16x2 per column)
static_assert(kLoaderThreads == 128, "loader threads: 64 per operand");
constexpr int kOpLoaders = kLoaderThreads / 2;
constexpr int kBSplitThreads = kBSplitWarps * 32;
static_assert(kBSplitThreads == 256, "B split: 256 threads x 4 row groups");
static_assert(kTmemA + kAStages * kAStageCols <= kTmemCols, "TMEM budget");

// Shared-memory plan per B mode and N-tile width.  TMA delivery is latency bound (~2 us
// per box under load, tools/tma_bw_probe.cu), so the plan maximises bytes in flight:
//   fp32 B : raw slots hold an A and a B k-block, the B split fills bf16 stages;
//   pre-split B (OP_W16_*): raw slots hold A only, and the B stages -- filled by TMA
//            straight from the bf16 planes -- are deeper.
// A 64-wide N tile (NB = 64) halves every B buffer, which buys more slots.
template <int BMODE, int NB = BN>
struct Cfg {
  static constexpr bool kW16 = mode_is_w16(BMODE);
  static constexpr int kBTile = NB * BKS * 2;                   // bf16 hi (or lo) stage tile
  static constexpr int kStageBytes = 2 * kBTile;                // B hi + B lo
  static constexpr int kRawSlots = kW16 ? (NB == BN ? 4 : 6) : (NB == BN ? 4 : 6);
  static constexpr int kRawBytes = kW16 ? kRawTile : kRawTile + NB * BKR * 4;
  static constexpr int kBStages = kW16 ? (NB == BN ? 4 : 6) : (NB == BN ? 3 : 4);
  // pre-split-B kernels store the output through smem + TMA: two 32x32 fp32 blocks per epilogue warp
  static constexpr int kEpiBytes = kW16 ? kEpiWarps * 2 * 32 * 32 * 4 : 0;
  static constexpr int kStatBytes = kW16 ? kEpiWarps * 2 * 32 * 4 : 0;  // per-quarter (mean, M2) x 32 cols
  static constexpr int kNumBars = 2 * kRawSlots + 2 * kAStages + 2 * kBStages + 2 * kAccStages;
  static constexpr int kSmemBytes =
      kRawSlots * kRawBytes + kBStages * kStageBytes + kEpiBytes + kStatBytes + 1024 + 8 * kNumBars + 16;
  static_assert(kSmemBytes <= 232448, "shared memory budget");
};

MONET_DEV void cp_async_mbar_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// two fp32 -> packed bf16x2 (lo half = first argument), round to nearest even
MONET_DEV uint32_t pack_bf16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
// split a pair: hi2 = bf16x2(a, b); lo2 = bf16x2(a - hi(a), b - hi(b))
MONET_DEV void split_pair(float a, float b, uint32_t& hi2, uint32_t& lo2) {
  hi2 = pack_bf16x2(a, b);
  const float ah = __uint_as_float(hi2 << 16);
  const float bh = __uint_as_float(hi2 & 0xFFFF0000u);
  lo2 = pack_bf16x2(a - ah, b - bh);
}

template <int N>
MONET_DEV void tmem_st(uint32_t taddr, const uint32_t (&r)[N]);

template <>
MONET_DEV void tmem_st<16>(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
MONET_DEV void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// D[tmem] (+)= A[tmem] * B[smem]^T, kind::f16 (bf16 in, fp32 accumulate); one CTA,
// or (PR) the CTA pair: M = 256, A rows / B columns split across the two CTAs.
template <bool PR>
MONET_DEV void mma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  if constexpr (PR) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate));
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate));
  }
}

__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, int b_mn_major) {
  return (1u << 4)                 // D format F32
         | (1u << 7)               // A format BF16
         | (1u << 10)              // B format BF16
         | ((uint32_t)b_mn_major << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// B stage tile descriptors (bf16, SWIZZLE_128B), k16 slice kk (0..3).
//   K-major : rows n (128B = 64 k each), 8-row groups every 1024 B; k16 = +32 B
//   MN-major: 64-element MN chunks of 64 k-rows x 128 B (8 KB, LBO), 8-row
//             k groups every 1024 B (SBO); k16 = 16 rows = +2048 B
MONET_DEV uint64_t b_desc(uint32_t tile, bool mn, int kk) {
  if (mn) return smem_desc(tile + kk * 2048, BKS * 128, 1024, 2);
  return smem_desc(tile + kk * 32, 16, 1024, 2);
}

// byte offset of bf16 element (n, k) inside a B stage tile (k in 0..63)
MONET_DEV uint32_t b_off_kmajor(int n, int k) {
  const int g = k >> 3;  // 16B granule = 8 bf16
  return n * 128 + (((g ^ (n & 7)) << 4) | ((k & 7) << 1));
}
MONET_DEV uint32_t b_off_mnmajor(int n, int k) {
  const int g = (n & 63) >> 3;
  return (n >> 6) * (BKS * 128) + k * 128 + (((g ^ (k & 7)) << 4) | ((n & 7) << 1));
}

MONET_DEV void tile_range(const GemmParams& p, int tile, int& mt, int& nt, int& kb0, int& nstage) {
  int sp;
  tile_coords(p, tile, mt, nt, sp);
  int kb1;
  kb_range(p, sp, kb0, kb1);
  nstage = (kb1 - kb0 + 1) / 2;  // kb_per_split is even; only the last split may be odd -> zero-padded
}


// ------------------------------------------------------------------ loaders
MONET_DEV void mbar_arrive_tx(uint64_t* bar, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(tx) : "memory");
}
MONET_DEV void tma_2d(uint32_t dst, const CUtensorMap* m, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
          "r"(dst),
      "l"(m), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
MONET_DEV void tma_3d(uint32_t dst, const CUtensorMap* m, int x, int y, int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(dst),
      "l"(m), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}
// TMA store / reduce-add of a 32 x 32 fp32 smem block (SWIZZLE_128B) to the output map
// {N, M, splits}: rows past M are clipped per split
MONET_DEV void tma_store_3d(const CUtensorMap* m, uint32_t src, int x, int y, int z, bool add) {
  if (add)
    asm volatile("cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(m),
                 "r"(src), "r"(x), "r"(y), "r"(z)
                 : "memory");
  else
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(m),
                 "r"(src), "r"(x), "r"(y), "r"(z)
                 : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N>
MONET_DEV void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
MONET_DEV void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

MONET_DEV void tma_4d(uint32_t dst, const CUtensorMap* m, int c0, int c1, int c2, int c3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
      "%5}], [%6];" ::"r"(dst),
      "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}
MONET_DEV void tma_5d(uint32_t dst, const CUtensorMap* m, int c0, int c1, int c2, int c3, int c4, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, "
      "%6}], [%7];" ::"r"(dst),
      "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(bar))
      : "memory");
}
// im2col: coordinates {c, w, h, n} of the base pixel, offsets {w, h} of the filter tap
MONET_DEV void tma_im2col(uint32_t dst, const CUtensorMap* m, int c, int w, int h, int n, int ow, int oh,
                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
      "%5}], [%6], {%7, %8};" ::"r"(dst),
      "l"(m), "r"(c), "r"(w), "r"(h), "r"(n), "r"(smem_u32(bar)), "h"((uint16_t)ow), "h"((uint16_t)oh)
      : "memory");
}

// Address of the 4-element group starting at (row, k) -- generic fallback with
// divisions.  K-major modes: k..k+3 contiguous; MN-major: row..row+3 contiguous.
// Returns nullptr for padding / out-of-range groups (zero fill).
template <int MODE>
MONET_DEV const float* group_ptr(const GemmParams& p, const Operand& op, int row, int k) {
  const ConvGeom& g = p.g;
  if (row >= op.rows || k >= p.Kd) return nullptr;
  if constexpr (MODE == OP_KMAJOR) {
    return op.ptr + (long long)row * op.ld + k;
  } else if constexpr (MODE == OP_MNMAJOR) {
    const int kh = k / op.kdiv, kl = k - kh * op.kdiv;
    const int th = p.ph.on ? p.ph.tap[kh] : kh;  // phase dgrad: phase tap -> filter tap
    return op.ptr + th * op.ks1 + (long long)kl * op.ld + row;
  } else if constexpr (MODE == OP_IM2COL_FPROP) {
    const int q = row % g.Q, t = row / g.Q, pp = t % g.P, n = t / g.P;
    const int tap = k / g.C, c = k - tap * g.C, r = tap / g.S, s = tap - r * g.S;
    const int h = pp * g.sh - g.ph + r, w = q * g.sw - g.pw + s;
    if ((unsigned)h >= (unsigned)g.H || (unsigned)w >= (unsigned)g.W) return nullptr;
    return op.ptr + (((long long)n * g.H + h) * g.W + w) * g.C + c;
  } else if constexpr (MODE == OP_IM2COL_DGRAD) {
    if (p.ph.on) {
      const int j = row % p.ph.Wp, t = row / p.ph.Wp, i = t % p.ph.Hp, n = t / p.ph.Hp;
      const int tp = k / g.K, ko = k - tp * g.K;
      const int pp = i + p.ph.dr[tp], q = j + p.ph.ds[tp];
      if ((unsigned)pp >= (unsigned)g.P || (unsigned)q >= (unsigned)g.Q) return nullptr;
      return op.ptr + (((long long)n * g.P + pp) * g.Q + q) * g.K + ko;
    }
    const int w = row % g.W, t = row / g.W, h = t % g.H, n = t / g.H;
    const int tap = k / g.K, ko = k - tap * g.K, r = tap / g.S, s = tap - r * g.S;
    const int hp = h + g.ph - r, wp = w + g.pw - s;
    if (hp < 0 || wp < 0) return nullptr;
    const int pp = hp / g.sh, q = wp / g.sw;
    if (pp * g.sh != hp || q * g.sw != wp || pp >= g.P || q >= g.Q) return nullptr;
    return op.ptr + (((long long)n * g.P + pp) * g.Q + q) * g.K + ko;
  } else {  // OP_IM2COL_WGRAD: rows (tap, c), k = output pixel
    const int tap = row / g.C, c = row - tap * g.C, r = tap / g.S, s = tap - r * g.S;
    const int q = k % g.Q, t = k / g.Q, pp = t % g.P, n = t / g.P;
    const int h = pp * g.sh - g.ph + r, w = q * g.sw - g.pw + s;
    if ((unsigned)h >= (unsigned)g.H || (unsigned)w >= (unsigned)g.W) return nullptr;
    return op.ptr + (((long long)n * g.H + h) * g.W + w) * g.C + c;
  }
}

// Raw k-block layouts in smem (what the splitters read):
//   K-major : 128 rows x 128 B, SWIZZLE_128B (16B chunk c of row r at
//             r*128 + ((c ^ (r & 7)) << 4)) -- TMA tiled / im2col box layout
//   MN-major: segment-major, `seg` rows per segment (128, or C = 32 / 64 for a
//             wgrad tile spanning several taps): element (row, k) at
//             (row / seg) * 32 * seg * 4 + k * seg * 4 + (row % seg) * 4
MONET_DEV uint32_t mn_off(int row, int kr, int seg) {
  const int sg = row / seg;
  return sg * (BKR * seg * 4) + kr * seg * 4 + (row - sg * seg) * 4;
}

// One operand's loader.  TMA operands: one elected thread (sub == 0) issues
// the whole k-block; fallback operands: 128 threads issue 16B cp.async groups.
template <int MODE>
struct Loader {
  static constexpr bool kMN = mode_is_mn(MODE);
  int row0, k0;
  int cw, chh, cn;          // im2col base pixel of the tile (FPROP / DGRAD)
  int kin0, tap_r, tap_s;   // k-block decomposition (FPROP / DGRAD)

  MONET_DEV void init(const GemmParams& p, const Operand& op, int row0_, int k0_) {
    const ConvGeom& g = p.g;
    row0 = row0_;
    k0 = k0_;
    if constexpr (MODE == OP_IM2COL_WGRAD) {
      if (op.tma == 4) tap_r = row0 / (g.S * g.C);  // tap view: first filter row of the n-tile
    }
    if (op.tma < 2) return;
    if constexpr (MODE == OP_IM2COL_FPROP || MODE == OP_IM2COL_DGRAD) {
      const bool fp = MODE == OP_IM2COL_FPROP;
      const bool phs = !fp && p.ph.on;
      const int X = fp ? g.Q : (phs ? p.ph.Wp : g.W), Y = fp ? g.P : (phs ? p.ph.Hp : g.H);
      const int x = row0 % X, t = row0 / X, y = t % Y;
      cn = t / Y;
      if (fp) {
        cw = x * g.sw - g.pw;
        chh = y * g.sh - g.ph;
      } else if (phs) {
        cw = x + p.ph.lo_w;
        chh = y + p.ph.lo_h;
      } else {
        cw = x - (g.S - 1 - g.pw);
        chh = y - (g.R - 1 - g.ph);
      }
      const int cx = fp ? g.C : g.K;
      const int tap = k0 / cx;
      kin0 = k0 - tap * cx;
      if (phs) {  // phase dgrad: tap_s walks the phase's tap list
        tap_r = 0;
        tap_s = tap;
      } else {
        tap_r = tap / g.S;
        tap_s = tap - tap_r * g.S;
      }
    }
  }

  // go == false: only advance the incremental im2col coordinates (another issuer owns kb)
  MONET_DEV void issue_tma(const GemmParams& p, const Operand& op, const CUtensorMap* m, int kb, uint8_t* tile,
                           uint64_t* bar, bool go = true) {
    const ConvGeom& g = p.g;
    const uint32_t dst = smem_u32(tile);
    const int k = kb * BKR;
    if constexpr (MODE == OP_KMAJOR) {
      if (go) mbar_arrive_tx(bar, op.rows_box * BKR * 4);
      if (go) tma_2d(dst, m, k, row0, bar);
    } else if constexpr (MODE == OP_MNMAJOR) {
      if (go) mbar_arrive_tx(bar, op.rows_box * BKR * 4);
      if (op.tma == 4) {  // wgrad tap view: dy as {kout, q, n*p}
        const int np = k / p.wv_q;
        if (go) tma_3d(dst, m, row0, k - np * p.wv_q, np, bar);
      } else if (op.kdiv >= p.Kd && !p.ph.on) {
        if (go) tma_2d(dst, m, row0, k, bar);
      } else {  // k = tap * kdiv + kout, kdiv % 32 == 0: tensor {rows, taps, kdiv}
        const int kh = k / op.kdiv;
        if (go) tma_3d(dst, m, row0, p.ph.on ? p.ph.tap[kh] : kh, k - kh * op.kdiv, bar);
      }
    } else if constexpr (MODE == OP_IM2COL_FPROP) {
      if (op.tma == 5) {  // fprop tap view: one box {32 (s, c), 128 q, filter row kb, p, n} per k-block
        if (go) mbar_arrive_tx(bar, BM * BKR * 4);
        const int t = row0 / p.fv_q;
        if (go) tma_5d(dst, m, 0, 0, kb, t % g.P, t / g.P, bar);
        return;
      }
      if (op.tma == 3) {  // C < 32: the k-block spans 32 / C filter taps, one C-channel box each
        if (go) mbar_arrive_tx(bar, BM * BKR * 4);
        const int ntb = BKR / g.C;
        for (int j = 0; j < ntb; ++j) {
          const bool valid = tap_r < g.R;
          if (go) tma_im2col(dst + j * (BM * g.C * 4), m, valid ? 0 : g.C, cw, chh, cn, valid ? tap_s : 0,
                     valid ? tap_r : 0, bar);
          if (++tap_s == g.S) {
            tap_s = 0;
            ++tap_r;
          }
        }
        return;
      }
    }
    if constexpr (MODE == OP_KMAJOR || MODE == OP_MNMAJOR) {
      // issued above
    } else if constexpr (MODE == OP_IM2COL_FPROP || MODE == OP_IM2COL_DGRAD) {
      if (go) mbar_arrive_tx(bar, BM * BKR * 4);
      const bool phs = MODE == OP_IM2COL_DGRAD && p.ph.on;
      if (k < p.Kd) {
        int ow, oh;
        if (MODE == OP_IM2COL_FPROP) {
          ow = tap_s;
          oh = tap_r;
        } else if (phs) {
          ow = p.ph.ds[tap_s] - p.ph.lo_w;
          oh = p.ph.dr[tap_s] - p.ph.lo_h;
        } else {
          ow = g.S - 1 - tap_s;
          oh = g.R - 1 - tap_r;
        }
        if (go) tma_im2col(dst, m, kin0, cw, chh, cn, ow, oh, bar);
      } else {  // zero-padded tail k-block: out-of-range channel coordinate -> zero fill
        if (go) tma_im2col(dst, m, MODE == OP_IM2COL_FPROP ? g.C : g.K, cw, chh, cn, 0, 0, bar);
      }
      const int cx = MODE == OP_IM2COL_FPROP ? g.C : g.K;
      kin0 += BKR;
      if (kin0 >= cx) {
        kin0 = 0;
        if (++tap_s == g.S && !phs) {
          tap_s = 0;
          ++tap_r;
        }
      }
    } else if (op.tma == 4) {  // wgrad tap view: one box {S*C, 32 q, R-segments, 1, 1}
      if (go) mbar_arrive_tx(bar, op.rows_box * BKR * 4);
      const int np = k / p.wv_q, pp = np % g.P;
      if (go) tma_5d(dst, m, 0, k - np * p.wv_q, tap_r, pp, np / g.P, bar);
    } else {  // IM2COL_WGRAD: rows (tap, c) in segments of op.seg channels, k = 32 output pixels
      const int seg = op.seg;
      if (go) mbar_arrive_tx(bar, op.rows_box * BKR * 4);
      const int q = k % g.Q, t = k / g.Q, pp = t % g.P, n = t / g.P;
      const int w0 = q * g.sw - g.pw, h0 = pp * g.sh - g.ph;
      for (int sg = 0; sg < op.rows_box / seg; ++sg) {
        const int row = row0 + sg * seg;
        const int tap = row / g.C, c = row - tap * g.C;
        const int r = tap / g.S, s = tap - r * g.S;
        // rows past R*S*C: the tap offset stays in range, the channel
        // coordinate is pushed out of bounds (zero fill)
        const bool valid = tap < g.R * g.S && k < p.Kd;
        if (go) tma_im2col(dst + sg * (BKR * seg * 4), m, valid ? c : g.C, w0, h0, n, valid ? s : 0, valid ? r : 0, bar);
      }
    }
  }

  MONET_DEV void issue_fallback(const GemmParams& p, const Operand& op, int kb, int sub, uint8_t* tile,
                                uint64_t* bar) {
    const int kk0 = kb * BKR;
#pragma unroll 2
    for (int i = 0; i < 16; ++i) {  // 64 threads x 16 groups of 16B = one 16 KB tile
      int row, k;
      uint32_t off;
      if constexpr (kMN) {
        const int kr = (sub >> 5) + 2 * i;
        const int r = 4 * (sub & 31);
        if (r >= op.rows_box) continue;  // the B half of a CTA pair covers 64 rows
        row = row0 + r;
        k = kk0 + kr;
        off = mn_off(r, kr, op.seg);
      } else {
        const int r = (sub >> 3) + 8 * i;
        if (r >= op.rows_box) continue;
        row = row0 + r;
        k = kk0 + 4 * (sub & 7);
        off = sw128_offset(r, sub & 7);
      }
      const float* src = group_ptr<MODE>(p, op, row, k);
      const uint32_t dst = smem_u32(tile + off);
      if (op.aligned || src == nullptr) {
        cp_async16(dst, src, op.ptr);
      } else {
        const int cnt = kMN ? op.rows - row : p.Kd - k;
#pragma unroll
        for (int e = 0; e < 4; ++e) cp_async4(dst + 4 * e, e < cnt ? src + e : op.ptr, e < cnt);
      }
    }
    cp_async_mbar_arrive(bar);
  }
};
// BN statistics of a 128-row output tile from the epilogue (the conv -> BN forward): after the
// warp has staged its 32x32 block in smem (SWIZZLE_128B, row r = lane r), lane l walks column l
// down the 32 rows -- conflict-free, a handful of registers -- summing around the block's first
// row (a pivot); the four warps' (mean, M2) meet in smem and warp 0 merges them in order (Chan)
// into stats[mt][0|1][n].  One named-barrier pair per 32-column chunk among the four epilogue
// warps.  Deterministic.
MONET_DEV void tile_stats(const GemmParams& p, const uint8_t* blk, float* sm, int row0, int quarter, int lane, int n0,
                          int mt) {
  const int rows_here = min(32, p.M - (row0 + quarter * 32));
  const int cc = lane >> 2, cw = (lane & 3) * 4;  // 16-B chunk and byte offset of column `lane`
  float mean = 0.f, m2 = 0.f;
  if (rows_here > 0) {
    const float piv = *reinterpret_cast<const float*>(blk + ((cc ^ 0) << 4) + cw);
    float s1 = 0.f, s2 = 0.f;
#pragma unroll 8
    for (int r = 1; r < 32; ++r) {
      if (r < rows_here) {
        const float d = *reinterpret_cast<const float*>(blk + r * 128 + ((cc ^ (r & 7)) << 4) + cw) - piv;
        s1 += d;
        s2 += d * d;
      }
    }
    const float inv = 1.f / (float)rows_here;
    mean = piv + s1 * inv;
    m2 = fmaxf(s2 - s1 * s1 * inv, 0.f);
  }
  sm[(quarter * 2) * 32 + lane] = mean;
  sm[(quarter * 2 + 1) * 32 + lane] = m2;
  asm volatile("bar.sync 1, 128;" ::: "memory");
  if (quarter == 0 && n0 + lane < p.N) {
    float n = 0.f, mu = 0.f, sq = 0.f;
#pragma unroll
    for (int qq = 0; qq < 4; ++qq) {
      const int c = min(32, p.M - (row0 + qq * 32));
      if (c <= 0) break;
      const float mb = sm[(qq * 2) * 32 + lane], sb = sm[(qq * 2 + 1) * 32 + lane];
      const float nn = n + (float)c, delta = mb - mu;
      mu += delta * ((float)c / nn);
      sq += sb + delta * delta * (n * (float)c / nn);
      n = nn;
    }
    p.stats[(long long)(mt * 2) * p.N + n0 + lane] = mu;
    p.stats[(long long)(mt * 2 + 1) * p.N + n0 + lane] = sq;
  }
  asm volatile("bar.sync 1, 128;" ::: "memory");
}

// Debug wait-time accounting (p.dbg_t != nullptr): counters per CTA
//   0 loader raw_empty, 3 MMA a_full, 4 MMA b_full, 5 MMA tempty, 6 epilogue tfull,
//   7 A-split st_empty, 8 A-split raw_full, 9 B-split st_empty, 10 B-split raw_full,
//   11 MMA issue (first MMA to commit, lane 0), 15 kernel cycles
#define TWAIT(slot, expr)                                   \
  do {                                                      \
    const long long t0_ = p.dbg_t ? clock64() : 0;          \
    expr;                                                   \
    if (p.dbg_t) twait[slot] += clock64() - t0_;            \
  } while (0)

// PR (CTA pair, cta_group::2): the two CTAs of a cluster compute a 256 x 128
// tile -- each splits its own 128 A rows into its own TMEM and 64 of the 128 B
// rows into its own smem; the leader (rank 0) issues M=256 MMAs that read both
// halves, commits are multicast to both CTAs, and the producer / epilogue
// arrivals the leader waits on come per warp from both CTAs.  Per SM the B
// traffic through shared memory halves (the limiter of the 1-CTA kernel).
//
// NB (N-tile width): 128, or 64 for problems with N <= 64 (64-channel convs):
// half the B rows and half the MMA width per stage, same A work.
// ST: the epilogue also leaves BN statistics (p.stats) -- its own instantiation, so the plain
// kernels carry none of that code (register allocation of the epilogue stays unchanged)
template <int AM, int BMODE, bool PR, int NB, bool ST = false>
__global__ void __launch_bounds__(kThreads, 1) gemm_bf16x3_kernel(const __grid_constant__ GemmParams p) {
  static_assert(NB == BN || (NB == 64 && !PR), "tile widths: 128 (1 CTA or pair), 64 (1 CTA)");
  constexpr bool a_mn = mode_is_mn(AM), b_mn = mode_is_mn(BMODE);
  using CF = Cfg<BMODE, NB>;
  constexpr bool kW16 = CF::kW16;
  constexpr int kRawSlots = CF::kRawSlots, kRawBytes = CF::kRawBytes, kBStages = CF::kBStages;
  constexpr int kBTile = CF::kBTile, kStageBytes = CF::kStageBytes;
  static_assert(!(kW16 && PR), "pre-split B: one CTA per tile");
  constexpr int kPairN = PR ? 2 : 1;          // CTAs per tile
  constexpr int kBRows = NB / kPairN;         // B rows this CTA splits
  constexpr int kBChunks = kBRows / 32;       // K-major 16B chunks per B-split thread per raw k-block
  constexpr int kTileM = BM * kPairN;
  extern __shared__ uint8_t smem_raw[];
  // 1024-B align by offsetting the __shared__ array itself (not via an integer
  // round trip) so the compiler keeps the shared address space: LDS / STS
  // instead of generic LD / ST in the splitters
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* raw = smem;                                  // kRawSlots x (A[, B]) fp32
  uint8_t* bst = smem + kRawSlots * kRawBytes;          // kBStages x (B hi, B lo) bf16
  uint8_t* epi_st = bst + kBStages * kStageBytes;       // epilogue staging (pre-split-B kernels)
  float* stat_sm = reinterpret_cast<float*>(epi_st + CF::kEpiBytes);  // BN statistics exchange
  uint64_t* bars = reinterpret_cast<uint64_t*>(epi_st + CF::kEpiBytes + CF::kStatBytes);
  uint64_t* raw_full = bars;                            // loaders -> splitters
  uint64_t* raw_empty = raw_full + kRawSlots;           // splitters -> loaders
  uint64_t* a_full = raw_empty + kRawSlots;             // A-split -> MMA
  uint64_t* b_full = a_full + kAStages;                 // B-split (or pre-split B TMA) -> MMA
  uint64_t* a_empty = b_full + kBStages;                // MMA commit -> A-split
  uint64_t* b_empty = a_empty + kAStages;               // MMA commit -> B-split / B loader
  uint64_t* tfull = b_empty + kBStages;                 // MMA commit -> epilogue
  uint64_t* tempty = tfull + kAccStages;                // epilogue -> MMA
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + kAccStages);

  const int warp = warp_id();
  const int lane = lane_id();
  const int n_tiles_total = p.m_tiles * p.n_tiles * p.splits;
  const uint32_t rank = PR ? cluster_ctarank() : 0u;
  const int unit0 = PR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;  // persistent tile loop: one unit per pair
  const int n_units = PR ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  // arrivals the MMA issuer waits on: per warp, to the leader CTA's barrier
  auto arrive_leader = [&](uint64_t* bar) {
    __syncwarp();
    if (lane == 0) {
      if constexpr (PR)
        mbar_arrive_cluster(mapa_shared(bar, 0));
      else
        mbar_arrive(bar);
    }
  };
#ifdef MONET_DEBUG
  const int dm = p.dbg_mode;
#else
  constexpr int dm = 0;
#endif
  long long twait[16] = {0};
  float* const dbg_a = p.dbg_a;  // hoisted: loop-invariant kernel parameters
  float* const dbg_b = p.dbg_b;
  const long long t_start = clock64();

  if (threadIdx.x == 0) {
    for (int s = 0; s < kRawSlots; ++s) {
      mbar_init(&raw_full[s], (p.a.tma ? 1 : kOpLoaders) + (kW16 ? 0 : (p.b.tma ? 1 : kOpLoaders)));
      // one A half (+ all of B) per item
      mbar_init(&raw_empty[s], (kASplitWarps / 2 + (kW16 ? 0 : kBSplitWarps)) * 32);
    }
    for (int s = 0; s < kAStages; ++s) {
      mbar_init(&a_full[s], kASplitWarps * kPairN);
      mbar_init(&a_empty[s], 1);
    }
    for (int s = 0; s < kBStages; ++s) {
      mbar_init(&b_full[s], kW16 ? 1 : kBSplitWarps * kPairN);
      mbar_init(&b_empty[s], 1);
    }
    for (int a = 0; a < kAccStages; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], kEpiWarps * kPairN);
    }
    mbar_fence_init();
  }
  if (warp == kWarpMma) {
    if constexpr (PR)
      tmem_alloc_pair(tmem_slot, kTmemCols);
    else
      tmem_alloc(tmem_slot, kTmemCols);
  }
  tc_fence_before();
  if constexpr (PR)
    cluster_sync();  // the peer's barriers are initialised before any remote arrive
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp < kLoaderWarps) {
    // ---------------------------------------------------------------- loaders
    const int sub = threadIdx.x % kOpLoaders;
    const bool is_b = threadIdx.x >= kOpLoaders;
    if constexpr (kW16) {
      // pre-split B: one thread streams each 64-deep stage's bf16 hi / lo boxes straight
      // into the B stage tiles (K-major: one box per plane; MN-major: 64-channel chunks x
      // two 32-deep k halves per plane)
      // two issuers (lane 0 of each B loader warp) taking alternate stages; one for the sub-pixel
      // phase GEMMs of a strided dgrad (with two, those came out wrong and non-deterministic once
      // CTAs ran several tiles -- tools/dgrad_phase_check.py; cause not isolated)
      const int niss = ((dm & 16) || p.ph.on) ? 1 : 2;
      if (is_b && (sub & 31) == 0 && (sub >> 5) < niss) {
        const int iss = sub >> 5;
        int sitem = 0;
        for (int tile = unit0; tile < n_tiles_total; tile += n_units) {
          int mt, nt, kb0, nst;
          tile_range(p, tile, mt, nt, kb0, nst);
          const int n0 = nt * p.n_pitch;
          for (int s = 0; s < nst; ++s, ++sitem) {
            if ((sitem % niss) != iss) continue;
            const int sb = sitem % kBStages;
            TWAIT(0, mbar_wait(&b_empty[sb], ((sitem / kBStages) & 1) ^ 1));
            const uint32_t hi = smem_u32(bst + sb * kStageBytes), lo = hi + kBTile;
            uint64_t* bar = &b_full[sb];
            const int k0 = (kb0 + 2 * s) * BKR;
            if constexpr (BMODE == OP_W16_KMAJOR) {
              mbar_arrive_tx(bar, 2 * p.b.rows_box * 128);
              tma_3d(hi, &p.tma_b, k0, n0, 0, bar);
              tma_3d(lo, &p.tma_b, k0, n0, 1, bar);
            } else {
              const int nch = (p.b.rows_box + 63) / 64;
              mbar_arrive_tx(bar, 2 * 2 * nch * (BKR * 128));
              for (int h = 0; h < 2; ++h) {
                const int k = k0 + h * BKR;
                int tap = 0, ko = p.b.kdiv;  // past Kd (odd tail of the last split): zero fill
                if (k < p.Kd) {
                  const int kh = k / p.b.kdiv;
                  ko = k - kh * p.b.kdiv;
                  tap = p.ph.on ? p.ph.tap[kh] : kh;
                }
                for (int c = 0; c < nch; ++c) {
                  const uint32_t off = c * (BKS * 128) + h * (BKR * 128);
                  tma_4d(hi + off, &p.tma_b, n0 + 64 * c, tap, ko, 0, bar);
                  tma_4d(lo + off, &p.tma_b, n0 + 64 * c, tap, ko, 1, bar);
                }
              }
            }
          }
        }
      }
    }
    const Operand& op = is_b ? p.b : p.a;
    // TMA operands: lane 0 of each of the operand's two warps issues every other k-block --
    // a thread issues about one box per ~500 clk (tools/tma_bw_probe.cu), so one issuer
    // would cap delivery near 16 KB / 500 clk per SM; pre-split B is streamed above
    const bool active = (kW16 && is_b) ? false : (!op.tma || (sub & 31) == 0);
    const int issuer = op.tma ? sub >> 5 : 0;
    Loader<AM> la;
    Loader<BMODE> lb;
    int item = 0;
    for (int tile = active ? unit0 : n_tiles_total; tile < n_tiles_total; tile += n_units) {
      int mt, nt, kb0, nst;
      tile_range(p, tile, mt, nt, kb0, nst);
      if (is_b) {
        if constexpr (!kW16) lb.init(p, p.b, nt * p.n_pitch + (int)rank * kBRows, kb0 * BKR);
      } else
        la.init(p, p.a, mt * kTileM + (int)rank * BM, kb0 * BKR);
      for (int kb = kb0; kb < kb0 + 2 * nst; ++kb, ++item) {
        const int slot = item % kRawSlots;
        if (!op.tma || (item & 1) == issuer) TWAIT(0, mbar_wait(&raw_empty[slot], ((item / kRawSlots) & 1) ^ 1));
        uint8_t* base = raw + slot * kRawBytes;
        if (is_b) {
          if constexpr (!kW16) {
            if (op.tma)
              lb.issue_tma(p, op, &p.tma_b, kb, base + kRawTile, &raw_full[slot], (item & 1) == issuer);
            else
              lb.issue_fallback(p, op, kb, sub, base + kRawTile, &raw_full[slot]);
          }
        } else {
          if (op.tma)
            la.issue_tma(p, op, &p.tma_a, kb, base, &raw_full[slot], (item & 1) == issuer);
          else
            la.issue_fallback(p, op, kb, sub, base, &raw_full[slot]);
        }
      }
    }
    cp_async_wait<0>();
  } else if (warp < kWarpBSplit) {
    // ---------------------------------------------------------------- A split -> TMEM
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t lane_sel = (uint32_t)(quarter * 32) << 16;
    const int half = (warp - kWarpASplit) >> 2;  // which raw k-block of each stage this warp splits
    int stage_item = 0;
    for (int tile = unit0; tile < n_tiles_total; tile += n_units) {
      int mt, nt, kb0, nst;
      tile_range(p, tile, mt, nt, kb0, nst);
      const int item_kb0 = kb0;
      for (int s = 0; s < nst; ++s, ++stage_item) {
        const int stage = stage_item % kAStages;
        TWAIT(7, mbar_wait(&a_empty[stage], ((stage_item / kAStages) & 1) ^ 1));
        tc_fence_after();
        const uint32_t a_hi = tmem_base + lane_sel + kTmemA + stage * kAStageCols;
        do {  // a block (the debug skip's continue leaves it)
          const int item = 2 * stage_item + half;
          const int slot = item % kRawSlots;
          TWAIT(8, mbar_wait(&raw_full[slot], (item / kRawSlots) & 1));
          if (dm & 1) {
            mbar_arrive(&raw_empty[slot]);
            continue;
          }
          const uint8_t* rt = raw + slot * kRawBytes;
          float v[32];
          if constexpr (a_mn) {  // segment-major (mn_off): p.a.seg rows per segment
            const int seg = p.a.seg, sg = row / seg;
            const uint8_t* base = rt + sg * (BKR * seg * 4) + (row - sg * seg) * 4;
#pragma unroll
            for (int k = 0; k < 32; ++k) v[k] = *reinterpret_cast<const float*>(base + k * seg * 4);
          } else if (p.a.tma == 3) {  // chunk-major: tap box j holds C channels per row
            const int cb = p.g.C * 4;
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              const int e = 4 * c, j = e / p.g.C, ch = e - j * p.g.C;
              const float4 q = *reinterpret_cast<const float4*>(rt + j * (BM * cb) + row * cb + ch * 4);
              v[4 * c] = q.x;
              v[4 * c + 1] = q.y;
              v[4 * c + 2] = q.z;
              v[4 * c + 3] = q.w;
            }
          } else {
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              const float4 q = *reinterpret_cast<const float4*>(rt + sw128_offset(row, c));
              v[4 * c] = q.x;
              v[4 * c + 1] = q.y;
              v[4 * c + 2] = q.z;
              v[4 * c + 3] = q.w;
            }
          }
          if (dbg_a != nullptr) {
            const long long kpad = (long long)((p.Kd + 63) / 64) * 64;
            const int kb = (item_kb0 + 2 * s + half);
            const int m = mt * kTileM + (int)rank * BM + row;
            if (m < p.M)
              for (int k = 0; k < 32; ++k) dbg_a[m * kpad + kb * 32 + k] = v[k];
          }
          uint32_t hi[16], lo[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) split_pair(v[2 * j], v[2 * j + 1], hi[j], lo[j]);
          // release the raw slot only once every loaded value has been consumed:
          // the next TMA into it is an async-proxy write that is not ordered
          // behind LDS still in flight
          mbar_arrive(&raw_empty[slot]);
          tmem_st<16>(a_hi + half * 16, hi);
          tmem_st<16>(a_hi + 32 + half * 16, lo);
        } while (0);
        tmem_st_wait();
        tc_fence_before();
        arrive_leader(&a_full[stage]);
      }
    }
  } else if (warp < kWarpEpi) {
    // ---------------------------------------------------------------- B split -> smem bf16
    if constexpr (!kW16) {  // (pre-split B needs no split: these warps idle)
    const int t = threadIdx.x - kWarpBSplit * 32;  // 0..255
    int item = 0, stage_item = 0;
    for (int tile = unit0; tile < n_tiles_total; tile += n_units) {
      int mt, nt, kb0, nst;
      tile_range(p, tile, mt, nt, kb0, nst);
      for (int s = 0; s < nst; ++s, ++stage_item) {
        const int stage = stage_item % kBStages;
        TWAIT(9, mbar_wait(&b_empty[stage], ((stage_item / kBStages) & 1) ^ 1));
        uint8_t* bhi = bst + stage * kStageBytes;
        uint8_t* blo = bhi + kBTile;
#pragma unroll 1
        for (int half = 0; half < 2; ++half, ++item) {
          const int slot = item % kRawSlots;
          TWAIT(10, mbar_wait(&raw_full[slot], (item / kRawSlots) & 1));
          if (dm & 2) {
            mbar_arrive(&raw_empty[slot]);
            continue;
          }
          const uint8_t* rt = raw + slot * kRawBytes + kRawTile;
          // K-major: a warp covers rows {0,4,1,5}+base so that the two rows of
          // one 16-lane STS.64 phase land in opposite swizzle halves.
          // MN-major: 4-row group g of k-rows kr0 + kstep * i.
          const int w8 = t >> 5, l = t & 31;
          const int rbase = 8 * (w8 >> 1) + 2 * (w8 & 1) + (((l >> 3) & 1) << 2) + (l >> 4);
          constexpr int kGroups = kBRows / 4, kStep = 256 / kGroups;
          const int g = t % kGroups, kr0 = t / kGroups;
          float4 q[kBChunks];
#pragma unroll
          for (int i = 0; i < kBChunks; ++i) {
            uint32_t off;
            if constexpr (b_mn) {
              off = mn_off(4 * g, kr0 + kStep * i, p.b.seg);
            } else {
              off = sw128_offset(rbase + 32 * i, t & 7);
            }
            q[i] = *reinterpret_cast<const float4*>(rt + off);
          }
          if (dbg_b != nullptr) {
            const long long kpad = (long long)((p.Kd + 63) / 64) * 64;
            const int kb = kb0 + 2 * s + half;
            for (int i = 0; i < kBChunks; ++i) {
              const float e[4] = {q[i].x, q[i].y, q[i].z, q[i].w};
              for (int j = 0; j < 4; ++j) {
                int n, k;
                if (b_mn) {
                  n = 4 * g + j;
                  k = kr0 + kStep * i;
                } else {
                  n = rbase + 32 * i;
                  k = 4 * (t & 7) + j;
                }
                n += nt * p.n_pitch + (int)rank * kBRows;
                if (n < p.N) dbg_b[n * kpad + kb * 32 + k] = e[j];
              }
            }
          }
#pragma unroll
          for (int i = 0; i < kBChunks; ++i) {
            uint2 h, lw;
            split_pair(q[i].x, q[i].y, h.x, lw.x);
            split_pair(q[i].z, q[i].w, h.y, lw.y);
            uint32_t off;
            if constexpr (b_mn) {
              off = b_off_mnmajor(4 * g, 32 * half + kr0 + kStep * i);
            } else {
              off = b_off_kmajor(rbase + 32 * i, 32 * half + 4 * (t & 7));
            }
            *reinterpret_cast<uint2*>(bhi + off) = h;
            *reinterpret_cast<uint2*>(blo + off) = lw;
          }
          mbar_arrive(&raw_empty[slot]);  // after all loaded values are consumed (see A split)
        }
        fence_proxy_async_smem();
        arrive_leader(&b_full[stage]);
      }
    }
    }  // !kW16
  } else if (warp < kWarpMma) {
    // ---------------------------------------------------------------- epilogue
    const int quarter = warp & 3;
    int acc = 0;
    uint32_t acc_phase = 0;
    int epi_stores = 0;  // TMA-store epilogue: bulk stores issued by this warp
    for (int tile = unit0; tile < n_tiles_total; tile += n_units) {
      int mt, nt, sp, kb0, kb1;
      tile_coords(p, tile, mt, nt, sp);
      kb_range(p, sp, kb0, kb1);
      const int nst = (kb1 - kb0 + 1) / 2;
      const int nchunks = (nst + p.chunk_stages - 1) / p.chunk_stages;
      const int m = mt * kTileM + (int)rank * BM + quarter * 32 + lane;
      long long out_row = m;  // phase dgrad: scatter row (n, i, j) to dx[n][i*sh + a][j*sw + b]
      bool row_ok = m < p.M;
      if (p.ph.on && m < p.M) {
        const int j = m % p.ph.Wp, t = m / p.ph.Wp, i = t % p.ph.Hp, n = t / p.ph.Hp;
        out_row = ((long long)n * p.g.H + i * p.g.sh + p.ph.a) * p.g.W + j * p.g.sw + p.ph.b;
      }
      if (p.fv_q) {  // fprop tap view: row (n, p, q < fv_q); q >= Q are padding rows
        const int q = m % p.fv_q;
        row_ok = row_ok && q < p.g.Q;
        out_row = (long long)(m / p.fv_q) * p.g.Q + q;
      }
      for (int chunk = 0; chunk < nchunks; ++chunk) {
        // later chunks (and accumulate mode) add with fire-and-forget vector
        // reductions: no read-back latency, and one thread owns each element,
        // so the order of the adds is fixed (deterministic)
        const bool add_old = chunk > 0 || p.epi == EPI_ACCUM;
        const bool add_bias = p.bias != nullptr && chunk == 0 && p.epi == EPI_STORE;
        TWAIT(6, mbar_wait(&tfull[acc], acc_phase));
        tc_fence_after();
        if constexpr (kW16) {
          if (p.c_tma) {
            // 32x32 blocks staged in smem (SWIZZLE_128B: conflict-free row writes) and stored by one
            // TMA per block -- full 128-B lines instead of 16-B pieces of 32 rows per instruction.
            // A later chunk's reduce-add waits for the earlier flushes of the tile to land, so the
            // adds to an element happen in chunk order (deterministic).
            if (chunk > 0 && lane == 0) bulk_wait_all();
            __syncwarp();
            const int mrow = mt * kTileM + quarter * 32, zs = p.epi == EPI_PARTIAL ? sp : 0;
            for (int cc = 0; cc < NB / 32; ++cc) {
              float v[32];
              tmem_ld32(tmem_base + acc * NB + cc * 32 + ((uint32_t)(quarter * 32) << 16), v);
              const int n0 = nt * p.n_pitch + cc * 32;
              if (n0 >= p.N) continue;  // a trailing chunk of a partial n-tile: nothing to store
              if (add_bias) {
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] += (n0 + j < p.N) ? __ldg(p.bias + n0 + j) : 0.f;
              }
              // the warp's two staging blocks alternate per store (not per chunk: skipped chunks
              // would break the pairing); wait until the store two back has read its block
              uint8_t* blk = epi_st + (quarter * 2 + (epi_stores & 1)) * 4096;
              ++epi_stores;
              if (lane == 0) bulk_wait_read<1>();
              __syncwarp();
#pragma unroll
              for (int c = 0; c < 8; ++c)
                *reinterpret_cast<float4*>(blk + lane * 128 + ((c ^ (lane & 7)) << 4)) =
                    make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
              fence_proxy_async_smem();
              __syncwarp();
              if (lane == 0 && !(dm & 8)) tma_store_3d(&p.tma_c, smem_u32(blk), n0, mrow, zs, add_old);
              if constexpr (ST) tile_stats(p, blk, stat_sm, mt * kTileM, quarter, lane, n0, mt);
            }
            tc_fence_before();
            arrive_leader(&tempty[acc]);
            if (++acc == kAccStages) {
              acc = 0;
              acc_phase ^= 1;
            }
            continue;
          }
        }
        for (int cc = 0; cc < NB / 32; ++cc) {
          float v[32];
          tmem_ld32(tmem_base + acc * NB + cc * 32 + ((uint32_t)(quarter * 32) << 16), v);
          const int n0 = nt * p.n_pitch + cc * 32;
          if (row_ok && n0 < p.N && cc * 32 < p.n_pitch && !(dm & 8)) {
            float* dst;
            long long ld;
            if (p.epi == EPI_PARTIAL) {
              dst = p.ws + (long long)sp * p.M * p.N + (long long)m * p.N + n0;
              ld = p.N;
            } else {
              dst = p.c + out_row * p.ldc + n0;
              ld = p.ldc;
            }
            const int ncols = min(min(32, p.N - n0), p.n_pitch - cc * 32);
            if (p.c_trans && p.epi != EPI_PARTIAL) {
              // transposed result: column n0 + j is a row of c; the 32 lanes hold consecutive m,
              // so every j is one coalesced 128-B store (or reduction)
              float* col = p.c + (long long)n0 * p.ldc + m;
#pragma unroll
              for (int j = 0; j < 32; ++j) {
                if (j < ncols) {
                  if (add_old)
                    atomicAdd(col + (long long)j * p.ldc, v[j]);
                  else
                    col[(long long)j * p.ldc] = v[j];
                }
              }
            } else {
            if (add_bias) {
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] += j < ncols ? __ldg(p.bias + n0 + j) : 0.f;
            }
            const bool vec = (ncols == 32) && ((ld & 3) == 0) && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0);
            if (vec) {
#pragma unroll
              for (int j = 0; j < 32; j += 4) {
                if (add_old) {
                  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst + j), "f"(v[j]),
                               "f"(v[j + 1]), "f"(v[j + 2]), "f"(v[j + 3])
                               : "memory");
                } else {
                  *reinterpret_cast<float4*>(dst + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
                }
              }
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j) {
                if (j < ncols) {
                  if (add_old)
                    atomicAdd(dst + j, v[j]);
                  else
                    dst[j] = v[j];
                }
              }
            }
            }  // not transposed
          }
          __syncwarp();
        }
        tc_fence_before();
        arrive_leader(&tempty[acc]);
        if (++acc == kAccStages) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (rank == 0) {
    // ---------------------------------------------------------------- MMA issuer (leader CTA)
    const uint32_t idesc = idesc_bf16(kTileM, NB, b_mn ? 1 : 0);
    int stage_item = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    auto wait = [&](uint64_t* bar, uint32_t ph) {
      if constexpr (PR)
        mbar_wait_cluster(bar, ph);
      else
        mbar_wait(bar, ph);
    };
    for (int tile = unit0; tile < n_tiles_total; tile += n_units) {
      int mt, nt, kb0, nst;
      tile_range(p, tile, mt, nt, kb0, nst);
      for (int c0 = 0; c0 < nst; c0 += p.chunk_stages) {
        const int c1 = min(nst, c0 + p.chunk_stages);
        TWAIT(5, wait(&tempty[acc], acc_phase ^ 1));
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * NB;
        for (int s = c0; s < c1; ++s, ++stage_item) {
          const int stage = stage_item % kAStages, bstage = stage_item % kBStages;
          TWAIT(3, wait(&a_full[stage], (stage_item / kAStages) & 1));
          TWAIT(4, wait(&b_full[bstage], (stage_item / kBStages) & 1));
          tc_fence_after();
          if (lane == 0) {
            const long long t_issue = p.dbg_t ? clock64() : 0;
            const uint32_t a_hi = tmem_base + kTmemA + stage * kAStageCols;
            const uint32_t a_lo = a_hi + 32;
            const uint32_t bhi = smem_u32(bst + bstage * kStageBytes);
            const uint32_t blo = bhi + kBTile;
#pragma unroll
            for (int kk = 0; kk < ((dm & 4) ? 0 : BKS / 16); ++kk) {
              const uint32_t first = (s == c0 && kk == 0) ? 0u : 1u;
              mma_bf16_ts<PR>(d_tmem, a_lo + kk * 8, b_desc(bhi, b_mn, kk), idesc, first);
              mma_bf16_ts<PR>(d_tmem, a_hi + kk * 8, b_desc(blo, b_mn, kk), idesc, 1u);
              mma_bf16_ts<PR>(d_tmem, a_hi + kk * 8, b_desc(bhi, b_mn, kk), idesc, 1u);
            }
            if constexpr (PR) {
              mma_commit_pair(&a_empty[stage]);
              mma_commit_pair(&b_empty[bstage]);
              if (s == c1 - 1) mma_commit_pair(&tfull[acc]);
            } else {
              mma_commit(&a_empty[stage]);
              mma_commit(&b_empty[bstage]);
              if (s == c1 - 1) mma_commit(&tfull[acc]);
            }
            if (p.dbg_t) twait[11] += clock64() - t_issue;
          }
          __syncwarp();
        }
        if (++acc == kAccStages) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  }

  if constexpr (kW16) {
    if (warp >= kWarpEpi && warp < kWarpMma && lane == 0 && p.c_tma) bulk_wait_all();  // stores read smem / land
  }
  if (p.dbg_t) {  // one representative thread per role reports its waits
    const bool rep = threadIdx.x == 0 || threadIdx.x == kWarpASplit * 32 || threadIdx.x == kWarpBSplit * 32 ||
                     threadIdx.x == kWarpEpi * 32 || threadIdx.x == kWarpMma * 32;
    if (rep) {
      twait[15] = clock64() - t_start;
      for (int i = 0; i < 16; ++i)
        if (twait[i] && (i != 15 || threadIdx.x == kWarpMma * 32)) atomicAdd(p.dbg_t + i, (unsigned long long)twait[i]);
    }
  }
  tc_fence_before();
  if constexpr (PR)
    cluster_sync();  // the leader's MMAs read this CTA's TMEM / smem until the end
  else
    __syncthreads();
  if (warp == kWarpMma) {
    tc_fence_after();
    if constexpr (PR)
      tmem_dealloc_pair(tmem_base, kTmemCols);
    else
      tmem_dealloc(tmem_base, kTmemCols);
  }
}
#undef TWAIT

}  // namespace bx3
}  // namespace monet
