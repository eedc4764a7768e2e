// monet_profile_variant: the on-device profiler's C entry point (SURVEY.md §8b,
// R3).  Times one operator variant on its own synthetic buffers with CUDA events
// and reports the workspace it takes -- the two numbers a catalog variant carries
// (costmodel.py:85-181: `cost` as an integer, units.py:61-62; `workspace_bytes`).
// Unlike the kernels, the profiler allocates: it owns its operands and frees them.
#include <algorithm>
#include <cstring>
#include <functional>
#include <vector>

#include "../../include/monet_b200.h"
#include "common.cuh"

namespace {

// deterministic operand fill in [-1, 1) (splitmix hash of the index): random-looking
// data, so the tensor pipe and HBM see realistic switching activity
__global__ void prof_fill_kernel(float* p, long long n, unsigned salt) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    unsigned long long z = (unsigned long long)i * 0x9E3779B97F4A7C15ull + salt;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    p[i] = (float)((z >> 40) & 0xFFFFFF) / 8388608.0f - 1.0f;
  }
}

struct Bufs {
  std::vector<void*> ptrs;
  cudaStream_t st;
  int err = 0;
  float* get(size_t bytes, unsigned salt, float offset = 0.f) {
    void* p = nullptr;
    bytes = std::max<size_t>(bytes, 16);
    if (cudaMallocAsync(&p, bytes, st) != cudaSuccess) {
      err = -(int)cudaErrorMemoryAllocation;
      return nullptr;
    }
    ptrs.push_back(p);
    const long long n = (long long)(bytes / 4);
    prof_fill_kernel<<<(int)std::min<long long>((n + 255) / 256, 4096), 256, 0, st>>>(static_cast<float*>(p), n, salt);
    if (offset != 0.f) {  // positive-definite per-channel parameters (gamma, invstd)
      std::vector<float> h(n, offset);
      cudaMemcpyAsync(p, h.data(), bytes / 4 * 4, cudaMemcpyHostToDevice, st);
      cudaStreamSynchronize(st);
    }
    return static_cast<float*>(p);
  }
  ~Bufs() {
    for (void* p : ptrs) cudaFreeAsync(p, st);
    cudaStreamSynchronize(st);
  }
};

}  // namespace

extern "C" int monet_profile_variant(const monet_prof_desc* d, int variant, int iters, int64_t* ns, size_t* ws_bytes,
                                     void* stream) {
  if (!d || iters < 1 || !ns) return -(int)cudaErrorInvalidValue;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Bufs B;
  B.st = st;
  size_t ws = 0;
  const int pass = d->pass;
  if (pass < MONET_PASS_FWD || pass > MONET_PASS_BWD) return -(int)cudaErrorInvalidValue;
  if (d->op != MONET_OP_CONV && pass != MONET_PASS_FWD && pass != MONET_PASS_BWD) return -(int)cudaErrorInvalidValue;
  // one launch of the variant; returns 0 or a negative error
  std::function<int()> run;
  if (d->op == MONET_OP_CONV) {
    const monet_conv_desc* c = &d->conv;
    if (c->c % 4 || c->k % 4) return -(int)cudaErrorInvalidValue;
    const size_t xb = (size_t)c->n * c->h * c->w * c->c * 4, yb = (size_t)c->n * c->p * c->q * c->k * 4;
    const size_t wb = (size_t)c->k * c->r * c->s * c->c * 4;
    ws = monet_conv_ws_bytes(variant, pass, c);
    float *x = B.get(xb, 1), *w = B.get(wb, 2), *y = B.get(yb, 3), *wsp = B.get(ws, 4);
    float *dx = pass != MONET_PASS_FWD ? B.get(xb, 5) : nullptr, *dw = pass != MONET_PASS_FWD ? B.get(wb, 6) : nullptr;
    // the weights' bf16 split as an executor keeps it (monet_conv_*_w16): split once, untimed
    const int64_t wn = (int64_t)(wb / 4), wn8 = (wn + 7) / 8 * 8;
    uint16_t* whi = reinterpret_cast<uint16_t*>(B.get((size_t)wn8 * 4, 7));
    if (B.err) return B.err;
    uint16_t* wlo = whi + wn8;
    if (int e = monet_split_bf16(w, whi, wlo, wn, st)) return e;
    const bool need_dx = d->conv_needs_dx != 0;
    float* stats = (pass == MONET_PASS_FWD && d->fused_stats) ? B.get(monet_conv_stats_bytes(c), 8) : nullptr;
    if (B.err) return B.err;
    run = [=]() -> int {  // BWD: dgrad (if the input has a gradient) + wgrad; DGRAD / WGRAD: one pass
      if (pass == MONET_PASS_FWD && stats)
        return monet_conv_fwd_w16_stats(variant, c, x, w, whi, wlo, nullptr, y, stats, wsp, ws, st);
      if (pass == MONET_PASS_FWD) return monet_conv_fwd_w16(variant, c, x, w, whi, wlo, nullptr, y, wsp, ws, st);
      if ((pass == MONET_PASS_BWD && need_dx) || pass == MONET_PASS_DGRAD)
        if (int e = monet_conv_dgrad_w16(variant, c, y, w, whi, wlo, dx, 0, wsp, ws, st)) return e;
      if (pass == MONET_PASS_DGRAD) return 0;
      return monet_conv_wgrad(variant, c, x, y, dw, 0, wsp, ws, st);
    };
  } else if (d->op == MONET_OP_RELU) {
    const int64_t n = d->rows * d->c;
    float *x = B.get(n * 4, 1), *y = B.get(n * 4, 2), *dy = B.get(n * 4, 3), *dx = B.get(n * 4, 4);
    uint32_t* m = reinterpret_cast<uint32_t*>(B.get((n + 31) / 32 * 4, 5));
    if (B.err) return B.err;
    run = [=]() -> int {
      if (pass == MONET_PASS_FWD) return monet_relu_fwd(x, y, m, n, st);
      if (variant == MONET_BWD_MASK) return monet_relu_bwd_mask(m, dy, dx, n, 0, st);
      return variant == MONET_BWD_OUT ? monet_relu_bwd_out(y, dy, dx, n, 0, st) : monet_relu_bwd_in(x, dy, dx, n, 0, st);
    };
  } else if (d->op == MONET_OP_BN || d->op == MONET_OP_BNRELU) {
    const int64_t rows = d->rows;
    const int c = d->c;
    if (c % 4) return -(int)cudaErrorInvalidValue;
    const size_t nb = (size_t)rows * c * 4;
    float *x = B.get(nb, 1), *y = B.get(nb, 2), *dy = B.get(nb, 3), *dx = B.get(nb, 4);
    float *g = B.get(c * 4, 5, 1.f), *b = B.get(c * 4, 6), *mean = B.get(c * 4, 7), *inv = B.get(c * 4, 8, 1.f);
    float *rm = B.get(c * 4, 9), *rv = B.get(c * 4, 10, 1.f), *dg = B.get(c * 4, 11), *db = B.get(c * 4, 12);
    float* scratch = B.get(monet_bn_scratch_bytes(rows, c), 13);
    // conv-provided statistics: tile stats [T][2][c] (+ merge partials), positive M2
    const long long T = (rows + 127) / 128;
    const size_t sb = ((size_t)T * 2 * c * 4 + 255) / 256 * 256 + ((size_t)((T + 31) / 32) * 3 * c * 8 + 255) / 256 * 256;
    float* stats = d->fused_stats ? B.get(sb, 14, 2.f) : nullptr;
    if (B.err) return B.err;
    const bool fused = d->op == MONET_OP_BNRELU;
    run = [=]() -> int {
      if (pass == MONET_PASS_FWD && stats) {
        if (int e = monet_bn_stats_finalize(stats, rows, c, 1e-5f, 0.1f, 1, mean, inv, rm, rv, st)) return e;
        return fused ? monet_bnrelu_fwd_replay(x, y, g, b, mean, inv, rows, c, st)
                     : monet_bn_fwd_replay(x, y, g, b, mean, inv, rows, c, st);
      }
      if (pass == MONET_PASS_FWD)
        return fused ? monet_bnrelu_fwd_train(x, y, g, b, mean, inv, rm, rv, rows, c, 1e-5f, 0.1f, 1, scratch, st)
                     : monet_bn_fwd_train(x, y, g, b, mean, inv, rm, rv, rows, c, 1e-5f, 0.1f, 1, scratch, st);
      if (fused) return monet_bnrelu_bwd(x, dy, dx, 0, g, b, mean, inv, dg, db, rows, c, scratch, st);
      return variant == MONET_BWD_OUT ? monet_bn_bwd_out(y, dy, dx, 0, g, b, inv, dg, db, rows, c, scratch, st)
                                      : monet_bn_bwd_in(x, dy, dx, 0, g, mean, inv, dg, db, rows, c, scratch, st);
    };
  } else {
    return -(int)cudaErrorInvalidValue;
  }
  // warm-up (also sets kernel attributes outside the timed region), then the
  // median of three event-timed groups of `iters` launches
  for (int i = 0; i < 2; ++i)
    if (int e = run()) return e;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float t[3];
  int rc = 0;
  for (int r = 0; r < 3 && !rc; ++r) {
    cudaEventRecord(a, st);
    for (int i = 0; i < iters && !rc; ++i) rc = run();
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&t[r], a, b);
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  if (rc) return rc;
  std::sort(t, t + 3);
  *ns = std::max<int64_t>(1, (int64_t)((double)t[1] * 1e6 / iters + 0.5));
  if (ws_bytes) *ws_bytes = ws;
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : -(int)e;
}
