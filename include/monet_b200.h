/* monet_b200.h — C ABI of the B200 MONeT execution engine (libmonet_b200.so).
 *
 * The reference has exactly one boundary on this path: the executor contract
 * `simulate(schedule, g, catalog) -> Trace` (pkg/src/remsched/schedule.py:320)
 * whose per-step `record()` (schedule.py:338-342) stands for "run this
 * operator variant".  Every entry point below is one such operator variant,
 * the arena planner the ledger's alloc/free events drive, or the profiler
 * that fills the catalog (`Catalog`, costmodel.py:30-73; workspace bytes and
 * costs per variant, costmodel.py:85-181).  The Python executor
 * (paper_2010_14501_b200/engine.py) binds these with ctypes; INTEGRATION.md
 * shows the binding a remsched maintainer would add.
 *
 * Conventions: plain pointers to device memory (fp32 NHWC activations, KRSC
 * conv weights), sizes in elements unless named *_bytes, `stream` is a
 * cudaStream_t passed as void*.  Return 0 on success, a negative
 * -cudaError_t on failure; no C++ exception crosses this boundary.  Kernels
 * never allocate: workspace and scratch come from the caller (the budgeted
 * arena), sized by the *_ws_bytes / *_scratch_bytes queries.
 * `accumulate` selects dx = f(dy) (0, first consumer allocates the gradient,
 * schedule.py:445-449) or dx += f(dy) (1, later consumers).
 */
#ifndef MONET_B200_H
#define MONET_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Convolution geometry, NHWC input [n,h,w,c], KRSC weight [k,r,s,c],
 * NHWC output [n,p,q,k].  c and k must be multiples of 4. */
typedef struct {
  int n, h, w, c, k, r, s, p, q, stride_h, stride_w, pad_h, pad_w;
} monet_conv_desc;

/* conv variants (catalog ForwardVariant / BackwardVariant names):
 *   MONET_CONV_IMPLICIT  "implicit"  tcgen05 bf16x3 implicit GEMM (fp32 = bf16 hi + lo, three
 *                                    MMAs, ~1e-5 relative), A operand staged in TMEM
 *   MONET_CONV_SPLITK    "splitk"    as implicit, plus split-K over the reduction with
 *                                    fp32 partials in workspace (honest ws/speed trade)
 *   MONET_CONV_TF32      "tf32"      single-pass TF32 (faster, ~1e-3 relative error; tests only)
 *   MONET_CONV_TF32X3    "tf32x3"    3xTF32 all-shared-memory kernel (round-1 baseline)
 *   MONET_CONV_PAIR      "pair"      retired (returns -cudaErrorNotSupported): CTA pairs measured
 *                                    15-25 % slower than one CTA per tile */
enum { MONET_CONV_IMPLICIT = 0, MONET_CONV_SPLITK = 1, MONET_CONV_TF32 = 2, MONET_CONV_TF32X3 = 3,
       MONET_CONV_PAIR = 4 };
enum { MONET_PASS_FWD = 0, MONET_PASS_DGRAD = 1, MONET_PASS_WGRAD = 2, MONET_PASS_BWD = 3 };

/* --- library --------------------------------------------------------------- */
const char* monet_version(void);
int monet_device_check(void); /* 0 if the current device is sm_100 */
/* device-to-device byte copy on `stream` (staging the input batch into the arena,
 * the loss seed); the executor needs no other CUDA runtime entry point */
int monet_copy_async(void* dst, const void* src, size_t bytes, void* stream);
/* (The operand-dump and wait-counter hooks of the GEMM exist only in the debug build,
 * libmonet_b200_dbg.so, `python -m paper_2010_14501_b200.build --debug`; not part of this ABI.) */

/* --- data-parallel gradient exchange (SURVEY.md §8b "Comm", §8e) ----------------------
 * One communicator per GPU process (NCCL, resolved at run time from the process's own
 * libnccl.so.2).  Rank 0 creates the unique id (monet_comm_unique_id_bytes() bytes), the
 * caller broadcasts it (torch.distributed), every rank calls monet_comm_init.
 * monet_allreduce_bucket forks the in-place fp32 sum of one gradient bucket off `stream`
 * onto the communicator's own stream, ordered after everything already enqueued on
 * `stream` (the backward kernels that finalize the bucket), so it overlaps the remaining
 * backward stages; monet_comm_join makes `stream` wait for every bucket forked since the
 * last join (before the optimizer).  All of it is stream-ordered and CUDA-graph
 * capturable.  NCCL failures return -(1000 + ncclResult_t). */
typedef struct monet_comm monet_comm;
size_t monet_comm_unique_id_bytes(void);
int monet_comm_unique_id(void* id_out);
int monet_comm_init(const void* unique_id, int rank, int nranks, monet_comm** out);
int monet_comm_destroy(monet_comm* comm);
int monet_allreduce_bucket(monet_comm* comm, float* buf, size_t count, void* stream);
int monet_comm_join(monet_comm* comm, void* stream);

/* --- profiler (R3: fills the catalog's variant costs and workspace, costmodel.py:85-181) ---
 * monet_profile_variant times one operator variant on synthetic operands it allocates
 * and frees itself: two warm-up launches, then the median of three CUDA-event-timed
 * groups of `iters` launches on `stream`.  *ns = nanoseconds per launch (an integer,
 * units.py:61-62 forbids fractional costs in a catalog), *ws_bytes = the workspace the
 * variant takes from the arena (conv: monet_conv_ws_bytes of that variant and pass; 0 for
 * the local operators, whose scratch lives in the fixed region).
 *   op  MONET_OP_CONV   pass FWD (forward), BWD (dgrad, if conv_needs_dx, + wgrad), or DGRAD /
 *                       WGRAD alone (a split conv's two backward nodes); variant = MONET_CONV_*;
 *                       desc in `conv`
 *       MONET_OP_RELU   pass FWD (with the 1-bit mask) or BWD with variant MONET_BWD_IN /
 *                       _OUT / _MASK; rows * c elements
 *       MONET_OP_BN     pass FWD (train: statistics + apply) or BWD (MONET_BWD_IN / _OUT)
 *       MONET_OP_BNRELU fused BN+ReLU: FWD, or BWD (MONET_BWD_IN, from x) */
enum { MONET_OP_CONV = 0, MONET_OP_RELU = 1, MONET_OP_BN = 2, MONET_OP_BNRELU = 3 };
enum { MONET_BWD_IN = 0, MONET_BWD_OUT = 1, MONET_BWD_MASK = 2 };
typedef struct {
  int op, pass;
  monet_conv_desc conv;
  int conv_needs_dx; /* 0 when the conv reads the network input (no dgrad) */
  int64_t rows;      /* local ops: [rows, c] NHWC */
  int c;
  int fused_stats;   /* FWD: conv -> BN statistics handed over (monet_conv_fwd_w16_stats;
                        BN / BNRELU: monet_bn_stats_finalize + the replay apply) */
} monet_prof_desc;
int monet_profile_variant(const monet_prof_desc* d, int variant, int iters, int64_t* ns, size_t* ws_bytes,
                          void* stream);

/* --- convolution (K1-K3; replaces conv entries of Catalog, costmodel.py:30-44) */
size_t monet_conv_ws_bytes(int variant, int pass, const monet_conv_desc* d);
int monet_conv_fwd(int variant, const monet_conv_desc* d, const float* x, const float* w, float* y, void* ws,
                   size_t ws_bytes, void* stream);
int monet_conv_dgrad(int variant, const monet_conv_desc* d, const float* dy, const float* w, float* dx,
                     int accumulate, void* ws, size_t ws_bytes, void* stream);
int monet_conv_wgrad(int variant, const monet_conv_desc* d, const float* x, const float* dy, float* dw,
                     int accumulate, void* ws, size_t ws_bytes, void* stream);

/* conv with a per-output-channel bias (VGG-style convs): the bias is added in the
 * GEMM epilogue (split-K: in the partial-sum reduce).  Its gradient is
 * monet_bias_grad over dy ([rows = n*p*q, k]); scratch = monet_bn_scratch_bytes(rows, k). */
int monet_conv_fwd_bias(int variant, const monet_conv_desc* d, const float* x, const float* w, const float* bias,
                        float* y, void* ws, size_t ws_bytes, void* stream);
int monet_bias_grad(const float* dy, float* db, int64_t rows, int c, int accumulate, void* scratch, void* stream);

/* Pre-split weights: the bf16x3 GEMM splits every fp32 operand element into
 * hi = bf16(x), lo = bf16(x - hi) (round to nearest even).  The weights change only at
 * the optimizer step, so an executor keeps their split in two bf16 planes (w_hi, w_lo:
 * the same element offsets as w) refreshed once per step, and the conv forward / input
 * gradient load them by TMA straight into the MMA tiles (no per-tile B split).  Results
 * are bit-identical to monet_conv_fwd[_bias] / monet_conv_dgrad, which these fall back to
 * when the shape or alignment does not allow it (w_hi == NULL: always).  bias may be NULL.
 * split_bf16_segments: table (device memory) holds nseg x {src_off, dst_off, count}
 * (elements), max_count >= every count. */
int monet_conv_fwd_w16(int variant, const monet_conv_desc* d, const float* x, const float* w, const uint16_t* w_hi,
                       const uint16_t* w_lo, const float* bias, float* y, void* ws, size_t ws_bytes, void* stream);
int monet_conv_dgrad_w16(int variant, const monet_conv_desc* d, const float* dy, const float* w, const uint16_t* w_hi,
                         const uint16_t* w_lo, float* dx, int accumulate, void* ws, size_t ws_bytes, void* stream);
int monet_split_bf16(const float* src, uint16_t* hi, uint16_t* lo, int64_t n, void* stream);

/* Conv -> BN forward without re-reading the conv output: monet_conv_fwd_w16_stats is
 * monet_conv_fwd_w16 that also leaves per-128-row-tile BN statistics (mean, M2 per output
 * channel) in `stats` (monet_conv_stats_bytes(d) bytes) -- from the GEMM epilogue when each
 * tile is final in one accumulation chain, else from one extra pass over y.  The following
 * BN's training forward is monet_bn_stats_finalize (batch mean / invstd and the running-stat
 * update, merged in fp64 in a fixed order: deterministic) + the BN's *_fwd_replay apply. */
size_t monet_conv_stats_bytes(const monet_conv_desc* d);
int monet_conv_fwd_w16_stats(int variant, const monet_conv_desc* d, const float* x, const float* w,
                             const uint16_t* w_hi, const uint16_t* w_lo, const float* bias, float* y, void* stats,
                             void* ws, size_t ws_bytes, void* stream);
int monet_bn_stats_finalize(const void* stats, int64_t rows, int c, float eps, float momentum, int update_running,
                            float* mean, float* invstd, float* running_mean, float* running_var, void* stream);
int monet_split_bf16_segments(const float* src, uint16_t* hi, uint16_t* lo, const int64_t* table, int nseg,
                              int64_t max_count, void* stream);

/* --- dropout (VGG / MobileNet-V2 / GoogleNet classifiers) ------------------------
 * keep(i) <=> splitmix64(seed*0x9E3779B97F4A7C15 + salt*0xD1B54A32D192ED03 + i) >> 40 >= floor(p*2^24),
 * i = element index in NHWC order; y = keep ? x / (1-p) : 0.  The mask is never stored:
 * backward and recomputes regenerate it from *seed (device memory, read at run time),
 * which monet_seed_advance increments once per training step. */
int monet_dropout_fwd(const float* x, float* y, int64_t n, float p, const unsigned long long* seed, uint64_t salt,
                      void* stream);
int monet_dropout_bwd(const float* dy, float* dx, int64_t n, float p, const unsigned long long* seed, uint64_t salt,
                      int accumulate, void* stream);
int monet_seed_advance(unsigned long long* seed, void* stream);

/* --- transposed conv (UNet up-sampling) --------------------------------------------
 * The adjoint of the conv described by d: d's input is the transposed conv's OUTPUT y
 * [n][h][w][c], d's output its INPUT x [n][p][q][k]; weights KRSC (torch [in][out][R][S]
 * with in = k, out = c).  Forward = the conv dgrad kernel (+ bias), input gradient = the conv
 * forward kernel (optionally accumulating), weight gradient = the conv wgrad kernel. */
size_t monet_convT_ws_bytes(int variant, int pass, const monet_conv_desc* d);
int monet_convT_fwd(int variant, const monet_conv_desc* d, const float* x, const float* w, const float* bias, float* y,
                    void* ws, size_t ws_bytes, void* stream);
int monet_convT_bwd(int variant, const monet_conv_desc* d, const float* x, const float* w, const float* dy, float* dx,
                    int dx_accumulate, float* dw, void* ws, size_t ws_bytes, void* stream);

/* --- channel concat (GoogLeNet inception outputs) ---------------------------------
 * NHWC channel-slice copy: dst[pix][dst_off + j] (+)= src[pix][src_off + j], j < count
 * (all channel counts and offsets multiples of 4).  Concat forward = one call per input
 * into its channel range; backward = one call per input taking its slice of dy. */
int monet_channel_copy(const float* src, int src_c, int src_off, float* dst, int dst_c, int dst_off, int count,
                       int64_t pixels, int accumulate, void* stream);

/* --- depthwise conv (groups = C; MobileNet-V2) ------------------------------------
 * NHWC, d->k == d->c, R*S <= 9, weights [R][S][C].  HBM-bound direct kernels.
 * wgrad reduces in two fixed-order levels through ws (monet_dwconv_ws_bytes). */
size_t monet_dwconv_ws_bytes(const monet_conv_desc* d);
int monet_dwconv_fwd(const monet_conv_desc* d, const float* x, const float* w, float* y, void* stream);
int monet_dwconv_dgrad(const monet_conv_desc* d, const float* dy, const float* w, float* dx, int accumulate,
                       void* stream);
int monet_dwconv_wgrad(const monet_conv_desc* d, const float* x, const float* dy, float* dw, void* ws,
                       size_t ws_bytes, void* stream);

/* --- dense layer (fc) -------------------------------------------------------- */
size_t monet_linear_ws_bytes(int variant, int pass, int n, int in_f, int out_f);
int monet_linear_fwd(int variant, const float* x, const float* w, const float* b, float* y, int n, int in_f,
                     int out_f, void* ws, size_t ws_bytes, void* stream);
int monet_linear_bwd(int variant, const float* x, const float* w, const float* dy, float* dx, int dx_accumulate,
                     float* dw, float* db, int n, int in_f, int out_f, void* ws, size_t ws_bytes, void* stream);

/* --- ReLU with packed sign bitmask (K4/K5) -------------------------------------
 * mask: ceil(n/32) uint32 words, bit b of word w <-> element 32w+b; nullable. */
int monet_relu_fwd(const float* x, float* y, uint32_t* mask, int64_t n, void* stream);
int monet_relu_bwd_mask(const uint32_t* mask, const float* dy, float* dx, int64_t n, int accumulate, void* stream);
int monet_relu_bwd_out(const float* y, const float* dy, float* dx, int64_t n, int accumulate, void* stream);
int monet_relu_bwd_in(const float* x, const float* dy, float* dx, int64_t n, int accumulate, void* stream);

/* ReLU6 = hardtanh(0, 6) (MobileNet-V2): y = min(max(x, 0), 6); mask bit = the gradient
 * gate 0 < x < 6, so the backward from the mask is monet_relu_bwd_mask. */
int monet_relu6_fwd(const float* x, float* y, uint32_t* mask, int64_t n, void* stream);
int monet_relu6_bwd_out(const float* y, const float* dy, float* dx, int64_t n, int accumulate, void* stream);
int monet_relu6_bwd_in(const float* x, const float* dy, float* dx, int64_t n, int accumulate, void* stream);

/* --- BatchNorm, training mode, [rows = n*h*w, c] (K6-K8) ----------------------
 * scratch: monet_bn_scratch_bytes(rows, c) bytes of caller memory. */
size_t monet_bn_scratch_bytes(int64_t rows, int c);
int monet_bn_fwd_train(const float* x, float* y, const float* gamma, const float* beta, float* saved_mean,
                       float* saved_invstd, float* running_mean, float* running_var, int64_t rows, int c, float eps,
                       float momentum, int update_running, void* scratch, void* stream);
/* recompute: reuses saved statistics, never touches running stats */
int monet_bn_fwd_replay(const float* x, float* y, const float* gamma, const float* beta, const float* saved_mean,
                        const float* saved_invstd, int64_t rows, int c, void* stream);
int monet_bn_bwd_in(const float* x, const float* dy, float* dx, int accumulate, const float* gamma,
                    const float* saved_mean, const float* saved_invstd, float* dgamma, float* dbeta, int64_t rows,
                    int c, void* scratch, void* stream);
/* output-activated: xhat = (y - beta) / gamma, |gamma| clamped to >= 1e-12 */
int monet_bn_bwd_out(const float* y, const float* dy, float* dx, int accumulate, const float* gamma,
                     const float* beta, const float* saved_invstd, float* dgamma, float* dbeta, int64_t rows, int c,
                     void* scratch, void* stream);

/* --- fused BN+ReLU (K9 / K10): z = relu(BN(x)), the BN output never exists -----
 * Backward from the BN input x: the ReLU gate [BN(x) > 0] is recomputed with the
 * forward's exact expression (relu(y) alone cannot give dx). */
int monet_bnrelu_fwd_train(const float* x, float* z, const float* gamma, const float* beta, float* saved_mean,
                           float* saved_invstd, float* running_mean, float* running_var, int64_t rows, int c,
                           float eps, float momentum, int update_running, void* scratch, void* stream);
int monet_bnrelu_fwd_replay(const float* x, float* z, const float* gamma, const float* beta, const float* saved_mean,
                            const float* saved_invstd, int64_t rows, int c, void* stream);
int monet_bnrelu_bwd(const float* x, const float* dz, float* dx, int accumulate, const float* gamma,
                     const float* beta, const float* saved_mean, const float* saved_invstd, float* dgamma,
                     float* dbeta, int64_t rows, int c, void* scratch, void* stream);

/* fused BN+ReLU6 (MobileNet-V2's expand / depthwise blocks): z = min(max(BN(x), 0), 6); the
 * backward recomputes the gate 0 < BN(x) < 6 from x and the saved statistics. */
int monet_bnrelu6_fwd_train(const float* x, float* z, const float* gamma, const float* beta, float* saved_mean,
                            float* saved_invstd, float* running_mean, float* running_var, int64_t rows, int c,
                            float eps, float momentum, int update_running, void* scratch, void* stream);
int monet_bnrelu6_fwd_replay(const float* x, float* z, const float* gamma, const float* beta,
                             const float* saved_mean, const float* saved_invstd, int64_t rows, int c, void* stream);
int monet_bnrelu6_bwd(const float* x, const float* dz, float* dx, int accumulate, const float* gamma,
                      const float* beta, const float* saved_mean, const float* saved_invstd, float* dgamma,
                      float* dbeta, int64_t rows, int c, void* scratch, void* stream);

/* fused BN + residual add + ReLU (a bottleneck's last BN feeding its join): z = max(BN(x) + skip, 0),
 * the BN output never exists.  Backward gate from z (gate_from_out = 1, gate_src = z) or recomputed
 * from x and skip (0, gate_src = skip); writes / accumulates dx and dskip in one pass. */
int monet_bnaddrelu_fwd_train(const float* x, const float* skip, float* z, const float* gamma, const float* beta,
                              float* saved_mean, float* saved_invstd, float* running_mean, float* running_var,
                              int64_t rows, int c, float eps, float momentum, int update_running, void* scratch,
                              void* stream);
int monet_bnaddrelu_fwd_replay(const float* x, const float* skip, float* z, const float* gamma, const float* beta,
                               const float* saved_mean, const float* saved_invstd, int64_t rows, int c, void* stream);
int monet_bnaddrelu_bwd(const float* x, const float* gate_src, int gate_from_out, const float* dz, float* dx,
                        int acc_x, float* dskip, int acc_skip, const float* gamma, const float* beta,
                        const float* saved_mean, const float* saved_invstd, float* dgamma, float* dbeta, int64_t rows,
                        int c, void* scratch, void* stream);

/* --- residual add / gradient pass-through (K12) --------------------------- */
int monet_add_fwd(const float* a, const float* b, float* y, int64_t n, void* stream);
int monet_grad_pass(const float* dy, float* dx, int64_t n, float scale, int accumulate, void* stream);
/* fused residual join + ReLU: z = max(a + b, 0); backward gates dz by z > 0
 * (output-activated) or by a + b > 0 (input-activated) and writes / adds both
 * input gradients in one pass */
int monet_addrelu_fwd(const float* a, const float* b, float* z, int64_t n, void* stream);
int monet_addrelu_bwd_out(const float* z, const float* dz, float* da, int acc_a, float* db, int acc_b, int64_t n,
                          void* stream);
int monet_addrelu_bwd_in(const float* a, const float* b, const float* dz, float* da, int acc_a, float* db, int acc_b,
                         int64_t n, void* stream);

/* --- pooling (K11, K13) ----------------------------------------------------- */
int monet_maxpool_fwd(const monet_conv_desc* d, const float* x, float* y, uint8_t* idx8, void* stream);
int monet_maxpool_bwd(const monet_conv_desc* d, const uint8_t* idx8, const float* x, const float* dy, float* dx,
                      int accumulate, void* stream);
int monet_avgpool_fwd(const float* x, float* y, int n, int hw, int c, void* stream);
int monet_avgpool_bwd(const float* dy, float* dx, int n, int hw, int c, int accumulate, void* stream);

/* --- loss and optimizer (K13) ----------------------------------------------- */
size_t monet_xent_scratch_bytes(int n);
int monet_xent_fwd(const float* logits, const int32_t* labels, float* loss, int n, int classes, void* scratch,
                   void* stream);
int monet_xent_bwd(const float* logits, const int32_t* labels, const float* dloss, float* dlogits, int n,
                   int classes, int accumulate, void* stream);
int monet_sgd_step(float* w, const float* g, float* momentum_buf, int64_t n, float lr, float momentum,
                   float weight_decay, float grad_scale, int first_step, void* stream);

/* --- generic tcgen05 GEMM (test / profiler access) ---------------------------
 * C[m,n] (=|+=) sum_k A[m,k] B[n,k]; a_mn/b_mn select MN-major operands. */
int monet_gemm(int variant, const float* a, int a_mn, int64_t lda, const float* b, int b_mn, int64_t ldb, float* c,
               int64_t ldc, int m, int n, int k, int accumulate, void* ws, size_t ws_bytes, void* stream);
size_t monet_gemm_ws_bytes(int variant, int m, int n, int k);

/* --- budget-capped arena: static offset planning (R2) -------------------------
 * Blocks i = 0..count-1 live over ledger events [t_alloc[i], t_free[i]).
 * Writes offsets (aligned to `align`) so that no two simultaneously live
 * blocks overlap and returns the arena high-water mark in *peak_bytes.
 * Returns -12 (ENOMEM) when the plan exceeds capacity_bytes (0 = no cap). */
int monet_arena_plan(int64_t count, const int64_t* sizes, const int64_t* t_alloc, const int64_t* t_free,
                     int64_t align, int64_t capacity_bytes, int64_t* offsets, int64_t* peak_bytes);

/* --- host ILP: exact 0-1 branch-and-bound (replaces solver.solve, solver.py:441) ---
 * Same propagation, bound (+ capacity surrogate), branch order, dives and
 * limits as the reference, so decisions are bit-exact; costs are integers
 * (the objective scaled by the lcm of its denominators), 128-bit values are
 * (hi, lo) int64 pairs.  See paper_2010_14501_b200/solver.py for the packing. */
void* monet_bnb_create(int n_vars, int n_rows, const int* row_ptr, const int* row_var, const int64_t* row_coef,
                       const int64_t* row_rhs, const int* row_is_eq, int n_fix, const int* fix_var, const int* fix_val,
                       int n_obj, const int* obj_var, const int64_t* obj_cost128, int n_fwd, int n_bwd, int n_re,
                       const int* grp_ptr, const int* grp_var, const int64_t* grp_cost128, const int* re_rvar);
int monet_bnb_set_surrogate(void* h, int64_t cap_base, int n_stages, const int64_t* grad, const int* var_ptr,
                            const int* var_db, const int64_t* var_ws, const int* dep_ptr, const int* dep_idx,
                            int n_storables, const int64_t* size, const int64_t* recost, const int* rcol);
void monet_bnb_destroy(void* h);
int monet_bnb_propagate(void* h, int n_partial, const int* pvar, const int* pval, signed char* out);
int monet_bnb_lower_bound(void* h, int n_partial, const int* pvar, const int* pval, int64_t scale, int64_t* out128);
/* opts: node_limit (-1 none), telemetry_every, dive_bound, most_tight, gap_num, gap_den (0 none), scale.
 * Returns 0 optimal, 1 feasible-gap, 2 infeasible, 3 timeout-no-incumbent. */
int monet_bnb_solve(void* h, const int64_t* opts, double time_limit_s, const int* order, int n_order,
                    const signed char* pref, int has_inc, const int64_t* inc_obj128, const signed char* inc_vals,
                    int64_t* nodes_out, int64_t* res128);
int monet_bnb_best(void* h, signed char* out);
int monet_bnb_n_events(void* h);
int monet_bnb_event(void* h, int i, int* kinds, int64_t* counts, int64_t* vals128);

#ifdef __cplusplus
}
#endif
#endif /* MONET_B200_H */
