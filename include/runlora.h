/*
 * runlora.h — C ABI of the B200 (sm_100a) RunLoRA hot path.
 *
 * The operation (arXiv 2312.03415, PAPER.md):
 *   forward   Y  = X W + (X A) B          (forward1, Eq. 1)
 *             Y  = X (W + A B)            (forward2, Eq. 2)
 *   backward  dA = Xᵀ dY Bᵀ,  dB = Aᵀ Xᵀ dY,  dX = dY Wᵀ + dY Bᵀ Aᵀ   (Eq. 3)
 *             evaluated by one of the bracketings backward1..backward5
 *             (Algorithms 1-5); backward6..8 exist for
 *             cost queries only.
 *   cost      Table 1, exact integers; Eq. 5 parameter-reduction
 *             predicate r(i+o) < io.
 *   select    "best forward and backward computation graph based on FLOPs and
 *             time estimations" (abstract, P:5).
 * Nothing from X·A is saved between forward and backward: every backward
 * entry point takes only X, W, A, B, dY.
 *
 * Notation: n = b·s tokens, k = input dim (paper i), m = output dim (paper o),
 * r = rank.  All matrices are ROW-MAJOR, contiguous, in the paper's orientation:
 *   X[n,k]  W[k,m]  A[k,r]  B[r,m]  Y,dY[n,m]  dX[n,k]  dA[k,r]  dB[r,m]
 *
 * Pointers:
 *   - Every matrix pointer passed to forward/backward/select is a DEVICE pointer
 *     (cudaMalloc / caching allocator memory of the handle's device) unless the
 *     parameter name ends in _host (pinned or pageable host memory).
 *   - Device pointers must be 16-byte aligned.
 *   - The caller owns every buffer, including the workspace; the library never
 *     allocates device memory on the forward/backward path.  The handle owns only
 *     host-side caches (TMA descriptors, plans, profiling events).
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *     All calls are asynchronous and stream-ordered; argument validation is
 *     synchronous and happens before anything is launched.
 *
 * Dtypes: RUNLORA_F32 computes every product in true fp32 FFMA (no TF32);
 * RUNLORA_BF16 reads bf16 operands, accumulates in fp32 on the tcgen05 tensor
 * cores and stores Y, dX and the rank-r intermediates in bf16 (X·A and dY·Bᵀ as
 * one block per K-split, summed in fp32 by the tensor cores where they are used,
 * DESIGN.md R16); W+AB is formed in fp32 and rounded once (R10).  For
 * bf16, k, m and r must be multiples of 8 (TMA needs 16-byte row strides) —
 * otherwise RUNLORA_ERR_ALIGNMENT.
 *
 * Concurrency: any host thread may call into a handle; the calls that enqueue
 * work or touch the handle's caches are serialised by a per-handle mutex (held
 * only while the call enqueues; time-mode selection holds it while it measures).
 * Calls for different streams may run concurrently on the device if every stream
 * uses its own workspace.  Every launch of a call goes to the caller's stream (one
 * programmatic-dependent-launch chain, no internal streams or events).
 *
 * Errors: a non-zero runlora_status_t; runlora_last_error() returns a
 * thread-local message naming the offending argument(s).  No C++ exception
 * crosses this boundary.  Asynchronous device faults surface at the caller's
 * next synchronisation.
 */
#ifndef RUNLORA_H_
#define RUNLORA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RUNLORA_ABI_VERSION 2

typedef enum {
  RUNLORA_OK = 0,
  RUNLORA_ERR_INVALID_ARG = 1,      /* null pointer, n/k/m/r <= 0, bad enum */
  RUNLORA_ERR_SHAPE = 2,            /* inconsistent shapes */
  RUNLORA_ERR_DTYPE = 3,            /* unsupported dtype combination */
  RUNLORA_ERR_UNSUPPORTED_VARIANT = 4, /* backward6..8 passed to an execute call */
  RUNLORA_ERR_OVERFLOW = 5,         /* FLOP count does not fit in uint64 */
  RUNLORA_ERR_ALIGNMENT = 6,        /* pointer not 16B aligned, or bf16 k/m/r not multiple of 8 */
  RUNLORA_ERR_WORKSPACE = 7,        /* workspace smaller than runlora_workspace_size() */
  RUNLORA_ERR_CUDA = 8,             /* a CUDA runtime/driver call or launch failed */
  RUNLORA_ERR_TIMING = 9,           /* time-based selection could not measure */
  RUNLORA_ERR_DEVICE = 10           /* device is not sm_100 (B200) */
} runlora_status_t;

typedef enum { RUNLORA_F32 = 0, RUNLORA_BF16 = 1 } runlora_dtype_t;

/* Forward variant numbers: 1 = forward1 (Eq. 1), 2 = forward2 (Eq. 2).
 * Backward variant numbers: 1..8 = backwardN; 1..5 executable. */
typedef enum { RUNLORA_BY_FLOPS = 0, RUNLORA_BY_TIME = 1, RUNLORA_HYBRID = 2 } runlora_criterion_t;

typedef struct {
  int64_t n, k, m, r;   /* tokens (b·s), in (i), out (o), rank */
  int32_t dtype;        /* runlora_dtype_t of X, W, A, B, dY, Y, dX */
} runlora_shape_t;

typedef struct {
  int32_t fwd;                 /* chosen forward variant (1|2) */
  int32_t bwd;                 /* chosen backward variant (1..5) */
  int32_t criterion;           /* runlora_criterion_t used */
  int32_t param_reduction;     /* Eq. 5 holds (1) or not (0); a violation is not an error */
  uint64_t flops_fwd[3];       /* index = variant number; [0] unused */
  uint64_t flops_bwd[9];       /* index = variant number 1..8; [0] unused */
  float time_fwd_us[3];        /* median device time per candidate; NaN if not timed */
  float time_bwd_us[9];
  int32_t flops_fwd_pick;      /* the FLOP-criterion pick, always reported */
  int32_t flops_bwd_pick;
} runlora_plan_t;

/* Device operand set for time-based selection (all device pointers, caller-owned;
 * Y, dX, dA, dB are overwritten while candidates are timed). */
typedef struct {
  const void *X, *W, *A, *B, *dY;
  void *Y, *dX, *dA, *dB;
  int32_t grad_dtype;          /* runlora_dtype_t of dA/dB */
} runlora_operands_t;

typedef struct runlora_handle_s* runlora_handle_t;

/* Per-kernel profile record (runlora_profile_read). */
typedef struct {
  char name[48];
  uint64_t launches;
  double total_ms;   /* sum of CUDA-event durations of this kernel's launches */
} runlora_kernel_stat_t;

/* ---------------------------------------------------------------- lifetime */
const char* runlora_version(void);
/* Creates a handle bound to CUDA `device`; fails with RUNLORA_ERR_DEVICE unless
 * the device is compute capability 10.0 (sm_100a code only). */
runlora_status_t runlora_create(runlora_handle_t* out, int device);
runlora_status_t runlora_destroy(runlora_handle_t h);

/* -------------------------------------------------------------- cost model
 * Table 1 as printed, exact uint64 arithmetic (overflow-checked).
 * is_backward = 0: variant in {1,2}; is_backward = 1: variant in {1..8}.
 * dtype is ignored. */
runlora_status_t runlora_flops(const runlora_shape_t* s, int is_backward, int variant, uint64_t* out);
/* Eq. 5: 1 iff r(k+m) < k·m. */
int runlora_param_reduction(const runlora_shape_t* s);
/* Bytes of device workspace that runlora_forward(fwd) and runlora_backward(bwd)
 * (and the split _params/_input pair) need for shape s.  fwd or bwd may be 0 to
 * size only the other.  The same workspace may be reused across calls. */
runlora_status_t runlora_workspace_size(const runlora_shape_t* s, int fwd, int bwd, size_t* bytes);

/* ---------------------------------------------------------------- selector
 * RUNLORA_BY_FLOPS: argmin of Table 1 over {F1,F2} and {B1..B5}, ties to the
 *   lowest index ("with flops criterion").  `ops`, workspace, stream unused.
 * RUNLORA_BY_TIME: every executable candidate is run on `ops` on `stream`
 *   (3 warm-up rounds, 15 timed rounds, candidates interleaved; one rep = 4
 *   back-to-back calls between CUDA events; median); forward and backward timed
 *   independently; argmin of the medians (within 1 %: fewer FLOPs wins).  Needs a workspace of
 *   runlora_workspace_size(s, 2, 4) bytes or more (the largest candidate set).
 *   Blocks the calling thread until timing is done.
 * RUNLORA_HYBRID: as TIME but only candidates within 2x of the FLOP minimum.
 * The FLOP pick is always reported in flops_*_pick.  Plans are cached in the
 * handle per (shape, criterion). */
runlora_status_t runlora_select(runlora_handle_t h, const runlora_shape_t* s, int criterion,
                                const runlora_operands_t* ops, void* workspace, size_t ws_bytes,
                                void* stream, runlora_plan_t* out);

/* ----------------------------------------------------------------- execute
 * Y[n,m] is overwritten.  fwd in {1,2}. */
runlora_status_t runlora_forward(runlora_handle_t h, int fwd, const runlora_shape_t* s,
                                 const void* X, const void* W, const void* A, const void* B, void* Y,
                                 void* workspace, size_t ws_bytes, void* stream);

/* dX[n,k] (nullable: skipped), dA[k,r], dB[r,m].  bwd in {1..5}.
 * grad_dtype: dtype of dA/dB (RUNLORA_F32 or RUNLORA_BF16; must be RUNLORA_F32
 * when s->dtype is RUNLORA_F32).  accumulate != 0 adds into dA/dB instead of
 * overwriting (micro-batch accumulation); dA/dB are reduced over all n tokens in
 * fp32 before the single rounding to grad_dtype. */
runlora_status_t runlora_backward(runlora_handle_t h, int bwd, const runlora_shape_t* s,
                                  const void* X, const void* W, const void* A, const void* B,
                                  const void* dY, void* dX, void* dA, void* dB, int grad_dtype,
                                  int accumulate, void* workspace, size_t ws_bytes, void* stream);

/* Split backward for data-parallel overlap: _params computes dA, dB (and, for
 * backward1..3, leaves Z1 = dY·Bᵀ — and for backward1 A repeated per Z1 block —
 * in the workspace); _input computes dX and must follow the _params call of the
 * same variant/shape with the same workspace on the same stream (for backward4/5
 * _input is self-contained).  runlora_backward == _params then _input. */
runlora_status_t runlora_backward_params(runlora_handle_t h, int bwd, const runlora_shape_t* s,
                                         const void* X, const void* W, const void* A, const void* B,
                                         const void* dY, void* dA, void* dB, int grad_dtype, int accumulate,
                                         void* workspace, size_t ws_bytes, void* stream);
runlora_status_t runlora_backward_input(runlora_handle_t h, int bwd, const runlora_shape_t* s,
                                        const void* X, const void* W, const void* A, const void* B,
                                        const void* dY, void* dX, void* workspace, size_t ws_bytes,
                                        void* stream);

/* forward2 in two halves (Eq. 2; "forward2" computes X(W + AB)):
 *   runlora_wprime_t:       Wpt = (W + A·B)ᵀ, [m, k] bf16 row-major (fp32 accumulation, one
 *                           rounding; the identity-tail GEMM forward2 itself runs)
 *   runlora_forward_wprime: Y = X·W' reading Wpt (the main GEMM forward2 itself runs)
 * Together they are runlora_forward(2) bit for bit.  For callers that reuse W' while A and B
 * are unchanged — the micro-batches of one gradient-accumulation step — and so build it once
 * per step instead of once per call; keeping Wpt valid (rebuilding it after A or B change) is
 * the caller's job.  Wpt: caller device memory, m·k bf16, 16-byte aligned.  bf16 shapes only
 * (else RUNLORA_ERR_DTYPE).  runlora_wprime_t needs no workspace; runlora_forward_wprime needs
 * runlora_workspace_size(s, 2, 0) bytes.  runlora_wprime_t_wq: the same from a quantized W
 * (Wq, scale, diag below; m a multiple of 16).  Asynchronous on `stream`. */
runlora_status_t runlora_wprime_t(runlora_handle_t h, const runlora_shape_t* s, const void* W, const void* A,
                                  const void* B, void* Wpt, void* stream);
runlora_status_t runlora_wprime_t_wq(runlora_handle_t h, const runlora_shape_t* s, const void* Wq,
                                     const float* scale, const void* diag, const void* A, const void* B, void* Wpt,
                                     void* stream);
runlora_status_t runlora_forward_wprime(runlora_handle_t h, const runlora_shape_t* s, const void* X, const void* Wpt,
                                        void* Y, void* workspace, size_t ws_bytes, void* stream);

/* End-to-end step from HOST buffers: H2D copies of X_host and dY_host into the
 * device staging buffers X, dY; forward(fwd) into Y; backward(bwd) into dX, dA,
 * dB; then, if `exchange` is non-NULL, exchange(exchange_user, stream) is called on
 * the calling thread (the data-parallel allreduce of dA, dB is enqueued there, so
 * the host copies below receive the summed gradients); then D2H copies of dA, dB
 * into dA_host, dB_host (and of Y / dX when Y_host / dX_host are non-NULL).
 * Everything is enqueued on `stream`; the call returns without synchronising.
 * W, A, B are device pointers (resident parameters).  Every argument (variants,
 * pointers, workspace) is validated before the first copy is enqueued. */
typedef void (*runlora_exchange_fn)(void* user, void* stream);
typedef struct {
  int32_t fwd, bwd, grad_dtype, accumulate;
  const void *X_host, *dY_host;          /* host inputs  */
  void *Y_host, *dX_host;                /* host outputs, nullable */
  void *dA_host, *dB_host;               /* host outputs */
  const void *W, *A, *B;                 /* device parameters */
  void *X, *dY, *Y, *dX, *dA, *dB;       /* device staging buffers */
  runlora_exchange_fn exchange;          /* nullable (ABI version 2) */
  void* exchange_user;
} runlora_host_step_t;
runlora_status_t runlora_step_host(runlora_handle_t h, const runlora_shape_t* s, const runlora_host_step_t* st,
                                   void* workspace, size_t ws_bytes, void* stream);

/* ---------------------------------------------- quantized frozen weight (QLoRA-style)
 * "functionality to work with quantized model weights to fine-tune models in fashion of
 * QLoRA" (no format given).  Format (R18): FP8 E4M3 (OCP E4M3FN: bias 7,
 * max 448, no infinities) with one power-of-two scale per output column:
 *   e[j]     = clamp(ceil(log2(max_i |W[i, j]| / 448)), -16, 15)   (0 for an all-zero column)
 *   scale[j] = 2^e[j],  Wq[i, j] = e4m3_rn_satfinite(W[i, j] / scale[j])   (Wq: k x m bytes)
 *   W~[i, j] = e4m3(Wq[i, j]) · scale[j]   (exact — what the hot path multiplies by)
 *   diag     = m x 128 bytes, E5M2: row j holds 2^e[j] at column j mod 128, zeros elsewhere
 *              (the scale as a diagonal matrix the tensor cores multiply Wq by)
 * runlora_quantize_w_e4m3: W bf16 [k, m] (device) -> Wq, scale, diag (device; 16-byte aligned,
 *   m a multiple of 16).  Asynchronous on `stream`.
 * runlora_forward_wq / runlora_backward_wq: as runlora_forward / runlora_backward with W
 *   given as (Wq, scale, diag); only those persist between calls (about half of the bf16 W).
 *   The dequantization rides in the tensor cores: forward2's W'ᵀ and backward4/5's W' are
 *   built straight from the 1-byte Wq by one GEMM whose FP8 tail multiplies Wq by the scale
 *   diagonal (kind::f8f6f4, exact) into the same accumulator as A·B, D = bf16(A·B + W~);
 *   forward1 and backward1..3, which multiply by W~ itself, get it from the same GEMM without
 *   the A·B part, written after the regular workspace.  m must be a multiple of 16, else
 *   RUNLORA_ERR_ALIGNMENT.  Workspace: runlora_workspace_size_wq bytes. */
runlora_status_t runlora_quantize_w_e4m3(runlora_handle_t h, int64_t k, int64_t m, const void* W, void* Wq,
                                         float* scale, void* diag, void* stream);
runlora_status_t runlora_workspace_size_wq(const runlora_shape_t* s, int fwd, int bwd, size_t* bytes);
runlora_status_t runlora_forward_wq(runlora_handle_t h, int fwd, const runlora_shape_t* s, const void* X,
                                    const void* Wq, const float* scale, const void* diag, const void* A,
                                    const void* B, void* Y, void* workspace, size_t ws_bytes, void* stream);
runlora_status_t runlora_backward_wq(runlora_handle_t h, int bwd, const runlora_shape_t* s, const void* X,
                                     const void* Wq, const float* scale, const void* diag, const void* A,
                                     const void* B, const void* dY, void* dX, void* dA, void* dB, int grad_dtype,
                                     int accumulate, void* workspace, size_t ws_bytes, void* stream);

/* ---------------------------------------------- data-parallel exchange (one-shot allreduce)
 * The DP exchange step (token-sharded ranks; a8 reduces the per-rank
 * adapter gradients dA = Xᵀ·dY·Bᵀ, dB = Aᵀ·Xᵀ·dY, which are sums over tokens, Eq. 3):
 *   out[i] = sum_{p = 0 .. P-1} peers[p][i]      (fp32, i < n, rank order 0, 1, .., P-1)
 * read directly from the P ranks' device buffers (peer pointers valid in this process:
 * CUDA IPC / torch symmetric memory, NVLink P2P loads).  Every rank that calls it with the
 * same peers gets a bit-identical result.  peers: HOST array of P device pointers (16-byte
 * aligned, n floats each, 1 <= P <= 16); out: this rank's device buffer (16-byte aligned),
 * not one of the peers'.  Ordering across ranks is the caller's: every rank's writes to its
 * buffer must be visible before any rank's call (a cross-rank barrier on `stream`), and no
 * buffer may be rewritten until every rank's call has finished (a second barrier).
 * Asynchronous on `stream`.  Errors: INVALID_ARG (P, n, null/aliased pointers), ALIGNMENT. */
runlora_status_t runlora_allreduce_sum_f32(runlora_handle_t h, const float* const* peers, int P, float* out,
                                           int64_t n, void* stream);

/* ------------------------------------ fused data-parallel exchange (issued by the dX GEMM)
 * The a8 exchange step fused into the backward: with the tokens sharded
 * over P ranks, dA = Xᵀ·dY·Bᵀ and dB = Aᵀ·Xᵀ·dY of the full batch are the sums of the ranks'
 * partial sums (Eq. 3 sums over tokens).  runlora_backward_exchange runs the backward
 * like runlora_backward, but the idle warps of its dX GEMM launch — concurrently with that
 * GEMM's mainloop — sum this rank's token-split slabs in fixed order into its exchange buffer,
 * publish each 64-row chunk to every rank (flag stores over NVLink), wait for every rank's
 * chunk, and write dA, dB = the rank-order sum over ranks (peer loads: bit-identical on every
 * rank), or the switch-side sum multimem.ld_reduce when a multicast address is given (NVLS).
 * No NCCL call, no extra launch.  Every rank must call it for the same shape, variant and
 * epoch, on GPUs that run concurrently (never several ranks on one GPU).
 *
 * runlora_exchange_sizes: bytes of each rank's exchange buffer (2 epoch halves of r·(k+m)
 *   fp32) and flag array (ceil((k+m)/64)·P uint32) — allocate both in memory every rank can
 *   address (CUDA IPC / torch symmetric memory), the flags zero-initialised.
 * runlora_exchange_create: this rank's view: bufs / flags = HOST arrays of P device pointers
 *   (rank order, as mapped in this process), mc = multicast address of the buffers or NULL.
 *   Allocates a small device descriptor (setup time, not on the forward/backward path).
 * runlora_backward_exchange: grad_dtype must be RUNLORA_F32, dX non-NULL (the exchange rides
 *   on the dX GEMM), bf16 operands; epoch = 1, 2, 3, ... per exchange (same on every rank; the
 *   buffer half alternates with it, so consecutive steps never overwrite what a slow peer
 *   still reads).  Errors as runlora_backward, plus INVALID_ARG for a bad exchange/epoch. */
typedef struct runlora_exchange_s* runlora_exchange_t;
runlora_status_t runlora_exchange_sizes(int64_t k, int64_t m, int64_t r, int P, size_t* buf_bytes,
                                        size_t* flag_bytes);
runlora_status_t runlora_exchange_create(runlora_handle_t h, int P, int rank, int64_t k, int64_t m, int64_t r,
                                         void* const* bufs, void* const* flags, void* mc, runlora_exchange_t* out);
runlora_status_t runlora_exchange_destroy(runlora_exchange_t x);
runlora_status_t runlora_backward_exchange(runlora_handle_t h, int bwd, const runlora_shape_t* s, const void* X,
                                           const void* W, const void* A, const void* B, const void* dY, void* dX,
                                           void* dA, void* dB, int grad_dtype, int accumulate, runlora_exchange_t x,
                                           uint32_t epoch, void* workspace, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------- tracing
 * When enabled, every kernel the library launches is bracketed by CUDA events
 * on its stream; runlora_profile_read synchronises those events and returns
 * per-kernel totals (and resets them when reset != 0). */
runlora_status_t runlora_profile_enable(runlora_handle_t h, int enable);
runlora_status_t runlora_profile_read(runlora_handle_t h, runlora_kernel_stat_t* stats, int max_stats,
                                      int* count, int reset);
/* Number of kernels this handle has launched since creation. */
uint64_t runlora_launch_count(runlora_handle_t h);

const char* runlora_status_string(runlora_status_t st);
const char* runlora_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* RUNLORA_H_ */
