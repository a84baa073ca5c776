// C ABI of the RunLoRA hot path (include/runlora.h): validation, Table 1 cost
// model, selector, and the launch sequence of every forward/backward variant.
//
// Variant sequences (bf16; every product is one tcgen05 launch, see tc_gemm.cuh):
//   forward1:  Z2 = X·A                      [proj, split-K -> reduce -> bf16]
//                     Y  = [X | Z2]·[W ; B]         [main GEMM, concat-K tail]
//   forward2:  W' = W + A·B                  [K = r, epilogue adds W, bf16]
//                     Y  = X·W'                     [main GEMM]
//   backward1 (Alg.1): Z1 = dY·Bᵀ; Z2 = X·A; dA = Xᵀ·Z1; dB = Z2ᵀ·dY;
//                     dX = [dY | Z1]·[Wᵀ ; Aᵀ]
//   backward2 (Alg.2): Z1; Z2' = Xᵀ·dY; dA = Xᵀ·Z1; dB = Aᵀ·Z2'; dX as B1
//   backward3 (Alg.3): Z1; Z2'; dA = Z2'·Bᵀ; dB = Aᵀ·Z2'; dX as B1
//   backward4 (Alg.4): Z2'; dA = Z2'·Bᵀ; dB = Aᵀ·Z2'; W' = W+AB; dX = dY·W'ᵀ
//   backward5 (Alg.5): Z1; Z2; dA = Xᵀ·Z1; dB = Z2ᵀ·dY; W' = W+AB; dX = dY·W'ᵀ
// dB is produced as dBᵀ = (·)ᵀ·(·) so that the rank sits on the MMA's N axis and is
// transposed by the split-K reducer.  fp32 (RUNLORA_F32) runs the same algorithm
// lines with the fp32 SIMT GEMM (true FFMA; the 1e-5 tolerance excludes TF32).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>
#include <algorithm>

#include "internal.h"
#include "tc_gemm.cuh"

using namespace runlora;

struct runlora_handle_s {
  Ctx* ctx;
};

struct runlora_exchange_s {
  XDesc* d_desc;  // device copy
  int P, rank, device;
  int64_t k, m, r;
};

namespace {

thread_local std::string g_last_error;

runlora_status_t fail(runlora_status_t st, const std::string& msg) {
  g_last_error = msg;
  return st;
}

#define RL_TRY(expr)                       \
  do {                                     \
    runlora_status_t _st = (expr);         \
    if (_st != RUNLORA_OK) return _st;     \
  } while (0)

// Makes the handle's device (and its primary context) current on the calling thread —
// callers such as PyTorch's autograd engine run the backward on their own threads, where
// the driver-API TMA encoder would otherwise see no current context — and restores the
// previously selected device afterwards.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    cudaSetDevice(dev);
    if (prev == dev) prev = -1;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

bool mul_ok(unsigned __int128 v) { return v <= (unsigned __int128)UINT64_MAX; }

runlora_status_t check_shape(const runlora_shape_t* s) {
  if (!s) return fail(RUNLORA_ERR_INVALID_ARG, "shape is NULL");
  if (s->n <= 0 || s->k <= 0 || s->m <= 0 || s->r <= 0) {
    char b[160];
    snprintf(b, sizeof b, "n, k, m, r must all be >= 1 (got n=%lld k=%lld m=%lld r=%lld)", (long long)s->n,
             (long long)s->k, (long long)s->m, (long long)s->r);
    return fail(RUNLORA_ERR_INVALID_ARG, b);
  }
  if (s->dtype != RUNLORA_F32 && s->dtype != RUNLORA_BF16) return fail(RUNLORA_ERR_DTYPE, "dtype must be F32 or BF16");
  const int64_t lim = (int64_t)1 << 31;
  if (s->n >= lim || s->k >= lim || s->m >= lim || s->r >= lim)
    return fail(RUNLORA_ERR_INVALID_ARG, "each of n, k, m, r must be < 2^31");
  if (s->dtype == RUNLORA_BF16 && ((s->k | s->m | s->r) & 7)) {
    char b[160];
    snprintf(b, sizeof b, "bf16 needs k, m, r multiples of 8 for 16-byte TMA row strides (k=%lld m=%lld r=%lld)",
             (long long)s->k, (long long)s->m, (long long)s->r);
    return fail(RUNLORA_ERR_ALIGNMENT, b);
  }
  return RUNLORA_OK;
}

runlora_status_t check_ptr(const void* p, const char* name, bool nullable = false) {
  if (!p) {
    if (nullable) return RUNLORA_OK;
    return fail(RUNLORA_ERR_INVALID_ARG, std::string(name) + " is NULL");
  }
  if (reinterpret_cast<uintptr_t>(p) & 15) return fail(RUNLORA_ERR_ALIGNMENT, std::string(name) + " is not 16-byte aligned");
  return RUNLORA_OK;
}

runlora_status_t cuda_fail(cudaError_t e, const char* what) {
  char b[256];
  snprintf(b, sizeof b, "%s: %s", what, cudaGetErrorString(e));
  return fail(RUNLORA_ERR_CUDA, b);
}

// ------------------------------------------------------------ Table 1
runlora_status_t flops_of(const runlora_shape_t* s, int is_backward, int v, uint64_t* out) {
  typedef unsigned __int128 u;
  const u n = (u)s->n, i = (u)s->k, o = (u)s->m, r = (u)s->r;
  u f;
  if (!is_backward) {
    if (v == 1) f = 2 * n * (i * o + r * i + o * r);
    else if (v == 2) f = 2 * (i * o * r + n * o * i);
    else return fail(RUNLORA_ERR_INVALID_ARG, "forward variant must be 1 or 2 (P:62-64)");
  } else {
    switch (v) {
      case 1: f = 2 * n * (2 * o * r + 3 * i * r + o * i); break;
      case 2: f = 2 * n * (o * r + 2 * i * r + 2 * i * o) + 2 * i * o * r; break;
      case 3: f = 2 * n * (2 * i * o + o * r + i * r) + 4 * i * r * o; break;
      case 4: f = 2 * (2 * n * i * o + 3 * i * o * r); break;
      case 5: f = 2 * n * (2 * o * r + 2 * i * r + o * i) + 2 * i * o * r; break;
      case 6: f = 2 * n * (2 * o * r + 2 * i * r + 2 * o * i) + 4 * i * o * r; break;
      case 7:
      case 8: f = 2 * n * (o * r + i * r + 2 * o * i) + 4 * i * o * r; break;
      default: return fail(RUNLORA_ERR_INVALID_ARG, "backward variant must be 1..8 (P:84-94)");
    }
  }
  if (!mul_ok(f)) return fail(RUNLORA_ERR_OVERFLOW, "FLOP count exceeds uint64");
  *out = (uint64_t)f;
  return RUNLORA_OK;
}

size_t al(size_t x) { return (x + 255) & ~size_t(255); }
DeviceMat mat(const void* p, int64_t rows, int64_t cols) { return DeviceMat{p, rows, cols, cols}; }

// -------------------------------------------------------------- skinny plans
// A "skinny" product has a rank-r output axis: out[rows, r] = A_op[rows, K]·B_op[K, r].
// One launch runs up to two of them (e.g. Z1 and Z2 together).  With enough row tiles
// to fill the GPU they write bf16 directly; otherwise they split K (the long axis)
// into fp32 partial slabs reduced in fixed order by one reducer launch (deterministic).
constexpr int kSmTarget = 148;  // fixed so that workspace sizes are device-independent
constexpr int kMaxSplits = 32;

struct Skinny {
  DeviceMat a;
  bool a_mn;
  DeviceMat b;
  bool b_mn;
  int64_t rows, K, r;
  void* out;
  bool out_bf16;
  int64_t ldo;
  bool transpose, accumulate;
};

int skinny_bn(int64_t r, bool b_mn) {
  if (b_mn) return r <= 16 ? 16 : r <= 32 ? 32 : r <= 64 ? 64 : r <= 128 ? 128 : 256;
  static const int opts[] = {16, 32, 48, 64, 128, 256};
  for (int o : opts)
    if (r <= o) return o;
  return 256;
}

struct SkinnyPlan {
  int n;             // jobs
  bool direct;       // outputs written by the GEMM epilogue (no partials)
  int BN[2], Npad[2], splits[2], kps[2];
  size_t p_off[2];   // byte offsets of the partial slabs in the workspace P region
  size_t p_bytes;    // total partial bytes
};

bool can_direct(const Skinny& j) { return j.out_bf16 && !j.transpose && !j.accumulate && j.ldo == j.r; }

SkinnyPlan plan_skinny(const Skinny* jobs, int n) {
  SkinnyPlan p{};
  p.n = n;
  int64_t tiles = 0, kb_max = 0;
  bool direct_ok = true;
  for (int i = 0; i < n; ++i) {
    p.BN[i] = skinny_bn(jobs[i].r, jobs[i].b_mn);
    const int64_t ntn = (jobs[i].r + p.BN[i] - 1) / p.BN[i];
    p.Npad[i] = (int)(ntn * p.BN[i]);
    tiles += ((jobs[i].rows + kBM - 1) / kBM) * ntn;
    kb_max = std::max<int64_t>(kb_max, (jobs[i].K + kBK - 1) / kBK);
    direct_ok = direct_ok && can_direct(jobs[i]);
  }
  // enough row tiles (>= 2/3 of the SMs busy) -> no split, direct bf16 epilogue;
  // otherwise the smallest split that fills one wave of CTA slots (2 per SM for these
  // HBM-bound kernels): fewer splits = smaller fp32 slabs and a cheaper reducer.
  p.direct = direct_ok && 3 * tiles >= 2 * kSmTarget;
  int64_t s = 1;
  if (!p.direct) {
    s = std::max<int64_t>(1, (2 * kSmTarget) / std::max<int64_t>(tiles, 1));
    s = std::min<int64_t>(s, std::min<int64_t>(kMaxSplits, kb_max));
  }
  size_t off = 0;
  for (int i = 0; i < n; ++i) {
    const int64_t kb = (jobs[i].K + kBK - 1) / kBK;
    const int64_t si = std::min<int64_t>(s, kb);
    p.kps[i] = (int)((kb + si - 1) / si);
    p.splits[i] = (int)((kb + p.kps[i] - 1) / p.kps[i]);
    p.p_off[i] = off;
    if (!p.direct) off += al((size_t)p.splits[i] * (size_t)jobs[i].rows * (size_t)p.Npad[i] * 4);
  }
  p.p_bytes = off;
  return p;
}

GemmReq base_req(int M, int N, KernelId kid) {
  GemmReq q;
  memset(&q, 0, sizeof q);
  q.M = M;
  q.N = N;
  q.splits = 1;
  q.cg = 1;
  q.kid = kid;
  return q;
}

// Split (!direct) plans reduce their fp32 slabs inside the same launch: the last split of
// each output tile to finish sums the slabs in split order (Prob::fixup, deterministic).
// The fix-up counters (per output tile) are zeroed by a memset node ahead of the launch —
// this path serves shapes off the hot configurations (small n, backward2..4); the backward1/5
// hot path zeroes them inside its projection launch instead (grads_tok_bf16).  With `defer`
// the slabs are not reduced here: their ReduceJobs are returned for the idle warps of the dX
// GEMM launch that follows (do_backward).
runlora_status_t run_skinny(Ctx& c, const Skinny* jobs, int n, float* P, int* counters, KernelId kid,
                            cudaStream_t st, std::vector<ReduceJob>* defer = nullptr) {
  const SkinnyPlan p = plan_skinny(jobs, n);
  GemmReq q[2];
  int ntiles = 0;
  for (int i = 0; i < n; ++i) {
    const Skinny& j = jobs[i];
    q[i] = base_req((int)j.rows, p.direct ? (int)j.r : p.Npad[i], kid);
    q[i].a = j.a;
    q[i].a_mn = j.a_mn;
    q[i].b = j.b;
    q[i].b_mn = j.b_mn;
    q[i].K1 = (int)j.K;
    q[i].BN = p.BN[i];
    q[i].a_stream_once = true;
    float* Pi = reinterpret_cast<float*>(reinterpret_cast<char*>(P) + p.p_off[i]);
    if (p.direct) {
      q[i].out_mode = OUT_BF16;
      q[i].D = j.out;
      q[i].ldd = j.ldo;
    } else {
      q[i].out_mode = OUT_F32;
      q[i].D = Pi;
      q[i].ldd = p.Npad[i];
      q[i].split_stride = j.rows * (int64_t)p.Npad[i];
      q[i].splits = p.splits[i];
      q[i].kb_per_split = p.kps[i];
      if (defer) {  // reduced by the idle warps of a later launch (see do_backward)
        defer->push_back(ReduceJob{Pi, p.splits[i], j.rows * (int64_t)p.Npad[i], (int)j.rows, (int)j.r, p.Npad[i],
                                   j.out, j.out_bf16 ? 1 : 0, j.ldo, j.transpose ? 1 : 0, j.accumulate ? 1 : 0});
        continue;
      }
      q[i].fixup = true;
      q[i].counters = counters + ntiles;
      q[i].fx_out = j.out;
      q[i].fx_ldo = j.ldo;
      q[i].fx_cols = (int)j.r;
      q[i].fx_transpose = j.transpose;
      q[i].fx_accumulate = j.accumulate;
      q[i].fx_bf16 = j.out_bf16;
      ntiles += (int)(((j.rows + kBM - 1) / kBM) * (p.Npad[i] / p.BN[i]));
    }
  }
  if (!p.direct && ntiles > 0) {
    cudaError_t e = cudaMemsetAsync(counters, 0, sizeof(int) * (size_t)ntiles, st);
    if (e != cudaSuccess) return cuda_fail(e, "fix-up counter reset");
  }
  std::string err;
  cudaError_t e = launch_tc_gemm(c, q, n, st, &err);
  if (e != cudaSuccess) return fail(RUNLORA_ERR_CUDA, err.empty() ? cudaGetErrorString(e) : err);
  return RUNLORA_OK;
}

// Job builders (names follow Alg. 1-5).
Skinny job_Z1(const runlora_shape_t& s, const void* dY, const void* B, void* z1) {  // Z1 = dY·Bᵀ
  return Skinny{mat(dY, s.n, s.m), false, mat(B, s.r, s.m), false, s.n, s.m, s.r, z1, true, s.r, false, false};
}
Skinny job_Z2(const runlora_shape_t& s, const void* X, const void* A, void* z2) {  // Z2 = X·A
  return Skinny{mat(X, s.n, s.k), false, mat(A, s.k, s.r), true, s.n, s.k, s.r, z2, true, s.r, false, false};
}
Skinny job_dA_tok(const runlora_shape_t& s, const void* X, const void* z1, void* dA, bool gb, bool acc) {
  return Skinny{mat(X, s.n, s.k), true, mat(z1, s.n, s.r), true, s.k, s.n, s.r, dA, gb, s.r, false, acc};
}
Skinny job_dB_tok(const runlora_shape_t& s, const void* dY, const void* z2, void* dB, bool gb, bool acc) {
  return Skinny{mat(dY, s.n, s.m), true, mat(z2, s.n, s.r), true, s.m, s.n, s.r, dB, gb, s.m, true, acc};
}
Skinny job_dA_dense(const runlora_shape_t& s, const void* z2d, const void* B, void* dA, bool gb, bool acc) {
  return Skinny{mat(z2d, s.k, s.m), false, mat(B, s.r, s.m), false, s.k, s.m, s.r, dA, gb, s.r, false, acc};
}
Skinny job_dB_dense(const runlora_shape_t& s, const void* z2d, const void* A, void* dB, bool gb, bool acc) {
  return Skinny{mat(z2d, s.k, s.m), true, mat(A, s.k, s.r), true, s.m, s.k, s.r, dB, gb, s.m, true, acc};
}

// Backward1/5 adapter gradients (Alg. 1 lines 1-4 / Alg. 5 lines 1-4)
// in two launches that keep every CTA slot streaming:
//   projections   Z1 = dY·Bᵀ, Z2 = X·A, split over K (m for Z1, k for Z2) into sz bf16
//                 partials stored side by side, Zp = [Z_0 | .. | Z_{sz-1}] (n x sz*r), so no
//                 split-K fix-up sits on the epilogue path;
//   reductions    dA = Xᵀ·Z1 = Σ_s Xᵀ·Z1_s and dBᵀ = dYᵀ·Z2: ONE MMA against all blocks
//                 (N = sz*r), the epilogue folds the sz column blocks in fixed order; split
//                 over tokens into fp32 slabs summed by the deterministic reducer.
// backward1's dX tail then reads Zp against A repeated sz times (Σ_s Z1_s·Aᵀ).
// The plan is a pure function of the shape (and environment), so backward_input knows
// which Z1 layout backward_params left in the workspace.
struct ZPlan {
  bool ok;
  int sz, kpz[2];        // projection K-splits (Z1, Z2 alike) and k-blocks per split
  int szf, kpzf;         // forward1's Z2 = X·A alone: its K-split and k-blocks per split
  int bn_z[2];           // MMA N of the projections
  int bn_t;              // MMA N of the reductions (sz * r when the partials are folded)
  int tsplits, kpt;      // token-reduction splits and k-blocks (64 tokens) per split
  size_t off[2], bytes;  // fp32 slab regions: dA, dB
};

ZPlan plan_z(const runlora_shape_t& s) {
  ZPlan f{};
  if (s.dtype != RUNLORA_BF16) return f;
  const int64_t n = s.n, k = s.k, m = s.m, r = s.r;
  const int64_t mt = (n + kBM - 1) / kBM;
  const int64_t nkb_n = (n + kBK - 1) / kBK;
  f.bn_z[0] = skinny_bn(r, false);  // Z1: B_op = Bᵀ from B [r, m] (K-major)
  f.bn_z[1] = skinny_bn(r, true);   // Z2: B_op = A [k, r] (MN-major)
  if (r > f.bn_z[0] || r > f.bn_z[1]) return f;  // one n tile per projection
  // sz: split K only while the projections' 2*mt row tiles leave SMs idle (2*mt*sz <= one
  // wave of 2 CTAs/SM), within sz*r in {16, 32, 64} — 128 for r = 64 — (a legal MN-major tile
  // width that keeps the reductions on the 2-CTA/SM kernel) and r a fold width (8, 16, 32,
  // 64).  At C2 (mt = 64) this gives sz = 2 for r = 16 (projections 41 -> 34 µs) and for
  // r = 64 (40 -> 27 µs; the reductions +2 µs and backward1's dX tail one more k-block:
  // steps 0.958-0.967x, profiles/r02/ab_z64.jsonl).  env RUNLORA_ZSPLIT64=0: sz = 1 at r = 64.
  const int64_t kbz[2] = {(m + kBK - 1) / kBK, (k + kBK - 1) / kBK};
  int sz = 1;
  static const bool split64 = getenv("RUNLORA_ZSPLIT64") == nullptr || atoi(getenv("RUNLORA_ZSPLIT64")) != 0;
  if ((r == 8 || r == 16 || r == 32 || (r == 64 && split64)) && 2 * mt < 148) {
    for (int c = 2; c <= 8 && 2 * mt * c <= 2 * 148; c *= 2) {
      if (c * r > (r == 64 ? 128 : 64)) break;
      bool even = true;
      for (int i = 0; i < 2; ++i) {
        const int64_t kp = (kbz[i] + c - 1) / c;
        even = even && (kbz[i] + kp - 1) / kp == c;
      }
      if (!even) break;
      sz = c;
    }
  }
  if (const char* e = getenv("RUNLORA_ZSPLIT")) sz = std::max(1, atoi(e));
  f.sz = sz;
  // forward1 runs Z2 alone (mt row tiles): the same rule with half the tiles
  int szf = 1;
  if ((r == 8 || r == 16 || r == 32) && mt < 148) {
    for (int c = 2; c <= 8 && mt * c <= 2 * 148; c *= 2) {
      if (c * r > 64) break;
      const int64_t kp = (kbz[1] + c - 1) / c;
      if ((kbz[1] + kp - 1) / kp != c) break;
      szf = c;
    }
  }
  f.szf = szf;
  f.kpzf = (int)((kbz[1] + szf - 1) / szf);
  for (int i = 0; i < 2; ++i) {
    f.kpz[i] = (int)((kbz[i] + sz - 1) / sz);
    if ((kbz[i] + f.kpz[i] - 1) / f.kpz[i] != sz) return f;
  }
  f.bn_t = sz > 1 ? (int)(sz * r) : skinny_bn(r, true);
  if (r > f.bn_t || f.bn_t > 256) return f;
  // without K-split blocks the projections need enough row tiles to stream from every SM;
  // otherwise the fp32 split-K path (run_skinny + reducer) is the better plan
  if (sz == 1 && 3 * 2 * mt < 2 * 148) return f;
  // token splits: as many as fit in one wave of CTA slots
  const int64_t tiles = (k + kBM - 1) / kBM + (m + kBM - 1) / kBM;
  int64_t ts = std::max<int64_t>(1, (2 * 148) / tiles);
  ts = std::min<int64_t>({ts, 32, nkb_n});
  f.kpt = (int)((nkb_n + ts - 1) / ts);
  f.tsplits = (int)((nkb_n + f.kpt - 1) / f.kpt);
  const size_t w = sz > 1 ? (size_t)r : (size_t)f.bn_t;  // slab row width (folded: r)
  size_t off = 0;
  f.off[0] = off;
  off += al((size_t)f.tsplits * (size_t)k * w * 4);
  f.off[1] = off;
  off += al((size_t)f.tsplits * (size_t)m * w * 4);
  f.bytes = off;
  f.ok = true;
  return f;
}

size_t partial_need(const runlora_shape_t& s) {
  // every skinny launch group any variant issues; the P region covers the largest
  const void* d = reinterpret_cast<const void*>(256);
  void* o = reinterpret_cast<void*>(256);
  Skinny g[8][2] = {
      {job_Z2(s, d, d, o), job_Z2(s, d, d, o)},            // forward1: Z2 alone (slot 1 unused)
      {job_Z1(s, d, d, o), job_Z2(s, d, d, o)},            // B1/B5 projections
      {job_dA_tok(s, d, d, o, true, false), job_dB_tok(s, d, d, o, true, false)},
      {job_Z1(s, d, d, o), job_Z1(s, d, d, o)},            // B2/B3 projection alone
      {job_dA_tok(s, d, d, o, true, false), job_dB_dense(s, d, d, o, true, false)},
      {job_dA_dense(s, d, d, o, true, false), job_dB_dense(s, d, d, o, true, false)},
  };
  const int counts[8] = {1, 2, 2, 1, 2, 2, 0, 0};
  size_t need = 0;
  for (int i = 0; i < 6; ++i) need = std::max(need, plan_skinny(g[i], counts[i]).p_bytes);
  const ZPlan f = plan_z(s);
  if (f.ok) need = std::max(need, f.bytes);
  return need;
}

// ------------------------------------------------------------ workspace layout
// Split-K plan of a main GEMM with fewer 256x256 tiles than CTA pairs (small n: the
// K loop of a lone tile is latency-bound): splits so that the units fill about one wave
// of pairs, fp32 slabs [split][M][N], summed in fixed order into bf16 by the reducer.
struct MainSplit {
  int splits, kps;
};
MainSplit main_split(int64_t M, int64_t N, int64_t K) {
  const int64_t units = ((M + 255) / 256) * ((N + 255) / 256);
  const int64_t nkb = (K + kBK - 1) / kBK;
  MainSplit ms{1, (int)nkb};
  if (units >= 74 || nkb < 8) return ms;
  int64_t sp = std::min<int64_t>({74 / units, 8, nkb / 4});
  if (sp < 2) return ms;
  ms.kps = (int)((nkb + sp - 1) / sp);
  ms.splits = (int)((nkb + ms.kps - 1) / ms.kps);
  return ms;
}
size_t main_split_bytes(const runlora_shape_t& s) {
  const MainSplit a = main_split(s.n, s.m, s.k), b = main_split(s.n, s.k, s.m);
  return std::max(a.splits > 1 ? al((size_t)a.splits * s.n * s.m * 4) : 0,
                  b.splits > 1 ? al((size_t)b.splits * s.n * s.k * 4) : 0);
}

struct Layout {
  size_t z1, z2, arep, brep, cnt, wp, p, pm, total;
};

// Split fix-up counters: one int per output tile of a split rank-r launch (both problems).
size_t counter_count(const runlora_shape_t& s) {
  const int64_t rows = std::max({s.n, s.k, s.m});
  return (size_t)(2 * ((rows + kBM - 1) / kBM) * ((s.r + 15) / 16) + 64);
}

// Z1, Z2: n x r (or n x sz*r partial blocks, see ZPlan); arep: A repeated sz times along its
// columns (k x sz*r, backward1's dX tail against Z1's blocks); brep: B stacked szf times
// (szf*r x m, forward1's Y tail against Z2's blocks) — both written by the idle warps of the
// projection launch before them; cnt: split fix-up counters.
Layout layout_of(const runlora_shape_t& s) {
  const size_t es = s.dtype == RUNLORA_BF16 ? 2 : 4;
  const int64_t n = s.n, k = s.k, m = s.m, r = s.r;
  const ZPlan f = plan_z(s);
  const size_t zc = (size_t)r * (f.ok ? f.sz : 1);                       // Z1 (and backward Z2)
  const size_t zc2 = (size_t)r * (f.ok ? std::max(f.sz, f.szf) : 1);    // Z2 (forward1 too)
  Layout L;
  L.z1 = 0;
  L.z2 = al((size_t)n * zc * es);
  L.arep = L.z2 + al((size_t)n * zc2 * es);
  L.brep = L.arep + (f.ok && f.sz > 1 ? al((size_t)k * zc * es) : 0);
  L.cnt = L.brep + (f.ok && f.szf > 1 ? al((size_t)m * r * f.szf * es) : 0);
  L.wp = L.cnt + al(4 * counter_count(s));
  L.p = L.wp + al((size_t)k * m * es);
  L.pm = L.p + (s.dtype == RUNLORA_BF16 ? partial_need(s) : 0);  // main-GEMM split-K slabs after
  L.total = L.pm + (s.dtype == RUNLORA_BF16 ? main_split_bytes(s) : 0);  // the rank-r ones (see main_gemm)
  return L;
}

struct Bufs {
  void *z1, *z2, *arep, *brep, *wp;
  int* cnt;   // split fix-up counters
  float* P;   // rank-r split-K slabs
  float* Pm;  // main-GEMM split-K slabs
};

runlora_status_t bind_ws(const runlora_shape_t& s, void* ws, size_t ws_bytes, Bufs* b) {
  Layout L = layout_of(s);
  if (!ws) return fail(RUNLORA_ERR_INVALID_ARG, "workspace is NULL");
  if (reinterpret_cast<uintptr_t>(ws) & 255) return fail(RUNLORA_ERR_ALIGNMENT, "workspace must be 256-byte aligned");
  if (ws_bytes < L.total) {
    char buf[160];
    snprintf(buf, sizeof buf, "workspace too small: %zu bytes given, %zu needed", ws_bytes, L.total);
    return fail(RUNLORA_ERR_WORKSPACE, buf);
  }
  char* base = static_cast<char*>(ws);
  b->z1 = base + L.z1;
  b->z2 = base + L.z2;
  b->arep = base + L.arep;
  b->brep = base + L.brep;
  b->cnt = reinterpret_cast<int*>(base + L.cnt);
  b->wp = base + L.wp;
  b->P = reinterpret_cast<float*>(base + L.p);
  b->Pm = reinterpret_cast<float*>(base + L.pm);
  return RUNLORA_OK;
}

runlora_status_t gemm(Ctx& c, const GemmReq& q, cudaStream_t st) {
  std::string err;
  cudaError_t e = launch_tc_gemm(c, &q, 1, st, &err);
  if (e != cudaSuccess) return fail(RUNLORA_ERR_CUDA, err.empty() ? cudaGetErrorString(e) : err);
  return RUNLORA_OK;
}

// W' = W + A·B  (k×m, bf16, formed in fp32 in TMEM and rounded once; Eq. 2).
// ONE GEMM D = [A | I]·[B ; W_rows(tile)]: the K = r product plus a block-diagonal identity
// tail that brings W's rows of the output tile into the same fp32 accumulator through the
// tensor cores (1.0·w is exact), so the epilogue is a plain (TMA) store.
runlora_status_t wprime_bf16(Ctx& c, const runlora_shape_t& s, const void* W, const void* A, const void* B, void* Wp,
                             cudaStream_t st) {
  GemmReq q = base_req((int)s.k, (int)s.m, KID_GEMM_WPRIME);
  q.a = mat(A, s.k, s.r);  // A_op[M=k, K=r], K-major
  q.b = mat(B, s.r, s.m);  // B_op[K=r, N=m] stored [K, N]: MN-major
  q.b_mn = true;
  q.K1 = (int)s.r;
  q.a2 = mat(c.identity(), 128, 128);
  q.b2 = mat(W, s.k, s.m);  // B2_op[K=i, N=j] = W[i, j]: MN-major, rows of the tile
  q.K2 = 128;
  q.tail_diag = true;
  q.out_mode = OUT_BF16;
  q.D = Wp;
  q.ldd = s.m;
  q.BN = 256;
  q.tma_store = c.tma_store_wprime();
  return gemm(c, q, st);
}

// W'ᵀ = (W + A·B)ᵀ  (m×k, bf16) for forward2: stored K-major for the Y GEMM's B operand
// (the tensor cores stream K-major B faster than MN-major B).  GEMM M = m,
// N = k: D[j, i] = Σ_r B[r, j]·A[i, r] + Σ_j' I[j, j']·W[i, j'] — A_op = Bᵀ (B stored [r, m]:
// MN-major), B_op = Aᵀ (A stored [k, r]: K-major); the tail B operand W[i][j'] is K-major
// (K = j' contiguous), read at this tile's rows j' = m0.. (I is symmetric, so it serves as
// the MN-major A operand too).
runlora_status_t wprime_t_bf16(Ctx& c, const runlora_shape_t& s, const void* W, const void* A, const void* B,
                               void* Wpt, cudaStream_t st) {
  GemmReq q = base_req((int)s.m, (int)s.k, KID_GEMM_WPRIME);
  q.a = mat(B, s.r, s.m);
  q.a_mn = true;
  q.b = mat(A, s.k, s.r);
  q.b_mn = false;
  q.K1 = (int)s.r;
  q.a2 = mat(c.identity(), 128, 128);
  q.b2 = mat(W, s.k, s.m);
  q.K2 = 128;
  q.tail_diag = true;
  q.out_mode = OUT_BF16;
  q.D = Wpt;
  q.ldd = s.k;
  q.BN = 256;
  q.tma_store = c.tma_store_wprime();
  return gemm(c, q, st);
}

// ------------------------------------------------------------ quantized W (R18)
// Wq [k, m] E4M3 bytes with one power-of-two scale 2^e[j] per column; D [m, 128] E5M2 bytes:
// row j holds 2^e[j] at column j mod 128 (the scale diagonal, built by the quantizer).
struct QW {
  const void* q;
  const float* scale;
  const void* diag;
};

// W' = W~ + A·B (transposed = false: [k, m], the dX operand of backward4/5), W'ᵀ (transposed:
// [m, k], forward2's B operand), or W~ alone (ab = false: the x1 variants' W) straight from
// the 1-byte Wq: ONE GEMM whose FP8 tail multiplies Wq by the E5M2 scale diagonal (kind::
// f8f6f4) into the same fp32 accumulator as A·B — W~ = e4m3 · 2^e is exact — so the epilogue
// is the plain bf16 TMA store: D = bf16(fp32(A·B) + W~), W read as 1 byte per element.
runlora_status_t wprime_q(Ctx& c, const runlora_shape_t& s, const QW& w, const void* A, const void* B, void* D,
                          bool transposed, bool ab, cudaStream_t st) {
  GemmReq q = base_req((int)(transposed ? s.m : s.k), (int)(transposed ? s.k : s.m),
                       ab ? KID_GEMM_WPRIME : KID_DEQUANT);
  if (!ab) {  // W~ only: no main K (the main operands are never loaded)
    q.a = mat(c.identity(), 128, 128);
    q.b = mat(c.identity(), 128, 128);
    q.b_mn = true;
    q.K1 = 0;
  } else if (transposed) {  // D[j, i] = Σ_r B[r, j]·A[i, r] + Σ_j' diag[j, j']·Wq[i, j']
    q.a = mat(B, s.r, s.m);
    q.a_mn = true;
    q.b = mat(A, s.k, s.r);
    q.K1 = (int)s.r;
  } else {  // D[i, j] = Σ_r A[i, r]·B[r, j] + Σ_j' Wq[i, j']·diag[j', j]
    q.a = mat(A, s.k, s.r);
    q.b = mat(B, s.r, s.m);
    q.b_mn = true;
    q.K1 = (int)s.r;
  }
  const DeviceMat wq{w.q, s.k, s.m, s.m}, dg{w.diag, s.m, 128, 128};  // bytes
  q.BN = 256;
  q.tail_fp8 = transposed ? 1 : 2;
  q.a2 = transposed ? dg : wq;
  q.b2 = transposed ? wq : dg;
  q.K2 = transposed ? 128 : q.BN;
  q.out_mode = OUT_BF16;
  q.D = D;
  q.ldd = transposed ? s.k : s.m;
  q.tma_store = true;
  return gemm(c, q, st);
}

// ------------------------------------------------------------ 512-wide main-GEMM tiles
// A 256x512 pair tile (two N = 256 MMAs per k-step sharing the A tile) moves 25 % fewer TMA
// bytes per FLOP than a 256x256 one, and the main GEMM's time tracks those bytes (DESIGN.md
// §5); its 512 accumulator columns leave no second TMEM buffer (the kernel's 8 epilogue
// warps read the whole tile into registers and release TMEM before storing), and big tiles
// quantise coarsely on 74 pairs (C2: 256 tiles = 3.46 rounds).  So output rows [0, rows_big) run as 512-wide tiles and
// the rest as 256-wide ones in the same launch (two problems).  rows_big minimises the
// busiest pair's summed unit cost under the kernel's static round-robin assignment (unit u
// -> pair u mod 74).  Cost of a 512-wide tile in 256-wide tile times: a + e / K, fitted to
// gemm_bench runs at 131072 x 2048 x K, K = 2048 / 4096 / 8192 (1.744 / 1.741 / 1.729: a =
// 1.72, e = 41 — with the tile held in registers the epilogue is nearly hidden; before, the
// exposed epilogue made it 1.87 at K = 2048).  Cached per shape.
struct WideSplit {
  int rows_big;  // multiple of 256; 0 = no 512-wide tiles
  double cost, cost_small_only;
};

// decode_unit's raster (tc_gemm.cuh) on the host: unit -> (row tile, column tile)
static void host_unit_tile(int u, int mt, int nt, int G, int* m_blk, int* n_blk) {
  const int band = u / (G * nt);
  const int m_first = band * G;
  const int g_rows = std::min(G, mt - m_first);
  const int r = u - band * G * nt;
  *m_blk = m_first + r % g_rows;
  *n_blk = r / g_rows;
}

WideSplit wide_split(Ctx& c, const GemmReq& q) {
  WideSplit w{0, 0, 0};
  if (!c.main_wide() || q.cg != 2 || q.a_mn || q.b_mn || q.splits > 1 || q.out_mode != OUT_BF16) return w;
  const int G = raster_rows(q);
  const int K = q.K1 + q.K2;
  const int pairs = (c.num_sms() - (q.overlaps_comm ? c.comm_sms() : 0)) / 2;  // launch_tc_gemm's grid
  const auto key = std::make_tuple(q.M, q.N, K, G, pairs);
  auto& cache = c.wide_cache();
  if (auto it = cache.find(key); it != cache.end()) {
    w.rows_big = it->second;
    return w;
  }
  const int mt = (q.M + 255) / 256;
  const int ntb = (q.N + 511) / 512, nts = (q.N + 255) / 256;
  const bool ragged = (int64_t)ntb * 512 - q.N >= 256;  // last 512-wide column tile has one half
  const double cb = c.wide_cost_a() + c.wide_cost_e() / K, cs = 1.0;
  std::vector<double> load(pairs);
  auto simulate = [&](int rb) {
    std::fill(load.begin(), load.end(), 0.0);
    const int ub = rb * ntb, us = (mt - rb) * nts;
    for (int u = 0; u < ub; ++u) {
      int mb, nb;
      host_unit_tile(u, rb, ntb, G, &mb, &nb);
      load[u % pairs] += (ragged && nb == ntb - 1) ? cs : cb;
    }
    for (int u = 0; u < us; ++u) load[(ub + u) % pairs] += cs;
    return *std::max_element(load.begin(), load.end());
  };
  w.cost_small_only = simulate(0);
  w.cost = w.cost_small_only;
  // the 256-wide remainder only ever needs to fill the last round or two
  const int lo = std::max(1, mt - (3 * pairs + nts - 1) / nts);
  // from all-wide down; a narrower split must win clearly (4 %): in a mixed launch the
  // 256-wide tiles cost more than the model's 1.0 (C3 8192x11008x4096: model 17.15 vs 17.68
  // rounds for 27 wide row tiles vs all 32, measured 480.3 vs 472.1 µs)
  for (int rb = mt; rb >= lo; --rb) {
    const double t = simulate(rb);
    if (t < w.cost * (w.rows_big ? 0.96 : 0.995)) w.cost = t, w.rows_big = rb * 256;
  }
  cache[key] = w.rows_big;
  return w;
}

static DeviceMat rows_from(const DeviceMat& m, int64_t r0) {
  return DeviceMat{static_cast<const char*>(m.ptr) + r0 * m.ld * 2, m.rows - r0, m.cols, m.ld};
}

// One main-GEMM launch: 512-wide tiles for rows [0, rows_big) and 256-wide ones below
// (wide_split), or plain 256-wide tiles.
runlora_status_t gemm_wide_or_narrow(Ctx& c, const GemmReq& q, cudaStream_t st) {
  const WideSplit w = wide_split(c, q);
  static const bool dbg = getenv("RUNLORA_DEBUG_WIDE") != nullptr;
  if (dbg)
    fprintf(stderr, "[runlora] main GEMM %dx%dx%d: 512-wide rows %d, est. %.2f vs %.2f (256-wide only)\n", q.M, q.N,
            q.K1 + q.K2, w.rows_big, w.cost, w.cost_small_only);
  if (w.rows_big == 0) return gemm(c, q, st);
  GemmReq r[2] = {q, q};
  const int rb = std::min(w.rows_big, q.M);
  r[0].BN = 512;
  r[0].M = rb;
  r[0].a.rows = rb;
  if (r[0].K2 > 0) r[0].a2.rows = rb;
  r[0].tma_store = true;  // the exposed epilogue: full-line bulk stores
  int nreq = 1;
  if (rb < q.M) {
    r[1].M = q.M - rb;
    r[1].a = rows_from(q.a, rb);
    if (q.K2 > 0) r[1].a2 = rows_from(q.a2, rb);
    r[1].D = static_cast<char*>(q.D) + (int64_t)rb * q.ldd * 2;
    r[1].tma_store = true;
    nreq = 2;
  }
  std::string err;
  cudaError_t e = launch_tc_gemm(c, r, nreq, st, &err);
  if (e != cudaSuccess) return fail(RUNLORA_ERR_CUDA, err.empty() ? cudaGetErrorString(e) : err);
  return RUNLORA_OK;
}

// Runs a main GEMM (bf16 D = q.D, ld q.ldd), split over K into fp32 slabs in the P region
// and reduced when main_split says so, or as 512-/256-wide tiles when wide_split says so.
runlora_status_t main_gemm(Ctx& c, GemmReq q, Bufs& b, cudaStream_t st) {
  const MainSplit ms = main_split(q.M, q.N, q.K1);
  if (ms.splits <= 1) {
    return gemm_wide_or_narrow(c, q, st);
  }
  void* out = q.D;
  const int64_t ldo = q.ldd;
  q.out_mode = OUT_F32;
  q.tma_store = false;
  q.D = b.Pm;
  q.ldd = q.N;
  q.split_stride = (int64_t)q.M * q.N;
  q.splits = ms.splits;
  q.kb_per_split = ms.kps;
  RL_TRY(gemm(c, q, st));
  ReduceJob rj{b.Pm, ms.splits, (int64_t)q.M * q.N, q.M, q.N, q.N, out, 1, ldo, 0, 0};
  cudaError_t e = launch_splitk_reduce(c, &rj, 1, st);
  if (e != cudaSuccess) return cuda_fail(e, "splitk_reduce launch");
  return RUNLORA_OK;
}

// The dominant Y / dX GEMMs: 256x256 tiles on CTA pairs (cta_group::2) unless disabled.
GemmReq main_req(Ctx& c, int M, int N) {
  GemmReq q = base_req(M, N, KID_GEMM_MAIN);
  q.BN = 256;
  q.cg = c.main_cg();
  q.out_mode = OUT_BF16;
  q.tma_store = c.tma_store_main() && q.cg == 2;
  return q;
}

// ------------------------------------------------------------ bf16 variants
runlora_status_t forward_bf16(Ctx& c, int v, const runlora_shape_t& s, const void* X, const void* W, const void* A,
                              const void* B, void* Y, Bufs& b, cudaStream_t st, const QW* qw = nullptr) {
  const int64_t n = s.n, k = s.k, m = s.m, r = s.r;
  GemmReq q = main_req(c, (int)n, (int)m);
  q.a = mat(X, n, k);
  q.a_mn = false;
  q.K1 = (int)k;
  q.b_mn = true;
  q.D = Y;
  q.ldd = m;
  if (v == 1) {
    // Z2 = X·A (never saved for the backward), then Y = [X | Z2]·[W ; B]
    q.b = mat(W, k, m);
    const ZPlan f = plan_z(s);
    if (f.ok && f.szf > 1) {
      // Z2 as szf K-split bf16 blocks (every CTA slot streams X, no reducer), then
      // Y = [X | Z2_0 | .. | Z2_{szf-1}]·[W ; B ; .. ; B]: B stacked szf times (one 64-wide
      // tail k-block), written by the Z2 launch's idle warps
      const int zc = (int)(r * f.szf);
      const ReduceJob rep = repeat_job(B, 1, (int)(r * m), f.szf, b.brep);
      GemmReq z = base_req((int)n, (int)r, KID_GEMM_PROJ);
      z.a = mat(X, n, k);
      z.b = mat(A, k, r);
      z.b_mn = true;
      z.K1 = (int)k;
      z.BN = f.bn_z[1];
      z.a_stream_once = true;
      z.out_mode = OUT_BF16;
      z.D = b.z2;
      z.ldd = zc;
      z.split_stride = r;
      z.splits = f.szf;
      z.kb_per_split = f.kpzf;
      z.side = &rep;
      z.nside = 1;
      RL_TRY(gemm(c, z, st));
      q.a2 = mat(b.z2, n, zc);
      q.b2 = mat(b.brep, zc, m);
      q.K2 = zc;
    } else {
      Skinny j = job_Z2(s, X, A, b.z2);
      RL_TRY(run_skinny(c, &j, 1, b.P, b.cnt, KID_GEMM_PROJ, st));
      q.a2 = mat(b.z2, n, r);
      q.b2 = mat(B, r, m);
      q.K2 = (int)r;
    }
  } else {
    if (qw) RL_TRY(wprime_q(c, s, *qw, A, B, b.wp, true, true, st));  // W'ᵀ [m, k] from Wq
    else RL_TRY(wprime_t_bf16(c, s, W, A, B, b.wp, st));                // W'ᵀ [m, k]
    q.b = mat(b.wp, m, k);
    q.b_mn = false;
  }
  return main_gemm(c, q, b, st);
}

// forward2's second half on a W'ᵀ [m, k] the caller built (runlora_wprime_t) — the same main
// GEMM as forward_bf16(v = 2) issues, so the result is bit-identical.
runlora_status_t forward_from_wpt(Ctx& c, const runlora_shape_t& s, const void* X, const void* Wpt, void* Y, Bufs& b,
                                  cudaStream_t st) {
  GemmReq q = main_req(c, (int)s.n, (int)s.m);
  q.a = mat(X, s.n, s.k);
  q.a_mn = false;
  q.K1 = (int)s.k;
  q.b = mat(Wpt, s.m, s.k);
  q.b_mn = false;
  q.D = Y;
  q.ldd = s.m;
  return main_gemm(c, q, b, st);
}

// backward1/5 adapter gradients: projections launch, then reductions launch whose token-split
// slabs are summed in fixed order either by the reductions launch itself (the last split per
// output tile, Prob::fixup) or, with `defer`, by the idle warps of the dX GEMM launch that
// follows (no reducer launch either way; see ZPlan).
runlora_status_t grads_tok_bf16(Ctx& c, int v, const ZPlan& f, const runlora_shape_t& s, const void* X, const void* A,
                                const void* B, const void* dY, void* dA, void* dB, bool gb, bool acc, Bufs& b,
                                cudaStream_t st, std::vector<ReduceJob>* defer) {
  const int64_t n = s.n, k = s.k, m = s.m, r = s.r;
  const int zc = (int)(r * f.sz);  // columns of the partial-Z matrices
  const int tiles[2] = {(int)((k + kBM - 1) / kBM), (int)((m + kBM - 1) / kBM)};  // reduction output tiles
  std::string err;
  // projections: Zp[:, s*r:(s+1)*r] = K-split s of dY·Bᵀ / X·A (bf16); this launch also zeroes
  // the reductions' fix-up counters (after its PDL wait, so no earlier launch still uses them)
  GemmReq q[2];
  const DeviceMat za[2] = {mat(dY, n, m), mat(X, n, k)};
  const DeviceMat zb[2] = {mat(B, r, m), mat(A, k, r)};
  void* zout[2] = {b.z1, b.z2};
  for (int i = 0; i < 2; ++i) {
    GemmReq& g = q[i];
    g = base_req((int)n, (int)r, KID_GEMM_PROJ);
    g.a = za[i];
    g.b = zb[i];
    g.b_mn = i == 1;
    g.K1 = (int)(i == 0 ? m : k);
    g.BN = f.bn_z[i];
    g.a_stream_once = true;
    g.out_mode = OUT_BF16;
    g.D = zout[i];
    g.ldd = zc;
    g.split_stride = r;  // split s -> column block s
    g.splits = f.sz;
    g.kb_per_split = f.kpz[i];
  }
  if (!defer) {
    q[0].zero_ptr = b.cnt;
    q[0].zero_n = tiles[0] + tiles[1];
  }
  // backward1's dX tail needs A repeated per Z1 block: written by this launch's idle warps
  const ReduceJob rep = repeat_job(A, (int)k, (int)r, f.sz, b.arep);
  if (v == 1 && f.sz > 1) {
    q[0].side = &rep;
    q[0].nside = 1;
  }
  cudaError_t e = launch_tc_gemm(c, q, 2, st, &err);
  if (e != cudaSuccess) return fail(RUNLORA_ERR_CUDA, err.empty() ? cudaGetErrorString(e) : err);
  // reductions: dA = Σ_s Xᵀ·Z1_s, dBᵀ = Σ_s dYᵀ·Z2_s (token splits -> fp32 slabs, fixed-order
  // in-kernel fix-up into dA [k, r] and dB [r, m] (transposed), fp32 or bf16, = or +=)
  const DeviceMat ta[2] = {mat(X, n, k), mat(dY, n, m)};
  const int64_t rows[2] = {k, m};
  void* outs[2] = {dA, dB};
  for (int i = 0; i < 2; ++i) {
    GemmReq& g = q[i];
    g = base_req((int)rows[i], f.sz > 1 ? f.bn_t : (int)r, KID_GEMM_TOKRED);
    g.a = ta[i];
    g.a_mn = true;
    g.b = mat(zout[i], n, zc);
    g.b_mn = true;
    g.K1 = (int)n;
    g.BN = f.bn_t;
    g.a_stream_once = true;
    float* P = reinterpret_cast<float*>(reinterpret_cast<char*>(b.P) + f.off[i]);
    g.D = P;
    g.splits = f.tsplits;
    g.kb_per_split = f.kpt;
    if (f.sz > 1) {
      g.out_mode = OUT_F32_FOLD;
      g.fold = f.sz;
      g.fold_w = (int)r;
      g.ldd = r;
    } else {
      g.out_mode = OUT_F32;
      g.ldd = f.bn_t;  // plain slabs keep the padded tile width
    }
    g.split_stride = rows[i] * g.ldd;
    if (defer) {  // the idle warps of the dX GEMM launch reduce the slabs (do_backward)
      defer->push_back(ReduceJob{P, f.tsplits, g.split_stride, (int)rows[i], (int)r, g.ldd, outs[i], gb ? 1 : 0,
                                 i == 0 ? r : m, i == 1 ? 1 : 0, acc ? 1 : 0});
      continue;
    }
    g.fixup = true;
    g.counters = b.cnt + (i == 0 ? 0 : tiles[0]);
    g.fx_out = outs[i];
    g.fx_ldo = i == 0 ? r : m;
    g.fx_cols = (int)r;
    g.fx_transpose = i == 1;
    g.fx_accumulate = acc;
    g.fx_bf16 = gb;
  }
  e = launch_tc_gemm(c, q, 2, st, &err);
  if (e != cudaSuccess) return fail(RUNLORA_ERR_CUDA, err.empty() ? cudaGetErrorString(e) : err);
  return RUNLORA_OK;
}

runlora_status_t params_bf16(Ctx& c, int v, const runlora_shape_t& s, const void* X, const void* A, const void* B,
                             const void* dY, void* dA, void* dB, bool gb, bool acc, Bufs& b, cudaStream_t st,
                             std::vector<ReduceJob>* defer = nullptr) {
  const int64_t n = s.n, k = s.k, m = s.m;
  if (v == 1 || v == 5) {  // Alg. 1 / Alg. 5: Z1, Z2 | dA = Xᵀ·Z1, dB = Z2ᵀ·dY
    const ZPlan f = plan_z(s);
    if (f.ok) return grads_tok_bf16(c, v, f, s, X, A, B, dY, dA, dB, gb, acc, b, st, defer);
    Skinny pj[2] = {job_Z1(s, dY, B, b.z1), job_Z2(s, X, A, b.z2)};
    RL_TRY(run_skinny(c, pj, 2, b.P, b.cnt, KID_GEMM_PROJ, st));
    Skinny tj[2] = {job_dA_tok(s, X, b.z1, dA, gb, acc), job_dB_tok(s, dY, b.z2, dB, gb, acc)};
    return run_skinny(c, tj, 2, b.P, b.cnt, KID_GEMM_TOKRED, st, defer);
  }
  if (v == 2 || v == 3) {  // Z1 = dY·Bᵀ
    Skinny j = job_Z1(s, dY, B, b.z1);
    RL_TRY(run_skinny(c, &j, 1, b.P, b.cnt, KID_GEMM_PROJ, st));
  }
  {  // Z2' = Xᵀ·dY (k×m): A_op = Xᵀ (MN-major X), B_op = dY (MN-major)
    GemmReq q = base_req((int)k, (int)m, KID_GEMM_DENSE_XTDY);
    q.a = mat(X, n, k);
    q.a_mn = true;
    q.b = mat(dY, n, m);
    q.b_mn = true;
    q.K1 = (int)n;
    q.out_mode = OUT_BF16;
    q.D = b.wp;
    q.ldd = m;
    q.BN = 256;
    q.cg = c.main_cg();
    RL_TRY(gemm(c, q, st));
  }
  if (v == 2) {  // dA = Xᵀ·Z1, dB = Aᵀ·Z2'
    Skinny j[2] = {job_dA_tok(s, X, b.z1, dA, gb, acc), job_dB_dense(s, b.wp, A, dB, gb, acc)};
    return run_skinny(c, j, 2, b.P, b.cnt, KID_GEMM_SMALL, st, defer);
  }
  // v = 3, 4: dA = Z2'·Bᵀ, dB = Aᵀ·Z2'
  Skinny j[2] = {job_dA_dense(s, b.wp, B, dA, gb, acc), job_dB_dense(s, b.wp, A, dB, gb, acc)};
  return run_skinny(c, j, 2, b.P, b.cnt, KID_GEMM_SMALL, st, defer);
}

runlora_status_t input_bf16(Ctx& c, int v, const runlora_shape_t& s, const void* W, const void* A, const void* B,
                            const void* dY, void* dX, Bufs& b, cudaStream_t st, const QW* qw = nullptr,
                            const std::vector<ReduceJob>* side = nullptr, const void* xdesc = nullptr,
                            unsigned xepoch = 0) {
  const int64_t n = s.n, k = s.k, m = s.m, r = s.r;
  GemmReq q = main_req(c, (int)n, (int)k);
  if (side && !side->empty()) {  // the adapter gradients' slabs, reduced by this launch's idle warps
    q.side = side->data();
    q.nside = (int)side->size();
    q.xdesc = xdesc;             // ... and exchanged across ranks (runlora_backward_exchange)
    q.xepoch = xepoch;
  }
  q.overlaps_comm = true;  // backward_input runs while backward_params' allreduce is in flight
  q.a = mat(dY, n, m);
  q.a_mn = false;
  q.b_mn = false;
  q.K1 = (int)m;
  q.D = dX;
  q.ldd = k;
  if (v <= 3) {  // dX = [dY | Z1]·[Wᵀ ; Aᵀ]
    q.b = mat(W, k, m);  // B_op[K=m, N=k] = Wᵀ stored [N, K] = W: K-major
    q.a2 = mat(b.z1, n, r);
    q.b2 = mat(A, k, r);  // Aᵀ stored [N=k, K=r] = A: K-major
    q.K2 = (int)r;
    const ZPlan f = plan_z(s);
    if (v == 1 && f.ok && f.sz > 1) {
      // backward1's adapter-gradient pass left Z1 as sz partial blocks: dY·Wᵀ + Σ_s Z1_s·Aᵀ =
      // [dY | Z1_0 | .. | Z1_{sz-1}]·[Wᵀ ; Aᵀ ; .. ; Aᵀ] (A repeated by the projection launch)
      const int zc = (int)(r * f.sz);
      q.a2 = mat(b.z1, n, zc);
      q.b2 = mat(b.arep, k, zc);
      q.K2 = zc;
    }
  } else {  // dX = dY·W'ᵀ
    if (qw) RL_TRY(wprime_q(c, s, *qw, A, B, b.wp, false, true, st));  // W' [k, m] from Wq
    else RL_TRY(wprime_bf16(c, s, W, A, B, b.wp, st));
    q.b = mat(b.wp, k, m);
  }
  return main_gemm(c, q, b, st);
}

// ------------------------------------------------------------ fp32 variants
runlora_status_t sg(Ctx& c, int M, int N, int K, const void* A, int64_t sa0, int64_t sa1, const void* B, int64_t sb0,
                    int64_t sb1, void* C, int64_t ldc, const void* Cadd, int64_t ldadd, bool acc, cudaStream_t st) {
  cudaError_t e = launch_sgemm(c, M, N, K, (const float*)A, sa0, sa1, (const float*)B, sb0, sb1, (float*)C, ldc,
                               (const float*)Cadd, ldadd, acc, st);
  if (e != cudaSuccess) return cuda_fail(e, "sgemm launch");
  return RUNLORA_OK;
}

runlora_status_t forward_f32(Ctx& c, int v, const runlora_shape_t& s, const void* X, const void* W, const void* A,
                             const void* B, void* Y, Bufs& b, cudaStream_t st) {
  const int n = (int)s.n, k = (int)s.k, m = (int)s.m, r = (int)s.r;
  if (v == 1) {
    RL_TRY(sg(c, n, r, k, X, k, 1, A, r, 1, b.z2, r, nullptr, 0, false, st));   // Z2 = X·A
    RL_TRY(sg(c, n, m, k, X, k, 1, W, m, 1, Y, m, nullptr, 0, false, st));      // Y = X·W
    return sg(c, n, m, r, b.z2, r, 1, B, m, 1, Y, m, nullptr, 0, true, st);    // Y += Z2·B
  }
  RL_TRY(sg(c, k, m, r, A, r, 1, B, m, 1, b.wp, m, W, m, false, st));         // W' = W + A·B
  return sg(c, n, m, k, X, k, 1, b.wp, m, 1, Y, m, nullptr, 0, false, st);     // Y = X·W'
}

runlora_status_t params_f32(Ctx& c, int v, const runlora_shape_t& s, const void* X, const void* A, const void* B,
                            const void* dY, void* dA, void* dB, bool acc, Bufs& b, cudaStream_t st) {
  const int n = (int)s.n, k = (int)s.k, m = (int)s.m, r = (int)s.r;
  if (v == 1 || v == 2 || v == 3 || v == 5)
    RL_TRY(sg(c, n, r, m, dY, m, 1, B, 1, m, b.z1, r, nullptr, 0, false, st));  // Z1 = dY·Bᵀ
  if (v == 1 || v == 5) RL_TRY(sg(c, n, r, k, X, k, 1, A, r, 1, b.z2, r, nullptr, 0, false, st));  // Z2 = X·A
  if (v == 2 || v == 3 || v == 4)
    RL_TRY(sg(c, k, m, n, X, 1, k, dY, m, 1, b.wp, m, nullptr, 0, false, st));  // Z2' = Xᵀ·dY
  if (v == 1 || v == 2 || v == 5)
    RL_TRY(sg(c, k, r, n, X, 1, k, b.z1, r, 1, dA, r, nullptr, 0, acc, st));     // dA = Xᵀ·Z1
  else
    RL_TRY(sg(c, k, r, m, b.wp, m, 1, B, 1, m, dA, r, nullptr, 0, acc, st));     // dA = Z2'·Bᵀ
  if (v == 1 || v == 5)
    RL_TRY(sg(c, r, m, n, b.z2, 1, r, dY, m, 1, dB, m, nullptr, 0, acc, st));    // dB = Z2ᵀ·dY
  else
    RL_TRY(sg(c, r, m, k, A, 1, r, b.wp, m, 1, dB, m, nullptr, 0, acc, st));     // dB = Aᵀ·Z2'
  return RUNLORA_OK;
}

runlora_status_t input_f32(Ctx& c, int v, const runlora_shape_t& s, const void* W, const void* A, const void* B,
                           const void* dY, void* dX, Bufs& b, cudaStream_t st) {
  const int n = (int)s.n, k = (int)s.k, m = (int)s.m, r = (int)s.r;
  if (v <= 3) {
    RL_TRY(sg(c, n, k, m, dY, m, 1, W, 1, m, dX, k, nullptr, 0, false, st));   // dX = dY·Wᵀ
    return sg(c, n, k, r, b.z1, r, 1, A, 1, r, dX, k, nullptr, 0, true, st);   // dX += Z1·Aᵀ
  }
  RL_TRY(sg(c, k, m, r, A, r, 1, B, m, 1, b.wp, m, W, m, false, st));        // W' = W + A·B
  return sg(c, n, k, m, dY, m, 1, b.wp, 1, m, dX, k, nullptr, 0, false, st);  // dX = dY·W'ᵀ
}

// ------------------------------------------------------------ entry helpers
runlora_status_t check_handle(runlora_handle_t h) {
  if (!h || !h->ctx) return fail(RUNLORA_ERR_INVALID_ARG, "handle is NULL");
  return RUNLORA_OK;
}

runlora_status_t post_launch() {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
  return RUNLORA_OK;
}

using CallLock = std::lock_guard<std::recursive_mutex>;

runlora_status_t validate_forward(runlora_handle_t h, int fwd, const runlora_shape_t* s, const void* X, const void* W,
                                  const void* A, const void* B, const void* Y) {
  RL_TRY(check_handle(h));
  RL_TRY(check_shape(s));
  if (fwd != 1 && fwd != 2) return fail(RUNLORA_ERR_INVALID_ARG, "forward variant must be 1 or 2 (P:62-64)");
  RL_TRY(check_ptr(X, "X"));
  RL_TRY(check_ptr(W, "W"));
  RL_TRY(check_ptr(A, "A"));
  RL_TRY(check_ptr(B, "B"));
  RL_TRY(check_ptr(Y, "Y"));
  return RUNLORA_OK;
}

runlora_status_t do_forward(runlora_handle_t h, int fwd, const runlora_shape_t* s, const void* X, const void* W,
                            const void* A, const void* B, void* Y, void* ws, size_t ws_bytes, void* stream) {
  RL_TRY(validate_forward(h, fwd, s, X, W, A, B, Y));
  Bufs b;
  RL_TRY(bind_ws(*s, ws, ws_bytes, &b));
  CallLock lk(h->ctx->call_mu);
  DeviceGuard dg(h->ctx->device());
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (s->dtype == RUNLORA_BF16) RL_TRY(forward_bf16(*h->ctx, fwd, *s, X, W, A, B, Y, b, st));
  else RL_TRY(forward_f32(*h->ctx, fwd, *s, X, W, A, B, Y, b, st));
  return post_launch();
}

runlora_status_t check_bwd_common(runlora_handle_t h, int bwd, const runlora_shape_t* s) {
  RL_TRY(check_handle(h));
  RL_TRY(check_shape(s));
  if (bwd >= 6 && bwd <= 8)
    return fail(RUNLORA_ERR_UNSUPPORTED_VARIANT,
                "backward6..8 are cost-model only: the paper implements only the first five (P:96-98)");
  if (bwd < 1 || bwd > 8) return fail(RUNLORA_ERR_INVALID_ARG, "backward variant must be 1..5");
  return RUNLORA_OK;
}

runlora_status_t validate_params(runlora_handle_t h, int bwd, const runlora_shape_t* s, const void* X,
                                 const void* A, const void* B, const void* dY, const void* dA, const void* dB,
                                 int grad_dtype) {
  RL_TRY(check_bwd_common(h, bwd, s));
  RL_TRY(check_ptr(X, "X"));
  RL_TRY(check_ptr(A, "A"));
  RL_TRY(check_ptr(B, "B"));
  RL_TRY(check_ptr(dY, "dY"));
  RL_TRY(check_ptr(dA, "dA"));
  RL_TRY(check_ptr(dB, "dB"));
  if (grad_dtype != RUNLORA_F32 && grad_dtype != RUNLORA_BF16) return fail(RUNLORA_ERR_DTYPE, "grad_dtype must be F32 or BF16");
  if (s->dtype == RUNLORA_F32 && grad_dtype != RUNLORA_F32)
    return fail(RUNLORA_ERR_DTYPE, "fp32 operands need fp32 adapter gradients");
  return RUNLORA_OK;
}

runlora_status_t validate_input(runlora_handle_t h, int bwd, const runlora_shape_t* s, const void* W, const void* A,
                                const void* B, const void* dY, const void* dX) {
  RL_TRY(check_bwd_common(h, bwd, s));
  RL_TRY(check_ptr(W, "W"));
  RL_TRY(check_ptr(A, "A"));
  RL_TRY(check_ptr(B, "B"));
  RL_TRY(check_ptr(dY, "dY"));
  RL_TRY(check_ptr(dX, "dX"));
  return RUNLORA_OK;
}

runlora_status_t do_params(runlora_handle_t h, int bwd, const runlora_shape_t* s, const void* X, const void* W,
                           const void* A, const void* B, const void* dY, void* dA, void* dB, int grad_dtype,
                           int accumulate, void* ws, size_t ws_bytes, void* stream,
                           std::vector<ReduceJob>* defer = nullptr) {
  (void)W;
  RL_TRY(validate_params(h, bwd, s, X, A, B, dY, dA, dB, grad_dtype));
  Bufs b;
  RL_TRY(bind_ws(*s, ws, ws_bytes, &b));
  CallLock lk(h->ctx->call_mu);
  DeviceGuard dg(h->ctx->device());
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (s->dtype == RUNLORA_BF16)
    RL_TRY(params_bf16(*h->ctx, bwd, *s, X, A, B, dY, dA, dB, grad_dtype == RUNLORA_BF16, accumulate != 0, b, st,
                       defer));
  else
    RL_TRY(params_f32(*h->ctx, bwd, *s, X, A, B, dY, dA, dB, accumulate != 0, b, st));
  return post_launch();
}

runlora_status_t do_input(runlora_handle_t h, int bwd, const runlora_shape_t* s, const void* W, const void* A,
                          const void* B, const void* dY, void* dX, void* ws, size_t ws_bytes, void* stream,
                          const std::vector<ReduceJob>* side = nullptr) {
  RL_TRY(validate_input(h, bwd, s, W, A, B, dY, dX));
  Bufs b;
  RL_TRY(bind_ws(*s, ws, ws_bytes, &b));
  CallLock lk(h->ctx->call_mu);
  DeviceGuard dg(h->ctx->device());
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (s->dtype == RUNLORA_BF16) RL_TRY(input_bf16(*h->ctx, bwd, *s, W, A, B, dY, dX, b, st, nullptr, side));
  else RL_TRY(input_f32(*h->ctx, bwd, *s, W, A, B, dY, dX, b, st));
  return post_launch();
}

runlora_status_t do_backward(runlora_handle_t h, int bwd, const runlora_shape_t* s, const void* X, const void* W,
                             const void* A, const void* B, const void* dY, void* dX, void* dA, void* dB,
                             int grad_dtype, int accumulate, void* ws, size_t ws_bytes, void* stream) {
  // Everything is validated before the first launch (the split calls validate again).
  RL_TRY(validate_params(h, bwd, s, X, A, B, dY, dA, dB, grad_dtype));
  if (dX) RL_TRY(validate_input(h, bwd, s, W, A, B, dY, dX));
  {
    Bufs b;
    RL_TRY(bind_ws(*s, ws, ws_bytes, &b));
  }
  CallLock lk(h->ctx->call_mu);
  // adapter gradients, then dX — one PDL chain.  With dX, the adapter gradients' split-K slabs
  // are reduced (fixed order) by the idle warps 2-3 of the dX GEMM launch, concurrently with
  // its mainloop; without dX (or in the split _params call) their own launch reduces them.
  static const bool side_ok = !getenv("RUNLORA_SIDE_REDUCE") || atoi(getenv("RUNLORA_SIDE_REDUCE")) != 0;
  std::vector<ReduceJob> side;
  RL_TRY(do_params(h, bwd, s, X, W, A, B, dY, dA, dB, grad_dtype, accumulate, ws, ws_bytes, stream,
                   side_ok && dX && s->dtype == RUNLORA_BF16 ? &side : nullptr));
  if (dX) RL_TRY(do_input(h, bwd, s, W, A, B, dY, dX, ws, ws_bytes, stream, &side));
  return RUNLORA_OK;
}

// ------------------------------------------------------------ selector
void fill_flops(const runlora_shape_t* s, runlora_plan_t* p) {
  for (int v = 1; v <= 2; ++v) flops_of(s, 0, v, &p->flops_fwd[v]);
  for (int v = 1; v <= 8; ++v) flops_of(s, 1, v, &p->flops_bwd[v]);
  int bf = 1, bb = 1;
  for (int v = 2; v <= 2; ++v)
    if (p->flops_fwd[v] < p->flops_fwd[bf]) bf = v;
  for (int v = 2; v <= 5; ++v)
    if (p->flops_bwd[v] < p->flops_bwd[bb]) bb = v;  // strict: ties keep the lowest index
  p->flops_fwd_pick = bf;
  p->flops_bwd_pick = bb;
  p->param_reduction = (s->r * (s->k + s->m) < s->k * s->m) ? 1 : 0;
}

float median(std::vector<float> v) {
  std::sort(v.begin(), v.end());
  const size_t n = v.size();
  return n % 2 ? v[n / 2] : 0.5f * (v[n / 2 - 1] + v[n / 2]);
}

}  // namespace

// ============================================================== exported ABI
extern "C" {

const char* runlora_version(void) { return "runlora-b200 0.1 (sm_100a, tcgen05/TMA)"; }

runlora_status_t runlora_create(runlora_handle_t* out, int device) {
  if (!out) return fail(RUNLORA_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  int major = 0, minor = 0;
  cudaError_t e = cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetAttribute");
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device);
  if (major != 10 || minor != 0) {
    char b[128];
    snprintf(b, sizeof b, "device %d is sm_%d%d; this library is built for sm_100a (B200) only", device, major, minor);
    return fail(RUNLORA_ERR_DEVICE, b);
  }
  try {
    runlora_handle_s* h = new runlora_handle_s;
    h->ctx = new Ctx(device);
    if (!h->ctx->identity()) {
      delete h->ctx;
      delete h;
      return fail(RUNLORA_ERR_CUDA, "device allocation of the handle's identity tile failed");
    }
    *out = h;
  } catch (...) {
    return fail(RUNLORA_ERR_INVALID_ARG, "allocation of handle failed");
  }
  return RUNLORA_OK;
}

runlora_status_t runlora_destroy(runlora_handle_t h) {
  if (!h) return RUNLORA_OK;
  delete h->ctx;
  delete h;
  return RUNLORA_OK;
}

runlora_status_t runlora_flops(const runlora_shape_t* s, int is_backward, int variant, uint64_t* out) {
  if (!s || !out) return fail(RUNLORA_ERR_INVALID_ARG, "shape/out is NULL");
  if (s->n <= 0 || s->k <= 0 || s->m <= 0 || s->r <= 0)
    return fail(RUNLORA_ERR_INVALID_ARG, "n, k, m, r must all be >= 1");
  return flops_of(s, is_backward, variant, out);
}

int runlora_param_reduction(const runlora_shape_t* s) {
  if (!s) return 0;
  typedef unsigned __int128 u;
  return ((u)s->r * ((u)s->k + (u)s->m) < (u)s->k * (u)s->m) ? 1 : 0;
}

runlora_status_t runlora_workspace_size(const runlora_shape_t* s, int fwd, int bwd, size_t* bytes) {
  RL_TRY(check_shape(s));
  if (!bytes) return fail(RUNLORA_ERR_INVALID_ARG, "bytes is NULL");
  if (fwd < 0 || fwd > 2) return fail(RUNLORA_ERR_INVALID_ARG, "fwd must be 0, 1 or 2");
  if (bwd < 0 || bwd > 8) return fail(RUNLORA_ERR_INVALID_ARG, "bwd must be 0..5");
  if (bwd >= 6) return fail(RUNLORA_ERR_UNSUPPORTED_VARIANT, "backward6..8 are cost-model only (P:96-98)");
  *bytes = layout_of(*s).total;  // one layout serves every variant
  return RUNLORA_OK;
}

runlora_status_t runlora_select(runlora_handle_t h, const runlora_shape_t* s, int criterion,
                                const runlora_operands_t* ops, void* ws, size_t ws_bytes, void* stream,
                                runlora_plan_t* out) {
  RL_TRY(check_shape(s));
  if (!out) return fail(RUNLORA_ERR_INVALID_ARG, "out is NULL");
  if (criterion < RUNLORA_BY_FLOPS || criterion > RUNLORA_HYBRID)
    return fail(RUNLORA_ERR_INVALID_ARG, "criterion must be BY_FLOPS, BY_TIME or HYBRID");
  runlora_plan_t p;
  memset(&p, 0, sizeof p);
  for (int v = 0; v < 3; ++v) p.time_fwd_us[v] = NAN;
  for (int v = 0; v < 9; ++v) p.time_bwd_us[v] = NAN;
  p.criterion = criterion;
  {
    uint64_t tmp;
    RL_TRY(flops_of(s, 1, 6, &tmp));  // overflow check of the largest rows
    RL_TRY(flops_of(s, 1, 4, &tmp));
  }
  fill_flops(s, &p);
  p.fwd = p.flops_fwd_pick;
  p.bwd = p.flops_bwd_pick;
  if (criterion == RUNLORA_BY_FLOPS) {
    *out = p;
    return RUNLORA_OK;
  }
  RL_TRY(check_handle(h));
  std::vector<int64_t> key = {s->n, s->k, s->m, s->r, s->dtype, criterion, ops ? ops->grad_dtype : -1};
  {
    std::lock_guard<std::mutex> g(h->ctx->plan_mu);
    auto it = h->ctx->plans.find(key);
    if (it != h->ctx->plans.end()) {
      *out = it->second;
      return RUNLORA_OK;
    }
  }
  if (!ops) return fail(RUNLORA_ERR_INVALID_ARG, "time-based selection needs device operands");
  CallLock lk(h->ctx->call_mu);  // the candidates are measured without interleaved calls
  DeviceGuard dg(h->ctx->device());
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaEvent_t e0, e1;
  if (cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess)
    return fail(RUNLORA_ERR_TIMING, "cudaEventCreate failed");
  // Candidates are timed round-robin (one rep of each per round) so that clock and power
  // drift under the 1 kW cap affects all of them alike; median of 15 rounds after 3.  A rep
  // is `inner` back-to-back calls between two events (their mean): a single call timed from
  // an idle GPU is dominated by launch latency at small shapes and misranks candidates
  // whose steady-state cost is lower.
  const int warm = 3, reps = 15, inner = 4;
  const uint64_t fmin = std::min(p.flops_fwd[1], p.flops_fwd[2]);
  uint64_t bmin = p.flops_bwd[1];
  for (int v = 2; v <= 5; ++v) bmin = std::min(bmin, p.flops_bwd[v]);
  std::vector<int> cands;  // 1..2 forward, 11..15 backward
  for (int v = 1; v <= 2; ++v)
    if (!(criterion == RUNLORA_HYBRID && p.flops_fwd[v] > 2 * fmin)) cands.push_back(v);
  for (int v = 1; v <= 5; ++v)
    if (!(criterion == RUNLORA_HYBRID && p.flops_bwd[v] > 2 * bmin)) cands.push_back(10 + v);
  std::vector<std::vector<float>> times(cands.size());
  runlora_status_t st_all = RUNLORA_OK;
  for (int i = 0; i < warm + reps && st_all == RUNLORA_OK; ++i) {
    for (size_t ci = 0; ci < cands.size() && st_all == RUNLORA_OK; ++ci) {
      const int v = cands[ci];
      cudaEventRecord(e0, st);
      for (int j = 0; j < inner && st_all == RUNLORA_OK; ++j) {
        if (v < 10)
          st_all = do_forward(h, v, s, ops->X, ops->W, ops->A, ops->B, ops->Y, ws, ws_bytes, stream);
        else
          st_all = do_backward(h, v - 10, s, ops->X, ops->W, ops->A, ops->B, ops->dY, ops->dX, ops->dA, ops->dB,
                               ops->grad_dtype, 0, ws, ws_bytes, stream);
      }
      cudaEventRecord(e1, st);
      if (st_all != RUNLORA_OK) break;
      if (cudaEventSynchronize(e1) != cudaSuccess) {
        st_all = fail(RUNLORA_ERR_TIMING, "event sync failed");
        break;
      }
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      if (i >= warm) times[ci].push_back(ms * 1000.f / inner);
    }
  }
  if (st_all == RUNLORA_OK) {
    for (size_t ci = 0; ci < cands.size(); ++ci) {
      const int v = cands[ci];
      if (v < 10) p.time_fwd_us[v] = median(times[ci]);
      else p.time_bwd_us[v - 10] = median(times[ci]);
    }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (st_all != RUNLORA_OK) return st_all;
  // argmin of the medians; candidates within 1 % of the fastest count as a tie (timer and
  // clock noise) and the tie goes to fewer FLOPs, then the lower index (R9).
  auto pick = [](const float* t, const uint64_t* fl, int lo, int hi) {
    int best = 0;
    for (int v = lo; v <= hi; ++v)
      if (!std::isnan(t[v]) && (best == 0 || t[v] < t[best])) best = v;
    if (best == 0) return 0;
    int sel = best;
    for (int v = lo; v <= hi; ++v)
      if (!std::isnan(t[v]) && t[v] <= 1.01f * t[best] && (fl[v] < fl[sel] || (fl[v] == fl[sel] && v < sel))) sel = v;
    return sel;
  };
  const int bf = pick(p.time_fwd_us, p.flops_fwd, 1, 2);
  const int bb = pick(p.time_bwd_us, p.flops_bwd, 1, 5);
  if (bf == 0 || bb == 0) return fail(RUNLORA_ERR_TIMING, "no candidate could be timed");
  p.fwd = bf;
  p.bwd = bb;
  {
    std::lock_guard<std::mutex> g(h->ctx->plan_mu);
    h->ctx->plans[key] = p;
  }
  *out = p;
  return RUNLORA_OK;
}

runlora_status_t runlora_forward(runlora_handle_t h, int fwd, const runlora_shape_t* s, const void* X, const void* W,
                                 const void* A, const void* B, void* Y, void* ws, size_t ws_bytes, void* stream) {
  return do_forward(h, fwd, s, X, W, A, B, Y, ws, ws_bytes, stream);
}

runlora_status_t runlora_backward(runlora_handle_t h, int bwd, const runlora_shape_t* s, const void* X, const void* W,
                                  const void* A, const void* B, const void* dY, void* dX, void* dA, void* dB,
                                  int grad_dtype, int accumulate, void* ws, size_t ws_bytes, void* stream) {
  return do_backward(h, bwd, s, X, W, A, B, dY, dX, dA, dB, grad_dtype, accumulate, ws, ws_bytes, stream);
}

runlora_status_t runlora_backward_params(runlora_handle_t h, int bwd, const runlora_shape_t* s, const void* X,
                                         const void* W, const void* A, const void* B, const void* dY, void* dA,
                                         void* dB, int grad_dtype, int accumulate, void* ws, size_t ws_bytes,
                                         void* stream) {
  return do_params(h, bwd, s, X, W, A, B, dY, dA, dB, grad_dtype, accumulate, ws, ws_bytes, stream);
}

runlora_status_t runlora_backward_input(runlora_handle_t h, int bwd, const runlora_shape_t* s, const void* X,
                                        const void* W, const void* A, const void* B, const void* dY, void* dX,
                                        void* ws, size_t ws_bytes, void* stream) {
  (void)X;
  return do_input(h, bwd, s, W, A, B, dY, dX, ws, ws_bytes, stream);
}

// ------------------------------------------------ forward2 in two halves
runlora_status_t runlora_wprime_t(runlora_handle_t h, const runlora_shape_t* s, const void* W, const void* A,
                                  const void* B, void* Wpt, void* stream) {
  RL_TRY(check_handle(h));
  RL_TRY(check_shape(s));
  if (s->dtype != RUNLORA_BF16) return fail(RUNLORA_ERR_DTYPE, "runlora_wprime_t: bf16 operands only");
  RL_TRY(check_ptr(W, "W"));
  RL_TRY(check_ptr(A, "A"));
  RL_TRY(check_ptr(B, "B"));
  RL_TRY(check_ptr(Wpt, "Wpt"));
  CallLock lk(h->ctx->call_mu);
  DeviceGuard dg(h->ctx->device());
  RL_TRY(wprime_t_bf16(*h->ctx, *s, W, A, B, Wpt, static_cast<cudaStream_t>(stream)));
  return post_launch();
}

runlora_status_t runlora_forward_wprime(runlora_handle_t h, const runlora_shape_t* s, const void* X, const void* Wpt,
                                        void* Y, void* ws, size_t ws_bytes, void* stream) {
  RL_TRY(check_handle(h));
  RL_TRY(check_shape(s));
  if (s->dtype != RUNLORA_BF16) return fail(RUNLORA_ERR_DTYPE, "runlora_forward_wprime: bf16 operands only");
  RL_TRY(check_ptr(X, "X"));
  RL_TRY(check_ptr(Wpt, "Wpt"));
  RL_TRY(check_ptr(Y, "Y"));
  Bufs b;
  RL_TRY(bind_ws(*s, ws, ws_bytes, &b));
  CallLock lk(h->ctx->call_mu);
  DeviceGuard dg(h->ctx->device());
  RL_TRY(forward_from_wpt(*h->ctx, *s, X, Wpt, Y, b, static_cast<cudaStream_t>(stream)));
  return post_launch();
}

// ------------------------------------------------ quantized frozen weight (R18)
runlora_status_t runlora_quantize_w_e4m3(runlora_handle_t h, int64_t k, int64_t m, const void* W, void* Wq,
                                         float* scale, void* diag, void* stream) {
  RL_TRY(check_handle(h));
  if (k <= 0 || m <= 0) return fail(RUNLORA_ERR_INVALID_ARG, "k and m must be >= 1");
  if (m & 15) return fail(RUNLORA_ERR_ALIGNMENT, "m must be a multiple of 16 (16-byte rows of Wq)");
  RL_TRY(check_ptr(W, "W"));
  RL_TRY(check_ptr(Wq, "Wq"));
  RL_TRY(check_ptr(scale, "scale"));
  RL_TRY(check_ptr(diag, "diag"));
  CallLock lk(h->ctx->call_mu);
  DeviceGuard dg(h->ctx->device());
  cudaError_t e = launch_quantize_w(*h->ctx, W, k, m, Wq, scale, diag, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "quantize launch");
  return RUNLORA_OK;
}

runlora_status_t runlora_allreduce_sum_f32(runlora_handle_t h, const float* const* peers, int P, float* out,
                                           int64_t n, void* stream) {
  RL_TRY(check_handle(h));
  if (!peers || P < 1 || P > kMaxPeers) return fail(RUNLORA_ERR_INVALID_ARG, "allreduce: need 1..16 peer buffers");
  if (n < 0) return fail(RUNLORA_ERR_INVALID_ARG, "allreduce: n must be >= 0");
  RL_TRY(check_ptr(out, "out"));
  for (int q = 0; q < P; ++q) {
    RL_TRY(check_ptr(peers[q], "peers[p]"));
    if (reinterpret_cast<uintptr_t>(peers[q]) & 15) return fail(RUNLORA_ERR_ALIGNMENT, "allreduce: peer buffers must be 16-byte aligned");
    if (peers[q] == out) return fail(RUNLORA_ERR_INVALID_ARG, "allreduce: out must not be a peer buffer");
  }
  if (reinterpret_cast<uintptr_t>(out) & 15) return fail(RUNLORA_ERR_ALIGNMENT, "allreduce: out must be 16-byte aligned");
  if (n == 0) return RUNLORA_OK;
  CallLock lk(h->ctx->call_mu);
  DeviceGuard dg(h->ctx->device());
  cudaError_t e = launch_allreduce_sum_f32(*h->ctx, peers, P, out, n, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "allreduce launch");
  return RUNLORA_OK;
}

runlora_status_t runlora_workspace_size_wq(const runlora_shape_t* s, int fwd, int bwd, size_t* bytes) {
  RL_TRY(runlora_workspace_size(s, fwd, bwd, bytes));
  if (s->dtype != RUNLORA_BF16) return fail(RUNLORA_ERR_DTYPE, "quantized W needs bf16 operands");
  *bytes += al((size_t)s->k * s->m * 2);  // W~ for the x1 variants, after the regular workspace
  return RUNLORA_OK;
}

namespace {
// Validates the quantized-W arguments; binds the regular workspace and the W~ region after it.
runlora_status_t bind_wq(runlora_handle_t h, const runlora_shape_t* s, const void* Wq, const float* scale,
                         const void* diag, void* ws, size_t ws_bytes, Bufs* b, void** wdq) {
  RL_TRY(check_handle(h));
  RL_TRY(check_shape(s));
  if (s->dtype != RUNLORA_BF16) return fail(RUNLORA_ERR_DTYPE, "quantized W needs bf16 operands");
  if (s->m & 15)
    return fail(RUNLORA_ERR_ALIGNMENT, "quantized W needs m a multiple of 16 (16-byte TMA row strides of the 1-byte Wq)");
  RL_TRY(check_ptr(Wq, "Wq"));
  RL_TRY(check_ptr(scale, "scale"));
  RL_TRY(check_ptr(diag, "diag"));
  if (!ws) return fail(RUNLORA_ERR_INVALID_ARG, "workspace is NULL");
  const size_t main = layout_of(*s).total;
  if (ws_bytes < main + al((size_t)s->k * s->m * 2)) {
    char buf[160];
    snprintf(buf, sizeof buf, "workspace too small for the quantized-W entry points: %zu bytes given, %zu needed",
             ws_bytes, main + al((size_t)s->k * s->m * 2));
    return fail(RUNLORA_ERR_WORKSPACE, buf);
  }
  RL_TRY(bind_ws(*s, ws, main, b));
  *wdq = static_cast<char*>(ws) + main;
  return RUNLORA_OK;
}
}  // namespace

// forward2 builds W'ᵀ straight from Wq (one fused launch); forward1 needs W~ itself as its
// main B operand: the same converter writes it into the workspace tail first.
runlora_status_t runlora_forward_wq(runlora_handle_t h, int fwd, const runlora_shape_t* s, const void* X,
                                    const void* Wq, const float* scale, const void* diag, const void* A,
                                    const void* B, void* Y, void* ws, size_t ws_bytes, void* stream) {
  Bufs b;
  void* wdq = nullptr;
  RL_TRY(bind_wq(h, s, Wq, scale, diag, ws, ws_bytes, &b, &wdq));
  RL_TRY(validate_forward(h, fwd, s, X, wdq, A, B, Y));
  CallLock lk(h->ctx->call_mu);
  DeviceGuard dg(h->ctx->device());
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const QW qw{Wq, scale, diag};
  if (fwd == 1) RL_TRY(wprime_q(*h->ctx, *s, qw, nullptr, nullptr, wdq, false, false, st));
  RL_TRY(forward_bf16(*h->ctx, fwd, *s, X, wdq, A, B, Y, b, st, fwd == 2 ? &qw : nullptr));
  return post_launch();
}

// forward2's first half from a quantized W: W'ᵀ = (W~ + A·B)ᵀ into caller memory (the same
// fused launch runlora_forward_wq(2) issues), for runlora_forward_wprime.
runlora_status_t runlora_wprime_t_wq(runlora_handle_t h, const runlora_shape_t* s, const void* Wq,
                                     const float* scale, const void* diag, const void* A, const void* B, void* Wpt,
                                     void* stream) {
  RL_TRY(check_handle(h));
  RL_TRY(check_shape(s));
  if (s->dtype != RUNLORA_BF16) return fail(RUNLORA_ERR_DTYPE, "quantized W needs bf16 operands");
  if (s->m & 15)
    return fail(RUNLORA_ERR_ALIGNMENT, "quantized W needs m a multiple of 16 (16-byte TMA row strides of the 1-byte Wq)");
  RL_TRY(check_ptr(Wq, "Wq"));
  RL_TRY(check_ptr(scale, "scale"));
  RL_TRY(check_ptr(diag, "diag"));
  RL_TRY(check_ptr(A, "A"));
  RL_TRY(check_ptr(B, "B"));
  RL_TRY(check_ptr(Wpt, "Wpt"));
  CallLock lk(h->ctx->call_mu);
  DeviceGuard dg(h->ctx->device());
  const QW qw{Wq, scale, diag};
  RL_TRY(wprime_q(*h->ctx, *s, qw, A, B, Wpt, true, true, static_cast<cudaStream_t>(stream)));
  return post_launch();
}

// backward4/5 build W' straight from Wq for dX; backward1..3 multiply dX by W~ itself
// (converter into the workspace tail); the adapter gradients never touch W.
runlora_status_t runlora_backward_wq(runlora_handle_t h, int bwd, const runlora_shape_t* s, const void* X,
                                     const void* Wq, const float* scale, const void* diag, const void* A,
                                     const void* B, const void* dY, void* dX, void* dA, void* dB, int grad_dtype,
                                     int accumulate, void* ws, size_t ws_bytes, void* stream) {
  Bufs b;
  void* wdq = nullptr;
  RL_TRY(bind_wq(h, s, Wq, scale, diag, ws, ws_bytes, &b, &wdq));
  RL_TRY(validate_params(h, bwd, s, X, A, B, dY, dA, dB, grad_dtype));
  if (dX) RL_TRY(validate_input(h, bwd, s, wdq, A, B, dY, dX));
  CallLock lk(h->ctx->call_mu);
  DeviceGuard dg(h->ctx->device());
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const QW qw{Wq, scale, diag};
  std::vector<ReduceJob> side;
  RL_TRY(params_bf16(*h->ctx, bwd, *s, X, A, B, dY, dA, dB, grad_dtype == RUNLORA_BF16, accumulate != 0, b, st,
                     dX ? &side : nullptr));
  if (dX) {
    if (bwd <= 3) RL_TRY(wprime_q(*h->ctx, *s, qw, nullptr, nullptr, wdq, false, false, st));
    RL_TRY(input_bf16(*h->ctx, bwd, *s, wdq, A, B, dY, dX, b, st, bwd >= 4 ? &qw : nullptr, &side));
  }
  return post_launch();
}

runlora_status_t runlora_step_host(runlora_handle_t h, const runlora_shape_t* s, const runlora_host_step_t* t,
                                   void* ws, size_t ws_bytes, void* stream) {
  RL_TRY(check_handle(h));
  RL_TRY(check_shape(s));
  if (!t) return fail(RUNLORA_ERR_INVALID_ARG, "step is NULL");
  if (!t->X_host || !t->dY_host || !t->dA_host || !t->dB_host)
    return fail(RUNLORA_ERR_INVALID_ARG, "X_host, dY_host, dA_host, dB_host must be non-NULL");
  // everything the forward and backward will check, before the first copy is enqueued
  RL_TRY(validate_forward(h, t->fwd, s, t->X, t->W, t->A, t->B, t->Y));
  RL_TRY(validate_params(h, t->bwd, s, t->X, t->A, t->B, t->dY, t->dA, t->dB, t->grad_dtype));
  if (t->dX) RL_TRY(validate_input(h, t->bwd, s, t->W, t->A, t->B, t->dY, t->dX));
  if (t->dX_host && !t->dX) return fail(RUNLORA_ERR_INVALID_ARG, "dX_host needs the device buffer dX");
  {
    Bufs b;
    RL_TRY(bind_ws(*s, ws, ws_bytes, &b));
  }
  CallLock lk(h->ctx->call_mu);
  DeviceGuard dg(h->ctx->device());
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t es = s->dtype == RUNLORA_BF16 ? 2 : 4;
  const size_t ges = t->grad_dtype == RUNLORA_BF16 ? 2 : 4;
  const size_t xb = (size_t)s->n * s->k * es, yb = (size_t)s->n * s->m * es;
  cudaError_t e;
  if ((e = cudaMemcpyAsync(t->X, t->X_host, xb, cudaMemcpyHostToDevice, st)) != cudaSuccess)
    return cuda_fail(e, "H2D X");
  if ((e = cudaMemcpyAsync(t->dY, t->dY_host, yb, cudaMemcpyHostToDevice, st)) != cudaSuccess)
    return cuda_fail(e, "H2D dY");
  RL_TRY(do_forward(h, t->fwd, s, t->X, t->W, t->A, t->B, t->Y, ws, ws_bytes, stream));
  RL_TRY(do_backward(h, t->bwd, s, t->X, t->W, t->A, t->B, t->dY, t->dX, t->dA, t->dB, t->grad_dtype, t->accumulate,
                     ws, ws_bytes, stream));
  if (t->exchange) t->exchange(t->exchange_user, stream);  // e.g. the DP allreduce of dA, dB
  if ((e = cudaMemcpyAsync(t->dA_host, t->dA, (size_t)s->k * s->r * ges, cudaMemcpyDeviceToHost, st)) != cudaSuccess)
    return cuda_fail(e, "D2H dA");
  if ((e = cudaMemcpyAsync(t->dB_host, t->dB, (size_t)s->r * s->m * ges, cudaMemcpyDeviceToHost, st)) != cudaSuccess)
    return cuda_fail(e, "D2H dB");
  if (t->Y_host && (e = cudaMemcpyAsync(t->Y_host, t->Y, yb, cudaMemcpyDeviceToHost, st)) != cudaSuccess)
    return cuda_fail(e, "D2H Y");
  if (t->dX_host && (e = cudaMemcpyAsync(t->dX_host, t->dX, xb, cudaMemcpyDeviceToHost, st)) != cudaSuccess)
    return cuda_fail(e, "D2H dX");
  return RUNLORA_OK;
}

runlora_status_t runlora_profile_enable(runlora_handle_t h, int enable) {
  RL_TRY(check_handle(h));
  CallLock lk(h->ctx->call_mu);
  h->ctx->profile_enable(enable != 0);
  return RUNLORA_OK;
}

runlora_status_t runlora_profile_read(runlora_handle_t h, runlora_kernel_stat_t* stats, int max_stats, int* count,
                                      int reset) {
  RL_TRY(check_handle(h));
  std::string err;
  CallLock lk(h->ctx->call_mu);
  DeviceGuard dg(h->ctx->device());
  if (!h->ctx->profile_read(stats, max_stats, count, reset != 0, &err)) return fail(RUNLORA_ERR_CUDA, err);
  return RUNLORA_OK;
}

uint64_t runlora_launch_count(runlora_handle_t h) { return (h && h->ctx) ? h->ctx->launches() : 0; }

const char* runlora_status_string(runlora_status_t st) {
  switch (st) {
    case RUNLORA_OK: return "ok";
    case RUNLORA_ERR_INVALID_ARG: return "invalid argument";
    case RUNLORA_ERR_SHAPE: return "shape mismatch";
    case RUNLORA_ERR_DTYPE: return "unsupported dtype";
    case RUNLORA_ERR_UNSUPPORTED_VARIANT: return "unsupported variant";
    case RUNLORA_ERR_OVERFLOW: return "FLOP count overflow";
    case RUNLORA_ERR_ALIGNMENT: return "alignment";
    case RUNLORA_ERR_WORKSPACE: return "workspace too small";
    case RUNLORA_ERR_CUDA: return "CUDA error";
    case RUNLORA_ERR_TIMING: return "timing failure";
    case RUNLORA_ERR_DEVICE: return "unsupported device";
  }
  return "unknown status";
}

const char* runlora_last_error(void) { return g_last_error.c_str(); }

}  // extern "C"

// ------------------------------------------------ fused data-parallel exchange (NEXT-2)
namespace {
void exchange_geometry(int64_t k, int64_t m, int64_t r, int P, size_t* half_elems, size_t* chunks, size_t* buf_bytes,
                       size_t* flag_bytes) {
  *half_elems = (((size_t)(k + m) * (size_t)r) + 63) & ~size_t(63);
  *chunks = (size_t)((k + m + kXChunkRows - 1) / kXChunkRows);
  *buf_bytes = 2 * *half_elems * sizeof(float);
  *flag_bytes = *chunks * (size_t)P * sizeof(unsigned);
}
}  // namespace

extern "C" {

runlora_status_t runlora_exchange_sizes(int64_t k, int64_t m, int64_t r, int P, size_t* buf_bytes,
                                        size_t* flag_bytes) {
  if (k <= 0 || m <= 0 || r <= 0 || (r & 3) || P < 1 || P > kXMaxPeers || !buf_bytes || !flag_bytes)
    return fail(RUNLORA_ERR_INVALID_ARG, "exchange: k, m, r >= 1 (r a multiple of 4), 1 <= P <= 16");
  size_t half, chunks;
  exchange_geometry(k, m, r, P, &half, &chunks, buf_bytes, flag_bytes);
  return RUNLORA_OK;
}

runlora_status_t runlora_exchange_create(runlora_handle_t h, int P, int rank, int64_t k, int64_t m, int64_t r,
                                         void* const* bufs, void* const* flags, void* mc, runlora_exchange_t* out) {
  RL_TRY(check_handle(h));
  if (!out) return fail(RUNLORA_ERR_INVALID_ARG, "exchange: out is NULL");
  *out = nullptr;
  size_t bb, fb, half, chunks;
  RL_TRY(runlora_exchange_sizes(k, m, r, P, &bb, &fb));
  if (rank < 0 || rank >= P) return fail(RUNLORA_ERR_INVALID_ARG, "exchange: rank must be in [0, P)");
  if (!bufs || !flags) return fail(RUNLORA_ERR_INVALID_ARG, "exchange: bufs / flags are NULL");
  exchange_geometry(k, m, r, P, &half, &chunks, &bb, &fb);
  XDesc d;
  memset(&d, 0, sizeof d);
  d.P = P;
  d.rank = rank;
  d.rows0 = (int)k;
  d.rows1 = (int)m;
  d.cols = (int)r;
  d.half_elems = (long long)half;
  for (int q = 0; q < P; ++q) {
    RL_TRY(check_ptr(bufs[q], "exchange buffer"));
    RL_TRY(check_ptr(flags[q], "exchange flags"));
    d.bufs[q] = static_cast<float*>(bufs[q]);
    d.flags[q] = static_cast<unsigned*>(flags[q]);
  }
  RL_TRY(check_ptr(mc, "exchange multicast address", true));
  d.mc = static_cast<float*>(mc);
  DeviceGuard dg(h->ctx->device());
  runlora_exchange_s* x = new runlora_exchange_s{nullptr, P, rank, h->ctx->device(), k, m, r};
  cudaError_t e = cudaMalloc(&x->d_desc, sizeof(XDesc));
  if (e == cudaSuccess) e = cudaMemcpy(x->d_desc, &d, sizeof(XDesc), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    if (x->d_desc) cudaFree(x->d_desc);
    delete x;
    return cuda_fail(e, "exchange descriptor");
  }
  *out = x;
  return RUNLORA_OK;
}

runlora_status_t runlora_exchange_destroy(runlora_exchange_t x) {
  if (!x) return RUNLORA_OK;
  DeviceGuard dg(x->device);
  cudaFree(x->d_desc);
  delete x;
  return RUNLORA_OK;
}

runlora_status_t runlora_backward_exchange(runlora_handle_t h, int bwd, const runlora_shape_t* s, const void* X,
                                           const void* W, const void* A, const void* B, const void* dY, void* dX,
                                           void* dA, void* dB, int grad_dtype, int accumulate, runlora_exchange_t x,
                                           uint32_t epoch, void* ws, size_t ws_bytes, void* stream) {
  RL_TRY(validate_params(h, bwd, s, X, A, B, dY, dA, dB, grad_dtype));
  if (!dX) return fail(RUNLORA_ERR_INVALID_ARG, "exchange: dX is required (the exchange rides on the dX GEMM)");
  RL_TRY(validate_input(h, bwd, s, W, A, B, dY, dX));
  if (s->dtype != RUNLORA_BF16 || grad_dtype != RUNLORA_F32)
    return fail(RUNLORA_ERR_DTYPE, "exchange: bf16 operands and fp32 adapter gradients");
  if (!x || x->k != s->k || x->m != s->m || x->r != s->r)
    return fail(RUNLORA_ERR_INVALID_ARG, "exchange: NULL or built for another (k, m, r)");
  if (epoch == 0) return fail(RUNLORA_ERR_INVALID_ARG, "exchange: epoch starts at 1");
  {
    Bufs b;
    RL_TRY(bind_ws(*s, ws, ws_bytes, &b));
  }
  CallLock lk(h->ctx->call_mu);
  std::vector<ReduceJob> side;
  RL_TRY(do_params(h, bwd, s, X, W, A, B, dY, dA, dB, grad_dtype, accumulate, ws, ws_bytes, stream, &side));
  if (side.size() != 2) return fail(RUNLORA_ERR_UNSUPPORTED_VARIANT, "exchange: the adapter gradients were not split");
  Bufs b;
  RL_TRY(bind_ws(*s, ws, ws_bytes, &b));
  DeviceGuard dg(h->ctx->device());
  RL_TRY(input_bf16(*h->ctx, bwd, *s, W, A, B, dY, dX, b, static_cast<cudaStream_t>(stream), nullptr, &side,
                    x->d_desc, epoch));
  return post_launch();
}

}  // extern "C"

// ------------------------------------------------------------ test hook
#include "../../include/runlora_testing.h"
extern "C" runlora_status_t runlora_debug_gemm(runlora_handle_t h, int M, int N, int K1, const void* A1, int a_mn,
                                               const void* B1, int b_mn, int K2, const void* A2, const void* B2,
                                               int out_mode, void* D, const void* Cin, int BN, int splits, int cg,
                                               void* stream) {
  RL_TRY(check_handle(h));
  if (M <= 0 || N <= 0 || K1 <= 0 || K2 < 0 || splits < 1) return fail(RUNLORA_ERR_INVALID_ARG, "bad gemm dims");
  GemmReq q = base_req(M, N, KID_GEMM_MAIN);
  q.cg = cg == 2 ? 2 : 1;
  q.a_stream_once = BN <= 64;  // rank-r style problem: eligible for the 2-CTA/SM variant
  q.a = a_mn ? mat(A1, K1, M) : mat(A1, M, K1);
  q.a_mn = a_mn != 0;
  q.b = b_mn ? mat(B1, K1, N) : mat(B1, N, K1);
  q.b_mn = b_mn != 0;
  q.K1 = K1;
  if (K2 > 0) {
    q.a2 = a_mn ? mat(A2, K2, M) : mat(A2, M, K2);
    q.b2 = b_mn ? mat(B2, K2, N) : mat(B2, N, K2);
    q.K2 = K2;
  }
  q.out_mode = out_mode;
  q.D = D;
  q.ldd = N;
  q.Cin = Cin;
  q.ldc = N;
  q.BN = BN;
  const int nk = (K1 + kBK - 1) / kBK;
  q.kb_per_split = (nk + splits - 1) / splits;
  q.splits = (nk + q.kb_per_split - 1) / q.kb_per_split;
  q.split_stride = (int64_t)M * N;
  // env RUNLORA_DEBUG_TMA_STORE=1: the TMA-store epilogue (plain bf16 output, 256/512-wide tiles)
  q.tma_store = getenv("RUNLORA_DEBUG_TMA_STORE") && out_mode == OUT_BF16 && q.splits <= 1 && BN >= 256;
  CallLock lk(h->ctx->call_mu);
  DeviceGuard dg(h->ctx->device());
  if (BN == 0) {  // the main GEMMs' launch: 512/256-wide split by the planner
    q.BN = 256;
    q.cg = 2;
    q.kid = KID_GEMM_MAIN;
    if (out_mode != OUT_BF16 || q.splits > 1) return fail(RUNLORA_ERR_INVALID_ARG, "debug_gemm: BN = 0 needs a bf16 output");
    RL_TRY(gemm_wide_or_narrow(*h->ctx, q, static_cast<cudaStream_t>(stream)));
    return post_launch();
  }
  RL_TRY(gemm(*h->ctx, q, static_cast<cudaStream_t>(stream)));
  return post_launch();
}

// Copies the debug timeline of the last traced launch (env RUNLORA_TRACE=<kernel id>) to
// host memory: 8 uint64 per unit (see GemmArgs::trace).  Returns the number of units copied.
extern "C" int runlora_debug_trace(runlora_handle_t h, unsigned long long* host, int max_units) {
  if (!h || !h->ctx || !h->ctx->trace || !host) return 0;
  const int n = std::min(max_units, Ctx::kTraceUnits);
  DeviceGuard dg(h->ctx->device());
  if (cudaMemcpy(host, h->ctx->trace, sizeof(unsigned long long) * 8 * n, cudaMemcpyDeviceToHost) != cudaSuccess)
    return 0;
  if (n == Ctx::kTraceUnits &&  // full buffer requested: the per-CTA records follow
      cudaMemcpy(host + 8ull * n, h->ctx->trace + 8ull * n, sizeof(unsigned long long) * 4 * 1024,
                 cudaMemcpyDeviceToHost) != cudaSuccess)
    return 0;
  return n;
}

// Launch timeline (env RUNLORA_LTRACE=1 at handle creation): copies the records of the
// launches since the last read — 8 uint64 per launch {min CTA entry, min ready, max ready,
// min exit, max exit, 0, 0, 0} (%globaltimer ns) and the kernel id of each — then resets.
// Synchronises the device.  Returns the number of launches copied.
extern "C" int runlora_debug_ltrace(runlora_handle_t h, unsigned long long* host, int* kids, int max_launches) {
  if (!h || !h->ctx || !host || !kids) return 0;
  CallLock lk(h->ctx->call_mu);
  DeviceGuard dg(h->ctx->device());
  return h->ctx->ltrace_read(host, kids, max_launches);
}

extern "C" int runlora_debug_wide_rows(runlora_handle_t h, int M, int N, int K, int b_mn) {
  if (!h || !h->ctx || M <= 0 || N <= 0 || K <= 0) return -1;
  CallLock lk(h->ctx->call_mu);
  GemmReq q = main_req(*h->ctx, M, N);
  q.K1 = K;
  q.b_mn = b_mn != 0;
  if (main_split(M, N, K).splits > 1) return 0;  // small-M split-K path (main_gemm)
  return wide_split(*h->ctx, q).rows_big;
}

extern "C" const char* runlora_debug_kernel_name(int kid) {
  return (kid >= 0 && kid < KID_COUNT) ? kKernelNames[kid] : "?";
}

extern "C" runlora_status_t runlora_debug_exchange_emulate(runlora_handle_t h, int P, int64_t k, int64_t m, int64_t r,
                                                           int splits, const float* const* sA,
                                                           const float* const* sB, float* const* dA,
                                                           float* const* dB, void* const* bufs, void* const* flags,
                                                           uint32_t epoch) {
  RL_TRY(check_handle(h));
  size_t bb, fb, half, chunks;
  RL_TRY(runlora_exchange_sizes(k, m, r, P, &bb, &fb));
  if (splits < 1 || epoch == 0 || !sA || !sB || !dA || !dB || !bufs || !flags)
    return fail(RUNLORA_ERR_INVALID_ARG, "exchange emulation: bad arguments");
  exchange_geometry(k, m, r, P, &half, &chunks, &bb, &fb);
  std::vector<XDesc> descs(P);
  std::vector<XSlabs> slabs(P);
  for (int q = 0; q < P; ++q) {
    XDesc& d = descs[q];
    memset(&d, 0, sizeof d);
    d.P = P;
    d.rank = q;
    d.rows0 = (int)k;
    d.rows1 = (int)m;
    d.cols = (int)r;
    d.half_elems = (long long)half;
    for (int p2 = 0; p2 < P; ++p2) {
      d.bufs[p2] = static_cast<float*>(bufs[p2]);
      d.flags[p2] = static_cast<unsigned*>(flags[p2]);
    }
    XSlabs& S = slabs[q];
    memset(&S, 0, sizeof S);
    S.P[0] = sA[q];
    S.P[1] = sB[q];
    S.split_stride[0] = k * r;
    S.split_stride[1] = m * r;
    S.ldp[0] = S.ldp[1] = r;
    S.ldo[0] = r;
    S.ldo[1] = m;
    S.out[0] = dA[q];
    S.out[1] = dB[q];
    S.splits[0] = S.splits[1] = splits;
  }
  CallLock lk(h->ctx->call_mu);
  DeviceGuard dg(h->ctx->device());
  cudaError_t e = launch_exchange_emulate(*h->ctx, P, descs.data(), slabs.data(), epoch);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return cuda_fail(e, "exchange emulation");
  return RUNLORA_OK;
}
