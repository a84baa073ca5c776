// tcgen05 / TMEM / TMA GEMM for sm_100a (kernel family K1/K2 of DESIGN.md).
//
// One launch runs up to two independent GEMM problems ("dual" launches fill the
// 148 SMs with e.g. Z1 = dY·Bᵀ and Z2 = X·A at once).  Each problem is
//
//   D[M,N] = A1[M,K1]·B1[K1,N]  (+ A2[M,K2]·B2[K2,N])       (concat-K tail)
//
// bf16 operands, fp32 accumulation in TMEM.  Every bf16 product of the paper's
// variants (Eq. 1-3, Alg. 1-5) is a problem of this kernel:
//   * Y = [X | XA]·[W ; B]           (forward1 fused)   A K-major, B MN-major
//   * Y = X·(W+AB)                   (forward2)          A K-major, B K-major (W'ᵀ)
//   * dX = [dY | dYBᵀ]·[Wᵀ ; Aᵀ]     (Alg. 1-3 last line)      A K-major, B K-major
//   * dX = dY·(W+AB)ᵀ                (Alg. 4-5 last line)      A K-major, B K-major
//   * Z1 = dY·Bᵀ, Z2 = X·A           (rank-r projections)      N = r; K-split bf16 blocks
//   * dA = Xᵀ·Z1, dBᵀ = dYᵀ·Z2       (token reductions, K = n) A and B MN-major, split-K,
//                                                              partial Z blocks folded
//   * W+AB, (W+AB)ᵀ                  (K = r plus an identity tail that adds W, tail_diag)
//
// Structure (persistent, warp-specialised, one CTA per SM; CG = 2 pairs two SMs
// of a cluster on one 256-row tile with tcgen05 cta_group::2):
//   warp 0 lane 0 : TMA producer (smem ring of STAGES {A,B} tiles, mbarrier full/empty)
//   warp 1 lane 0 : tcgen05.mma issuer (leader CTA only)
//   warp 2        : TMEM allocator (2 accumulator slots of min(BN_MAX, 256) columns: the
//                   epilogue of tile i overlaps the mainloop of tile i+1; BN_MAX = 512 pair
//                   tiles issue two N = 256 MMAs per k-step sharing the A tile and use both)
//   warps 2-3     : side jobs while the mainloop runs (slab reduction, column repeat, the
//                   fused DP exchange), else idle
//   warps 4..7    : epilogue (tcgen05.ld -> registers -> global, or -> swizzled smem ->
//                   TMA store for EPI = 3), TMEM lanes 32*(w%4)..; the 512-wide TMA-store
//                   kernel runs warps 4..11 (two per lane quarter, 128 columns each) with a
//                   setmaxnreg split, holding the whole tile in registers so TMEM is released
//                   before the stores (TileCfg::WIDE_HOLD)
// Tiles: 128 rows per CTA, bn columns (runtime, <= BN_MAX), K atoms of 64 (one 128-byte
// swizzle row of bf16), KS atoms per pipeline stage.  Shared-memory tiles use the 128B
// swizzle written by TMA:
//   K-major  tile: rows of 128 B (64 K-elements), 8-row atoms of 1024 B  -> SBO = 1024
//   MN-major tile: 64-element MN chunks, each a box of 64 K-rows x 128 B  -> LBO = 8192
//                  (MN chunk stride), SBO = 1024 (8 K-rows); a UMMA_K=16 step is +2048 B.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include "ptx.cuh"
#include "exchange.cuh"

namespace runlora {

enum OutMode : int { OUT_BF16 = 0, OUT_BF16_ADD = 1, OUT_F32 = 2, OUT_F32_FOLD = 4 };
// OUT_BF16 with splits: split s of the K reduction writes its own bf16 partial at
//                 D + s * split_stride (e.g. side-by-side column blocks of a partial matrix).
// OUT_F32_FOLD:   the accumulator's bn = fold * fold_w columns are fold column blocks whose sum
//                 (fixed block order, fp32) is the output: fp32 slab D[split][M][ldd], fold_w cols.
// OUT_BF16_ADD:   D[i, j] = acc[i, j] + Cin[i * ldc + j]

struct Prob {
  int M, N;              // output extent (epilogue masks rows >= M, cols >= N)
  int bn;                // MMA N of this problem (multiple of 16*CG; of 64*CG when b_mn)
  int k1, nk1;           // main operand K (elements) and K blocks of 64
  int k2, nk2;           // tail operand K and K blocks (0 = no tail)
  int kb_per_split, num_splits;
  int num_m_tiles, num_n_tiles;
  int units;             // num_m_tiles * num_n_tiles * num_splits
  int a_mn, b_mn;        // operand majorness (0 = K-major)
  int b_swz;             // MN-major B swizzle width in bytes (32, 64, 128); K-major operands use 128
  int a_3d, b_3d;        // MN-major operand loaded by one 3-D TMA box (all swizzle chunks at once)
  int snake;             // alternate the K direction between a CTA's consecutive units (L2 reuse)
  int raster_g;          // output tiles are visited in bands of raster_g row tiles (1: row-major)
  int out_mode;          // OutMode
  uint32_t idesc;        // tcgen05 instruction descriptor
  uint32_t stage_tx;     // TMA bytes per stage for the whole CTA group
  void* D;               // bf16 [M, ldd] or fp32 partial slabs [split][M][ldd]
  long long ldd;
  long long split_stride;
  const __nv_bfloat16* Cin;  // OUT_BF16_ADD: added matrix [M, ldc]
  long long ldc;
  uint64_t hint_a, hint_b;   // TMA L2 cache hints
  int fold, fold_w;  // OUT_F32_FOLD
  // Block-diagonal concat-K tail: the tail A operand is the 128x128 identity (A2, loaded at
  // M coordinate 0) and the tail B operand is read at K coordinate m0 + k, i.e. the rows of
  // B2 that belong to this tile's own M range.  D += I·B2[m0.., n0..] adds a matrix that is
  // indexed like the output (W + A·B: the add rides in the mainloop, exact in fp32).
  int tail_diag;
};

// Per-problem fields of the features added after the main GEMM was tuned, kept in their own
// array at the END of GemmArgs so that the kernel parameter offsets the main GEMMs' hot loops
// read stay where they were.
struct ProbX {
  // Split-K fix-up (fp32 slab modes): the last split of an output tile to finish sums the
  // num_splits slabs of that tile in split order (deterministic) and writes
  //   out[i, c] (or out[c, i] when fx_transpose) {=, +=} sum_s slab[s][i][c],  c < fx_cols,
  // as fp32 or bf16.  counters: one int per output tile, zero before the launch (the
  // launch that zeroes them is GemmArgs::zero_ptr of an earlier launch in the stream).
  // FP8 tail (quantized W, R18): W~ = e4m3(Wq) · 2^e[col] enters the SAME fp32
  // accumulator as A·B through kind::f8f6f4 MMAs (idesc2) against the E5M2 diagonal D of the
  // power-of-two column scales — exact, so the epilogue is the plain bf16 store and W is read
  // as 1 byte per element.  1: W'ᵀ tile (rows j): one tail block, A2 = D rows of this tile,
  // B2 = Wq rows of the tile's columns at K = j' (MMA N = bn).  2: W' / W~ tile (rows i): one
  // tail block per 128 columns h, A2 = Wq rows of this tile at K = n0 + 128 h, B2 = D rows
  // n0 + 128 h (MMA N = 128 into accumulator columns [128 h, +128)).  Both K-major.
  int tail_fp8;
  uint32_t idesc2;
  int fixup;
  int* counters;
  void* fx_out;
  long long fx_ldo;
  int fx_cols, fx_transpose, fx_accumulate, fx_bf16;
};

constexpr int kMaxProb = 2;  // problems per launch (dual launches); kernel params stay ~1.8 KB
constexpr int kTraceMaxUnits = 1 << 16;  // debug trace: unit records, then 4 words per CTA

// A fixed-order split-K reduction carried by a GEMM launch as a side job of its otherwise idle
// warps 2-3 (e.g. the adapter gradients' token-split slabs, reduced while the dX GEMM runs):
//   out[i, c] (or out[c, i] when transpose) {=, +=} sum_{s < splits} P[s][i][c],  c < cols.
struct SideJob {
  const float* P;
  long long split_stride, ldp, ldo;
  void* out;
  int splits, rows, cols, out_bf16, transpose, accumulate;
  int repeat;  // > 0: column repeat of a bf16 matrix instead (dst[i, t*cols + j] = src[i, j], t < repeat)
};

struct GemmArgs {
  Prob p[kMaxProb];
  int nprob;
  int total_units;
  int dbg;  // 0 normal; 1: no TMA (MMA-only); 2: no MMA (TMA-only); 3: as 1 + no stores; 4: as 1 + no epilogue;
            // 5: A loads only (MMA on stale B); 6: B loads only (stale A); 7: A loads on even
            // k-blocks only (75 % of the TMA bytes); 8: 512-wide tiles read TMEM but store nothing
  // Debug timeline (RUNLORA_TRACE): per unit u, trace[8u + {0: producer start, 2: last load
  // issued, 3: epilogue done, 4: CTA, 5: problem}] (%globaltimer ns).
  unsigned long long* trace;
  unsigned long long* ltrace;  // launch timeline slot (nullptr: off)
  int stages;                  // pipeline stages (0: the compiled maximum TileCfg::STAGES)
  int endj;                    // 512-wide tiles: k-blocks whose MMA 1 follows the tile's last MMA 0
  int* zero_ptr;               // zeroed by CTA 0 after the PDL wait (split fix-up counters of a
  int zero_n;                  // later launch in the stream), nullptr: none
  SideJob side[2];
  int nside;
  ProbX px[kMaxProb];
  // fused data-parallel exchange (exchange.cuh): with xdesc, side[0] / side[1] are the dA / dB
  // slab reductions and warps 2-3 reduce them ACROSS ranks (epoch: this exchange's number)
  const XDesc* xdesc;
  unsigned xepoch;
};

struct Tmaps {  // per problem: A1, B1, A2, B2, D (EPI = 3: TMA-store epilogue)
  CUtensorMap m[kMaxProb][5];
};

constexpr int kStgBufs = 4;  // EPI = 3 staging tiles per epilogue warp (a 256-wide tile's 4 stores never wait)
constexpr int kBM = 128;  // rows per CTA
constexpr int kMaxFixups = 64;  // split fix-ups one CTA can defer to the end of its unit loop
constexpr int kBK = 64;
constexpr int kWideRegsLow = 120;   // setmaxnreg of the 512-wide kernel's warp groups:
constexpr int kWideRegsHigh = 184;  // 128 x 104 + 256 x 200 = 384 x 168 (launch allocation)

// OCC = CTAs per SM (2 for the HBM-bound rank-r kernels: twice the TMA requests in flight).
// EPI = 3: TMA-store epilogue (bf16 tile staged per warp in swizzled smem).
// KS = 64-wide K atoms per pipeline stage (1 or 2): a stage holds KS A atoms then KS B atoms.
template <int BN_MAX, int CG, int OCC = 1, int EPI = 0, int KS = 1>
struct TileCfg {
  static constexpr uint32_t A_ATOM = kBM * kBK * 2;
  static constexpr uint32_t B_ATOM = (BN_MAX / CG) * kBK * 2;
  static constexpr uint32_t A_BYTES = KS * A_ATOM;
  static constexpr uint32_t B_BYTES = KS * B_ATOM;
  static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  // Epilogue warps: 4 (one per TMEM lane quarter), or 8 for the 512-wide TMA-store kernel —
  // two per lane quarter, each holding 128 columns of both accumulator slots in registers
  // (bf16 pairs, 128 registers per thread), so the whole tile leaves TMEM at TMEM-read speed
  // and its stores overlap the next tile's mainloop (warp-group register split: setmaxnreg).
  static constexpr bool WIDE_HOLD = BN_MAX > 256 && EPI == 3;
  static constexpr int EPI_WARPS = WIDE_HOLD ? 8 : 4;
  static constexpr int THREADS = 128 + 32 * EPI_WARPS;
  // EPI = 3: per epilogue warp STG_BUFS 32-row x 64-column bf16 staging tiles (128B swizzle)
  // (1 for the 512-wide kernel, whose 4 ring stages of 48 KB leave 32 KB for 8 warps)
  static constexpr int STG_BUFS = WIDE_HOLD ? 1 : kStgBufs;
  static constexpr uint32_t STG_BYTES = EPI == 3 ? EPI_WARPS * STG_BUFS * 4096 : 0;
  // up to ~225 KB of the 227 KB opt-in smem per SM (7 stages for the 256x256 pair tiles)
  static constexpr int STAGES_RAW = ((OCC == 1 ? 225 : 110) * 1024 - STG_BYTES) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 12 ? 12 : STAGES_RAW;
  static constexpr uint32_t TMEM_COLS = (2 * BN_MAX <= 32) ? 32 : (2 * BN_MAX <= 64) ? 64
                                        : (2 * BN_MAX <= 128) ? 128 : (2 * BN_MAX <= 256) ? 256 : 512;
  static constexpr bool FIXUP = CG == 1 && EPI == 0;  // kernels that compile the split fix-up
  static constexpr uint32_t SMEM_BYTES = STAGES * STAGE_BYTES + STG_BYTES + 1024 /*align*/ + 256 /*barriers*/ +
                                         (FIXUP ? 4 * kMaxFixups : 0) /*split fix-up list*/;
};

struct Unit {
  int prob, m_blk, n_blk, split;
};
__device__ __forceinline__ Unit decode_unit(const GemmArgs& g, int u) {
  Unit t;
  t.prob = 0;
  while (t.prob < kMaxProb - 1 && u >= g.p[t.prob].units) {
    u -= g.p[t.prob].units;
    ++t.prob;
  }
  const Prob& p = g.p[t.prob];
  const int per_split = p.num_m_tiles * p.num_n_tiles;
  t.split = u / per_split;
  int r = u - t.split * per_split;
  // Grouped raster: bands of G row tiles, row index fastest inside a band, so the CTAs
  // resident at any time cover a compact block of the output and the A and B tiles they
  // stream stay in L2 (walking whole rows of tiles streams all of B through L2 once per
  // wave, e.g. an 86 MiB W for the 11008-wide Llama MLP).  G = 1 (row-major walk) when
  // all of B fits comfortably in L2.
  const int G = p.raster_g;
  const int band = r / (G * p.num_n_tiles);
  const int m_first = band * G;
  const int g_rows = min(G, p.num_m_tiles - m_first);
  r -= band * G * p.num_n_tiles;
  t.m_blk = m_first + r % g_rows;
  t.n_blk = r / g_rows;
  return t;
}

// The i-th unit of CTA group `group` (static round-robin: units group, group + ngroups, ..),
// -1 past its last.  (Walking odd groups' units in reverse, to stagger the wide tiles'
// exposed epilogues, measured 12 µs slower at C2: it breaks the raster's L2 locality.)
__device__ __forceinline__ int unit_of(const GemmArgs& g, int group, int ngroups, int i) {
  const int u = group + i * ngroups;
  return u < g.total_units ? u : -1;
}

// MMAs of N = slot_w per k-step for a unit: 2 for a 512-wide tile unless its second half lies
// wholly past N (the ragged last column tile runs as one MMA, one B box, one TMEM slot).
__device__ __forceinline__ int unit_halves(const Prob& p, int n_blk, int slot_w) {
  return (p.bn > slot_w && n_blk * p.bn + slot_w < p.N) ? 2 : 1;
}

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

__device__ __forceinline__ void tmem_ld_32x32b_x16(uint32_t taddr, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}

// Stores `cnt` (16 or 32) fp32 accumulator values of one row segment per out_mode.
__device__ __forceinline__ void store_row_segment(const Prob& p, int split, int row, int col, const uint32_t* v,
                                                  int cnt) {
  if (p.out_mode == OUT_F32) {
    float* dst = static_cast<float*>(p.D) + split * p.split_stride + (long long)row * p.ldd + col;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      if (e * 4 < cnt && col + 4 * e < p.N) {
        float4 w = make_float4(__uint_as_float(v[4 * e]), __uint_as_float(v[4 * e + 1]),
                               __uint_as_float(v[4 * e + 2]), __uint_as_float(v[4 * e + 3]));
        *reinterpret_cast<float4*>(dst + 4 * e) = w;
      }
    }
  } else {
    __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(p.D) + split * p.split_stride + (long long)row * p.ldd + col;
    const bool add = p.out_mode == OUT_BF16_ADD;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if (e * 8 < cnt && col + 8 * e < p.N) {
        float f[8];
#pragma unroll
        for (int x = 0; x < 8; ++x) f[x] = __uint_as_float(v[8 * e + x]);
        if (add) {
          uint4 cv = *reinterpret_cast<const uint4*>(p.Cin + (long long)row * p.ldc + col + 8 * e);
          const __nv_bfloat162* c2 = reinterpret_cast<const __nv_bfloat162*>(&cv);
#pragma unroll
          for (int x = 0; x < 4; ++x) {
            float2 cf = __bfloat1622float2(c2[x]);
            f[2 * x] += cf.x;
            f[2 * x + 1] += cf.y;
          }
        }
        uint4 o;
        o.x = pack_bf16x2(f[0], f[1]);
        o.y = pack_bf16x2(f[2], f[3]);
        o.z = pack_bf16x2(f[4], f[5]);
        o.w = pack_bf16x2(f[6], f[7]);
        *reinterpret_cast<uint4*>(dst + 8 * e) = o;
      }
    }
  }
}


// Split-K fix-up of output tile (m_blk, n_blk) of problem p, run by the 4 epilogue warps of
// the CTA whose split arrived last (Prob::fixup), after its unit loop.  Thread = row; 16-column
// chunks; the slabs are summed in split order (deterministic), two splits' loads (8 x 16 B)
// in flight before any is added.
__device__ __forceinline__ void split_fixup(const Prob& p, const ProbX& px, int row, int n_blk) {
  if (row >= p.M) return;
  const int c_lo = n_blk * p.bn, c_hi = min(px.fx_cols, c_lo + p.bn);
  const float* base = static_cast<const float*>(p.D) + (long long)row * p.ldd;
  const long long ostep = px.fx_transpose ? px.fx_ldo : 1;
  const long long obase = px.fx_transpose ? (long long)row : (long long)row * px.fx_ldo;
  const int S = p.num_splits;
#pragma unroll 1
  for (int c0 = c_lo; c0 < c_hi; c0 += 16) {
    float a[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) a[e] = 0.f;
#pragma unroll 1
    for (int sp = 0; sp < S; sp += 2) {
      float4 v[8];
#pragma unroll
      for (int x = 0; x < 8; ++x)
        if (sp + (x >> 2) < S && c0 + 4 * (x & 3) < c_hi)
          v[x] = __ldcg(reinterpret_cast<const float4*>(base + (sp + (x >> 2)) * p.split_stride + c0 + 4 * (x & 3)));
#pragma unroll
      for (int x = 0; x < 8; ++x)
        if (sp + (x >> 2) < S && c0 + 4 * (x & 3) < c_hi) {
          float* t = a + 4 * (x & 3);
          t[0] += v[x].x, t[1] += v[x].y, t[2] += v[x].z, t[3] += v[x].w;
        }
    }
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      if (c0 + e >= c_hi) break;
      const long long o = obase + (long long)(c0 + e) * ostep;
      float val = a[e];
      if (px.fx_bf16) {
        __nv_bfloat16* d = static_cast<__nv_bfloat16*>(px.fx_out) + o;
        if (px.fx_accumulate) val += __bfloat162float(*d);
        *d = __float2bfloat16_rn(val);
      } else {
        float* d = static_cast<float*>(px.fx_out) + o;
        if (px.fx_accumulate) val += *d;
        *d = val;
      }
    }
  }
}

__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// SideJob reduction by `nthr` threads (index tid) across the grid: one (row, 4-column group)
// per item, the splits' float4 loads issued 8 at a time, summed in split order.
__device__ __forceinline__ void side_reduce(const GemmArgs& g, long long tid, long long nthr) {
  for (int j = 0; j < g.nside; ++j) {
    const SideJob& J = g.side[j];
    if (J.repeat > 0) {  // bf16 column repeat, 16-byte groups
      const int gc = J.cols >> 3;
      const long long total = (long long)J.rows * gc * J.repeat;
      const uint4* src = reinterpret_cast<const uint4*>(J.P);
      uint4* dst = static_cast<uint4*>(J.out);
      for (long long idx = tid; idx < total; idx += nthr) {
        const long long i = idx / ((long long)gc * J.repeat);
        dst[idx] = src[i * gc + (int)(idx % gc)];
      }
      continue;
    }
    const int groups = (J.cols + 3) >> 2;
    const long long total = (long long)J.rows * groups;
    for (long long idx = tid; idx < total; idx += nthr) {
      const int i = (int)(idx / groups), c0 = (int)(idx % groups) * 4;
      const float4* src = reinterpret_cast<const float4*>(J.P + (long long)i * J.ldp + c0);
      const long long st4 = J.split_stride >> 2;
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int s0 = 0; s0 < J.splits; s0 += 8) {
        float4 v[8];
#pragma unroll
        for (int x = 0; x < 8; ++x)
          if (s0 + x < J.splits) v[x] = __ldcg(src + (s0 + x) * st4);
#pragma unroll
        for (int x = 0; x < 8; ++x)
          if (s0 + x < J.splits) acc.x += v[x].x, acc.y += v[x].y, acc.z += v[x].z, acc.w += v[x].w;
      }
      const float a4[4] = {acc.x, acc.y, acc.z, acc.w};
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        if (c0 + x >= J.cols) break;
        const long long o = J.transpose ? (long long)(c0 + x) * J.ldo + i : (long long)i * J.ldo + c0 + x;
        float val = a4[x];
        if (J.out_bf16) {
          __nv_bfloat16* d = static_cast<__nv_bfloat16*>(J.out) + o;
          if (J.accumulate) val += __bfloat162float(*d);
          *d = __float2bfloat16_rn(val);
        } else {
          float* d = static_cast<float*>(J.out) + o;
          if (J.accumulate) val += *d;
          *d = val;
        }
      }
    }
  }
}

// EPI = 3: one 32-row x 64-column bf16 chunk of a warp (row = lane) -> its staging buffer
// (128B swizzle: 16-byte chunk e of row r at (e ^ (r & 7)) * 16) -> TMA store.  A buffer is
// reused only after the store issued NB chunks earlier has finished reading it.
template <int NB>
__device__ __forceinline__ void stage_store_chunk(const uint32_t (&v)[2][32], uint8_t* stg, int& st_it, int lane,
                                                  const CUtensorMap* dmap, int col, int row0) {
  const int buf = st_it % NB;
  if (st_it >= NB) {
    if (lane == 0) bulk_wait_read<NB - 1>();
    __syncwarp();
  }
  uint8_t* rowp = stg + buf * 4096 + lane * 128;
  const uint32_t sw = (uint32_t)lane & 7u;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const uint32_t* x = &v[e >> 2][8 * (e & 3)];
    uint4 o;
    o.x = pack_bf16x2(__uint_as_float(x[0]), __uint_as_float(x[1]));
    o.y = pack_bf16x2(__uint_as_float(x[2]), __uint_as_float(x[3]));
    o.z = pack_bf16x2(__uint_as_float(x[4]), __uint_as_float(x[5]));
    o.w = pack_bf16x2(__uint_as_float(x[6]), __uint_as_float(x[7]));
    *reinterpret_cast<uint4*>(rowp + ((e ^ sw) << 4)) = o;
  }
  fence_proxy_async_shared();
  __syncwarp();
  if (lane == 0) {
    tma_store_2d(dmap, stg + buf * 4096, col, row0);
    bulk_commit();
  }
  ++st_it;
}

// As stage_store_chunk for a chunk already packed to bf16 pairs (pk[x] = columns 2x, 2x+1).
template <int NB>
__device__ __forceinline__ void stage_store_packed(const uint32_t (&pk)[32], uint8_t* stg, int& st_it, int lane,
                                                   const CUtensorMap* dmap, int col, int row0) {
  const int buf = st_it % NB;
  if (st_it >= NB) {
    if (lane == 0) bulk_wait_read<NB - 1>();
    __syncwarp();
  }
  uint8_t* rowp = stg + buf * 4096 + lane * 128;
  const uint32_t sw = (uint32_t)lane & 7u;
#pragma unroll
  for (int e = 0; e < 8; ++e)
    *reinterpret_cast<uint4*>(rowp + ((e ^ sw) << 4)) = make_uint4(pk[4 * e], pk[4 * e + 1], pk[4 * e + 2], pk[4 * e + 3]);
  fence_proxy_async_shared();
  __syncwarp();
  if (lane == 0) {
    tma_store_2d(dmap, stg + buf * 4096, col, row0);
    bulk_commit();
  }
  ++st_it;
}

// EPI = 0: epilogue stores from registers; EPI = 3: TMA-store epilogue (plain bf16 outputs).
// KS: 64-wide K atoms per pipeline stage (TileCfg).
template <int BN_MAX, int CG, int OCC = 1, int EPI = 0, int KS = 1>
__global__ void __launch_bounds__(TileCfg<BN_MAX, CG, OCC, EPI, KS>::THREADS, OCC)
    tc_gemm_kernel(const __grid_constant__ Tmaps tm, const __grid_constant__ GemmArgs g) {
  using C = TileCfg<BN_MAX, CG, OCC, EPI, KS>;
  // features compiled only where they are used, so the main GEMMs' code (and its MMA issue
  // loop) stays as lean as before them: the FP8 identity tail and its scaling epilogue (W'
  // builds from a quantized W: single-CTA TMA-store kernel), the split fix-up (rank-r kernels)
  constexpr bool kFp8Tail = CG == 1 && EPI == 3;
  constexpr bool kFixup = C::FIXUP;
  constexpr bool kSide = KS == 1;  // side jobs ride on K-major launches (dX GEMM, projections)
  // runtime ring depth <= the compiled maximum (fewer stages leave shared memory to kernels
  // that should co-reside, e.g. NCCL's during an overlapped allreduce)
  const int STAGES = (g.stages > 0 && g.stages < C::STAGES) ? g.stages : C::STAGES;
  static_assert(BN_MAX % (16 * CG) == 0 && BN_MAX >= 16 && (BN_MAX <= 256 || (BN_MAX == 512 && CG == 2)), "UMMA N");
  // TMEM: two accumulator slots of SLOT_W columns.  A unit of bn <= SLOT_W uses one slot (the
  // epilogue of unit i overlaps the mainloop of unit i+1); a 512-wide pair tile (BN_MAX = 512:
  // two N = 256 MMAs per k-step sharing the A tile) uses both.
  constexpr int SLOT_W = BN_MAX <= 256 ? BN_MAX : 256;
  constexpr uint32_t kBHalf = (SLOT_W / CG) * 128;  // K-major B bytes of one MMA's columns per CTA

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * C::A_BYTES;
  // [A ring | B ring | EPI = 3 staging | barriers]
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * C::B_BYTES + C::STG_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  // split fix-up: the tiles this CTA's splits completed last (packed prob|n_blk|m_blk), reduced
  // after its unit loop, where the epilogue's registers are free (Prob::fixup)
  volatile int* fx_count = reinterpret_cast<volatile int*>(tmem_slot + 1);
  int* fx_list = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(full) + 256);
  if (threadIdx.x == 4 * 32) *fx_count = 0;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = CG == 2 ? cluster_ctarank() : 0;
  const bool leader = rank == 0;
  const int group = blockIdx.x / CG;
  const int ngroups = gridDim.x / CG;

  // debug timeline per CTA (after the units): {kernel entry, inputs ready (after PDL wait), exit, SM id}
  unsigned long long* ctrace = g.trace ? g.trace + 8ull * kTraceMaxUnits + 4ull * blockIdx.x : nullptr;
  if (ctrace && threadIdx.x == 0) ctrace[0] = globaltimer(), ctrace[3] = smid();
  if (threadIdx.x == 0) ltrace_mark(g.ltrace, 0);
  if (warp == 0 && lane == 0) {
    for (int q = 0; q < g.nprob; ++q)
      for (int j = 0; j < 4; ++j)
        if (j < 2 || g.p[q].nk2 > 0) tma_prefetch_desc(&tm.m[q][j]);
    if constexpr (EPI == 3)
      for (int q = 0; q < g.nprob; ++q) tma_prefetch_desc(&tm.m[q][4]);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], C::EPI_WARPS * CG);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<CG>(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync();
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // everything above overlapped the previous kernel's tail (PDL); inputs are read below
  pdl_wait();
  pdl_launch_dependents();
  if (g.zero_ptr && blockIdx.x == 0)
    for (int i = threadIdx.x; i < g.zero_n; i += blockDim.x) g.zero_ptr[i] = 0;
  if (ctrace && threadIdx.x == 0) ctrace[1] = globaltimer();
  if (threadIdx.x == 0) ltrace_mark(g.ltrace, 1);

  // Roles: warp group 0 = TMA producer (warp 0), MMA issuer (warp 1), side jobs (warps 2-3);
  // the other warps = epilogue.  The bodies are inlined lambdas so that the 512-wide
  // TMA-store kernel can wrap them in its warp-group register split while every other
  // kernel keeps the plain dispatch chain (its code generation unchanged).
  auto run_producer = [&]() __attribute__((always_inline)) {
    // ------------------------------------------------------------ TMA producer
    // The whole warp runs the loop (warp-uniform values); one elected lane issues.
    int stage = 0;
    uint32_t phase = 0;
    for (int i_u = 0;; ++i_u) {
      const int u = unit_of(g, group, ngroups, i_u);
      if (u < 0) break;
      const Unit t = decode_unit(g, u);
      const Prob& p = g.p[t.prob];
      const ProbX& px = g.px[t.prob];
      if (g.trace && lane == 0) {
        g.trace[8 * u + 0] = globaltimer();
        g.trace[8 * u + 4] = blockIdx.x;
        g.trace[8 * u + 5] = t.prob;
      }
      const int m0 = t.m_blk * (kBM * CG) + rank * kBM;
      const int nb = p.bn / CG;  // B columns held by this CTA
      const int n0 = t.n_blk * p.bn + rank * nb;
      const int nh = BN_MAX > SLOT_W ? unit_halves(p, t.n_blk, SLOT_W) : 1;
      const int kb0 = t.split * p.kb_per_split;
      const int kb1 = min(p.nk1, kb0 + p.kb_per_split);
      const int nmain = kb1 - kb0;
      const int nkb = nmain + (t.split == 0 ? p.nk2 : 0);
      const bool fp8_tail = kFp8Tail && px.tail_fp8;
      // snake: every other round of this CTA walks K backwards, starting where the data it
      // (and its neighbours) just streamed is still in L2
      const bool rev = p.snake && (i_u & 1);
      if (g.dbg == 1 || g.dbg == 3 || g.dbg == 4) continue;
      const int cw = p.b_swz >> 1;   // MN-major B chunk width (elements)
      const int cb = p.b_swz * kBK;  // MN-major B chunk bytes (64 K-rows)
      for (int i0 = 0; i0 < nkb; i0 += KS) {
        mbar_wait(&empty[stage], phase ^ 1);
        if (elect_one_sync()) {
          const int natoms = min(KS, nkb - i0);
          uint64_t* fb = &full[stage];
          const bool skip_a = g.dbg == 6 || (g.dbg == 7 && (i0 & 1));
          // a ragged 512-wide tile loads one B box per CTA
          const uint32_t full_tx = (BN_MAX > SLOT_W && p.bn > SLOT_W && nh == 1) ? p.stage_tx - CG * kBHalf : p.stage_tx;
          const uint32_t tx = g.dbg == 5 ? (uint32_t)(CG * kBM * kBK * 2)
                              : skip_a ? full_tx - (uint32_t)(CG * kBM * kBK * 2)
                              : (fp8_tail && px.tail_fp8 == 2 && i0 >= nmain) ? 2u * 128u * 128u  // two 16 KB boxes
                                                                             : full_tx;
          if (leader) mbar_arrive_expect_tx(fb, tx * (uint32_t)natoms);
          for (int at = 0; at < natoms; ++at) {
            const int i = i0 + at;
            uint8_t* a = sA + stage * C::A_BYTES + at * C::A_ATOM;
            uint8_t* b = sB + stage * C::B_BYTES + at * C::B_ATOM;
            const bool tail = i >= nmain;
            const bool diag = tail && p.tail_diag;
            const CUtensorMap* ta = &tm.m[t.prob][tail ? 2 : 0];
            const CUtensorMap* tb = &tm.m[t.prob][tail ? 3 : 1];
            const int ki = rev ? nmain - 1 - i : i;
            // K coordinates of the A and B boxes: main k-block, plain tail block, repeated
            // tail block (A2 column block s against B2 from K = 0), identity tail (B2 rows of
            // this tile)
            // (this loop sets the 256-wide kernels' TMA issue rate: one more parameter-dependent
            // select per atom here measured 5-8 % slower main GEMMs)
            const int kc = (tail ? (i - nmain) : (kb0 + ki)) * kBK;
            const int ma = diag ? 0 : m0;          // identity tail: rows of I
            const int kcb = diag ? m0 + kc : kc;   // identity tail: B2 rows of this tile
            if (fp8_tail && tail) {  // ProbX::tail_fp8 (expect_tx set below for mode 2)
              const int h = i - nmain;
              if (px.tail_fp8 == 1) {  // D rows m0.. (E5M2); Wq rows n0.. at K = m0 (E4M3)
                tma_load_2d<CG>(ta, fb, a, 0, m0, p.hint_a);
                tma_load_2d<CG>(tb, fb, b, m0, n0, p.hint_b);
              } else {                 // Wq rows m0.. at K = n0 + 128 h (E4M3); D rows n0 + 128 h (E5M2)
                tma_load_2d<CG>(ta, fb, a, n0 + 128 * h, m0, p.hint_a);
                tma_load_2d<CG>(tb, fb, b, 0, n0 + 128 * h, p.hint_b);
              }
              continue;
            }
            if (skip_a) {
            } else if (!p.a_mn) {
              tma_load_2d<CG>(ta, fb, a, kc, ma, p.hint_a);
            } else if (p.a_3d) {
              tma_load_3d<CG>(ta, fb, a, 0, kc, ma >> 6, p.hint_a);
            } else {
              tma_load_2d<CG>(ta, fb, a, ma, kc, p.hint_a);
              tma_load_2d<CG>(ta, fb, a + 8192, ma + 64, kc, p.hint_a);
            }
            if (g.dbg == 5) {
            } else if (!p.b_mn) {
              if (BN_MAX > SLOT_W && p.bn > SLOT_W) {
                // two MMAs of N = SLOT_W: this CTA holds columns [SLOT_W*h + rank*SLOT_W/CG, +SLOT_W/CG) of MMA h
                const int tn = t.n_blk * p.bn + (int)rank * (SLOT_W / CG);
                tma_load_2d<CG>(tb, fb, b, kcb, tn, p.hint_b);
                if (nh == 2) tma_load_2d<CG>(tb, fb, b + kBHalf, kcb, tn + SLOT_W, p.hint_b);
              } else {
                tma_load_2d<CG>(tb, fb, b, kcb, n0, p.hint_b);
              }
            } else if (p.b_3d) {
              tma_load_3d<CG>(tb, fb, b, 0, kcb, n0 / cw, p.hint_b);
            } else {
              for (int h = 0; h < nb / cw; ++h) tma_load_2d<CG>(tb, fb, b + h * cb, n0 + cw * h, kcb, p.hint_b);
            }
          }
        }
        __syncwarp();
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (g.trace && lane == 0) g.trace[8 * u + 2] = globaltimer();
    }
  };
  auto run_mma = [&]() __attribute__((always_inline)) {
    // ------------------------------------------------------------- MMA issuer
    // Whole warp in the loop so descriptors live in uniform registers; one elected
    // lane issues tcgen05.mma / tcgen05.commit.
    int stage = 0;
    uint32_t phase = 0;
    int sc = 0;                  // accumulator slots handed out so far (slot = sc & 1)
    uint32_t use0 = 0, use1 = 0;  // uses of slot 0 / 1 (mbarrier phase parity)
    for (int it = 0;; ++it) {
      const int u = unit_of(g, group, ngroups, it);
      if (u < 0) break;
      const Unit t = decode_unit(g, u);
      const Prob& p = g.p[t.prob];
      const ProbX& px = g.px[t.prob];
      const int kb0 = t.split * p.kb_per_split;
      const int kb1 = min(p.nk1, kb0 + p.kb_per_split);
      const int nmain = kb1 - kb0;
      const int nkb = nmain + (t.split == 0 ? p.nk2 : 0);
      // snake: every other round of this CTA walks K backwards, starting where the data it
      // (and its neighbours) just streamed is still in L2
      const bool rev = p.snake && (it & 1);
      const int nh = BN_MAX > SLOT_W ? unit_halves(p, t.n_blk, SLOT_W) : 1;
      const bool fp8_tail = kFp8Tail && px.tail_fp8;
      const int s0 = sc & 1;
      mbar_wait(&tempty[s0], ((s0 ? use1 : use0) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + (uint32_t)(s0 * SLOT_W);
      const uint32_t d_tmem1 = tmem_base + (uint32_t)((s0 ^ 1) * SLOT_W);
      const uint32_t a_step = p.a_mn ? 2048u : 32u;
      const uint32_t b_swz = p.b_mn ? (uint32_t)p.b_swz : 128u;
      const uint32_t b_step = p.b_mn ? 16u * b_swz : 32u;
      const uint64_t a_hi = smem_desc(0, p.a_mn ? 8192 : 16, 1024, 2u);
      const uint64_t b_hi = smem_desc(0, p.b_mn ? 64u * b_swz : 16u, 8u * b_swz, sw_layout_code(b_swz));
      // MMAs of k-block group i0 from ring slot st for the halves in hmask (bit h: MMA h)
      auto issue = [&](int st, int i0, int hmask) {
        const int natoms = min(KS, nkb - i0);
        for (int at = 0; at < natoms; ++at) {
          const int i = i0 + at;
          const int ki = rev ? nmain - 1 - i : i;
          const int kleft = (i < nmain) ? (p.k1 - (kb0 + ki) * kBK) : (p.k2 - (i - nmain) * kBK);
          const int ksteps = min(kBK / 16, (kleft + 15) >> 4);
          const uint32_t a_addr = smem_u32(sA + st * C::A_BYTES + at * C::A_ATOM);
          const uint32_t b_addr = smem_u32(sB + st * C::B_BYTES + at * C::B_ATOM);
          if (fp8_tail && i >= nmain) {
            // 4 K-steps of 32 FP8 elements (32 B along the 128-byte K rows) into the main
            // accumulator (mode 2: columns [128 h, +128)); starts it when there is no main K
            const uint64_t d8 = smem_desc(0, 16u, 1024u, 2u);
            const uint32_t dcol = px.tail_fp8 == 2 ? (uint32_t)(128 * (i - nmain)) : 0u;
            for (int j = 0; j < 4; ++j)
              umma_f8(d_tmem + dcol, d8 | (uint64_t)(((a_addr + 32 * j) >> 4) & 0x3FFF),
                      d8 | (uint64_t)(((b_addr + 32 * j) >> 4) & 0x3FFF), px.idesc2,
                      (nmain > 0 || j > 0) ? 1u : 0u);
            continue;
          }
          for (int j = 0; j < (g.dbg == 2 ? 0 : ksteps); ++j) {
            const uint64_t ad = a_hi | (uint64_t)(((a_addr + j * a_step) >> 4) & 0x3FFF);
            if (hmask & 1) {
              const uint64_t bd = b_hi | (uint64_t)(((b_addr + j * b_step) >> 4) & 0x3FFF);
              umma_f16<CG>(d_tmem, ad, bd, p.idesc, (i > 0 || j > 0) ? 1u : 0u);
            }
            if (BN_MAX > SLOT_W && (hmask & 2)) {
              const uint64_t bd1 = b_hi | (uint64_t)(((b_addr + kBHalf + j * b_step) >> 4) & 0x3FFF);
              umma_f16<CG>(d_tmem1, ad, bd1, p.idesc, (i > 0 || j > 0) ? 1u : 0u);
            }
          }
        }
      };
      int i_start = 0;
      if (BN_MAX > SLOT_W && nh == 2) {
        // Second slot still draining (the previous wide tile's epilogue releases slot s0
        // first): run MMA 0 alone on up to STAGES k-blocks, holding their ring slots, then
        // catch MMA 1 up on them once its slot is free.
        const uint32_t par1 = (((s0 ^ 1) ? use1 : use0) & 1) ^ 1;
        const int st0 = stage;
        int npre = 0;
        while (npre < STAGES && npre * KS < nkb) {
          const bool free1 = __shfl_sync(0xffffffffu, mbar_test(&tempty[s0 ^ 1], par1) ? 1 : 0, 0) != 0;
          if (free1) break;
          if (g.dbg != 1 && g.dbg != 3 && g.dbg != 4) mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (elect_one_sync()) issue(stage, npre * KS, 1);
          __syncwarp();
          ++npre;
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        mbar_wait(&tempty[s0 ^ 1], par1);
        tc_fence_after();
        for (int q2 = 0; q2 < npre; ++q2) {
          const int st = (st0 + q2) % STAGES;
          if (elect_one_sync()) {
            issue(st, q2 * KS, 2);
            umma_commit<CG>(&empty[st]);
          }
          __syncwarp();
        }
        i_start = npre * KS;
      }
      // 512-wide tile: its last `endj` k-blocks run MMA 0 first and hand slot s0 to the
      // epilogue, then MMA 1 on the same (held) ring slots — the epilogue reads slot s0 while
      // the tensor core finishes slot s0 ^ 1
      const int endj = (BN_MAX > SLOT_W && nh == 2 && KS == 1 && nkb - i_start > g.endj) ? g.endj : 0;
      for (int i0 = i_start; i0 < nkb - endj; i0 += KS) {
        if (g.dbg != 1 && g.dbg != 3 && g.dbg != 4) mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (elect_one_sync()) {
          issue(stage, i0, nh == 2 ? 3 : 1);
          umma_commit<CG>(&empty[stage]);  // frees the smem slot(s) when these MMAs retire
        }
        __syncwarp();
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (BN_MAX > SLOT_W && endj > 0) {
        const int st0 = stage;
        for (int j = 0; j < endj; ++j) {
          if (g.dbg != 1 && g.dbg != 3 && g.dbg != 4) mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (elect_one_sync()) issue(stage, nkb - endj + j, 1);
          __syncwarp();
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (elect_one_sync()) umma_commit<CG>(&tfull[s0]);
        __syncwarp();
        for (int j = 0; j < endj; ++j) {
          const int st = (st0 + j) % STAGES;
          if (elect_one_sync()) {
            issue(st, nkb - endj + j, 2);
            umma_commit<CG>(&empty[st]);
          }
          __syncwarp();
        }
        if (elect_one_sync()) umma_commit<CG>(&tfull[s0 ^ 1]);
        __syncwarp();
      } else {
        if (elect_one_sync()) {  // accumulator(s) ready for the epilogue(s)
          umma_commit<CG>(&tfull[s0]);
          if (nh == 2) umma_commit<CG>(&tfull[s0 ^ 1]);
        }
        __syncwarp();
      }
      for (int h = 0; h < nh; ++h) {
        if (s0 ^ h) ++use1;
        else ++use0;
      }
      sc += nh;
    }
  };
  auto run_side = [&]() __attribute__((always_inline)) {
    // ----------------------------------------------- side job of the idle warps
    if (g.xdesc) {
      XSlabs S;
      for (int j = 0; j < 2; ++j) {
        S.P[j] = g.side[j].P;
        S.split_stride[j] = g.side[j].split_stride;
        S.ldp[j] = g.side[j].ldp;
        S.ldo[j] = g.side[j].ldo;
        S.out[j] = g.side[j].out;
        S.splits[j] = g.side[j].splits;
      }
      S.out_bf16 = g.side[0].out_bf16;
      S.accumulate = g.side[0].accumulate;
      exchange_run(*g.xdesc, S, g.xepoch, threadIdx.x - 64, blockIdx.x, gridDim.x);
    } else {
      side_reduce(g, (long long)blockIdx.x * 64 + (threadIdx.x - 64), (long long)gridDim.x * 64);
    }
  };
  auto run_epilogue = [&]() __attribute__((always_inline)) {
    // --------------------------------------------------------------- epilogue
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int ew = warp - 4;  // epilogue warp: staging buffers; with 8 warps, ew >> 2 = column half
    constexpr int kEpiStep = C::EPI_WARPS / 4;
    const int hp = C::EPI_WARPS == 8 ? ew >> 2 : 0;
    int it = 0;
    int st_it = 0;  // EPI = 3: TMA stores issued by this warp
    int sc = 0;     // accumulator slots consumed (same sequence as the MMA issuer)
    uint32_t use0 = 0, use1 = 0;
    for (;; ++it) {
      const int u = unit_of(g, group, ngroups, it);
      if (u < 0) break;
      const Unit t = decode_unit(g, u);
      const Prob& p = g.p[t.prob];
      const ProbX& px = g.px[t.prob];
      const int m0 = t.m_blk * (kBM * CG) + rank * kBM;
      const int n0 = t.n_blk * p.bn;
      const int row = (g.dbg == 3) ? 0x7fffffff : m0 + q * 32 + lane;
      const int nh = BN_MAX > SLOT_W ? unit_halves(p, t.n_blk, SLOT_W) : 1;
      if constexpr (C::WIDE_HOLD) {
        if (nh == 2 && g.dbg != 4) {
          // 512-wide tile, 8 warps: this warp reads columns [128 hp, +128) of slot A (tile
          // columns [0, 256)) and of slot B (tile columns [256, 512)) into registers as bf16,
          // releasing each slot as soon as it is read; the stores follow while the next
          // tile's MMAs run.
          const int sA = sc & 1, sB = sA ^ 1;
          uint8_t* stg = smem + STAGES * C::STAGE_BYTES + ew * (C::STG_BUFS * 4096);
          const CUtensorMap* dmap = &tm.m[t.prob][4];
          const uint32_t t_lane = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + (uint32_t)(128 * hp);
          uint32_t held[4][32];  // [slot A c0, c1, slot B c0, c1] x 64 columns, bf16 pairs
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int sl = h ? sB : sA;
            mbar_wait(&tfull[sl], (sl ? use1 : use0) & 1);
            tc_fence_after();
#pragma unroll
            for (int c = 0; c < 2; ++c) {
              uint32_t v[2][32];
              tmem_ld_32x32b_x32(t_lane + (uint32_t)(sl * SLOT_W + 64 * c), v[0]);
              tmem_ld_32x32b_x32(t_lane + (uint32_t)(sl * SLOT_W + 64 * c + 32), v[1]);
              tmem_ld_wait();
              reg_fence32(v[0]);
              reg_fence32(v[1]);
#pragma unroll
              for (int x = 0; x < 32; ++x)
                held[2 * h + c][x] = pack_bf16x2(__uint_as_float(v[x >> 4][2 * (x & 15)]),
                                                 __uint_as_float(v[x >> 4][2 * (x & 15) + 1]));
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_remote<CG>(&tempty[sl], 0);
            if (sl) ++use1;
            else ++use0;
          }
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int col = n0 + (c >> 1) * SLOT_W + 128 * hp + 64 * (c & 1);
            if (col < p.N && g.dbg != 3 && g.dbg != 8)
              stage_store_packed<C::STG_BUFS>(held[c], stg, st_it, lane, dmap, col, m0 + q * 32);
          }
          sc += 2;
          if (g.trace && threadIdx.x == 4 * 32) g.trace[8 * u + 3] = globaltimer();
          continue;
        }
      }
      for (int h = 0; h < nh; ++h) {  // slot by slot: the first is released while the second drains
        const int sl = (sc & 1) ^ h;
        mbar_wait(&tfull[sl], (sl ? use1 : use0) & 1);
        tc_fence_after();
        const uint32_t t_row = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + (uint32_t)(sl * SLOT_W);
        const int bw = min(p.bn - h * SLOT_W, SLOT_W);  // columns of this slot
        const int nc = n0 + h * SLOT_W;                 // their first output column
        if (g.dbg == 4) {
        } else if (EPI == 3) {
          // bf16 tile -> per-warp swizzled smem staging -> TMA store (coalesced full-line
          // writes; rows >= M / cols >= N are clipped by the tensor map bounds).  64-column
          // chunks, STG_BUFS staging tiles per warp: a buffer is reused only after the store
          // issued STG_BUFS chunks earlier has finished reading it.
          uint8_t* stg = smem + STAGES * C::STAGE_BYTES + ew * (C::STG_BUFS * 4096);
          const int nch = min(bw, p.N - nc + 63) / 64;  // 64-column chunks inside N
          const CUtensorMap* dmap = &tm.m[t.prob][4];
#pragma unroll 1
          for (int i = hp; i < nch; i += kEpiStep) {
            uint32_t v[2][32];
            tmem_ld_32x32b_x32(t_row + 64 * i, v[0]);
            tmem_ld_32x32b_x32(t_row + 64 * i + 32, v[1]);
            tmem_ld_wait();
            reg_fence32(v[0]);
            reg_fence32(v[1]);
            stage_store_chunk<C::STG_BUFS>(v, stg, st_it, lane, dmap, nc + 64 * i, m0 + q * 32);
          }
        } else if (CG == 1 && p.out_mode == OUT_F32_FOLD) {  // token reductions only (single-CTA kernels)
          // sum of the fold column blocks (w = fold_w in {8, 16, 32, 64}), in block order
          float o[64];
#pragma unroll
          for (int x = 0; x < 64; ++x) o[x] = 0.f;
          const int w = p.fold_w;
#pragma unroll 1
          for (int c = 0; c < bw; c += 32) {
            uint32_t v[32];
            const bool full32 = bw - c >= 32;
            if (full32) tmem_ld_32x32b_x32(t_row + c, v);
            else tmem_ld_32x32b_x16(t_row + c, v);
            tmem_ld_wait();
            if (w == 64) {  // 32-column chunk c/32 is half (c/32) & 1 of its 64-wide block
              if ((c & 32) == 0) {
#pragma unroll
                for (int x = 0; x < 32; ++x) o[x] += __uint_as_float(v[x]);
              } else {
#pragma unroll
                for (int x = 0; x < 32; ++x) o[32 + x] += __uint_as_float(v[x]);
              }
            } else if (w == 32) {
#pragma unroll
              for (int x = 0; x < 32; ++x) o[x] += __uint_as_float(v[x]);
            } else if (w == 16) {
#pragma unroll
              for (int x = 0; x < 16; ++x) o[x] += __uint_as_float(v[x]);
              if (full32) {
#pragma unroll
                for (int x = 0; x < 16; ++x) o[x] += __uint_as_float(v[16 + x]);
              }
            } else {
#pragma unroll
              for (int b8 = 0; b8 < 4; ++b8) {
                if (b8 >= 2 && !full32) break;
#pragma unroll
                for (int x = 0; x < 8; ++x) o[x] += __uint_as_float(v[8 * b8 + x]);
              }
            }
          }
          if (row < p.M) {
            float* dst = static_cast<float*>(p.D) + t.split * p.split_stride + (long long)row * p.ldd;
#pragma unroll
            for (int e = 0; e < 16; ++e)
              if (4 * e < w) *reinterpret_cast<float4*>(dst + 4 * e) = make_float4(o[4 * e], o[4 * e + 1], o[4 * e + 2], o[4 * e + 3]);
          }
        } else if (bw % 32 == 0) {
#pragma unroll 1
          for (int c = 0; c < bw; c += 32) {
            if (nc + c >= p.N) break;  // warp-uniform
            uint32_t v[32];
            tmem_ld_32x32b_x32(t_row + c, v);
            tmem_ld_wait();
            if (row < p.M) store_row_segment(p, t.split, row, nc + c, v, 32);
          }
        } else {
#pragma unroll 1
          for (int c = 0; c < bw; c += 16) {
            if (nc + c >= p.N) break;
            uint32_t v[32];
            tmem_ld_32x32b_x16(t_row + c, v);
            tmem_ld_wait();
            if (row < p.M) store_row_segment(p, t.split, row, nc + c, v, 16);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote<CG>(&tempty[sl], 0);  // leader's barrier
        if (sl) ++use1;
        else ++use0;
      }
      sc += nh;
      if (kFixup && px.fixup) {
        // split-K fix-up: count this split's arrival at its output tile once all 128 rows of
        // the slab are stored; the last split to arrive reduces the tile (after the loop)
        __threadfence();
        epi_bar();
        if (threadIdx.x == 4 * 32 &&
            atomicAdd(&px.counters[t.m_blk * p.num_n_tiles + t.n_blk], 1) == p.num_splits - 1)
          fx_list[(*fx_count)++] = (t.prob << 24) | (t.n_blk << 16) | t.m_blk;
      }
      if (g.trace && threadIdx.x == 4 * 32) g.trace[8 * u + 3] = globaltimer();
    }
    if constexpr (EPI == 3) {
      if (lane == 0) bulk_wait_all();  // stores complete before the CTA retires
      __syncwarp();
    }
    if constexpr (kFixup) {
      epi_bar();
      const int nfx = *fx_count;
      if (nfx > 0) {
        __threadfence();  // the other splits' slab rows (fenced before their arrival counts)
        for (int f = 0; f < nfx; ++f) {
          const int e = fx_list[f];
          const Prob& p = g.p[e >> 24];
          const ProbX& px = g.px[e >> 24];
          const int m_blk = e & 0xFFFF, n_blk = (e >> 16) & 0xFF;
          split_fixup(p, px, m_blk * kBM + q * 32 + lane, n_blk);
        }
      }
    }
  };
  if constexpr (C::WIDE_HOLD) {
    // 384 threads x 168 registers: warp group 0 gives registers to the two epilogue warp
    // groups (held tile + staging); the reallocation opens each branch so that the compiler
    // allocates each region against its own limit
    if (warp < 4) {
      setmaxnreg_dec<kWideRegsLow>();
      if (warp == 0) run_producer();
      else if (warp == 1 && leader) run_mma();
      else if (kSide && (warp == 2 || warp == 3) && g.nside > 0) run_side();
    } else {
      setmaxnreg_inc<kWideRegsHigh>();
      run_epilogue();
    }
  } else {
    if (warp == 0) run_producer();
    else if (warp == 1 && leader) run_mma();
    else if (kSide && (warp == 2 || warp == 3) && g.nside > 0) run_side();
    else if (warp >= 4) run_epilogue();
  }
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync();
  else __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<CG>(tmem_base, C::TMEM_COLS);
  }
  if (ctrace && threadIdx.x == 64) ctrace[2] = globaltimer();
  if (threadIdx.x == 64) ltrace_mark(g.ltrace, 2);
}

}  // namespace runlora
