// tcgen05 / TMEM / TMA GEMM for sm_100a (kernel family K1/K2 of DESIGN.md).
//
//   D[M,N] = A1[M,K1]·B1[K1,N]  (+ A2[M,K2]·B2[K2,N])       (concat-K tail)
//
// bf16 operands, fp32 accumulation in TMEM.  Every product of the paper's
// variants (Eq. 1-3, Alg. 1-5) that runs in bf16 is one launch
// of this template:
//   * Y = [X | XA]·[W ; B]           (forward1 fused)   A K-major, B MN-major
//   * Y = X·(W+AB)                   (forward2)          A K-major, B MN-major
//   * dX = [dY | dYBᵀ]·[Wᵀ ; Aᵀ]     (Alg. 1-3 last line)      A K-major, B K-major
//   * dX = dY·(W+AB)ᵀ                (Alg. 4-5 last line)      A K-major, B K-major
//   * Z = X·A, Z = dY·Bᵀ             (rank-r projections)      N = r (padded)
//   * dA = Xᵀ·Z1, dBᵀ = dYᵀ·Z2       (token reductions, K = n) A and B MN-major, split-K
//   * W+AB                           (K = r, epilogue adds W)
//
// Structure (persistent, warp-specialised, one CTA per SM):
//   warp 0 lane 0 : TMA producer      (smem ring of STAGES {A,B} tiles, mbarrier full/empty)
//   warp 1 lane 0 : tcgen05.mma issuer (single thread, accumulator in TMEM)
//   warp 2        : TMEM allocator (2 accumulators of BN columns: epilogue of tile i
//                   overlaps the mainloop of tile i+1)
//   warps 4..7    : epilogue (tcgen05.ld -> registers -> global), TMEM lanes 32*(w%4)..
// Tiles: BM = 128 rows, BN columns, BK = 64 (one 128-byte swizzle row of bf16).
// Shared-memory tiles use the 128B swizzle written by TMA and read by UMMA:
//   K-major  tile: rows of 128 B (64 K-elements), 8-row atoms of 1024 B  -> SBO = 1024
//   MN-major tile: 64-element MN chunks, each a box of 64 K-rows x 128 B  -> LBO = 8192 (MN chunk
//                  stride), SBO = 1024 (8 K-rows); one UMMA_K=16 step advances 2048 B.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include "ptx.cuh"

namespace runlora {

enum OutMode : int { OUT_BF16 = 0, OUT_BF16_ADD = 1, OUT_F32 = 2 };

struct GemmArgs {
  int M, N;              // output extent (epilogue masks rows >= M, cols >= N)
  int k1, nk1;           // main operand K (elements) and K blocks of 64
  int k2, nk2;           // tail operand K (elements) and K blocks (0 = no tail)
  int kb_per_split;      // main K blocks per split
  int num_m_tiles, num_n_tiles, num_splits;
  int out_mode;          // OutMode
  void* D;               // bf16 [M, ldd] or fp32 partial slabs [split][M][ldd]
  long long ldd;
  long long split_stride;  // elements between fp32 split slabs
  const __nv_bfloat16* Cin;  // OUT_BF16_ADD: added matrix, [M, ldc]
  long long ldc;
  uint64_t hint_a, hint_b;   // TMA L2 cache hints
};

constexpr int kBM = 128;
constexpr int kBK = 64;
constexpr int kGemmThreads = 256;

template <int BN>
struct TileCfg {
  static constexpr uint32_t A_BYTES = kBM * kBK * 2;
  static constexpr uint32_t B_BYTES = BN * kBK * 2;
  static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES_RAW = (200 * 1024) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
  static constexpr uint32_t TMEM_COLS = (2 * BN <= 32) ? 32 : (2 * BN <= 64) ? 64 : (2 * BN <= 128) ? 128
                                        : (2 * BN <= 256) ? 256 : 512;
  static constexpr uint32_t SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
};

struct Unit {
  int m_blk, n_blk, split;
};
__device__ __forceinline__ Unit decode_unit(const GemmArgs& g, int u) {
  Unit t;
  t.n_blk = u % g.num_n_tiles;
  int q = u / g.num_n_tiles;
  t.m_blk = q % g.num_m_tiles;
  t.split = q / g.num_m_tiles;
  return t;
}

template <int CH>
__device__ __forceinline__ void tmem_ld_chunk(uint32_t taddr, uint32_t (&v)[32]);
template <>
__device__ __forceinline__ void tmem_ld_chunk<32>(uint32_t taddr, uint32_t (&v)[32]) {
  tmem_ld_32x32b_x32(taddr, v);
}
template <>
__device__ __forceinline__ void tmem_ld_chunk<16>(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

template <int BN, bool A_MN, bool B_MN>
__global__ void __launch_bounds__(kGemmThreads, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmA2, const __grid_constant__ CUtensorMap tmB2,
                   const GemmArgs g) {
  using C = TileCfg<BN>;
  constexpr int STAGES = C::STAGES;
  constexpr uint32_t IDESC = idesc_bf16(kBM, BN, A_MN, B_MN);
  constexpr int CH = (BN % 32 == 0) ? 32 : 16;
  static_assert(!B_MN || BN % 64 == 0, "MN-major B needs 64-column swizzle chunks");
  static_assert(BN % 16 == 0 && BN >= 16 && BN <= 256, "UMMA N for M=128");

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * C::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * C::B_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    if (g.nk2 > 0) {
      tma_prefetch_desc(&tmA2);
      tma_prefetch_desc(&tmB2);
    }
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int total = g.num_m_tiles * g.num_n_tiles * g.num_splits;

  if (warp == 0 && lane == 0) {
    // ------------------------------------------------------------ TMA producer
    int stage = 0;
    uint32_t phase = 0;
    for (int u = blockIdx.x; u < total; u += gridDim.x) {
      const Unit t = decode_unit(g, u);
      const int m0 = t.m_blk * kBM, n0 = t.n_blk * BN;
      const int kb0 = t.split * g.kb_per_split;
      const int kb1 = min(g.nk1, kb0 + g.kb_per_split);
      const int nmain = kb1 - kb0;
      const int nkb = nmain + (t.split == 0 ? g.nk2 : 0);
      for (int i = 0; i < nkb; ++i) {
        mbar_wait(&empty[stage], phase ^ 1);
        uint8_t* a = sA + stage * C::A_BYTES;
        uint8_t* b = sB + stage * C::B_BYTES;
        mbar_arrive_expect_tx(&full[stage], C::STAGE_BYTES);
        const bool tail = i >= nmain;
        const CUtensorMap* ta = tail ? &tmA2 : &tmA;
        const CUtensorMap* tb = tail ? &tmB2 : &tmB;
        const int kc = (tail ? (i - nmain) : (kb0 + i)) * kBK;
        if constexpr (!A_MN) {
          tma_load_2d(ta, &full[stage], a, kc, m0, g.hint_a);
        } else {
          tma_load_2d(ta, &full[stage], a, m0, kc, g.hint_a);
          tma_load_2d(ta, &full[stage], a + 8192, m0 + 64, kc, g.hint_a);
        }
        if constexpr (!B_MN) {
          tma_load_2d(tb, &full[stage], b, kc, n0, g.hint_b);
        } else {
#pragma unroll
          for (int h = 0; h < BN / 64; ++h) tma_load_2d(tb, &full[stage], b + h * 8192, n0 + 64 * h, kc, g.hint_b);
        }
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ------------------------------------------------------------- MMA issuer
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int u = blockIdx.x; u < total; u += gridDim.x, ++it) {
      const Unit t = decode_unit(g, u);
      const int kb0 = t.split * g.kb_per_split;
      const int kb1 = min(g.nk1, kb0 + g.kb_per_split);
      const int nmain = kb1 - kb0;
      const int nkb = nmain + (t.split == 0 ? g.nk2 : 0);
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      for (int i = 0; i < nkb; ++i) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        const int kleft = (i < nmain) ? (g.k1 - (kb0 + i) * kBK) : (g.k2 - (i - nmain) * kBK);
        const int ksteps = min(kBK / 16, (kleft + 15) >> 4);
        const uint32_t a_addr = smem_u32(sA + stage * C::A_BYTES);
        const uint32_t b_addr = smem_u32(sB + stage * C::B_BYTES);
        for (int j = 0; j < ksteps; ++j) {
          const uint64_t ad = A_MN ? smem_desc_sw128(a_addr + j * 2048, 8192, 1024)
                                   : smem_desc_sw128(a_addr + j * 32, 16, 1024);
          const uint64_t bd = B_MN ? smem_desc_sw128(b_addr + j * 2048, 8192, 1024)
                                   : smem_desc_sw128(b_addr + j * 32, 16, 1024);
          umma_f16(d_tmem, ad, bd, IDESC, (i > 0 || j > 0) ? 1u : 0u);
        }
        umma_commit(&empty[stage]);  // frees the smem slot when these MMAs retire
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      umma_commit(&tfull[acc]);  // accumulator ready for the epilogue
    }
  } else if (warp >= 4) {
    // --------------------------------------------------------------- epilogue
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    int it = 0;
    for (int u = blockIdx.x; u < total; u += gridDim.x, ++it) {
      const Unit t = decode_unit(g, u);
      const int m0 = t.m_blk * kBM, n0 = t.n_blk * BN;
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int row = m0 + q * 32 + lane;
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN;
#pragma unroll 1
      for (int c = 0; c < BN / CH; ++c) {
        const int col = n0 + c * CH;
        if (col >= g.N) break;  // warp-uniform
        uint32_t v[32];
        tmem_ld_chunk<CH>(t_row + c * CH, v);
        tmem_ld_wait();
        if (row < g.M) {
          if (g.out_mode == OUT_F32) {
            float* dst = static_cast<float*>(g.D) + t.split * g.split_stride + (long long)row * g.ldd + col;
#pragma unroll
            for (int e = 0; e < CH / 4; ++e) {
              if (col + 4 * e < g.N) {
                float4 w = make_float4(__uint_as_float(v[4 * e]), __uint_as_float(v[4 * e + 1]),
                                       __uint_as_float(v[4 * e + 2]), __uint_as_float(v[4 * e + 3]));
                *reinterpret_cast<float4*>(dst + 4 * e) = w;
              }
            }
          } else {
            __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(g.D) + (long long)row * g.ldd + col;
            const bool add = g.out_mode == OUT_BF16_ADD;
            const __nv_bfloat16* cin = add ? g.Cin + (long long)row * g.ldc + col : nullptr;
#pragma unroll
            for (int e = 0; e < CH / 8; ++e) {
              if (col + 8 * e < g.N) {
                float f[8];
#pragma unroll
                for (int x = 0; x < 8; ++x) f[x] = __uint_as_float(v[8 * e + x]);
                if (add) {
                  uint4 cv = *reinterpret_cast<const uint4*>(cin + 8 * e);
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
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
}

}  // namespace runlora
