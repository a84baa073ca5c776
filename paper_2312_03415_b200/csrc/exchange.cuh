// Fused adapter-gradient exchange: the data-parallel
// allreduce of the packed fp32 adapter gradients issued from the reduction of their own
// token-split slabs, by the idle warps 2-3 of the dX GEMM launch — so the exchange over
// NVLink overlaps the GEMM's mainloop, with no NCCL kernel and no extra launch.
//
// dA = Xᵀ·dY·Bᵀ and dB = Aᵀ·Xᵀ·dY are sums over tokens (Eq. 3), so with the
// tokens sharded over P ranks the full-batch gradient is the sum of the ranks' partial sums.
// Per chunk of 64 gradient rows (rows [0, k) are dA, rows [k, k+m) are dBᵀ; r columns each):
//   1. fixed-order sum of this rank's token-split slabs -> this rank's exchange buffer
//      (half epoch & 1, so a slow peer can still read the previous step's half);
//   2. release: the chunk's flag in EVERY rank's flag array <- epoch (peer stores);
//   3. acquire: wait until all P ranks' flags for the chunk reached epoch;
//   4. rank-order sum of the P ranks' chunks (peer loads, NVLink), or one switch-side
//      reduction multimem.ld_reduce over the buffers' multicast address (NVLS);
//   5. write dA / dB (dB transposed back), fp32 or bf16, = or +=.
// With peer loads the result is bit-identical on every rank and run to run (fixed order).
// Deadlock freedom: every chunk's CTA is resident (persistent launches) on every rank, and a
// chunk's publication (1, 2) never waits on anything.
#pragma once
#include <cstdint>
#include <cuda_bf16.h>

namespace runlora {

constexpr int kXMaxPeers = 16;
constexpr int kXChunkRows = 64;

// Device-resident descriptor of one rank's view of the exchange (runlora_exchange_create).
struct XDesc {
  int P, rank;
  int rows0, rows1, cols;          // k, m, r
  long long half_elems;            // floats per epoch half of an exchange buffer
  float* bufs[kXMaxPeers];         // each rank's exchange buffer, as mapped in this process
  unsigned* flags[kXMaxPeers];     // each rank's flag array [chunks][P]
  float* mc;                       // multicast address of the buffers (nullptr: peer loads)
};

__device__ __forceinline__ void x_bar() { asm volatile("bar.sync 2, 64;" ::: "memory"); }

__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ float4 ld_relaxed_sys_v4(const float* p) {
  float4 v;
  asm volatile("ld.relaxed.sys.global.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ float4 multimem_ld_reduce_v4(const float* p) {
  float4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p)
               : "memory");
  return v;
}

// Local slabs of the two gradient parts: fp32 [splits][rows][ldp], the first `cols` columns.
struct XSlabs {
  const float* P[2];
  long long split_stride[2], ldp[2], ldo[2];
  void* out[2];
  int splits[2];
  int out_bf16, accumulate;
};

__device__ __forceinline__ void x_store(const XSlabs& S, int part, int i, int c, float v) {
  const long long o = part == 0 ? (long long)i * S.ldo[0] + c : (long long)c * S.ldo[1] + i;  // dB transposed
  if (S.out_bf16) {
    __nv_bfloat16* d = static_cast<__nv_bfloat16*>(S.out[part]) + o;
    if (S.accumulate) v += __bfloat162float(*d);
    *d = __float2bfloat16_rn(v);
  } else {
    float* d = static_cast<float*>(S.out[part]) + o;
    if (S.accumulate) v += *d;
    *d = v;
  }
}

// One rank's exchange, by 64 threads (tid) of each of `ncta` CTAs (cta).
__device__ __forceinline__ void exchange_run(const XDesc& X, const XSlabs& S, unsigned epoch, int tid, int cta,
                                             int ncta) {
  const int rows = X.rows0 + X.rows1, cols = X.cols;
  const int chunks = (rows + kXChunkRows - 1) / kXChunkRows;
  const long long hoff = (long long)(epoch & 1u) * X.half_elems;
  float* mine = X.bufs[X.rank] + hoff;
  for (int c = cta; c < chunks; c += ncta) {
    const int row = c * kXChunkRows + tid;
    const int part = row < X.rows0 ? 0 : 1;
    const int i = part == 0 ? row : row - X.rows0;
    // 1. this rank's partial: fixed split order
    if (row < rows) {
      const float* src = S.P[part] + (long long)i * S.ldp[part];
      for (int c4 = 0; c4 < cols; c4 += 4) {
        float4 acc = __ldcg(reinterpret_cast<const float4*>(src + c4));
        for (int s = 1; s < S.splits[part]; ++s) {
          const float4 v = __ldcg(reinterpret_cast<const float4*>(src + s * S.split_stride[part] + c4));
          acc.x += v.x, acc.y += v.y, acc.z += v.z, acc.w += v.w;
        }
        *reinterpret_cast<float4*>(mine + (long long)row * cols + c4) = acc;
      }
    }
    x_bar();
    // 2./3. publish the chunk to every rank, then wait for every rank's
    if (tid == 0) {
      __threadfence_system();
      for (int q = 0; q < X.P; ++q) st_release_sys(X.flags[q] + (long long)c * X.P + X.rank, epoch);
      for (int q = 0; q < X.P; ++q) {
        const unsigned* f = X.flags[X.rank] + (long long)c * X.P + q;
        while ((int)(ld_acquire_sys(f) - epoch) < 0) __nanosleep(64);
      }
    }
    x_bar();
    // 4./5. the sum over ranks, in rank order (or the switch's reduction)
    if (row < rows) {
      for (int c4 = 0; c4 < cols; c4 += 4) {
        const long long e = hoff + (long long)row * cols + c4;
        float4 acc;
        if (X.mc) {
          acc = multimem_ld_reduce_v4(X.mc + e);
        } else {
          acc = ld_relaxed_sys_v4(X.bufs[0] + e);
          for (int q = 1; q < X.P; ++q) {
            const float4 v = ld_relaxed_sys_v4(X.bufs[q] + e);
            acc.x += v.x, acc.y += v.y, acc.z += v.z, acc.w += v.w;
          }
        }
        x_store(S, part, i, c4, acc.x);
        x_store(S, part, i, c4 + 1, acc.y);
        x_store(S, part, i, c4 + 2, acc.z);
        x_store(S, part, i, c4 + 3, acc.w);
      }
    }
  }
}

}  // namespace runlora
