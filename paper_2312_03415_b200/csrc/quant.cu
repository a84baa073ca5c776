// Quantized frozen weight (QLoRA-style; format:
// DESIGN.md reading R18): W ≈ 2^e[j] · e4m3(Wq[i, j]) with one power-of-two scale per output
// column.  Four HBM-bound kernels:
//   colmax      amax[j] <- bits of max_i |W[i, j]|          (atomicMax on non-negative floats)
//   quantize    Wq[i, j] = e4m3_rn_satfinite(W[i, j] / 2^e[j]),
//               e[j] = clamp(ceil(log2(amax_j / 448)), -16, 15) (0 for an all-zero column)
//   finalize    scale[j] <- 2^e[j]
//   diagonal    D[j, c] = (c == j mod 128) ? e5m2(2^e[j]) : 0     (m x 128 bytes)
// The way back, W~ = e4m3(Wq) · 2^e (exact), is not a kernel of its own: the tcgen05 GEMM
// multiplies Wq by the E5M2 diagonal D in its FP8 tail (runlora.cu wprime_q, tc_gemm.cuh
// Prob::tail_fp8), inside the W' / W'ᵀ / W~ builds.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_fp8.h>

#include "internal.h"
#include "ptx.cuh"

namespace runlora {
namespace {

// e = clamp(ceil(log2(fp32(amax / 448))), -16, 15), 0 for amax = 0 (oracle/quant.py scale_exponent)
__device__ __forceinline__ int scale_exp(float amax) {
  if (!(amax > 0.f)) return 0;
  int e;
  const float m = frexpf(__fdiv_rn(amax, 448.f), &e);  // x = m · 2^e, m in [0.5, 1)
  const int c = m == 0.5f ? e - 1 : e;
  return c < -16 ? -16 : c > 15 ? 15 : c;
}
__device__ __forceinline__ float col_scale(float amax) { return __int_as_float((scale_exp(amax) + 127) << 23); }

// grid (ceil(m/256), row_splits): thread = one column, a strided share of the rows
__global__ void __launch_bounds__(256) colmax_kernel(const __nv_bfloat16* __restrict__ W, int64_t k, int64_t m,
                                                     unsigned* __restrict__ amax_bits) {
  pdl_wait();
  pdl_launch_dependents();
  const int64_t j = blockIdx.x * 256ll + threadIdx.x;
  if (j >= m) return;
  float a = 0.f;
  for (int64_t i = blockIdx.y; i < k; i += gridDim.y) a = fmaxf(a, fabsf(__bfloat162float(W[i * m + j])));
  atomicMax(amax_bits + j, __float_as_uint(a));  // non-negative floats order like their bits
}

// 8 consecutive elements of a row per thread
__global__ void __launch_bounds__(256) quantize_kernel(const __nv_bfloat16* __restrict__ W, int64_t k, int64_t m,
                                                       const unsigned* __restrict__ amax_bits, uint8_t* __restrict__ Wq) {
  pdl_wait();
  pdl_launch_dependents();
  const int64_t groups = m / 8, total = k * groups;
  for (int64_t g = blockIdx.x * 256ll + threadIdx.x; g < total; g += (int64_t)gridDim.x * 256) {
    const int64_t i = g / groups, j0 = (g % groups) * 8;
    const uint4 raw = *reinterpret_cast<const uint4*>(W + i * m + j0);
    const __nv_bfloat16* w = reinterpret_cast<const __nv_bfloat16*>(&raw);
    uint8_t q[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float s = col_scale(__uint_as_float(amax_bits[j0 + e]));
      q[e] = (uint8_t)__nv_cvt_float_to_fp8(__fdiv_rn(__bfloat162float(w[e]), s), __NV_SATFINITE, __NV_E4M3);
    }
    *reinterpret_cast<uint2*>(Wq + i * m + j0) = *reinterpret_cast<const uint2*>(q);
  }
}

__global__ void __launch_bounds__(256) finalize_scale_kernel(float* __restrict__ scale, int64_t m) {
  pdl_wait();
  pdl_launch_dependents();
  const int64_t j = blockIdx.x * 256ll + threadIdx.x;
  if (j < m) scale[j] = col_scale(scale[j]);  // amax bits (as float) -> scale
}

// m rows of 128 bytes; thread = 16 bytes of a row: zeros except the E5M2 code of 2^e[j] at
// column j mod 128 (e5m2: bias 15, 2 mantissa bits; 2^-15 and 2^-16 are subnormals)
__global__ void __launch_bounds__(256) diag_kernel(const float* __restrict__ scale, int64_t m, uint4* __restrict__ D) {
  pdl_wait();
  pdl_launch_dependents();
  const int64_t total = m * 8;
  for (int64_t t = blockIdx.x * 256ll + threadIdx.x; t < total; t += (int64_t)gridDim.x * 256) {
    const int64_t j = t >> 3;
    const int c0 = (int)(t & 7) * 16, cj = (int)(j & 127);
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (cj >= c0 && cj < c0 + 16) {
      const int e = (int)((__float_as_uint(scale[j]) >> 23) & 0xFF) - 127;
      const uint32_t code = e >= -14 ? (uint32_t)(e + 15) << 2 : e == -15 ? 0x02u : 0x01u;
      uint32_t w[4] = {0u, 0u, 0u, 0u};
      w[(cj - c0) >> 2] = code << (8 * ((cj - c0) & 3));
      v = make_uint4(w[0], w[1], w[2], w[3]);
    }
    D[t] = v;
  }
}

template <typename... KArgs, typename... Args>
cudaError_t launch(Ctx& ctx, KernelId kid, void (*kern)(KArgs...), dim3 grid, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = ctx.pdl() ? 1 : 0;
  ctx.launch_begin(s, kid);
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
  ctx.launch_end(s);
  return e;
}

unsigned elem_blocks(Ctx& ctx, int64_t total_threads) {
  // one resident wave (4 blocks of 256 threads per SM, any register count up to 64), grid-stride beyond it
  const int64_t b = (total_threads + 255) / 256, cap = (int64_t)ctx.num_sms() * 4;
  return (unsigned)(b < cap ? (b > 0 ? b : 1) : cap);
}

}  // namespace

cudaError_t launch_quantize_w(Ctx& ctx, const void* W, int64_t k, int64_t m, void* Wq, float* scale, void* diag,
                              cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(scale, 0, sizeof(float) * m, s);
  if (e != cudaSuccess) return e;
  const unsigned cols = (unsigned)((m + 255) / 256);
  const unsigned splits = (unsigned)std::max<int64_t>(1, std::min<int64_t>(k, (ctx.num_sms() * 8 + cols - 1) / cols));
  e = launch(ctx, KID_QUANT, colmax_kernel, dim3(cols, splits), s, static_cast<const __nv_bfloat16*>(W), k, m,
             reinterpret_cast<unsigned*>(scale));
  if (e != cudaSuccess) return e;
  e = launch(ctx, KID_QUANT, quantize_kernel, dim3(elem_blocks(ctx, k * (m / 8))), s,
             static_cast<const __nv_bfloat16*>(W), k, m, reinterpret_cast<const unsigned*>(scale),
             static_cast<uint8_t*>(Wq));
  if (e != cudaSuccess) return e;
  e = launch(ctx, KID_QUANT, finalize_scale_kernel, dim3(cols), s, scale, m);
  if (e != cudaSuccess) return e;
  return launch(ctx, KID_QUANT, diag_kernel, dim3(elem_blocks(ctx, m * 8)), s, static_cast<const float*>(scale), m,
                static_cast<uint4*>(diag));
}

}  // namespace runlora
