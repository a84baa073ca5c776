// Quantized frozen weight (QLoRA-style; format:
// DESIGN.md reading R18): W ≈ scale[j] · e4m3(Wq[i, j]) with one fp32 scale per output
// column.  Three HBM-bound kernels:
//   colmax      scale[j] <- bits of max_i |W[i, j]|           (atomicMax on non-negative floats)
//   quantize    Wq[i, j] = e4m3_rn_satfinite(W[i, j] / s[j]),  s[j] = amax > 0 ? amax/448 : 1
//   finalize    scale[j] <- s[j]
// The way back, W~[i, j] = bf16_rn(fp32(e4m3(Wq[i, j])) · scale[j]), is not a kernel of its own:
// the tcgen05 GEMM's FP8 identity tail does it inside the W' / W'ᵀ / W~ builds (runlora.cu
// wprime_q, tc_gemm.cuh Prob::tail_fp8).
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_fp8.h>

#include "internal.h"
#include "ptx.cuh"

namespace runlora {
namespace {

__device__ __forceinline__ float col_scale(float amax) { return amax > 0.f ? __fdiv_rn(amax, 448.f) : 1.f; }

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

cudaError_t launch_quantize_w(Ctx& ctx, const void* W, int64_t k, int64_t m, void* Wq, float* scale, cudaStream_t s) {
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
  return launch(ctx, KID_QUANT, finalize_scale_kernel, dim3(cols), s, scale, m);
}

}  // namespace runlora
