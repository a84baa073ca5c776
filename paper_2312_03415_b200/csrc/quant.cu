// Quantized frozen weight (QLoRA-style; format:
// DESIGN.md reading R18): W ≈ scale[j] · e4m3(Wq[i, j]) with one fp32 scale per output
// column.  Three HBM-bound kernels:
//   colmax      scale[j] <- bits of max_i |W[i, j]|           (atomicMax on non-negative floats)
//   quantize    Wq[i, j] = e4m3_rn_satfinite(W[i, j] / s[j]),  s[j] = amax > 0 ? amax/448 : 1
//   finalize    scale[j] <- s[j]
//   dequantize  W~[i, j] = bf16_rn(fp32(e4m3(Wq[i, j])) · scale[j])   (16 elements per thread)
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

// Each thread owns one group of `per` (16, or 8 when m % 16 != 0) columns — its scales stay
// in registers — and walks the rows with a stride of (threads / column groups).
__global__ void __launch_bounds__(256) dequantize_kernel(const uint8_t* __restrict__ Wq, const float* __restrict__ scale,
                                                         int64_t k, int64_t m, __nv_bfloat16* __restrict__ W,
                                                         unsigned long long* lt) {
  if (threadIdx.x == 0) ltrace_mark(lt, 0);
  pdl_wait();
  pdl_launch_dependents();
  if (threadIdx.x == 0) ltrace_mark(lt, 1);
  const int per = (m & 15) ? 8 : 16;
  const int64_t groups = m / per;
  const int64_t tid = blockIdx.x * 256ll + threadIdx.x, nthr = (int64_t)gridDim.x * 256;
  const int64_t rstride = nthr / groups;
  if (rstride > 0 && tid < rstride * groups) {
    const int64_t j0 = (tid % groups) * per;
    float s[16];
#pragma unroll
    for (int e = 0; e < 16; e += 4) {
      if (e < per) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(scale + j0 + e));
        s[e] = v.x, s[e + 1] = v.y, s[e + 2] = v.z, s[e + 3] = v.w;
      }
    }
    for (int64_t i = tid / groups; i < k; i += rstride) {
      uint8_t q[16];
      if (per == 16) *reinterpret_cast<uint4*>(q) = __ldg(reinterpret_cast<const uint4*>(Wq + i * m + j0));
      else *reinterpret_cast<uint2*>(q) = __ldg(reinterpret_cast<const uint2*>(Wq + i * m + j0));
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (h * 8 >= per) break;
        uint4 out;
        __nv_bfloat162* o = reinterpret_cast<__nv_bfloat162*>(&out);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int c = 8 * h + 2 * e;
          const float x0 = __half2float(__half(__nv_cvt_fp8_to_halfraw(q[c], __NV_E4M3))) * s[c];
          const float x1 = __half2float(__half(__nv_cvt_fp8_to_halfraw(q[c + 1], __NV_E4M3))) * s[c + 1];
          o[e] = __floats2bfloat162_rn(x0, x1);
        }
        *reinterpret_cast<uint4*>(W + i * m + j0 + 8 * h) = out;
      }
    }
  } else if (rstride == 0) {  // more column groups than threads: grid-stride over everything
    for (int64_t g = tid; g < k * groups; g += nthr) {
      const int64_t i = g / groups, j0 = (g % groups) * per;
      for (int e = 0; e < per; ++e) {
        const float x = __half2float(__half(__nv_cvt_fp8_to_halfraw(Wq[i * m + j0 + e], __NV_E4M3))) * scale[j0 + e];
        W[i * m + j0 + e] = __float2bfloat16_rn(x);
      }
    }
  }
  if (threadIdx.x == 0) ltrace_mark(lt, 2);
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

cudaError_t launch_dequantize_w(Ctx& ctx, const void* Wq, const float* scale, int64_t k, int64_t m, void* W,
                                cudaStream_t s) {
  return launch(ctx, KID_DEQUANT, dequantize_kernel, dim3(elem_blocks(ctx, k * (m / ((m & 15) ? 8 : 16)))), s,
                static_cast<const uint8_t*>(Wq), scale, k, m, static_cast<__nv_bfloat16*>(W),
                ctx.ltrace_slot(KID_DEQUANT));
}

}  // namespace runlora
