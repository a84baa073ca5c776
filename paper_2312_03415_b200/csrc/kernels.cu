// Kernel instantiations and launchers: tcgen05 GEMM family, split-K reducer,
// fp32 SIMT GEMM.  See tc_gemm.cuh for the GEMM design.
#include <cuda_bf16.h>

#include <string>

#include "internal.h"
#include "tc_gemm.cuh"

namespace runlora {

const char* const kKernelNames[KID_COUNT] = {
    "gemm_main",      "gemm_wprime", "gemm_proj",        "gemm_tokred",
    "gemm_dense_xtdy", "gemm_small",  "splitk_reduce", "sgemm_f32",
};

namespace {

constexpr int kMaxDevices = 64;

template <int BN, bool AM, bool BM>
cudaError_t run_tc(Ctx& ctx, const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& ta2,
                   const CUtensorMap& tb2, const GemmArgs& g, int units, cudaStream_t s) {
  auto kern = tc_gemm_kernel<BN, AM, BM>;
  static bool attr_set[kMaxDevices] = {};
  const int dev = ctx.device();
  if (dev < kMaxDevices && !attr_set[dev]) {
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TileCfg<BN>::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr_set[dev] = true;
  }
  const int grid = units < ctx.num_sms() ? units : ctx.num_sms();
  kern<<<grid, kGemmThreads, TileCfg<BN>::SMEM_BYTES, s>>>(ta, tb, ta2, tb2, g);
  return cudaGetLastError();
}

template <bool AM, bool BM>
cudaError_t dispatch_bn(Ctx& ctx, int BN, const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& ta2,
                        const CUtensorMap& tb2, const GemmArgs& g, int units, cudaStream_t s) {
  if constexpr (BM) {
    switch (BN) {
      case 64: return run_tc<64, AM, BM>(ctx, ta, tb, ta2, tb2, g, units, s);
      case 128: return run_tc<128, AM, BM>(ctx, ta, tb, ta2, tb2, g, units, s);
      case 256: return run_tc<256, AM, BM>(ctx, ta, tb, ta2, tb2, g, units, s);
      default: return cudaErrorInvalidValue;
    }
  } else {
    switch (BN) {
      case 16: return run_tc<16, AM, BM>(ctx, ta, tb, ta2, tb2, g, units, s);
      case 32: return run_tc<32, AM, BM>(ctx, ta, tb, ta2, tb2, g, units, s);
      case 48: return run_tc<48, AM, BM>(ctx, ta, tb, ta2, tb2, g, units, s);
      case 64: return run_tc<64, AM, BM>(ctx, ta, tb, ta2, tb2, g, units, s);
      case 128: return run_tc<128, AM, BM>(ctx, ta, tb, ta2, tb2, g, units, s);
      case 256: return run_tc<256, AM, BM>(ctx, ta, tb, ta2, tb2, g, units, s);
      default: return cudaErrorInvalidValue;
    }
  }
}

// ------------------------------------------------------------ split-K reduce
__global__ void splitk_reduce_kernel(const float* __restrict__ P, int splits, long long sstride, int rows, int cols,
                                     long long ldp, void* __restrict__ out, int out_bf16, long long ldo,
                                     int transpose, int accumulate) {
  const long long total = (long long)rows * cols;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(idx / cols), j = (int)(idx % cols);
    const float* p = P + (long long)i * ldp + j;
    float acc = 0.f;
    for (int sp = 0; sp < splits; ++sp) acc += p[sp * sstride];  // fixed order: deterministic
    const long long o = transpose ? (long long)j * ldo + i : (long long)i * ldo + j;
    if (out_bf16) {
      __nv_bfloat16* d = static_cast<__nv_bfloat16*>(out) + o;
      if (accumulate) acc += __bfloat162float(*d);
      *d = __float2bfloat16_rn(acc);
    } else {
      float* d = static_cast<float*>(out) + o;
      if (accumulate) acc += *d;
      *d = acc;
    }
  }
}

// ------------------------------------------------------------ fp32 SIMT GEMM
// 64x64 output tile per 256-thread CTA, 4x4 per thread, K step 16; true FP32 FFMA.
__global__ void __launch_bounds__(256) sgemm_kernel(int M, int N, int K, const float* __restrict__ A, long long sa0,
                                                    long long sa1, const float* __restrict__ B, long long sb0,
                                                    long long sb1, float* __restrict__ C, long long ldc,
                                                    const float* __restrict__ Cadd, long long ldadd,
                                                    int accumulate) {
  __shared__ float As[16][64 + 4];
  __shared__ float Bs[16][64 + 4];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
  float c[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += 16) {
    for (int e = threadIdx.x; e < 1024; e += 256) {
      const int i = e >> 4, kk = e & 15;
      const int gi = m0 + i, gk = k0 + kk;
      As[kk][i] = (gi < M && gk < K) ? A[gi * sa0 + gk * sa1] : 0.f;
      const int kb = e >> 6, j = e & 63;
      const int gkb = k0 + kb, gj = n0 + j;
      Bs[kb][j] = (gkb < K && gj < N) ? B[gkb * sb0 + gj * sb1] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        a[x] = As[kk][ty * 4 + x];
        b[x] = Bs[kk][tx * 4 + x];
      }
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) c[x][y] = fmaf(a[x], b[y], c[x][y]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    const int gi = m0 + ty * 4 + x;
    if (gi >= M) continue;
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      const int gj = n0 + tx * 4 + y;
      if (gj >= N) continue;
      float v = c[x][y];
      if (Cadd) v += Cadd[gi * ldadd + gj];
      if (accumulate) v += C[gi * ldc + gj];
      C[gi * ldc + gj] = v;
    }
  }
}

}  // namespace

cudaError_t launch_tc_gemm(Ctx& ctx, const GemmReq& r, cudaStream_t s, std::string* err) {
  CUtensorMap ta, tb, ta2, tb2;
  const int a_box = r.a_mn ? 64 : kBM;
  const int b_box = r.b_mn ? 64 : r.BN;
  if (!ctx.tmap(r.a, a_box, &ta, err) || !ctx.tmap(r.b, b_box, &tb, err)) return cudaErrorInvalidValue;
  if (r.K2 > 0) {
    if (!ctx.tmap(r.a2, a_box, &ta2, err) || !ctx.tmap(r.b2, b_box, &tb2, err)) return cudaErrorInvalidValue;
  } else {
    ta2 = ta;
    tb2 = tb;
  }
  GemmArgs g{};
  g.M = r.M;
  g.N = r.N;
  g.k1 = r.K1;
  g.nk1 = (r.K1 + kBK - 1) / kBK;
  g.k2 = r.K2;
  g.nk2 = r.K2 > 0 ? (r.K2 + kBK - 1) / kBK : 0;
  g.kb_per_split = r.splits > 1 ? r.kb_per_split : g.nk1;
  g.num_m_tiles = (r.M + kBM - 1) / kBM;
  g.num_n_tiles = (r.N + r.BN - 1) / r.BN;
  g.num_splits = r.splits > 1 ? r.splits : 1;
  g.out_mode = r.out_mode;
  g.D = r.D;
  g.ldd = r.ldd;
  g.split_stride = r.split_stride;
  g.Cin = static_cast<const __nv_bfloat16*>(r.Cin);
  g.ldc = r.ldc;
  g.hint_a = r.a_stream_once ? kEvictFirst : kEvictNormal;
  g.hint_b = kEvictLast;
  const int units = g.num_m_tiles * g.num_n_tiles * g.num_splits;
  if (units <= 0) return cudaSuccess;
  ctx.launch_begin(s, r.kid);
  cudaError_t e;
  if (!r.a_mn && !r.b_mn)
    e = dispatch_bn<false, false>(ctx, r.BN, ta, tb, ta2, tb2, g, units, s);
  else if (!r.a_mn && r.b_mn)
    e = dispatch_bn<false, true>(ctx, r.BN, ta, tb, ta2, tb2, g, units, s);
  else if (r.a_mn && r.b_mn)
    e = dispatch_bn<true, true>(ctx, r.BN, ta, tb, ta2, tb2, g, units, s);
  else
    e = cudaErrorNotSupported;  // MN-major A with K-major B is not used by any variant
  ctx.launch_end(s);
  if (e != cudaSuccess && err) *err = std::string("tc_gemm launch: ") + cudaGetErrorString(e);
  return e;
}

cudaError_t launch_splitk_reduce(Ctx& ctx, const float* P, int splits, int64_t split_stride, int rows, int cols,
                                 int64_t ldp, void* out, bool out_bf16, int64_t ldo, bool transpose,
                                 bool accumulate, cudaStream_t s) {
  const long long total = (long long)rows * cols;
  if (total <= 0) return cudaSuccess;
  long long blocks = (total + 255) / 256;
  const long long cap = (long long)ctx.num_sms() * 8;
  if (blocks > cap) blocks = cap;
  ctx.launch_begin(s, KID_SPLITK_REDUCE);
  splitk_reduce_kernel<<<(unsigned)blocks, 256, 0, s>>>(P, splits, split_stride, rows, cols, ldp, out, out_bf16 ? 1 : 0,
                                                        ldo, transpose ? 1 : 0, accumulate ? 1 : 0);
  ctx.launch_end(s);
  return cudaGetLastError();
}

cudaError_t launch_sgemm(Ctx& ctx, int M, int N, int K, const float* A, int64_t sa0, int64_t sa1, const float* B,
                         int64_t sb0, int64_t sb1, float* C, int64_t ldc, const float* Cadd, int64_t ldadd,
                         bool accumulate, cudaStream_t s) {
  dim3 grid((N + 63) / 64, (M + 63) / 64);
  ctx.launch_begin(s, KID_SGEMM_F32);
  sgemm_kernel<<<grid, 256, 0, s>>>(M, N, K, A, sa0, sa1, B, sb0, sb1, C, ldc, Cadd, ldadd, accumulate ? 1 : 0);
  ctx.launch_end(s);
  return cudaGetLastError();
}

}  // namespace runlora
