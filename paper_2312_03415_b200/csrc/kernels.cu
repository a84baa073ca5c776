// Kernel instantiations and launchers: tcgen05 GEMM family, split-K reducer,
// fp32 SIMT GEMM.  See tc_gemm.cuh for the GEMM design.
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "internal.h"
#include "tc_gemm.cuh"

namespace runlora {

const char* const kKernelNames[KID_COUNT] = {
    "gemm_main",      "gemm_wprime", "gemm_proj",        "gemm_tokred",
    "gemm_dense_xtdy", "gemm_small",  "splitk_reduce", "sgemm_f32", "quantize_w", "dequantize_w",
    "allreduce_sum",
};

namespace {

constexpr int kMaxDevices = 64;

// Plain launch with the programmatic-dependent-launch attribute (when enabled).
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(Ctx& ctx, void (*kern)(KArgs...), dim3 grid, dim3 block, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = ctx.pdl() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

template <int BN, int CG, int OCC = 1, int EPI = 0, int KS = 1>
cudaError_t run_tc(Ctx& ctx, const Tmaps& tm, GemmArgs& g, cudaStream_t s, int sms) {
  auto kern = tc_gemm_kernel<BN, CG, OCC, EPI, KS>;
  using TC = TileCfg<BN, CG, OCC, EPI, KS>;
  constexpr uint32_t smem_max = TC::SMEM_BYTES;
  const int stages = (g.stages > 0 && g.stages < TC::STAGES) ? g.stages : TC::STAGES;
  const uint32_t smem = smem_max - (uint32_t)(TC::STAGES - stages) * TC::STAGE_BYTES;
  static bool attr_set[kMaxDevices] = {};
  const int dev = ctx.device();
  if (dev < kMaxDevices && !attr_set[dev]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_max);
    if (e != cudaSuccess) return e;
    // the whole unified L1/shared array as shared memory, so OCC = 2 CTAs are co-resident
    e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
    attr_set[dev] = true;
  }
  int groups_max = sms * OCC / CG;  // persistent grid over the SMs this launch may use
  // debug (env RUNLORA_MAX_CTAS): cap the persistent grid of the non-main kernels, e.g. to
  // measure what a few SMs' worth of CTAs stream
  static const int max_ctas = getenv("RUNLORA_MAX_CTAS") ? atoi(getenv("RUNLORA_MAX_CTAS")) : 0;
  if (max_ctas > 0 && CG == 1 && BN < 256) groups_max = std::min(groups_max, max_ctas);
  const int groups = g.total_units < groups_max ? g.total_units : groups_max;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(groups * CG);
  cfg.blockDim = dim3(TC::THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (CG > 1) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = CG;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  if (ctx.pdl()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, tm, g);
  static const bool dbg_launch = getenv("RUNLORA_DEBUG_LAUNCH") != nullptr;
  if (dbg_launch) {
    int occ = -1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, TC::THREADS, smem);
    fprintf(stderr, "[runlora] tc_gemm<%d,%d,%d,%d,%d> grid %d smem %u occupancy/SM %d units %d: %s\n", BN, CG, OCC,
            EPI, KS, groups * CG, smem, occ, g.total_units, cudaGetErrorString(e));
  }
  return e;
}

cudaError_t dispatch_tc(Ctx& ctx, int bn_max, int cg, bool occ2, bool tma_store, const Tmaps& tm, GemmArgs& g,
                        cudaStream_t s, int sms) {
  if (tma_store) {
    if (cg == 1 && bn_max == 256) return run_tc<256, 1, 1, 3>(ctx, tm, g, s, sms);
    if (cg == 2 && bn_max == 256) return run_tc<256, 2, 1, 3>(ctx, tm, g, s, sms);
    if (cg == 2 && bn_max == 512) return run_tc<512, 2, 1, 3>(ctx, tm, g, s, sms);
    return cudaErrorNotSupported;
  }
  if (cg == 2) {
    // MN-major operands stream through TMA as 3-D boxes: two 64-wide K atoms per stage
    // (half the barrier/TMA-issue round trips) measured 8 % faster for MN-major B
    // (8192x4096x4096: 180 vs 197 µs) and neutral for K-major operands (168 µs both).
    static const int ks_env = getenv("RUNLORA_MAIN_KS") ? atoi(getenv("RUNLORA_MAIN_KS")) : 0;
    const bool ks2 = ks_env ? ks_env == 2 : (g.p[0].a_mn || g.p[0].b_mn);
    if (bn_max == 512) return run_tc<512, 2>(ctx, tm, g, s, sms);
    if (bn_max == 256 && ks2) return run_tc<256, 2, 1, 0, 2>(ctx, tm, g, s, sms);
    if (bn_max == 256) return run_tc<256, 2>(ctx, tm, g, s, sms);
    if (bn_max == 128) return run_tc<128, 2>(ctx, tm, g, s, sms);
    return cudaErrorInvalidValue;
  }
  if (occ2) {
    switch (bn_max) {
      case 16: return run_tc<16, 1, 2>(ctx, tm, g, s, sms);
      case 32: return run_tc<32, 1, 2>(ctx, tm, g, s, sms);
      case 48: return run_tc<48, 1, 2>(ctx, tm, g, s, sms);
      case 64: return run_tc<64, 1, 2>(ctx, tm, g, s, sms);
      case 128: return run_tc<128, 1, 2>(ctx, tm, g, s, sms);
      default: break;
    }
  }
  switch (bn_max) {
    case 16: return run_tc<16, 1>(ctx, tm, g, s, sms);
    case 32: return run_tc<32, 1>(ctx, tm, g, s, sms);
    case 48: return run_tc<48, 1>(ctx, tm, g, s, sms);
    case 64: return run_tc<64, 1>(ctx, tm, g, s, sms);
    case 128: return run_tc<128, 1>(ctx, tm, g, s, sms);
    case 256: return run_tc<256, 1>(ctx, tm, g, s, sms);
    default: return cudaErrorInvalidValue;
  }
}

// ------------------------------------------------------------ split-K reduce
struct ReduceArgs {
  ReduceJob j[2];
  long long total0, total;
  unsigned long long* ltrace;
};

// One thread per (row i, 4-column group): float4 loads of every split slab in fixed
// split order (deterministic), 4 slabs in flight at a time.  Column groups vary fastest
// so a warp reads contiguous 512 B of each slab.
__global__ void __launch_bounds__(256, 4) splitk_reduce_kernel(const __grid_constant__ ReduceArgs a) {
  if (threadIdx.x == 0) ltrace_mark(a.ltrace, 0);
  pdl_wait();
  pdl_launch_dependents();
  if (threadIdx.x == 0) ltrace_mark(a.ltrace, 1);
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < a.total;
       idx += (long long)gridDim.x * blockDim.x) {
    const bool second = idx >= a.total0;
    const ReduceJob& J = a.j[second ? 1 : 0];
    const long long e = second ? idx - a.total0 : idx;
    const int groups = (J.cols + 3) >> 2;
    const int i = (int)(e / groups);
    const int c0 = (int)(e % groups) * 4;
    const float4* p = reinterpret_cast<const float4*>(J.P + (long long)i * J.ldp + c0);
    const long long st4 = J.split_stride / 4;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s0 = 0; s0 < J.splits; s0 += 8) {
      float4 v[8];  // up to 8 slabs in flight, then summed in split order
#pragma unroll
      for (int x = 0; x < 8; ++x)
        if (s0 + x < J.splits) v[x] = __ldg(p + (s0 + x) * st4);
#pragma unroll
      for (int x = 0; x < 8; ++x) {
        if (s0 + x < J.splits) {
          acc.x += v[x].x;
          acc.y += v[x].y;
          acc.z += v[x].z;
          acc.w += v[x].w;
        }
      }
    }
    const float a4[4] = {acc.x, acc.y, acc.z, acc.w};
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      if (c0 + x >= J.cols) break;
      const long long o = J.transpose ? (long long)(c0 + x) * J.ldo + i : (long long)i * J.ldo + c0 + x;
      float v = a4[x];
      if (J.out_bf16) {
        __nv_bfloat16* d = static_cast<__nv_bfloat16*>(J.out) + o;
        if (J.accumulate) v += __bfloat162float(*d);
        *d = __float2bfloat16_rn(v);
      } else {
        float* d = static_cast<float*>(J.out) + o;
        if (J.accumulate) v += *d;
        *d = v;
      }
    }
  }
  if (threadIdx.x == 0) ltrace_mark(a.ltrace, 2);
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
  pdl_wait();
  pdl_launch_dependents();
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

int raster_rows(const GemmReq& r) {
  // Unit order (decode_unit): G = 1 walks row tiles (every column tile of a row band of one
  // tile), G >= the row-tile count walks column tiles, values between walk bands of G row
  // tiles.  env RUNLORA_RASTER_G overrides.
  static const int raster_env = getenv("RUNLORA_RASTER_G") ? atoi(getenv("RUNLORA_RASTER_G")) : 0;
  if (raster_env > 0) return raster_env;
  const double K = (double)(r.K1 + r.K2);
  const double a_bytes = 2.0 * (double)r.M * K, b_bytes = 2.0 * (double)r.N * K;
  if (b_bytes <= 48e6) return 1;  // all of B stays in L2: row order streams A once
  // The main GEMMs keep the SMALLER operand L2-resident and stream the other once: C3's Y
  // GEMM 8192x11008x4096 (A 64 MB, B 90 MB) column order 476 µs vs 482 at G = 16 and 486 in
  // row order; its dX GEMM 8192x4096x11008 (A 180 MB, B 90 MB) row order 449.5 µs vs 455.7
  // at G = 16 (tools/gemm_bench.py, RUNLORA_RASTER_G sweep, profiles/r02/raster_sweep.txt)
  if (r.kid == KID_GEMM_MAIN && a_bytes < b_bytes && a_bytes <= 100e6) return std::max(1, (r.M + 127) / 128);
  if (r.kid == KID_GEMM_MAIN && b_bytes <= 100e6) return 1;
  return 16;  // neither fits: bands of 16 row tiles
}

cudaError_t launch_tc_gemm(Ctx& ctx, const GemmReq* reqs, int nreq, cudaStream_t s, std::string* err) {
  if (nreq < 1 || nreq > kMaxProb) return cudaErrorInvalidValue;
  Tmaps tm;
  GemmArgs g;
  memset(&g, 0, sizeof g);
  const int cg = reqs[0].cg > 1 ? 2 : 1;
  const bool tma_store = reqs[0].tma_store;
  int bn_max = 0;
  for (int q = 0; q < nreq; ++q) {
    const GemmReq& r = reqs[q];
    if ((r.cg > 1 ? 2 : 1) != cg || r.tma_store != tma_store) return cudaErrorInvalidValue;
    if (r.BN > 256 && (r.BN != 512 || cg != 2 || r.b_mn || r.splits > 1 || r.tail_diag ||
                       !(r.out_mode == OUT_BF16 || r.out_mode == OUT_F32))) {
      if (err) *err = "tc_gemm: 512-wide tiles need a CTA pair, K-major B and a plain output";
      return cudaErrorInvalidValue;
    }
    if (r.tma_store && (r.out_mode != OUT_BF16 || r.BN < 256 || r.splits > 1)) {
      if (err) *err = "tc_gemm: TMA-store epilogue needs a plain bf16 output with 256- or 512-wide tiles";
      return cudaErrorInvalidValue;
    }
    // MN-major B: 128B swizzle in 64-column chunks, or one 16/32-column chunk (32B/64B swizzle)
    const int nb = std::min(r.BN, 256) / cg;  // B columns per CTA and MMA (512-wide: two MMAs)
    const int b_swz = !r.b_mn ? 128 : (nb % 64 == 0 ? 128 : nb == 32 ? 64 : nb == 16 ? 32 : 0);
    if (r.BN % (16 * cg) != 0 || b_swz == 0) {
      if (err) *err = "tc_gemm: illegal tile width for operand majorness";
      return cudaErrorInvalidValue;
    }
    const int a_box = r.a_mn ? 64 : kBM;
    const int b_box = r.b_mn ? 64 : nb;
    // MN-major operands whose contiguous extent is a whole number of swizzle chunks are
    // fetched with ONE 3-D TMA box per stage instead of one 2-D box per chunk.
    const int b_cw = b_swz / 2;
    static const bool tma3d = getenv("RUNLORA_TMA3D") == nullptr || atoi(getenv("RUNLORA_TMA3D")) != 0;
    const bool a3 = tma3d && r.a_mn && r.a.cols % 64 == 0 && (r.K2 == 0 || r.a2.cols % 64 == 0);
    const bool b3 = tma3d && r.b_mn && nb > b_cw && r.b.cols % b_cw == 0 && (r.K2 == 0 || r.b2.cols % b_cw == 0);
    if (!ctx.tmap(r.a, a_box, &tm.m[q][0], err, 128, a3 ? 2 : 0) ||
        !ctx.tmap(r.b, b_box, &tm.m[q][1], err, b_swz, b3 ? nb / b_cw : 0))
      return cudaErrorInvalidValue;
    if (r.tail_fp8) {  // Wq (E4M3) and the scale diagonal (E5M2), 128-byte K rows
      const bool ok = (r.tail_fp8 == 1 || r.tail_fp8 == 2) && cg == 1 && r.BN == 256 && r.tma_store &&
                      r.K2 == (r.tail_fp8 == 1 ? 128 : r.BN) && !r.tail_diag;
      if (!ok || !ctx.tmap(r.a2, 128, &tm.m[q][2], err, 128, 0, 1) ||
          !ctx.tmap(r.b2, r.tail_fp8 == 1 ? r.BN : 128, &tm.m[q][3], err, 128, 0, 1)) {
        if (err && err->empty()) *err = "tc_gemm: the FP8 tail needs 256-wide single-CTA tiles and the TMA store";
        return cudaErrorInvalidValue;
      }    } else if (r.K2 > 0) {
      if (!ctx.tmap(r.a2, a_box, &tm.m[q][2], err, 128, a3 ? 2 : 0) ||
          !ctx.tmap(r.b2, b_box, &tm.m[q][3], err, b_swz, b3 ? nb / b_cw : 0))
        return cudaErrorInvalidValue;
    } else {
      tm.m[q][2] = tm.m[q][0];
      tm.m[q][3] = tm.m[q][1];
    }
    if (r.tma_store) {  // D: box {64 columns, 32 rows}, 128B swizzle (one epilogue warp's chunk)
      const DeviceMat dm{r.D, (int64_t)r.M, (int64_t)r.N, r.ldd};
      if (!ctx.tmap(dm, 32, &tm.m[q][4], err, 128)) return cudaErrorInvalidValue;
    }
    Prob& p = g.p[q];
    ProbX& px = g.px[q];
    p.M = r.M;
    p.N = r.N;
    p.bn = r.BN;
    p.k1 = r.K1;
    p.nk1 = (r.K1 + kBK - 1) / kBK;
    p.k2 = r.K2;
    p.nk2 = r.K2 > 0 ? (r.K2 + kBK - 1) / kBK : 0;
    p.num_splits = r.splits > 1 ? r.splits : 1;
    p.kb_per_split = r.splits > 1 ? r.kb_per_split : p.nk1;
    p.num_m_tiles = (r.M + kBM * cg - 1) / (kBM * cg);
    p.num_n_tiles = (r.N + r.BN - 1) / r.BN;
    p.units = p.num_m_tiles * p.num_n_tiles * p.num_splits;
    p.a_mn = r.a_mn;
    p.b_mn = r.b_mn;
    p.b_swz = b_swz;
    p.a_3d = a3 ? 1 : 0;
    static const bool snake = getenv("RUNLORA_SNAKE") == nullptr || atoi(getenv("RUNLORA_SNAKE")) != 0;
    p.snake = (snake && r.splits <= 1 && r.kid == KID_GEMM_MAIN) ? 1 : 0;
    p.raster_g = raster_rows(r);
    p.b_3d = b3 ? 1 : 0;
    p.out_mode = r.out_mode;
    p.idesc = idesc_bf16(kBM * cg, std::min(r.BN, 256), r.a_mn, r.b_mn);
    p.stage_tx = (uint32_t)cg * (uint32_t)(kBM * kBK * 2 + (r.BN / cg) * kBK * 2);
    p.D = r.D;
    p.ldd = r.ldd;
    p.split_stride = r.split_stride;
    p.Cin = static_cast<const __nv_bfloat16*>(r.Cin);
    p.ldc = r.ldc;
    p.fold = r.fold;
    p.fold_w = r.fold_w;
    if (r.out_mode == OUT_F32_FOLD &&
        (!(r.fold_w == 8 || r.fold_w == 16 || r.fold_w == 32 || r.fold_w == 64) || r.fold * r.fold_w != r.BN ||
         r.BN > 256 || cg != 1)) {
      if (err) *err = "tc_gemm: OUT_F32_FOLD needs single-CTA tiles, fold_w in {8, 16, 32, 64} and BN = fold * fold_w";
      return cudaErrorInvalidValue;
    }
    p.tail_diag = r.tail_diag ? 1 : 0;
    if (r.tail_fp8) {  // mode 1: A2 = diagonal (E5M2), B2 = Wq; mode 2: A2 = Wq, B2 = diagonal
      px.tail_fp8 = r.tail_fp8;
      p.nk2 = r.tail_fp8 == 1 ? 1 : r.BN / 128;
      px.idesc2 = r.tail_fp8 == 1 ? idesc_f8(kBM, r.BN, kE5M2, kE4M3) : idesc_f8(kBM, 128, kE4M3, kE5M2);
    }
    if (r.fixup) {
      if (!(r.out_mode == OUT_F32 || r.out_mode == OUT_F32_FOLD) || cg != 1 || !r.counters || !r.fx_out ||
          r.ldd % 4 != 0 || r.tma_store) {
        if (err) *err = "tc_gemm: the split fix-up needs an fp32 slab output, single-CTA tiles and counters";
        return cudaErrorInvalidValue;
      }
      px.fixup = 1;
      px.counters = r.counters;
      px.fx_out = r.fx_out;
      px.fx_ldo = r.fx_ldo;
      px.fx_cols = r.fx_cols;
      px.fx_transpose = r.fx_transpose;
      px.fx_accumulate = r.fx_accumulate;
      px.fx_bf16 = r.fx_bf16;
    }
    p.hint_a = r.a_policy == 1 ? kEvictNormal : r.a_policy == 2 ? kEvictFirst
               : r.a_stream_once ? kEvictFirst : kEvictNormal;
    p.hint_b = kEvictLast;
    g.total_units += p.units;
    if (r.BN > bn_max) bn_max = r.BN;
  }
  g.nprob = nreq;
  if (reqs[0].nside < 0 || reqs[0].nside > 2) return cudaErrorInvalidValue;
  for (int j = 0; j < reqs[0].nside; ++j) {
    const ReduceJob& J = reqs[0].side[j];
    if (J.repeat > 0 ? (J.cols % 8 != 0) : (J.ldp % 4 || J.split_stride % 4))
      return cudaErrorInvalidValue;  // 16-byte groups / float4 slab reads
    g.side[j] = SideJob{J.P, J.split_stride, J.ldp, J.ldo, J.out, J.splits, J.rows, J.cols, J.out_bf16, J.transpose,
                        J.accumulate, J.repeat};
  }
  g.nside = reqs[0].nside;
  if (reqs[0].xdesc) {
    if (reqs[0].nside != 2 || reqs[0].side[0].transpose || !reqs[0].side[1].transpose) return cudaErrorInvalidValue;
    g.xdesc = static_cast<const XDesc*>(reqs[0].xdesc);
    g.xepoch = reqs[0].xepoch;
  }
  g.zero_ptr = reqs[0].zero_ptr;
  g.zero_n = reqs[0].zero_ptr ? reqs[0].zero_n : 0;
  g.trace = (ctx.trace && ctx.trace_kid == reqs[0].kid && g.total_units <= Ctx::kTraceUnits) ? ctx.trace : nullptr;
  g.ltrace = ctx.ltrace_slot(reqs[0].kid);
  g.stages = (reqs[0].kid == KID_GEMM_MAIN && reqs[0].overlaps_comm) ? ctx.main_stages() : 0;
  // RUNLORA_MAIN_STAGES < 7 asks the main GEMMs to leave shared memory for co-resident
  // kernels (NCCL's during an overlapped allreduce): the 512-wide kernel's 48 KB stages then
  // drop from 4 to 3 (frees 48 KB) instead of being clamped to the full ring
  if (g.stages > 0 && g.stages < 7 && bn_max > 256) g.stages = 3;
  if (const char* d = getenv("RUNLORA_DBG_GEMM")) g.dbg = atoi(d);
  {
    // 512-wide tiles: the last 3 k-blocks issue MMA 0 before MMA 1 so slot s0 drains under
    // MMA 1's tail (MMA-only run at 131072x2048x2048 554 -> 534 µs; steps 0.991-0.995x,
    // profiles/r02/ab_endj.jsonl); env RUNLORA_ENDJ=0 turns it off
    static const int endj = getenv("RUNLORA_ENDJ") ? atoi(getenv("RUNLORA_ENDJ")) : 3;
    const int st = g.stages > 0 ? g.stages : 4;
    g.endj = std::max(0, std::min(endj, st - 1));
  }
  for (int q = nreq; q < kMaxProb; ++q) g.p[q] = g.p[0], g.px[q] = g.px[0], g.p[q].units = 0;
  if (g.total_units <= 0) return cudaSuccess;
  // a CTA defers at most kMaxFixups split fix-ups to the end of its unit loop; beyond that
  // (never on the shapes of the configs) the slabs are reduced by the reducer kernel instead
  ReduceJob fallback[kMaxProb];
  int nfb = 0;
  const int min_groups = ctx.num_sms() / cg;
  if ((g.total_units + min_groups - 1) / min_groups > kMaxFixups) {
    for (int q = 0; q < nreq; ++q) {
      const Prob& p = g.p[q];
      ProbX& px = g.px[q];
      if (!px.fixup) continue;
      px.fixup = 0;
      fallback[nfb++] = ReduceJob{static_cast<const float*>(p.D), p.num_splits, p.split_stride, p.M, px.fx_cols, p.ldd,
                                  px.fx_out, px.fx_bf16, px.fx_ldo, px.fx_transpose, px.fx_accumulate};
    }
  }
  ctx.launch_begin(s, reqs[0].kid);
  // 2 CTAs per SM for the HBM-bound rank-r kernels; at 128 columns only for the token
  // reductions (r = 128: 42.6 -> 31.0 µs; the projections lost 38 -> 45 µs to the shallower ring)
  const bool occ2 = ctx.occ2() && reqs[0].a_stream_once && (bn_max <= 64 || reqs[0].kid == KID_GEMM_TOKRED);
  const int sms = ctx.num_sms() - ((reqs[0].kid == KID_GEMM_MAIN && reqs[0].overlaps_comm) ? ctx.comm_sms() : 0);
  cudaError_t e = dispatch_tc(ctx, bn_max, cg, occ2, tma_store, tm, g, s, sms);
  ctx.launch_end(s);
  if (e == cudaSuccess && nfb > 0) e = launch_splitk_reduce(ctx, fallback, nfb, s);
  if (e != cudaSuccess && err) *err = std::string("tc_gemm launch: ") + cudaGetErrorString(e);
  return e;
}

cudaError_t launch_splitk_reduce(Ctx& ctx, const ReduceJob* jobs, int njobs, cudaStream_t s) {
  ReduceArgs a;
  memset(&a, 0, sizeof a);
  a.j[0] = jobs[0];
  a.total0 = (long long)jobs[0].rows * ((jobs[0].cols + 3) / 4);
  a.total = a.total0;
  if (njobs > 1) {
    a.j[1] = jobs[1];
    a.total += (long long)jobs[1].rows * ((jobs[1].cols + 3) / 4);
  }
  if (a.total <= 0) return cudaSuccess;
  long long blocks = (a.total + 255) / 256;
  const long long cap = (long long)ctx.num_sms() * 16;
  if (blocks > cap) blocks = cap;
  a.ltrace = ctx.ltrace_slot(KID_SPLITK_REDUCE);
  ctx.launch_begin(s, KID_SPLITK_REDUCE);
  cudaError_t e = launch_pdl(ctx, splitk_reduce_kernel, dim3((unsigned)blocks), dim3(256), s, a);
  ctx.launch_end(s);
  return e;
}

cudaError_t launch_sgemm(Ctx& ctx, int M, int N, int K, const float* A, int64_t sa0, int64_t sa1, const float* B,
                         int64_t sb0, int64_t sb1, float* C, int64_t ldc, const float* Cadd, int64_t ldadd,
                         bool accumulate, cudaStream_t s) {
  dim3 grid((N + 63) / 64, (M + 63) / 64);
  ctx.launch_begin(s, KID_SGEMM_F32);
  cudaError_t e = launch_pdl(ctx, sgemm_kernel, grid, dim3(256), s, M, N, K, A, (long long)sa0, (long long)sa1, B,
                             (long long)sb0, (long long)sb1, C, (long long)ldc, Cadd, (long long)ldadd,
                             accumulate ? 1 : 0);
  ctx.launch_end(s);
  return e;
}

}  // namespace runlora
