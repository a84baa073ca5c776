// One-shot allreduce of the packed fp32 adapter gradients over peer memory (SURVEY §8(a)
// a8, §8(f) NEXT-2): out[i] = sum_{p = 0 .. P-1} peer_p[i] in fixed rank order, every rank
// reading all P ranks' buffers directly (NVLink P2P loads through unified virtual
// addresses, e.g. torch symmetric-memory buffers).  Fixed order => every rank computes the
// bit-identical sum, deterministic run to run.  HBM/NVLink-bound: P·n·4 bytes read, n·4
// written per rank.  The cross-rank ordering (all writes done before the reads; all reads
// done before a buffer is rewritten) is the caller's (include/runlora.h).
#include "internal.h"
#include "ptx.cuh"
#include "exchange.cuh"

namespace runlora {
namespace {

struct Peers {
  const float* p[kMaxPeers];
};

__global__ void __launch_bounds__(256) allreduce_sum_kernel(const __grid_constant__ Peers peers, int P, float* out,
                                                            int64_t n, unsigned long long* lt) {
  if (threadIdx.x == 0) ltrace_mark(lt, 0);
  pdl_wait();
  pdl_launch_dependents();
  if (threadIdx.x == 0) ltrace_mark(lt, 1);
  const int64_t nv = n / 4, stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv; i += stride) {
    float4 s = __ldcv(reinterpret_cast<const float4*>(peers.p[0]) + i);  // peers' data: bypass stale L1/L2 lines
    for (int q = 1; q < P; ++q) {
      const float4 v = __ldcv(reinterpret_cast<const float4*>(peers.p[q]) + i);
      s.x += v.x, s.y += v.y, s.z += v.z, s.w += v.w;
    }
    reinterpret_cast<float4*>(out)[i] = s;
  }
  for (int64_t i = 4 * nv + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    float s = __ldcv(peers.p[0] + i);
    for (int q = 1; q < P; ++q) s += __ldcv(peers.p[q] + i);
    out[i] = s;
  }
  if (threadIdx.x == 0) ltrace_mark(lt, 2);
}

}  // namespace

cudaError_t launch_allreduce_sum_f32(Ctx& ctx, const float* const* peers, int P, float* out, int64_t n,
                                     cudaStream_t s) {
  Peers pp{};
  for (int q = 0; q < P; ++q) pp.p[q] = peers[q];
  // one resident wave (4 blocks of 256 threads per SM), grid-stride beyond it
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((n / 4 + 255) / 256, (int64_t)ctx.num_sms() * 4));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)blocks);
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = ctx.pdl() ? 1 : 0;
  ctx.launch_begin(s, KID_ALLREDUCE);
  cudaError_t e = cudaLaunchKernelEx(&cfg, allreduce_sum_kernel, pp, P, out, n, ctx.ltrace_slot(KID_ALLREDUCE));
  ctx.launch_end(s);
  return e;
}

// ------------------------------------------------ fused exchange, P ranks emulated
namespace {
struct XEmuSlabs {
  XSlabs s[kXMaxPeers];
};
// block b plays rank b / per, as CTA b % per of that rank's exchange (64 threads: the two
// warps that run it inside the dX GEMM); cooperative launch, so all blocks are co-resident
__global__ void __launch_bounds__(64) exchange_emulate_kernel(const XDesc* descs, const __grid_constant__ XEmuSlabs sl,
                                                              int per, unsigned epoch) {
  const int q = blockIdx.x / per;
  exchange_run(descs[q], sl.s[q], epoch, threadIdx.x, blockIdx.x % per, per);
}
}  // namespace

cudaError_t launch_exchange_emulate(Ctx& ctx, int P, const XDesc* descs, const XSlabs* slabs, unsigned epoch) {
  XEmuSlabs sl;
  for (int q = 0; q < P; ++q) sl.s[q] = slabs[q];
  XDesc* d = nullptr;
  cudaError_t e = cudaMalloc(&d, sizeof(XDesc) * P);
  if (e != cudaSuccess) return e;
  e = cudaMemcpy(d, descs, sizeof(XDesc) * P, cudaMemcpyHostToDevice);
  const int chunks = (descs[0].rows0 + descs[0].rows1 + kXChunkRows - 1) / kXChunkRows;
  const int per = std::max(1, std::min(chunks, (ctx.num_sms() * 4) / P));  // all P*per blocks resident
  if (e == cudaSuccess) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(P * per));
    cfg.blockDim = dim3(64);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    ctx.launch_begin(nullptr, KID_ALLREDUCE);
    e = cudaLaunchKernelEx(&cfg, exchange_emulate_kernel, (const XDesc*)d, sl, per, epoch);
    ctx.launch_end(nullptr);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
  }
  cudaFree(d);
  return e;
}

}  // namespace runlora
