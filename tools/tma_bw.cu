// TMA streaming-bandwidth microbenchmark (design input for the HBM-bound rank-r kernels).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tma_bw tools/tma_bw.cu -lcuda
//   ./tma_bw
//
// Streams a [rows x cols] bf16 matrix (cols contiguous) from HBM into a shared-memory ring
// with cp.async.bulk.tensor and nothing else (the consumer only releases the slot), for
// several box shapes, CTAs/SM and traversal orders:
//   order 0 ("row band"):  CTA owns a band of `bh` rows and walks the columns (X·A pattern)
//   order 1 ("col band"):  CTA owns a band of columns and walks the rows (Xᵀ·Z pattern)
// A box is {64 cols (128 B, 128B swizzle), box_rows, chunks} (3-D when chunks > 1, i.e.
// box_rows rows x 128*chunks contiguous bytes).  Prints GB/s (median of 7, L2 flushed).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x)                                                                            \
  do {                                                                                   \
    cudaError_t e = (x);                                                                 \
    if (e != cudaSuccess) {                                                              \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);         \
      exit(1);                                                                           \
    }                                                                                    \
  } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

struct Args {
  int rows, cols, box_rows, chunks, stages, order;
  int ur, uc;  // unit tile: ur rows x uc cols; order 0 walks its columns fastest, order 1 its rows
  int units;
};

__global__ void __launch_bounds__(64) stream_kernel(const __grid_constant__ CUtensorMap tm, Args a, int* sink) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  const uint32_t box_bytes = 128u * a.box_rows * a.chunks;
  uint64_t* full = (uint64_t*)(sm + a.stages * box_bytes);
  uint64_t* empty = full + a.stages;
  if (threadIdx.x == 0) {
    for (int s = 0; s < a.stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int bw = 64 * a.chunks;  // box width (elements)
  if (threadIdx.x == 0) {
    int s = 0, ph = 0;
    for (int u = blockIdx.x; u < a.units; u += gridDim.x) {
      const int nur = a.cols / a.uc;
      const int ur0 = (u / nur) * a.ur, uc0 = (u % nur) * a.uc;
      const int nr = a.ur / a.box_rows, nc = a.uc / bw;
      for (int i = 0; i < nr * nc; ++i) {
          const int ir = a.order == 0 ? i / nc : i % nr;
          const int ic = a.order == 0 ? i % nc : i / nr;
          const int r0 = ur0 + ir * a.box_rows;
          const int c0 = uc0 + ic * bw;
          uint32_t done = 0;
          while (!done)
            asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                         : "=r"(done) : "r"(su32(&empty[s])), "r"(ph ^ 1));
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(box_bytes));
          if (a.chunks == 1)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                ::"r"(su32(sm + s * box_bytes)), "l"((uint64_t)&tm), "r"(su32(&full[s])), "r"(c0), "r"(r0) : "memory");
          else
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                ::"r"(su32(sm + s * box_bytes)), "l"((uint64_t)&tm), "r"(su32(&full[s])), "r"(0), "r"(r0), "r"(c0 / 64)
                : "memory");
          if (++s == a.stages) s = 0, ph ^= 1;
        }
    }
  } else if (threadIdx.x == 32) {
    int s = 0, ph = 0, acc = 0;
    for (int u = blockIdx.x; u < a.units; u += gridDim.x) {
      const int nr = a.ur / a.box_rows, nc = a.uc / bw;
      for (int i = 0; i < nr * nc; ++i) {
        uint32_t done = 0;
        while (!done)
          asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                       : "=r"(done) : "r"(su32(&full[s])), "r"(ph));
        acc += sm[s * box_bytes + 17];
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])));
        if (++s == a.stages) s = 0, ph ^= 1;
      }
    }
    if (acc == 123456789) *sink = acc;
  }
}

using EncFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                           const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                           CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  EncFn enc;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int rows = 65536, cols = 4096;  // 512 MiB bf16 (separates per-byte cost from launch ramp)
  void* buf;
  CK(cudaMalloc(&buf, (size_t)rows * cols * 2));
  CK(cudaMemset(buf, 1, (size_t)rows * cols * 2));
  void* flush;
  CK(cudaMalloc(&flush, 256 << 20));
  int* sink;
  CK(cudaMalloc(&sink, 4));
  CK(cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
  struct Cfg { int box_rows, chunks, order, ur, uc, occ, kb_smem; };
  std::vector<Cfg> cfgs = {
      // X·A pattern: unit = 128 rows x all columns, walk columns (current box: 128 rows x 128 B)
      {128, 1, 0, 128, 4096, 1, 200}, {128, 1, 0, 128, 4096, 2, 100}, {128, 1, 0, 128, 1024, 2, 100},
      {32, 4, 0, 128, 4096, 2, 100},  {32, 4, 0, 128, 4096, 1, 200},  {16, 8, 0, 128, 4096, 2, 100},
      {64, 2, 0, 128, 4096, 2, 100},  {8, 8, 0, 128, 4096, 2, 100},   {32, 8, 0, 128, 4096, 2, 100},
      {32, 4, 0, 32, 4096, 2, 100},
      // Xᵀ·Z pattern: unit = 2048 rows x 128 columns, walk rows (current box: 64 rows x 256 B)
      {64, 2, 1, 2048, 128, 2, 100},  {64, 2, 1, 2048, 128, 1, 200},  {32, 4, 1, 2048, 256, 2, 100},
      {128, 2, 1, 2048, 128, 2, 100}, {16, 8, 1, 2048, 512, 2, 100},  {64, 4, 1, 2048, 256, 2, 100},
      {64, 2, 1, 8192, 128, 2, 100},
  };
  for (const Cfg& c : cfgs) {
    CUtensorMap tm;
    cuuint64_t dims3[3] = {64, (cuuint64_t)rows, (cuuint64_t)cols / 64};
    cuuint64_t str3[2] = {(cuuint64_t)cols * 2, 128};
    cuuint32_t box3[3] = {64, (cuuint32_t)c.box_rows, (cuuint32_t)c.chunks};
    cuuint64_t dims2[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t str2[1] = {(cuuint64_t)cols * 2};
    cuuint32_t box2[2] = {64, (cuuint32_t)c.box_rows};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = c.chunks > 1
                     ? enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims3, str3, box3, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE)
                     : enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims2, str2, box2, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      printf("encode failed %d\n", (int)r);
      continue;
    }
    Args a;
    a.rows = rows;
    a.cols = cols;
    a.box_rows = c.box_rows;
    a.chunks = c.chunks;
    a.order = c.order;
    a.ur = c.ur;
    a.uc = c.uc;
    const int box_bytes = 128 * c.box_rows * c.chunks;
    a.stages = std::min(16, c.kb_smem * 1024 / box_bytes);
    a.units = (rows / c.ur) * (cols / c.uc);
    const size_t smem = (size_t)a.stages * box_bytes + 1024 + 256;
    const int grid = std::min(a.units, sms * c.occ);
    std::vector<float> ts;
    for (int it = 0; it < 9; ++it) {
      CK(cudaMemsetAsync(flush, it, 256 << 20));
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      stream_kernel<<<grid, 64, smem>>>(tm, a, sink);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (it >= 2) ts.push_back(ms);
    }
    CK(cudaGetLastError());
    std::sort(ts.begin(), ts.end());
    const float ms = ts[ts.size() / 2];
    printf("{\"order\": %d, \"box_rows\": %d, \"box_bytes_per_row\": %d, \"unit\": \"%dx%d\", \"occ\": %d, "
           "\"stages\": %d, \"grid\": %d, \"us\": %.2f, \"GBps\": %.0f}\n",
           c.order, c.box_rows, 128 * c.chunks, c.ur, c.uc, c.occ, a.stages, grid, ms * 1e3,
           (double)rows * cols * 2 / (ms * 1e-3) / 1e9);
  }
  return 0;
}
