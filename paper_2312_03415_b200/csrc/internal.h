// Internal interfaces between the ABI layer (runlora.cu) and the kernels.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <map>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/runlora.h"

namespace runlora {

// Kernel identities for launch counting / profiling.
enum KernelId : int {
  KID_GEMM_MAIN = 0,   // Y / dX GEMMs (dominant, tensor-bound)
  KID_GEMM_WPRIME,     // W + A·B (rank-r update, HBM-bound)
  KID_GEMM_PROJ,       // X·A, dY·Bᵀ (rank-r projections, HBM-bound; K-split bf16 partials)
  KID_GEMM_TOKRED,     // Xᵀ·Z1, dYᵀ·Z2 (token reductions, HBM-bound; folds Z's partials)
  KID_GEMM_DENSE_XTDY, // Xᵀ·dY (backward2..4 dense intermediate)
  KID_GEMM_SMALL,      // Z2'·Bᵀ, Z2'ᵀ·A (backward3/4 adapter grads)
  KID_SPLITK_REDUCE,   // fixed-order split-K reduction / cast / transpose
  KID_SGEMM_F32,       // fp32 SIMT GEMM (RUNLORA_F32 path)
  KID_QUANT,           // W -> FP8 E4M3 + per-column scales (column max, quantize, finalize)
  KID_DEQUANT,         // W~ = bf16(e4m3(Wq)·scale) via the FP8 identity-tail GEMM (x1 variants' W)
  KID_ALLREDUCE,       // one-shot fixed-order allreduce of [dA | dB] over peer pointers
  KID_COUNT
};
extern const char* const kKernelNames[KID_COUNT];

struct DeviceMat {  // row-major bf16 matrix view: element (i, j) at ptr[i*ld + j]
  const void* ptr;
  int64_t rows, cols, ld;
};

struct ReduceJob {
  const float* P;
  int splits;
  int64_t split_stride;
  int rows, cols;
  int64_t ldp;
  void* out;
  int out_bf16;
  int64_t ldo;
  int transpose, accumulate;
  // > 0: not a reduction but a column repeat (side jobs only): out[i, t*cols + j] = src[i, j]
  // for t < repeat, bf16 rows of `cols` (multiple of 8) elements, src = P (as bf16)
  int repeat;
};
inline ReduceJob repeat_job(const void* src, int rows, int cols, int reps, void* dst) {
  ReduceJob j{};
  j.P = static_cast<const float*>(src);
  j.rows = rows;
  j.cols = cols;
  j.out = dst;
  j.repeat = reps;
  return j;
}

struct GemmReq {
  int M, N;
  DeviceMat a;
  bool a_mn;       // false: a stored [M, K] (K-major); true: a stored [K, M] (MN-major)
  DeviceMat b;
  bool b_mn;       // false: b stored [N, K] (K-major); true: b stored [K, N] (MN-major)
  int K1;
  DeviceMat a2, b2;  // concat-K tail (same majors); K2 == 0: none
  int K2;
  int out_mode;      // OutMode
  void* D;
  int64_t ldd;
  int64_t split_stride;
  const void* Cin;
  int64_t ldc;
  int BN;
  int splits;        // >= 1 (only with OUT_F32)
  int kb_per_split;
  bool a_stream_once;  // A operand is read once (evict-first hint)
  int cg;              // 1: one CTA per 128-row tile; 2: CTA pair (cta_group::2) per 256-row tile
  KernelId kid;
  int fold, fold_w;  // OUT_F32_FOLD
  bool tail_diag;  // a2 = 128x128 identity, b2 read at the tile's own rows (see Prob)
  int a_policy;      // L2 policy of the A operand: 0 from a_stream_once, 1 normal, 2 evict-first
  bool tma_store;  // OUT_BF16 through the TMA-store epilogue (all problems of a launch alike)
  bool overlaps_comm;  // the dX GEMM, which a data-parallel allreduce overlaps: runs on the SMs
                       // minus Ctx::comm_sms (and on RUNLORA_MAIN_STAGES ring stages)
  // in-kernel split-K fix-up (Prob::fixup): the last split of each output tile reduces the
  // slabs into fx_out (the ReduceJob semantics); counters zeroed by an earlier launch
  bool fixup;
  int* counters;
  void* fx_out;
  int64_t fx_ldo;
  int fx_cols;
  bool fx_transpose, fx_accumulate, fx_bf16;
  int* zero_ptr;  // launch-level (first request): ints zeroed by CTA 0 after the PDL wait
  int zero_n;
  // launch-level (first request): up to 2 fixed-order split-K reductions run by the launch's
  // idle warps 2-3 (GemmArgs::side), e.g. the adapter-gradient slabs under the dX GEMM
  const ReduceJob* side;
  int nside;
  // fused data-parallel exchange (launch-level): side[0] / side[1] = the dA / dB slab
  // reductions, summed across ranks by the launch's idle warps (exchange.cuh)
  const void* xdesc;  // device XDesc
  unsigned xepoch;
  // FP8 tail (ProbX::tail_fp8): 1 = W'ᵀ tile (a2 = scale diagonal E5M2 [m, 128], b2 = Wq,
  // K2 = 128); 2 = W' / W~ tile (a2 = Wq, b2 = scale diagonal, K2 = BN); BN = 256, TMA store
  int tail_fp8;
};


class Ctx {
 public:
  explicit Ctx(int device);
  ~Ctx();
  int device() const { return device_; }
  int num_sms() const { return num_sms_; }
  int main_cg() const { return main_cg_; }  // CTA-group size of the Y / dX GEMMs (env RUNLORA_MAIN_CG)
  bool occ2() const { return occ2_; }  // 2 CTAs/SM for rank-r kernels (env RUNLORA_OCC2=0 disables)
  bool pdl() const { return pdl_; }    // programmatic dependent launch (env RUNLORA_PDL=0 disables)
  // 128x128 bf16 identity (device): A operand of the block-diagonal tail that adds W in W + A·B
  const void* identity() const { return identity_; }

  // debug timeline buffer (env RUNLORA_TRACE=<kernel id>): see GemmArgs::trace
  unsigned long long* trace = nullptr;
  unsigned long long* ltrace_ = nullptr;
  int ltrace_next_ = 0;
  std::vector<int> ltrace_kid_;
  int trace_kid = -1;
  static constexpr int kTraceUnits = 1 << 16;  // == kTraceMaxUnits (tc_gemm.cuh); + 4 words per CTA
  bool tma_store_main() const { return tma_store_main_; }
  // 512-wide pair tiles for the main GEMMs (env RUNLORA_MAIN_WIDE=0 disables).  Planner cost
  // of a 512-wide tile in 256-wide tile times: a + e / K (env RUNLORA_WIDE_COST="a,e").
  bool main_wide() const { return main_wide_; }
  double wide_cost_a() const { return wide_cost_a_; }
  double wide_cost_e() const { return wide_cost_e_; }
  std::map<std::tuple<int, int, int, int, int>, int>& wide_cache() { return wide_cache_; }
  // main-GEMM pipeline stages (env RUNLORA_MAIN_STAGES; 0 = all that fit = 7).  6 stages
  // cost ~1 % in a step (the GEMM alone: 166.9 µs either way; 5: 169, 4: 181) and leave
  // 32 KB of shared memory per SM, so NCCL's kernels can co-reside with the dX GEMM that
  // the data-parallel allreduce overlaps (bench.py sets 6 when it runs more than one rank).
  int main_stages() const { return main_stages_; }
  // SMs the dX GEMM (the one a data-parallel allreduce overlaps) leaves free for the
  // collective's kernels (env RUNLORA_COMM_SMS, even, default 0): the persistent main GEMM
  // holds ~63 K registers and ~225 KB of shared memory on every SM it runs on, so without free
  // SMs an NCCL kernel cannot start before the GEMM ends
  int comm_sms() const { return comm_sms_; }
  bool tma_store_wprime() const { return tma_store_wprime_; }

  // Encodes (or fetches from cache) a 2-D bf16 TMA descriptor with swz_bytes swizzle
  // (32, 64, 128): dims {cols, rows}, row stride ld*2 bytes, box {swz_bytes/2, box_rows}.
  // chunks > 0: 3-D view {swz/2, rows, cols/(swz/2)} (chunk stride swz bytes), box
  // {swz/2, box_rows, chunks} -> one TMA op fills `chunks` adjacent swizzle columns.
  bool tmap(const DeviceMat& m, int box_rows, CUtensorMap* out, std::string* err, int swz_bytes = 128,
            int chunks = 0, int elem_bytes = 2);  // elem_bytes 1: an E4M3 (uint8) matrix

  // Launch timeline (env RUNLORA_LTRACE=1): each launch gets a device slot of 8 words
  // {min CTA entry, min ready, max ready, min exit, max exit} (%globaltimer ns; "ready" =
  // after the PDL wait), filled by atomics from every CTA; see runlora_debug_ltrace.
  static constexpr int kLTraceSlots = 4096;
  unsigned long long* ltrace_slot(KernelId kid);
  int ltrace_read(unsigned long long* host, int* kids, int max_slots);

  // Profiling hooks around every launch.
  void launch_begin(cudaStream_t s, KernelId kid);
  void launch_end(cudaStream_t s);
  void profile_enable(bool on);
  bool profile_read(runlora_kernel_stat_t* stats, int max_stats, int* count, bool reset, std::string* err);
  uint64_t launches() const { return launches_.load(); }

  std::mutex plan_mu;
  std::map<std::vector<int64_t>, runlora_plan_t> plans;
  // Serialises every ABI call that enqueues work or touches the caches below (wide-tile
  // plans, launch-trace slots, profiling events): any host thread
  // may call into a handle (e.g. autograd runs the backward on its own thread).  Recursive:
  // time-mode selection and runlora_step_host call the forward/backward entry points.
  std::recursive_mutex call_mu;

 private:
  int device_;
  int num_sms_ = 148;
  int main_cg_ = 2;
  void* identity_ = nullptr;
  bool tma_store_main_ = false;   // env RUNLORA_TMA_STORE_MAIN=1
  bool main_wide_ = true;
  double wide_cost_a_ = 1.72, wide_cost_e_ = 41.0;
  std::map<std::tuple<int, int, int, int, int>, int> wide_cache_;  // (M, N, K, raster, pairs) -> rows_big
  int main_stages_ = 0;
  int comm_sms_ = 0;
  bool tma_store_wprime_ = true;  // env RUNLORA_TMA_STORE_WPRIME=0
  bool occ2_ = true;
  bool pdl_ = true;
  CUtensorMapL2promotion promo_mn_ = CU_TENSOR_MAP_L2_PROMOTION_L2_256B;  // 3-D (MN-major) boxes       // env RUNLORA_OCC2=0: one CTA per SM for the rank-r kernels too
  void* encode_fn_ = nullptr;
  struct TmapKey {
    const void* ptr;
    int64_t rows, cols, ld;
    int box_rows, swz, chunks, elem;
    bool operator==(const TmapKey& o) const {
      return ptr == o.ptr && rows == o.rows && cols == o.cols && ld == o.ld && box_rows == o.box_rows &&
             swz == o.swz && chunks == o.chunks && elem == o.elem;
    }
  };
  struct TmapKeyHash {
    size_t operator()(const TmapKey& k) const {
      size_t h = std::hash<const void*>()(k.ptr);
      for (int64_t v : {k.rows, k.cols, k.ld, (int64_t)k.box_rows, (int64_t)k.swz, (int64_t)k.chunks, (int64_t)k.elem})
        h = h * 1000003u ^ std::hash<int64_t>()(v);
      return h;
    }
  };
  std::mutex tmap_mu_;
  std::unordered_map<TmapKey, CUtensorMap, TmapKeyHash> tmaps_;
  bool profiling_ = false;
  std::atomic<uint64_t> launches_{0};
  struct Pending {
    KernelId kid;
    cudaEvent_t a, b;
  };
  std::vector<Pending> pending_;
  std::vector<cudaEvent_t> free_events_;
  KernelId cur_kid_ = KID_GEMM_MAIN;
  cudaEvent_t cur_start_ = nullptr;
  uint64_t stat_launches_[KID_COUNT] = {};
  double stat_ms_[KID_COUNT] = {};
  cudaEvent_t get_event();
};

// Kernel launchers (kernels.cu). Return cudaSuccess or the launch error.
// Row tiles per raster band of a tc_gemm problem (decode_unit in tc_gemm.cuh).
int raster_rows(const GemmReq& r);
cudaError_t launch_tc_gemm(Ctx& ctx, const GemmReq* reqs, int nreq, cudaStream_t s, std::string* err);
// Fixed-order sum of fp32 split-K slabs P[split][rows][ldp] (first `cols` columns) into
// out (fp32 or bf16; optionally transposed: out[j*ldo + i]; optionally accumulated).

cudaError_t launch_splitk_reduce(Ctx& ctx, const ReduceJob* jobs, int njobs, cudaStream_t s);
// Quantized frozen weight (quant.cu): W[k, m] bf16 -> Wq e4m3 bytes + scale[m] fp32, and back
// to bf16 (m multiple of 8, scale 16-byte aligned).
cudaError_t launch_quantize_w(Ctx& ctx, const void* W, int64_t k, int64_t m, void* Wq, float* scale, void* diag,
                              cudaStream_t s);
constexpr int kMaxPeers = 16;  // runlora_allreduce_sum_f32
struct XDesc;
struct XSlabs;
// P ranks' fused exchanges (exchange.cuh) in ONE cooperative launch on this GPU (testing):
// descs / slabs are host arrays of P (device descriptors are staged by the launcher).
cudaError_t launch_exchange_emulate(Ctx& ctx, int P, const XDesc* descs, const XSlabs* slabs, unsigned epoch);
cudaError_t launch_allreduce_sum_f32(Ctx& ctx, const float* const* peers, int P, float* out, int64_t n,
                                     cudaStream_t s);

// fp32 SIMT GEMM: C[i,j] = (acc ? C[i,j] : 0) + (Cadd ? Cadd[i,j] : 0) + sum_t A(i,t) B(t,j),
// A(i,t) = A[i*sa0 + t*sa1], B(t,j) = B[t*sb0 + j*sb1].
cudaError_t launch_sgemm(Ctx& ctx, int M, int N, int K, const float* A, int64_t sa0, int64_t sa1, const float* B,
                         int64_t sb0, int64_t sb1, float* C, int64_t ldc, const float* Cadd, int64_t ldadd,
                         bool accumulate, cudaStream_t s);

}  // namespace runlora
