// Per-handle host context: device facts, TMA descriptor cache, launch counting
// and CUDA-event kernel profiling.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "internal.h"

namespace runlora {

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

Ctx::Ctx(int device) : device_(device) {
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) == cudaSuccess && sms > 0) num_sms_ = sms;
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
      q == cudaDriverEntryPointSuccess)
    encode_fn_ = fn;
  if (const char* e = getenv("RUNLORA_MAIN_CG")) main_cg_ = atoi(e) == 1 ? 1 : 2;
  if (const char* e = getenv("RUNLORA_OCC2")) occ2_ = atoi(e) != 0;
  if (const char* e = getenv("RUNLORA_PDL")) pdl_ = atoi(e) != 0;
  if (const char* e = getenv("RUNLORA_L2PROMO_MN")) promo_mn_ = (CUtensorMapL2promotion)atoi(e);
  if (const char* e = getenv("RUNLORA_MAIN_STAGES")) main_stages_ = atoi(e) > 0 ? atoi(e) : 0;  // 0: all
  if (const char* e = getenv("RUNLORA_COMM_SMS")) comm_sms_ = std::max(0, std::min(atoi(e), num_sms_ - 2)) & ~1;
  if (const char* e = getenv("RUNLORA_TMA_STORE_MAIN")) tma_store_main_ = atoi(e) != 0;
  if (const char* e = getenv("RUNLORA_MAIN_WIDE")) main_wide_ = atoi(e) != 0;
  if (const char* e = getenv("RUNLORA_WIDE_COST")) {
    double a = 0, k = 0;
    if (sscanf(e, "%lf,%lf", &a, &k) == 2 && a > 0 && k >= 0) wide_cost_a_ = a, wide_cost_e_ = k;
  }
  if (const char* e = getenv("RUNLORA_TMA_STORE_WPRIME")) tma_store_wprime_ = atoi(e) != 0;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  if (const char* e = getenv("RUNLORA_LTRACE"); e && atoi(e) != 0) {
    std::vector<unsigned long long> init((size_t)kLTraceSlots * 8, 0ull);
    for (int i = 0; i < kLTraceSlots; ++i) init[8 * i] = init[8 * i + 1] = init[8 * i + 3] = ~0ull;
    if (cudaMalloc(&ltrace_, init.size() * 8) != cudaSuccess ||
        cudaMemcpy(ltrace_, init.data(), init.size() * 8, cudaMemcpyHostToDevice) != cudaSuccess)
      ltrace_ = nullptr;
  }
  if (const char* e = getenv("RUNLORA_TRACE")) {
    trace_kid = atoi(e);
    if (cudaMalloc(&trace, sizeof(unsigned long long) * (8 * kTraceUnits + 4 * 1024)) != cudaSuccess) trace = nullptr;
  }
  {
    std::vector<uint16_t> eye(128 * 128, 0);
    for (int i = 0; i < 128; ++i) eye[i * 128 + i] = 0x3F80;  // bf16 1.0
    if (cudaMalloc(&identity_, eye.size() * 2) != cudaSuccess ||
        cudaMemcpy(identity_, eye.data(), eye.size() * 2, cudaMemcpyHostToDevice) != cudaSuccess) {
      if (identity_) cudaFree(identity_);
      identity_ = nullptr;
    }
  }
  if (prev >= 0) cudaSetDevice(prev);
}

Ctx::~Ctx() {
  for (auto& p : pending_) {
    cudaEventDestroy(p.a);
    cudaEventDestroy(p.b);
  }
  for (auto e : free_events_) cudaEventDestroy(e);
  if (cur_start_) cudaEventDestroy(cur_start_);
  if (identity_) cudaFree(identity_);
  if (trace) cudaFree(trace);
  if (ltrace_) cudaFree(ltrace_);
}

bool Ctx::tmap(const DeviceMat& m, int box_rows, CUtensorMap* out, std::string* err, int swz, int chunks,
               int elem) {
  const TmapKey key{m.ptr, m.rows, m.cols, m.ld, box_rows, swz, chunks, elem};
  {
    std::lock_guard<std::mutex> g(tmap_mu_);
    auto it = tmaps_.find(key);
    if (it != tmaps_.end()) {
      *out = it->second;
      return true;
    }
  }
  if (!encode_fn_) {
    if (err) *err = "cuTensorMapEncodeTiled entry point unavailable";
    return false;
  }
  const cuuint32_t w = swz == 0 ? 256u / elem : (cuuint32_t)(swz / elem);  // swz 0: no swizzle, 256-byte rows
  cuuint64_t dims[3] = {(cuuint64_t)m.cols, (cuuint64_t)m.rows, 1};
  cuuint64_t strides[2] = {(cuuint64_t)m.ld * elem, 0};
  cuuint32_t box[3] = {w, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1u, 1u, 1u};
  cuuint32_t rank = 2;
  if (chunks > 0) {
    dims[0] = w;
    dims[2] = (cuuint64_t)(m.cols / w);
    strides[1] = (cuuint64_t)w * elem;
    box[2] = (cuuint32_t)chunks;
    rank = 3;
  }
  CUtensorMap tm;
  CUresult r = reinterpret_cast<EncodeTiledFn>(encode_fn_)(
      &tm, elem == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank,
      const_cast<void*>(m.ptr), dims, strides, box, estr,
      CU_TENSOR_MAP_INTERLEAVE_NONE,
      swz == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
      : swz == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
      : swz == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                  : CU_TENSOR_MAP_SWIZZLE_NONE,
      (chunks > 0 ? promo_mn_ : CU_TENSOR_MAP_L2_PROMOTION_L2_256B),
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    if (err) {
      char buf[256];
      snprintf(buf, sizeof buf, "cuTensorMapEncodeTiled failed (%d) for %lldx%lld ld=%lld box=%dx%d ptr=%p", (int)r,
               (long long)m.rows, (long long)m.cols, (long long)m.ld, swz / 2, box_rows, m.ptr);
      *err = buf;
    }
    return false;
  }
  std::lock_guard<std::mutex> g(tmap_mu_);
  if (tmaps_.size() > 4096) tmaps_.clear();
  tmaps_[key] = tm;
  *out = tm;
  return true;
}

unsigned long long* Ctx::ltrace_slot(KernelId kid) {
  if (!ltrace_ || ltrace_next_ >= kLTraceSlots) return nullptr;
  ltrace_kid_.push_back((int)kid);
  return ltrace_ + 8ull * (ltrace_next_++);
}

int Ctx::ltrace_read(unsigned long long* host, int* kids, int max_slots) {
  if (!ltrace_) return 0;
  const int n = std::min(max_slots, ltrace_next_);
  if (cudaDeviceSynchronize() != cudaSuccess ||
      cudaMemcpy(host, ltrace_, 8ull * 8 * n, cudaMemcpyDeviceToHost) != cudaSuccess)
    return 0;
  for (int i = 0; i < n; ++i) kids[i] = ltrace_kid_[i];
  std::vector<unsigned long long> init((size_t)kLTraceSlots * 8, 0ull);  // reset for the next window
  for (int i = 0; i < kLTraceSlots; ++i) init[8 * i] = init[8 * i + 1] = init[8 * i + 3] = ~0ull;
  cudaMemcpy(ltrace_, init.data(), init.size() * 8, cudaMemcpyHostToDevice);
  ltrace_next_ = 0;
  ltrace_kid_.clear();
  return n;
}

cudaEvent_t Ctx::get_event() {
  if (!free_events_.empty()) {
    cudaEvent_t e = free_events_.back();
    free_events_.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

void Ctx::launch_begin(cudaStream_t s, KernelId kid) {
  ++launches_;
  if (!profiling_) return;
  cur_kid_ = kid;
  cur_start_ = get_event();
  cudaEventRecord(cur_start_, s);
}

void Ctx::launch_end(cudaStream_t s) {
  if (!profiling_ || !cur_start_) return;
  cudaEvent_t b = get_event();
  cudaEventRecord(b, s);
  pending_.push_back({cur_kid_, cur_start_, b});
  cur_start_ = nullptr;
}

void Ctx::profile_enable(bool on) { profiling_ = on; }

bool Ctx::profile_read(runlora_kernel_stat_t* stats, int max_stats, int* count, bool reset, std::string* err) {
  for (auto& p : pending_) {
    if (cudaEventSynchronize(p.b) != cudaSuccess) {
      if (err) *err = "cudaEventSynchronize failed while reading profile";
      return false;
    }
    float ms = 0.f;
    cudaEventElapsedTime(&ms, p.a, p.b);
    stat_launches_[p.kid] += 1;
    stat_ms_[p.kid] += ms;
    free_events_.push_back(p.a);
    free_events_.push_back(p.b);
  }
  pending_.clear();
  int n = 0;
  for (int k = 0; k < KID_COUNT; ++k) {
    if (stat_launches_[k] == 0) continue;
    if (stats && n < max_stats) {
      memset(&stats[n], 0, sizeof(stats[n]));
      strncpy(stats[n].name, kKernelNames[k], sizeof(stats[n].name) - 1);
      stats[n].launches = stat_launches_[k];
      stats[n].total_ms = stat_ms_[k];
    }
    ++n;
  }
  if (count) *count = n;
  if (reset) {
    for (int k = 0; k < KID_COUNT; ++k) {
      stat_launches_[k] = 0;
      stat_ms_[k] = 0.0;
    }
  }
  return true;
}

}  // namespace runlora
