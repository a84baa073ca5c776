/*
 * runlora_testing.h — test hook of librunlora.so (not part of the stable ABI).
 *
 * runlora_debug_gemm runs ONE launch of the library's tcgen05 GEMM kernel
 * (the building block of every bf16 product of Eq. 1-3 / Alg. 1-5, PAPER.md
 * P:42-154) so that each operand-majorness / tile-width / split / epilogue
 * combination can be checked in isolation:
 *
 *   D[M,N] = A1·B1 (+ A2·B2)   bf16 operands, fp32 accumulation
 *   A1: a_mn == 0 -> stored [M, K1] row-major; a_mn == 1 -> stored [K1, M]
 *   B1: b_mn == 0 -> stored [N, K1] row-major; b_mn == 1 -> stored [K1, N]
 *   A2/B2: same majors with K2 (K2 == 0: no tail)
 *   out_mode 0: D bf16 [M, N]; 1: D bf16 = acc + Cin (bf16 [M, N]);
 *            2: D fp32 partial slabs [splits][M][N] (split-K over K1)
 *   BN: tile width (16, 32, 48, 64, 128, 256, 512 with cg = 2 and K-major B; MN-major B: 16, 32 or a
 *       multiple of 64); 0 = the main GEMMs' launch (cg = 2, bf16 output, 512/256-wide split by the planner).
 *   cg: 1 = one CTA per 128-row tile; 2 = CTA pair (tcgen05 cta_group::2) per 256-row tile.
 * All pointers are device pointers; rows are contiguous (ld = number of columns).
 */
#ifndef RUNLORA_TESTING_H_
#define RUNLORA_TESTING_H_
#include "runlora.h"
#ifdef __cplusplus
extern "C" {
#endif
runlora_status_t runlora_debug_gemm(runlora_handle_t h, int M, int N, int K1, const void* A1, int a_mn,
                                    const void* B1, int b_mn, int K2, const void* A2, const void* B2, int out_mode,
                                    void* D, const void* Cin, int BN, int splits, int cg, void* stream);
/* Debug timeline of the last launch of kernel id RUNLORA_TRACE (env, read at handle creation):
 * 8 uint64 per unit {producer start, dependencies met, last load issued, epilogue done (ns),
 * CTA index, problem index}; with max_units = 65536 the host buffer must hold 8*65536 + 4*1024 words:
 * 4 per CTA follow the unit records {kernel entry, inputs ready (after the PDL wait), exit}.
 * Returns the number of units copied (0 if tracing is off). */
int runlora_debug_trace(runlora_handle_t h, unsigned long long* host, int max_units);
/* Launch timeline (env RUNLORA_LTRACE=1 at handle creation): 8 uint64 per launch since the
 * last read {min CTA entry, min ready (after the PDL wait), max ready, min exit, max exit,
 * 0, 0, 0} (%globaltimer ns) and the launch's kernel id in kids[]; resets the record and
 * synchronises the device.  Returns the number of launches copied. */
int runlora_debug_ltrace(runlora_handle_t h, unsigned long long* host, int* kids, int max_launches);
const char* runlora_debug_kernel_name(int kid);
/* The main-GEMM tile split (DESIGN.md §5 "512-wide main-GEMM tiles"): for an M x N bf16
 * output with reduction length K and a K-major B operand (b_mn = 0), the number of leading
 * output rows the library runs as 256x512 pair tiles (a multiple of 256; 0 = 256-wide tiles
 * only, also when b_mn != 0 or env RUNLORA_MAIN_WIDE=0).  Host-only; -1 on a bad handle. */
int runlora_debug_wide_rows(runlora_handle_t h, int M, int N, int K, int b_mn);
/* The fused exchange (runlora_backward_exchange) with P ranks EMULATED on one GPU: one
 * cooperative launch runs every rank's exchange device code (its blocks wait on one another
 * only through the exchange flags, all co-resident).  Per rank q (HOST arrays of device
 * pointers): token-split slabs sA[q] [splits][k][r] and sB[q] [splits][m][r] (fp32), outputs
 * dA[q] [k, r] and dB[q] [r, m] (fp32), exchange buffers bufs[q] and zeroed flag arrays
 * flags[q] sized by runlora_exchange_sizes.  Deterministic: every dA[q] is the rank-order sum
 * of the ranks' split-order slab sums.  Synchronous. */
runlora_status_t runlora_debug_exchange_emulate(runlora_handle_t h, int P, int64_t k, int64_t m, int64_t r,
                                                int splits, const float* const* sA, const float* const* sB,
                                                float* const* dA, float* const* dB, void* const* bufs,
                                                void* const* flags, uint32_t epoch);
#ifdef __cplusplus
}
#endif
#endif
