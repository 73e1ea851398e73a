// common.cuh -- device-side types and integer helpers of libcrius (sm_100a).
//
// Nothing here is shared with the CPU oracle (oracle/); both follow SURVEY.md
// §N0-§N6 independently.  All decision-path arithmetic is integer: int64 ns,
// int64 bytes, beta in ns per MiB.  Every degree is a power of two, so every
// division of the formulas is a shift (§N0 "cdiv ... is (a + 2^e - 1) >> e").
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

// Device-side invariant checks, compiled in only with -DCRIUS_DEBUG (compute-
// sanitizer is unavailable on the GPU pool): a violated bound traps the kernel.
#ifdef CRIUS_DEBUG
#define CRIUS_CHECK(cond)                                                        \
  do {                                                                           \
    if (!(cond)) {                                                               \
      printf("CRIUS_CHECK failed: %s (%s:%d)\n", #cond, __FILE__, __LINE__);    \
      __trap();                                                                  \
    }                                                                            \
  } while (0)
#else
#define CRIUS_CHECK(cond) \
  do {                    \
  } while (0)
#endif

namespace crius {

constexpr int64_t kInf = INT64_MAX;
constexpr int kMaxTypes = 16;
constexpr int kMaxB = 16;
constexpr int kMaxDepth = 16;
constexpr int kMaxKmax = 6;
constexpr int kMaxSidx = 12;  // S up to 2^11 stages
constexpr int kMaxRanks = 8;  // ranks of one fused exchange (one NVSwitch node)

struct TypeParams {
  int32_t cap, gpn, lgpn, pad;
  int64_t mem, a_in, b_in, a_x, b_x;
};

// Everything a kernel needs about the problem, passed by value (~1.3 KB).
struct Params {
  int32_t T, J, K1;  // types, jobs, k_max + 1
  int32_t gpu_set, s_max, g_max, b_mode, nB, depth;
  int32_t lB[kMaxB];  // log2 of the configured B values (b_mode 1)
  int64_t TL;         // total layers
  TypeParams ty[kMaxTypes];
  const int32_t *ng, *gb, *kst, *L;
  const int64_t *off;
  const int32_t *c;  // [T][K1][TL]
  const int64_t *w, *act, *bnd, *tpv;
  const int32_t *tpn;
};

// Cell table, SoA (§N2 order).
struct Cells {
  int32_t *job, *type, *G, *S, *nplans;
  int64_t *plan_off;
  int64_t *unit_cell_begin, *unit_plan_begin, *unit_weight;  // [n_units+1]
};

struct CellResult {  // == crius_cell_result
  int64_t t_ns;
  int32_t plan;
  int32_t flags;
};

__host__ __device__ __forceinline__ int ilog2_pow2(uint32_t x) {
#ifdef __CUDA_ARCH__
  return 31 - __clz(x);
#else
  return 31 - __builtin_clz(x);
#endif
}

// Number of GPU counts of unit (j, t) and the gi-th one (§N2).
__device__ __forceinline__ int unit_num_G(const Params &P, int j, int t) {
  const int cap = P.ty[t].cap, ng = P.ng[j];
  if (P.gpu_set == 0) return (ng >= 2 && ng / 2 <= cap) + (ng <= cap) + (2 * ng <= cap);
  return ilog2_pow2(cap) + 1;
}
__device__ __forceinline__ int unit_G(const Params &P, int j, int t, int gi) {
  if (P.gpu_set == 1) return 1 << gi;
  const int cap = P.ty[t].cap, ng = P.ng[j];
  int cand[3] = {ng / 2, ng, 2 * ng};
  int first = (ng >= 2 && ng / 2 <= cap) ? 0 : 1;
  (void)cap;
  return cand[first + gi];
}

// ceil(a * b / 2^e) for a * b < 2^127, e in [1, 63], result < 2^64 (§N0: the
// alpha-beta numerators need 128-bit intermediates; __umul64hi + low product).
__device__ __forceinline__ uint64_t mul_shr_ceil(uint64_t a, uint64_t b, int e) {
  uint64_t lo = a * b;
  uint64_t hi = __umul64hi(a, b);
  const uint64_t add = (1ull << e) - 1;
  const uint64_t lo2 = lo + add;
  hi += (lo2 < lo);
  return (hi << (64 - e)) | (lo2 >> e);
}

// Warp-wide inclusive scan of int64 values.
__device__ __forceinline__ int64_t warp_incl_scan(int64_t x, int lane) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    int64_t y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x += y;
  }
  return x;
}

__device__ __forceinline__ int warp_max_int(int x) {
  return __reduce_max_sync(0xffffffffu, x);  // redux.sync: one instruction, no shuffle rounds
}

__device__ __forceinline__ int warp_sum_int(int x) {
  return (int)__reduce_add_sync(0xffffffffu, (unsigned)x);
}

// Warp-wide inclusive scan of int32 values (one shuffle per step).
__device__ __forceinline__ int warp_incl_scan32(int x, int lane) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x += y;
  }
  return x;
}

}  // namespace crius
