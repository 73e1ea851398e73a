// exchange.cuh -- receiver side of the fused all-gather (the
// "fused-collective option"): k_estimate's epilogue stores each Cell record
// straight into every rank's window over NVLink peer memory and its last CTA
// raises one arrival flag per receiving rank (estimate.cuh, exchange_signal);
// here a rank waits, on its stream, for the flags of every sender before the
// round reads the window.  Replaces estimate -> ncclAllGather -> k_compact
// with estimate(+P2P stores) -> k_xch_wait.
#pragma once
#include "common.cuh"

namespace crius {

#ifndef CRIUS_XCH_SPIN_NS
#define CRIUS_XCH_SPIN_NS 30000000000ll  // 30 s: a peer that never signals is a bug; trap, do not hang
#endif

// Thread r acquires flags[r] >= epoch (rank r's records of this step are
// visible); a bounded spin traps instead of hanging the device.
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long ns;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
  return ns;
}

__global__ void k_xch_wait(const int64_t *flags, int world, int64_t epoch) {
  const int r = threadIdx.x;
  if (r < world) {
    const unsigned long long t0 = global_ns();
    for (unsigned spins = 1;; ++spins) {
      int64_t v;
      asm volatile("ld.acquire.sys.global.s64 %0, [%1];" : "=l"(v) : "l"(flags + r) : "memory");
      if (v >= epoch) break;
      __nanosleep(128);
      if ((spins & 1023u) == 0 && global_ns() - t0 > (unsigned long long)CRIUS_XCH_SPIN_NS) __trap();
    }
  }
  __syncthreads();
}

}  // namespace crius
