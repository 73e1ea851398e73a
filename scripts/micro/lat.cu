// Latency microbenchmarks for the round kernel's building blocks (1 CTA).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t ord_double(double x) {
  if (x == 0.0) x = 0.0;
  const long long b = __double_as_longlong(x);
  return b < 0 ? ~(uint64_t)b : ((uint64_t)b | 0x8000000000000000ull);
}
__device__ __forceinline__ int warp_lex_argmin(bool valid, uint64_t k, uint32_t tie) {
  if (!__ballot_sync(0xffffffffu, valid)) return -1;
  const uint32_t hi = valid ? (uint32_t)(k >> 32) : 0xffffffffu;
  const uint32_t mhi = __reduce_min_sync(0xffffffffu, hi);
  valid = valid && hi == mhi;
  const uint32_t lo = valid ? (uint32_t)k : 0xffffffffu;
  const uint32_t mlo = __reduce_min_sync(0xffffffffu, lo);
  valid = valid && lo == mlo;
  const uint32_t tt = valid ? tie : 0xffffffffu;
  const uint32_t mtt = __reduce_min_sync(0xffffffffu, tt);
  valid = valid && tt == mtt;
  return __ffs(__ballot_sync(0xffffffffu, valid)) - 1;
}

__global__ void k_argmin(int nwarps_active, int iters, long long *out, int *sink) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (wid >= nwarps_active) return;
  double v = (lane * 7919 % 31) * 1.5 + wid;
  int acc = 0;
  __syncwarp();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    const int s = warp_lex_argmin(true, ord_double(v), lane);
    acc += s;
    v += (double)(s & 1);
  }
  long long t1 = clock64();
  if (lane == 0) out[wid] = t1 - t0;
  if (acc == 12345) sink[0] = acc;
}

__global__ void k_redux(int nwarps_active, int iters, long long *out, int *sink) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (wid >= nwarps_active) return;
  unsigned x = lane * 13 + wid;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = __reduce_min_sync(0xffffffffu, x) + lane;
  long long t1 = clock64();
  if (lane == 0) out[wid] = t1 - t0;
  if (x == 12345) sink[0] = x;
}

__global__ void k_lds(int nwarps_active, int iters, long long *out, int *sink, int generic) {
  __shared__ int buf[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) buf[i] = (i * 17 + 3) & 4095;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (wid >= nwarps_active) return;
  int *volatile gp = buf;  // defeat address-space inference when generic
  int *p = generic ? gp : buf;
  int x = lane;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = p[x];
  long long t1 = clock64();
  if (lane == 0) out[wid] = t1 - t0;
  if (x == 12345) sink[0] = x;
}

__global__ void k_bar(int iters, long long *out) {
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = t1 - t0;
}

__global__ void k_ddiv(int nwarps_active, int iters, long long *out, double *sink) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (wid >= nwarps_active) return;
  double x = 1.0 + lane;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = __ddiv_rn(x + 3.0, 1.0 + (double)(i & 7));
  long long t1 = clock64();
  if (lane == 0) out[wid] = t1 - t0;
  if (x == 12345.0) sink[0] = x;
}

__global__ void k_chain(int iters, long long *out, long long *sink, double *dsink) {
  // dependent single-warp chains: int IMAD, fp64 DADD
  long long x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = x * 3 + 1;
  long long t1 = clock64();
  double d = 1.0 + threadIdx.x;
  long long t2 = clock64();
  for (int i = 0; i < iters; ++i) d = __dadd_rn(d, 0.5);
  long long t3 = clock64();
  if (threadIdx.x == 0) {
    out[0] = t1 - t0;
    out[1] = t3 - t2;
  }
  if (x == 12345) sink[0] = x;
  if (d == 12345.0) dsink[0] = d;
}

int main() {
  long long *d_out, h[32];
  int *d_sink;
  double *d_ds;
  cudaMalloc(&d_out, 32 * 8);
  cudaMalloc(&d_sink, 4);
  cudaMalloc(&d_ds, 8);
  const int it = 1000;
  for (int nw : {1, 4, 8, 32}) {
    k_argmin<<<1, 1024>>>(nw, it, d_out, d_sink);
    cudaMemcpy(h, d_out, 8 * 32, cudaMemcpyDeviceToHost);
    printf("warp_lex_argmin  warps %2d : %.1f cycles/op\n", nw, h[0] / (double)it);
    k_redux<<<1, 1024>>>(nw, it, d_out, d_sink);
    cudaMemcpy(h, d_out, 8 * 32, cudaMemcpyDeviceToHost);
    printf("redux.min chain  warps %2d : %.1f cycles/op\n", nw, h[0] / (double)it);
    k_lds<<<1, 1024>>>(nw, it, d_out, d_sink, 0);
    cudaMemcpy(h, d_out, 8 * 32, cudaMemcpyDeviceToHost);
    printf("LDS chain        warps %2d : %.1f cycles/op\n", nw, h[0] / (double)it);
    k_lds<<<1, 1024>>>(nw, it, d_out, d_sink, 1);
    cudaMemcpy(h, d_out, 8 * 32, cudaMemcpyDeviceToHost);
    printf("generic LD chain warps %2d : %.1f cycles/op\n", nw, h[0] / (double)it);
    k_ddiv<<<1, 1024>>>(nw, it, d_out, d_ds);
    cudaMemcpy(h, d_out, 8 * 32, cudaMemcpyDeviceToHost);
    printf("ddiv chain       warps %2d : %.1f cycles/op\n", nw, h[0] / (double)it);
  }
  for (int nt : {256, 512, 1024}) {
    k_bar<<<1, nt>>>(it, d_out);
    cudaMemcpy(h, d_out, 8, cudaMemcpyDeviceToHost);
    printf("__syncthreads %4d thr   : %.1f cycles/op\n", nt, h[0] / (double)it);
  }
  k_chain<<<1, 32>>>(it, d_out, (long long *)d_sink, d_ds);
  cudaMemcpy(h, d_out, 16, cudaMemcpyDeviceToHost);
  printf("int64 IMAD chain (1 warp) : %.1f cycles/op\n", h[0] / (double)it);
  printf("fp64 DADD chain  (1 warp) : %.1f cycles/op\n", h[1] / (double)it);
  printf("err %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
