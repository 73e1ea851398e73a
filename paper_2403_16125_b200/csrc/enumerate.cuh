// enumerate.cuh -- K1: Cell enumeration on the device (PAPER.md
// :481-488 "Initializing Cells": G in {N_G/2, N_G, 2N_G}, S in {1,2,4,..}).
//
// Cells are generated per unit u = (job j, type t) = j*T + t in the order
// (G asc, S asc); a unit's Cells are contiguous and units are in (j, t) order,
// so Cell ids are global positions.  Three steps: per-unit closed-form counts,
// an exclusive scan (cells, plans, work weight), and a per-unit fill.
#pragma once
#include "common.cuh"

namespace crius {

struct UnitCounts {
  int64_t *ncells, *nplans, *weight;  // [n_units] (scanned in place into [n_units+1])
  int32_t *stats;                     // [0] max cells/unit, [1] max S, [2] max g
};

// Per-unit counts (one thread per unit).  weight = L*min(L,s_max)*ceil(log2 L)
// + sum_cells nplans*S: the DP probes plus the stage evaluations of the unit
// (SURVEY §8(e)), used to balance contiguous unit ranges across ranks.
__global__ void k_unit_count(Params P, UnitCounts U, int64_t n_units) {
  const int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (u >= n_units) return;
  const int j = (int)(u / P.T), t = (int)(u % P.T);
  const int L = P.L[j];
  const int nG = unit_num_G(P, j, t);
  int64_t nc = 0, np = 0, wt = 0;
  int smax = 0, gmax = 0;
  for (int gi = 0; gi < nG; ++gi) {
    const int G = unit_G(P, j, t, gi);
    const int lim = min(min(G, L), P.s_max);
    for (int S = 1; S <= lim; S <<= 1) {
      const int g = G / S;
      if (g > P.g_max) continue;
      const int np_c = (ilog2_pow2(g) + 1) * P.nB;
      nc += 1;
      np += np_c;
      wt += (int64_t)np_c * S;
      smax = max(smax, S);
      gmax = max(gmax, g);
    }
  }
  if (nc > 0) {
    int lg = 0;
    while ((1 << lg) < L) ++lg;
    wt += (int64_t)L * min(L, P.s_max) * max(lg, 1);
  }
  U.ncells[u] = nc;
  U.nplans[u] = np;
  U.weight[u] = wt;
  atomicMax(&U.stats[0], (int)nc);
  atomicMax(&U.stats[1], smax);
  atomicMax(&U.stats[2], gmax);
}

// ---- exclusive scan of three int64 arrays, in place, n -> n+1 entries -----
constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

struct Scan3 {
  int64_t *a[3];
};

__device__ __forceinline__ void block_excl_scan3(int64_t v[3], int64_t tot[3]) {
  __shared__ int64_t warp_sums[3][32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int64_t incl[3];
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    incl[q] = warp_incl_scan(v[q], lane);
    if (lane == 31) warp_sums[q][wid] = incl[q];
  }
  __syncthreads();
  if (wid == 0) {
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const int nw = blockDim.x >> 5;
      int64_t s = lane < nw ? warp_sums[q][lane] : 0;
      s = warp_incl_scan(s, lane);
      warp_sums[q][lane] = s;
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    const int64_t before = wid ? warp_sums[q][wid - 1] : 0;
    tot[q] = warp_sums[q][(blockDim.x >> 5) - 1];
    v[q] = before + incl[q] - v[q];
  }
  __syncthreads();
}

// Tile-local exclusive scan; tile totals to `sums` (length n_tiles).
__global__ void __launch_bounds__(kScanThreads) k_scan_tiles(Scan3 X, int64_t n, Scan3 sums) {
  const int64_t base = blockIdx.x * (int64_t)kScanTile + threadIdx.x * kScanItems;
  int64_t loc[3][kScanItems], v[3], tot[3];
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    v[q] = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
      loc[q][i] = base + i < n ? X.a[q][base + i] : 0;
      v[q] += loc[q][i];
    }
  }
  block_excl_scan3(v, tot);
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    int64_t run = v[q];
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
      if (base + i < n) X.a[q][base + i] = run;
      run += loc[q][i];
    }
    if (threadIdx.x == 0) sums.a[q][blockIdx.x] = tot[q];
  }
}

// Single block: exclusive scan of the tile sums (any length), grand total to [n_tiles].
__global__ void __launch_bounds__(kScanThreads) k_scan_sums(Scan3 S, int64_t n_tiles) {
  int64_t carry[3] = {0, 0, 0};
  for (int64_t b0 = 0; b0 < n_tiles; b0 += kScanThreads) {
    const int64_t i = b0 + threadIdx.x;
    int64_t v[3], tot[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) v[q] = i < n_tiles ? S.a[q][i] : 0;
    block_excl_scan3(v, tot);
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      if (i < n_tiles) S.a[q][i] = carry[q] + v[q];
      carry[q] += tot[q];
    }
  }
  if (threadIdx.x == 0)
#pragma unroll
    for (int q = 0; q < 3; ++q) S.a[q][n_tiles] = carry[q];
}

__global__ void k_scan_add(Scan3 X, int64_t n, Scan3 sums, int64_t n_tiles) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) {
    const int64_t tile = i / kScanTile;
#pragma unroll
    for (int q = 0; q < 3; ++q) X.a[q][i] += sums.a[q][tile];
  }
  if (i == 0)
#pragma unroll
    for (int q = 0; q < 3; ++q) X.a[q][n] = sums.a[q][n_tiles];
}

// Fill the Cell SoA (one thread per unit; its Cells are contiguous).
__global__ void k_unit_fill(Params P, Cells C, int64_t n_units) {
  const int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (u >= n_units) return;
  const int j = (int)(u / P.T), t = (int)(u % P.T);
  const int L = P.L[j];
  const int nG = unit_num_G(P, j, t);
  int64_t ci = C.unit_cell_begin[u], po = C.unit_plan_begin[u];
  for (int gi = 0; gi < nG; ++gi) {
    const int G = unit_G(P, j, t, gi);
    const int lim = min(min(G, L), P.s_max);
    for (int S = 1; S <= lim; S <<= 1) {
      const int g = G / S;
      if (g > P.g_max) continue;
      const int np_c = (ilog2_pow2(g) + 1) * P.nB;
      C.job[ci] = j;
      C.type[ci] = t;
      C.G[ci] = G;
      C.S[ci] = S;
      C.nplans[ci] = np_c;
      C.plan_off[ci] = po;
      ++ci;
      po += np_c;
    }
  }
}

// Round priority pi (A-18): jobs ordered by (submit, id) ascending.  Ids are
// unique, so the key order is total and no sort needs to be stable: tiles of
// kPrioTile jobs are sorted in shared memory (bitonic), then runs of doubling
// width are merged -- each element's output position is its rank in its own
// run plus the number of smaller keys in the partner run (binary search).
// pi[pos] = j and rank[j] = pos.
constexpr int kPrioTile = 2048;  // jobs per tile (1024 threads x 2)

struct PrioKey {
  int64_t sub, id;
  int32_t j;
};

__device__ __forceinline__ bool prio_less(int64_t s1, int64_t i1, int64_t s2, int64_t i2) {
  return s1 < s2 || (s1 == s2 && i1 < i2);
}

__global__ void __launch_bounds__(1024) k_prio_tiles(const int64_t *__restrict__ submit,
                                                     const int64_t *__restrict__ id, int32_t J,
                                                     int64_t *osub, int64_t *oid, int32_t *oj) {
  __shared__ int64_t ss[kPrioTile], si[kPrioTile];
  __shared__ int32_t sj[kPrioTile];
  const int base = blockIdx.x * kPrioTile;
  for (int i = threadIdx.x; i < kPrioTile; i += blockDim.x) {
    const int j = base + i;
    const bool in = j < J;
    ss[i] = in ? submit[j] : INT64_MAX;  // padding sorts last (ids break the tie)
    si[i] = in ? id[j] : INT64_MAX;
    sj[i] = in ? j : -1;
  }
  __syncthreads();
  for (int k = 2; k <= kPrioTile; k <<= 1)
    for (int d = k >> 1; d > 0; d >>= 1) {
      for (int i = threadIdx.x; i < kPrioTile; i += blockDim.x) {
        const int l = i ^ d;
        if (l > i) {
          const bool up = (i & k) == 0;
          const bool gt = prio_less(ss[l], si[l], ss[i], si[i]) ||
                          (ss[l] == ss[i] && si[l] == si[i] && sj[l] < sj[i]);
          if (gt == up) {
            const int64_t a = ss[i], b = si[i];
            const int32_t c = sj[i];
            ss[i] = ss[l];
            si[i] = si[l];
            sj[i] = sj[l];
            ss[l] = a;
            si[l] = b;
            sj[l] = c;
          }
        }
      }
      __syncthreads();
    }
  for (int i = threadIdx.x; i < kPrioTile; i += blockDim.x) {
    const int o = base + i;
    if (o < J) {
      osub[o] = ss[i];
      oid[o] = si[i];
      oj[o] = sj[i];
    }
  }
}

// Merge runs of width W (sorted) pairwise into runs of width 2W.
__global__ void k_prio_merge(const int64_t *__restrict__ isub, const int64_t *__restrict__ iid,
                             const int32_t *__restrict__ ij, int32_t J, int32_t W, int64_t *osub,
                             int64_t *oid, int32_t *oj) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= J) return;
  const int run = i / W, p = i - run * W;
  const int pb = (run ^ 1) * W;  // partner run [pb, pe)
  const int pe = min(pb + W, J);
  const int64_t s = isub[i], d = iid[i];
  int cnt = 0;
  if (pb < J) {  // number of partner keys below (s, d)
    int lo = pb, hi = pe;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (prio_less(isub[mid], iid[mid], s, d)) lo = mid + 1;
      else hi = mid;
    }
    cnt = lo - pb;
  }
  const int o = (run & ~1) * W + p + cnt;
  osub[o] = s;
  oid[o] = d;
  oj[o] = ij[i];
}

__global__ void k_priority_scatter(const int32_t *order, int32_t J, int32_t *pi, int32_t *rank) {
  const int pos = blockIdx.x * blockDim.x + threadIdx.x;
  if (pos < J) {
    const int j = order[pos];
    pi[pos] = j;
    rank[j] = pos;
  }
}

// Device-side profile validation, one block per job of [j0, j0 +
// gridDim.x): the job's max over c (every type and plane), min over c, and the
// per-layer sums; thread 0 then evaluates the overflow bounds of the plan
// cost and writes code[j]: 0 ok, 1 negative per-layer value, 2 L*max(c)*GB >=
// 2^52, 3 an alpha-beta numerator >= 2^63, 4 kst*sum(w) + GB*sum(act) >=
// 2^62, 5 the T_iter bound >= 2^62.  min_c collects the global min of c.
struct BoundArgs {
  int64_t amax, bmax;  // max alpha / beta over types and link classes
  int64_t p;           // g_max (tp, dp <= g <= g_max)
  int64_t bmax_list;   // b_mode 1: largest B; 0: B = 4 min(L, s_max)
};

__device__ __forceinline__ __int128 warp_sum128(__int128 x) {
  for (int d = 16; d > 0; d >>= 1) {
    const unsigned long long lo = __shfl_xor_sync(0xffffffffu, (unsigned long long)x, d);
    const long long hi = __shfl_xor_sync(0xffffffffu, (long long)(x >> 64), d);
    x += ((__int128)hi << 64) | (__int128)lo;
  }
  return x;
}

// blockDim.x == 64 (two warps)
__global__ void __launch_bounds__(64) k_profile_check(Params P, int j0, BoundArgs BA, int32_t *code,
                                                      int32_t *min_c) {
  typedef __int128 i128;
  __shared__ i128 s_sum[2][4];
  __shared__ int s_mx[2], s_mn[2], s_neg[2];
  __shared__ long long s_bm[2];
  const int j = j0 + blockIdx.x;
  const int64_t off = P.off[j];
  const int L = P.L[j];
  int mx = 0, mn = INT32_MAX, neg = 0;
  for (int tk = 0; tk < P.T * P.K1; ++tk) {
    const int32_t *row = P.c + (int64_t)tk * P.TL + off;
    for (int l = threadIdx.x; l < L; l += blockDim.x) {
      mx = max(mx, row[l]);
      mn = min(mn, row[l]);
    }
  }
  i128 W = 0, A = 0, V = 0, N = 0;  // exact: at most 4 values per thread, then 128-bit sums
  long long Bm = 0;
  for (int l = threadIdx.x; l < L; l += blockDim.x) {
    const int64_t w = P.w[off + l], a = P.act[off + l], bd = P.bnd[off + l], tv = P.tpv[off + l];
    const int32_t tn = P.tpn[off + l];
    neg |= (w < 0) | (a < 0) | (bd < 0) | (tv < 0) | (tn < 0);
    W += w;
    A += a;
    V += tv;
    N += tn;
    Bm = max(Bm, (long long)bd);
  }
  for (int d = 16; d > 0; d >>= 1) {
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, d));
    mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, d));
    neg |= __shfl_xor_sync(0xffffffffu, neg, d);
    Bm = max(Bm, __shfl_xor_sync(0xffffffffu, Bm, d));
  }
  W = warp_sum128(W);
  A = warp_sum128(A);
  V = warp_sum128(V);
  N = warp_sum128(N);
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    s_mx[wid] = mx;
    s_mn[wid] = mn;
    s_neg[wid] = neg;
    s_bm[wid] = Bm;
    s_sum[wid][0] = W;
    s_sum[wid][1] = A;
    s_sum[wid][2] = V;
    s_sum[wid][3] = N;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mx = max(s_mx[0], s_mx[1]);
    mn = min(s_mn[0], s_mn[1]);
    neg = s_neg[0] | s_neg[1];
    Bm = max(s_bm[0], s_bm[1]);
    const i128 Ws = s_sum[0][0] + s_sum[1][0], As = s_sum[0][1] + s_sum[1][1];
    const i128 Vs = s_sum[0][2] + s_sum[1][2], Ns = s_sum[0][3] + s_sum[1][3];
    atomicMin(min_c, mn);
    const i128 LIM52 = (i128)1 << 52, LIM62 = (i128)1 << 62, LIM63 = (i128)1 << 63, MIB = 1 << 20;
    const i128 GB = P.gb[j], Li = L, p = BA.p, amax = BA.amax, bmax = BA.bmax;
    int c = 0;
    if (neg) {
      c = 1;
    } else if (Li * mx * GB >= LIM52) {
      c = 2;
    } else if (2 * (p - 1) * GB * Vs >= LIM63 || p * GB * Bm >= LIM63 || 2 * (p - 1) * Ws >= LIM63) {
      c = 3;
    } else if ((i128)P.kst[j] * Ws + GB * As >= LIM62) {
      c = 4;
    } else {
      const i128 comp = GB * Li * mx;
      const i128 tpc = Ns * 2 * (p - 1) * amax + Li * (2 * (p - 1) * GB * Vs * bmax / MIB + 1);
      const i128 inb = Li * (amax + GB * Bm * bmax / MIB + 1 + (p - 1) * amax +
                             (p - 1) * GB * Bm * bmax / MIB + 1);
      const i128 X = comp + tpc + inb;
      const i128 sync = 2 * (p - 1) * amax + 2 * (p - 1) * Ws * bmax / MIB + 1;
      const i128 Bmax = BA.bmax_list ? (i128)BA.bmax_list : (i128)4 * min(L, P.s_max);
      if (Bmax * X + sync >= LIM62) c = 5;
    }
    code[j] = c;
  }
}

}  // namespace crius
