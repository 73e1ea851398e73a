// estimate.cuh -- K2+K3+K4 fused: per-unit stage DP, plan cost, per-Cell argmin.
//
// One warp owns one unit u = (job j, GPU type t) at a time (persistent warps,
// atomic work counter).  Every Cell of the unit shares the unit's profile rows,
// so the warp stages them ONCE as inclusive prefix sums in shared memory
// (coalesced loads: 32 consecutive layers per warp load), then:
//
//  K2  min-max stage DP over tp=1 per-layer compute for S = 1..S_top (SURVEY
//      §N3; "keeping the computation latency of each stage
//      similar"), O(log L) per DP entry: f[s-1][.] is non-decreasing and
//      P[i]-P[.] strictly decreasing (c >= 1), so the lowest argmin is one of
//      the two neighbours of the first k with f[s-1][k] >= P[i]-P[k] (R0, A-4);
//  K3  one lane per (Cell, plan): T_sigma, sync_sigma, mem_sigma of every stage
//      from prefix differences, T_iter = sum T + (B-1) max T + max sync (§N5;
//      PAPER.md:381-390 with the north_star steady-state term);
//  K4  segmented warp-shuffle min over (T_iter, p) per Cell; a Cell whose plans
//      span several 32-lane chunks carries its partial minimum (PAPER.md:386
//      "the best among them is taken as the Cell's estimation"; lowest p wins).
//
// No tensor cores: nothing here is a dense contraction (north_star).
#pragma once
#include "common.cuh"

namespace crius {

struct EstArgs {
  const int32_t *cG, *cS;
  const int64_t *plan_off, *ucb, *upb;
  int64_t unit_begin, unit_end;
  CellResult *out;
  int16_t *splits;
  int32_t split_stride;
  int32_t *work_counter;
  // per-warp shared-memory layout (byte offsets)
  int32_t Lp, K1e, Stop, maxCells;
  int32_t off_PC, off_PW, off_PA, off_PV, off_PN, off_BND, off_F, off_ARG, off_BD, off_CELL;
  int32_t warp_bytes;
};

// Inclusive prefix of a profile row into dst[0..L] (dst[0] = 0).
template <typename Src>
__device__ __forceinline__ void warp_prefix(int64_t *dst, const Src *__restrict__ src, int L,
                                            int lane) {
  int64_t carry = 0;
  if (lane == 0) dst[0] = 0;
  for (int b = 0; b < L; b += 32) {
    const int64_t x = (b + lane < L) ? (int64_t)__ldg(src + b + lane) : 0;
    const int64_t inc = warp_incl_scan(x, lane);
    if (b + lane < L) dst[b + lane + 1] = carry + inc;
    carry += __shfl_sync(0xffffffffu, inc, 31);
  }
}

struct UnitCtx {
  const int64_t *PC, *PW, *PA, *PV, *PN, *BND;
  const int16_t *BD;
  int32_t Lp, lGB, lgpn, b_mode, nB, kst;
  int64_t memt, a_in, b_in, a_x, b_x;
  const int32_t *lBv;
};

// T_iter of plan p of Cell (G, S) (§N5), or kInf when infeasible (A-12, memory).
__device__ __forceinline__ int64_t plan_time(const UnitCtx &U, int G, int S, int p) {
  const int lS = ilog2_pow2(S), lg = ilog2_pow2(G) - lS;
  int k, lB;
  if (U.b_mode == 0) {
    k = p;
    lB = lS + 2;  // B = 4S (GPipe)
  } else {
    k = p / U.nB;
    lB = U.lBv[p - k * U.nB];
  }
  const int ldp = lg - k;
  if (lB + ldp > U.lGB) return kInf;  // B * dp > GB: microbatch below one sample
  const int lmb = U.lGB - lB - ldp;   // mb = GB / (B dp)
  const uint64_t tp = 1ull << k, dp = 1ull << ldp;
  const bool tp_in = k <= U.lgpn, dp_in = lg <= U.lgpn;  // A-15
  const uint64_t a_tp = tp_in ? U.a_in : U.a_x, b_tp = tp_in ? U.b_in : U.b_x;
  const uint64_t a_dp = dp_in ? U.a_in : U.a_x, b_dp = dp_in ? U.b_in : U.b_x;
  const int64_t *PCk = U.PC + k * U.Lp;
  const int16_t *bd = U.BD + (S - 1) + lS;
  const int node_mask = lg < U.lgpn ? (1 << (U.lgpn - lg)) - 1 : 0;
  int a = 0;
  int64_t pc_a = 0, pv_a = 0, pn_a = 0, pw_a = 0, pa_a = 0;
  int64_t sumT = 0, maxT = 0, maxSync = 0;
  for (int s = 0; s < S; ++s) {
    const int e = bd[s + 1];
    const int64_t pc_e = PCk[e], pv_e = U.PV[e], pn_e = U.PN[e], pw_e = U.PW[e], pa_e = U.PA[e];
    const int64_t W = pw_e - pw_a, A = pa_e - pa_a;
    // mem = cdiv(kst W + (GB/dp) A, tp) <= mem_t  (A-13)
    const uint64_t mem = ((uint64_t)(U.kst * W + (A << (U.lGB - ldp))) + tp - 1) >> k;
    if (mem > (uint64_t)U.memt) return kInf;
    // comp = mb * sum c ; tpc = AR(tp, l_tp, mb sum tpv, sum tpn)
    uint64_t T = (uint64_t)(pc_e - pc_a) << lmb;
    if (k) {
      const uint64_t V = (uint64_t)(pv_e - pv_a) << lmb;
      T += (uint64_t)(pn_e - pn_a) * (2 * (tp - 1)) * a_tp + mul_shr_ceil(2 * (tp - 1) * V, b_tp, k + 20);
    }
    // inb = P2P(l_b, cdiv(mb bnd, tp)) + AG(tp, l_tp, mb bnd) for s >= 1
    if (s) {
      const uint64_t Vb = (uint64_t)U.BND[a - 1] << lmb;
      const bool b_in = (s & node_mask) != 0;
      T += (b_in ? U.a_in : U.a_x) + mul_shr_ceil((Vb + tp - 1) >> k, b_in ? U.b_in : U.b_x, 20);
      if (k) T += (tp - 1) * a_tp + mul_shr_ceil((tp - 1) * Vb, b_tp, k + 20);
    }
    // sync = AR(dp, l_dp, cdiv(W, tp), 1)
    if (ldp) {
      const uint64_t Wt = ((uint64_t)W + tp - 1) >> k;
      const uint64_t sy = 2 * (dp - 1) * a_dp + mul_shr_ceil(2 * (dp - 1) * Wt, b_dp, ldp + 20);
      maxSync = max(maxSync, (int64_t)sy);
    }
    sumT += (int64_t)T;
    maxT = max(maxT, (int64_t)T);
    a = e;
    pc_a = pc_e;
    pv_a = pv_e;
    pn_a = pn_e;
    pw_a = pw_e;
    pa_a = pa_e;
  }
  return sumT + (int64_t)((1ll << lB) - 1) * maxT + maxSync;
}

template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32) k_estimate(Params P, EstArgs A) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned char *base = smem + (size_t)wid * A.warp_bytes;
  int64_t *PC = (int64_t *)(base + A.off_PC);
  int64_t *PW = (int64_t *)(base + A.off_PW);
  int64_t *PA = (int64_t *)(base + A.off_PA);
  int64_t *PV = (int64_t *)(base + A.off_PV);
  int64_t *PN = (int64_t *)(base + A.off_PN);
  int64_t *BND = (int64_t *)(base + A.off_BND);
  int64_t *F0 = (int64_t *)(base + A.off_F), *F1 = F0 + A.Lp;
  uint8_t *ARG = (uint8_t *)(base + A.off_ARG);
  int16_t *BD = (int16_t *)(base + A.off_BD);
  int32_t *CG = (int32_t *)(base + A.off_CELL);
  int32_t *CS = CG + (A.maxCells + 1), *CP = CS + (A.maxCells + 1);
  const int Lp = A.Lp;
  const int64_t out_cell_base = A.ucb[A.unit_begin];

  for (;;) {
    int64_t u = 0;
    if (lane == 0) u = A.unit_begin + atomicAdd(A.work_counter, 1);
    u = __shfl_sync(0xffffffffu, u, 0);
    if (u >= A.unit_end) break;

    const int j = (int)(u / P.T), t = (int)(u % P.T);
    const int64_t cb = A.ucb[u];
    const int nc = (int)(A.ucb[u + 1] - cb);
    int16_t *split_out = A.splits ? A.splits + (u - A.unit_begin) * A.split_stride : nullptr;
    if (nc == 0) {
      if (split_out)
        for (int q = lane; q < A.split_stride; q += 32) split_out[q] = -1;
      continue;
    }
    const int64_t pb = A.upb[u];
    const int npu = (int)(A.upb[u + 1] - pb);
    const int L = P.L[j];
    const int64_t off = P.off[j];

    // ---- Cells of the unit -> shared memory
    int smax = 0, gmax = 0;
    for (int i = lane; i < nc; i += 32) {
      const int G = A.cG[cb + i], S = A.cS[cb + i];
      CG[i] = G;
      CS[i] = S;
      CP[i] = (int)(A.plan_off[cb + i] - pb);
      smax = max(smax, S);
      gmax = max(gmax, G / S);
    }
    if (lane == 0) CP[nc] = npu;
    smax = warp_max_int(smax);
    gmax = warp_max_int(gmax);
    const int K1u = ilog2_pow2(gmax) + 1;

    // ---- A3: prefix staging (HBM -> shared, once per unit)
    for (int k = 0; k < K1u; ++k)
      warp_prefix(PC + k * Lp, P.c + ((int64_t)t * P.K1 + k) * P.TL + off, L, lane);
    warp_prefix(PW, P.w + off, L, lane);
    warp_prefix(PA, P.act + off, L, lane);
    warp_prefix(PV, P.tpv + off, L, lane);
    warp_prefix(PN, P.tpn + off, L, lane);
    for (int l = lane; l < L; l += 32) BND[l] = __ldg(P.bnd + off + l);
    __syncwarp();

    // ---- K2: stage DP rows f[1..smax] over P0 = PC[0]
    const int64_t *P0 = PC;
    for (int i = lane; i <= L; i += 32) F0[i] = P0[i];
    __syncwarp();
    int64_t *fp = F0, *fc = F1;
    for (int s = 2; s <= smax; ++s) {
      uint8_t *arow = ARG + s * Lp;
      for (int i = s + lane; i <= L; i += 32) {
        const int64_t Pi = P0[i];
        int lo = s - 1, hi = i;  // first k in [s-1, i-1] with f[s-1][k] >= P[i]-P[k], else i
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (fp[mid] >= Pi - P0[mid])
            hi = mid;
          else
            lo = mid + 1;
        }
        int a;
        int64_t val;
        if (lo == s - 1) {
          a = lo;
          val = fp[lo];
        } else {
          const int64_t v0 = Pi - P0[lo - 1];  // value at k1-1 (its max is the stage term)
          if (lo == i) {
            a = lo - 1;
            val = v0;
          } else {
            const int64_t v1 = fp[lo];
            if (v0 <= v1) {
              a = lo - 1;
              val = v0;
            } else {
              a = lo;
              val = v1;
            }
          }
        }
        fc[i] = val;
        arow[i] = (uint8_t)a;
      }
      __syncwarp();
      int64_t *tmp = fp;
      fp = fc;
      fc = tmp;
    }

    // ---- R0 backtrack, one lane per S = 2^si
    const int nSi = ilog2_pow2(smax) + 1;
    if (lane < nSi) {
      const int S = 1 << lane;
      int16_t *bd = BD + (S - 1) + lane;
      bd[S] = (int16_t)L;
      int b = L;
      for (int s = S; s >= 2; --s) {
        b = ARG[s * Lp + b];
        bd[s - 1] = (int16_t)b;
      }
      bd[0] = 0;
    }
    __syncwarp();
    if (split_out) {
      const int used = (1 << nSi) - 1 + nSi;
      for (int q = lane; q < A.split_stride; q += 32) split_out[q] = q < used ? BD[q] : (int16_t)-1;
    }

    // ---- K3 + K4: every plan of every Cell of the unit, segmented argmin
    UnitCtx U;
    U.PC = PC;
    U.PW = PW;
    U.PA = PA;
    U.PV = PV;
    U.PN = PN;
    U.BND = BND;
    U.BD = BD;
    U.Lp = Lp;
    U.lGB = ilog2_pow2(P.gb[j]);
    U.lgpn = P.ty[t].lgpn;
    U.b_mode = P.b_mode;
    U.nB = P.nB;
    U.kst = P.kst[j];
    U.memt = P.ty[t].mem;
    U.a_in = P.ty[t].a_in;
    U.b_in = P.ty[t].b_in;
    U.a_x = P.ty[t].a_x;
    U.b_x = P.ty[t].b_x;
    U.lBv = P.lB;

    int carry_ci = -1, carry_p = 0;
    int64_t carry_T = kInf;
    for (int f0 = 0; f0 < npu; f0 += 32) {
      const int f = f0 + lane;
      const bool valid = f < npu;
      int ci = nc, p = 0;
      int64_t T = kInf;
      if (valid) {
        int lo = 0, hi = nc - 1;  // largest ci with CP[ci] <= f
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (CP[mid] <= f)
            lo = mid;
          else
            hi = mid - 1;
        }
        ci = lo;
        p = f - CP[ci];
        T = plan_time(U, CG[ci], CS[ci], p);
      }
      // segmented inclusive min-scan over (T, p); left lanes have lower p
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int64_t oT = __shfl_up_sync(0xffffffffu, T, d);
        const int op = __shfl_up_sync(0xffffffffu, p, d);
        const int oc = __shfl_up_sync(0xffffffffu, ci, d);
        if (lane >= d && oc == ci && oT <= T) {
          T = oT;
          p = op;
        }
      }
      const int next_ci = __shfl_down_sync(0xffffffffu, ci, 1);
      const bool tail = valid && (lane == 31 || next_ci != ci);
      if (tail && ci == carry_ci && carry_T <= T) {
        T = carry_T;
        p = carry_p;
      }
      const bool done = valid && (f + 1 == CP[ci + 1]);
      if (tail && done) {
        CellResult r;
        r.t_ns = T;
        r.plan = T == kInf ? -1 : p;
        r.flags = T == kInf ? 0 : 1;
        A.out[cb + ci - out_cell_base] = r;
      }
      const int c31 = __shfl_sync(0xffffffffu, ci, 31);
      const int64_t T31 = __shfl_sync(0xffffffffu, T, 31);
      const int p31 = __shfl_sync(0xffffffffu, p, 31);
      const bool open31 = __shfl_sync(0xffffffffu, (int)(valid && !done), 31);
      if (open31) {
        carry_ci = c31;
        carry_T = T31;
        carry_p = p31;
      } else {
        carry_ci = -1;
        carry_T = kInf;
      }
    }
    __syncwarp();
  }
}

}  // namespace crius
