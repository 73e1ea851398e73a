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
  int32_t off_CRAW, off_NRAW, off_POFF, off_ORD;
  int32_t warp_bytes;
  // NEXT-1 per-stage assembly (AMODE > 0): pipeline form, per-stage output
  int32_t form;            // 0: sum + (B-1) max; 1: sum + (B-1)(T_s* - T_comm,s*)
  int8_t *stage_tp;        // optional [cell][stage_stride] log2 tp of the best plan
  const int8_t *favor;     // AMODE 3 (tuner): [cell][stage_stride] log2 tp of the estimated plan
  int32_t stage_stride;
  int32_t off_ST, st_cap;  // per-warp stage table (st_cap entries)
  int32_t off_PS;          // NEXT-2 scratch: sorted gap bytes [Lp] i64, LF [Lp] i32, g [Stop] i32
  // fused exchange: every record is also stored at its GLOBAL
  // Cell index into each rank's window (peer memory over NVLink, xout[r]); the
  // last CTA to finish then raises flag xflag[r][x_rank] = x_epoch on every rank
  int32_t nx, x_rank;
  int64_t x_epoch;
  CellResult *xout[kMaxRanks];
  int64_t *xflag[kMaxRanks];
  uint32_t *x_done;        // CTA completion counter (the last CTA resets it)
  int32_t per_stage;       // b_mode 0 plan evaluation: one (Cell, k, stage) per lane
  int32_t global_out;      // records / splits at their global Cell / unit index (else
                           // relative to the launch's first Cell / unit)
};

// One Cell record: to the caller's chunk (local index) and, with the fused
// exchange, to every rank's window at the global index (16-byte P2P stores).
__device__ __forceinline__ void emit_result(const EstArgs &A, int64_t cell, int64_t base,
                                            const CellResult &r) {
  if (A.out) A.out[cell - base] = r;
  for (int q = 0; q < A.nx; ++q) A.xout[q][cell] = r;
}

// Fused exchange epilogue (all threads of the CTA).  Every CTA orders its own
// stores (bar.sync, then a system-scope fence by thread 0) before counting
// itself done; the last CTA fences again and release-stores the step's epoch
// into every rank's arrival slot for this rank: a receiver that acquires
// epoch there sees every record of this rank's Cell range (fence cumulativity).
__device__ __forceinline__ void exchange_signal(const EstArgs &A) {
  if (A.nx == 0) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    const uint32_t prev = atomicAdd(A.x_done, 1u);
    if (prev == gridDim.x - 1) {
      __threadfence_system();
      for (int q = 0; q < A.nx; ++q)
        asm volatile("st.release.sys.global.s64 [%0], %1;" ::"l"(A.xflag[q] + A.x_rank),
                     "l"(A.x_epoch)
                     : "memory");
      *A.x_done = 0u;  // next launch (stream-ordered) starts from zero
    }
  }
}

// A rank with an empty unit range still signals its (empty) contribution.
__global__ void k_xch_signal_only(EstArgs A) { exchange_signal(A); }

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

// ceil((hi:lo) / 2^e) for a 128-bit value whose result fits 64 bits; e <= 0
// means an exact left shift of the low word.
__device__ __forceinline__ uint64_t ceil_shr128(uint64_t hi, uint64_t lo, int e) {
  if (e <= 0) return lo << (-e);
  const uint64_t add = (1ull << e) - 1;
  const uint64_t lo2 = lo + add;
  hi += (lo2 < lo);
  return (hi << (64 - e)) | (lo2 >> e);
}

// T_iter of every microbatch count of one (Cell, k) group at once (§N5).  The
// per-stage memory filter and DP sync do not depend on B; mb = GB/(B dp) = 2^lmb,
// so every alpha-beta term is a 128-bit product formed once per stage (tpc: X,
// boundary send: Y, boundary all-gather: Z) followed, per B, by an exact
// ceil-shift.  Returns the best (T, p) of the group (lowest p on ties).
template <int NBG, bool kMemFeasible = false>
__device__ __forceinline__ int64_t plan_group_time(const UnitCtx &U, int G, int S, int k, int bg,
                                                   int &best_p) {
  const int lS = ilog2_pow2(S), lg = ilog2_pow2(G) - lS;
  const int ldp = lg - k;
  int lB[NBG], lmb[NBG];
  bool ok[NBG];
  bool any = false;
#pragma unroll
  for (int q = 0; q < NBG; ++q) {
    const int b = bg * NBG + q;
    lB[q] = U.b_mode == 0 ? lS + 2 : (b < U.nB ? U.lBv[b] : 0);
    lmb[q] = U.lGB - lB[q] - ldp;
    ok[q] = (U.b_mode == 0 ? q == 0 : b < U.nB) && lmb[q] >= 0;  // B dp <= GB (A-12)
    any |= ok[q];
  }
  if (!any) return kInf;
  const uint64_t tp = 1ull << k, dp = 1ull << ldp;
  const bool tp_in = k <= U.lgpn, dp_in = lg <= U.lgpn;  // A-15
  const uint64_t a_tp = tp_in ? U.a_in : U.a_x, b_tp = tp_in ? U.b_in : U.b_x;
  const uint64_t a_dp = dp_in ? U.a_in : U.a_x, b_dp = dp_in ? U.b_in : U.b_x;
  const int64_t *PCk = U.PC + k * U.Lp;
  const int16_t *bd = U.BD + (S - 1) + lS;
  const int node_mask = lg < U.lgpn ? (1 << (U.lgpn - lg)) - 1 : 0;
  int64_t sumT[NBG], maxT[NBG];
#pragma unroll
  for (int q = 0; q < NBG; ++q) sumT[q] = maxT[q] = 0;
  int64_t maxSync = 0;
  int a = 0;
  int64_t pc_a = 0, pv_a = 0, pn_a = 0, pw_a = 0, pa_a = 0;
  for (int s = 0; s < S; ++s) {
    const int e = bd[s + 1];
    const int64_t pc_e = PCk[e], pv_e = U.PV[e], pn_e = U.PN[e], pw_e = U.PW[e], pa_e = U.PA[e];
    const int64_t W = pw_e - pw_a, A = pa_e - pa_a, C = pc_e - pc_a;
    // mem = cdiv(kst W + (GB/dp) A, tp) <= mem_t  (A-13): B-independent;
    // the plain estimator's items start at the Cell's smallest memory-feasible k
    // (memory is monotone in k), so only the other modes check it here
    if (!kMemFeasible) {
      const uint64_t mem = ((uint64_t)(U.kst * W + (A << (U.lGB - ldp))) + tp - 1) >> k;
      if (mem > (uint64_t)U.memt) return kInf;
    }
    // sync = AR(dp, l_dp, cdiv(W, tp), 1): B-independent
    if (ldp) {
      const uint64_t Wt = ((uint64_t)W + tp - 1) >> k;
      const uint64_t sy = 2 * (dp - 1) * a_dp + mul_shr_ceil(2 * (dp - 1) * Wt, b_dp, ldp + 20);
      maxSync = max(maxSync, (int64_t)sy);
    }
    // tpc = N 2(tp-1) alpha + ceil(X 2^lmb / 2^(k+20)),  X = 2(tp-1) TPV beta
    uint64_t Xh = 0, Xl = 0, tpn_alpha = 0;
    if (k) {
      const uint64_t x = 2 * (tp - 1) * (uint64_t)(pv_e - pv_a);
      Xl = x * b_tp;
      Xh = __umul64hi(x, b_tp);
      tpn_alpha = (uint64_t)(pn_e - pn_a) * (2 * (tp - 1)) * a_tp;
    }
    // inb = P2P(l_b, cdiv(mb bnd, tp)) + AG(tp, l_tp, mb bnd):  Y = bnd beta_b, Z = (tp-1) bnd beta_tp
    uint64_t Yh = 0, Yl = 0, Zh = 0, Zl = 0, a_b = 0, b_b = 0, bnd = 0;
    if (s) {
      bnd = (uint64_t)U.BND[a - 1];
      const bool b_in = (s & node_mask) != 0;
      a_b = b_in ? U.a_in : U.a_x;
      b_b = b_in ? U.b_in : U.b_x;
      Yl = bnd * b_b;
      Yh = __umul64hi(bnd, b_b);
      if (k) {
        const uint64_t z = (tp - 1) * bnd;
        Zl = z * b_tp;
        Zh = __umul64hi(z, b_tp);
      }
    }
    // The B values of a group ascend, so mb = 2^lm descends and every term's
    // exponent e = k + 20 - lm grows from one B to the next: after the first
    // 128-bit ceil-shift the next is ceil(r / 2^(e - e_prev)) of the 64-bit
    // result (ceil(ceil(x / 2^a) / 2^b) = ceil(x / 2^(a+b)) for x >= 0).
    uint64_t rX = 0, rY = 0, rZ = 0;
    int pe = 0;
    bool chain = false, chainY = false;
#pragma unroll
    for (int q = 0; q < NBG; ++q) {
      if (!ok[q]) continue;
      const int lm = lmb[q];
      const int e = k + 20 - lm;
      const int d = e - pe;
      uint64_t T = (uint64_t)C << lm;
      if (k) {
        rX = chain ? (rX + (1ull << d) - 1) >> d : ceil_shr128(Xh, Xl, e);
        T += tpn_alpha + rX;
      }
      if (s) {
        if (lm >= k) {  // exponent 20 - (lm - k) == e
          rY = chainY ? (rY + (1ull << d) - 1) >> d : ceil_shr128(Yh, Yl, e);
          chainY = true;
          T += a_b + rY;
        } else {
          const int sh = k - lm;
          T += a_b + mul_shr_ceil((bnd + (1ull << sh) - 1) >> sh, b_b, 20);
        }
        if (k) {
          rZ = chain ? (rZ + (1ull << d) - 1) >> d : ceil_shr128(Zh, Zl, e);
          T += (tp - 1) * a_tp + rZ;
        }
      }
      chain = true;
      pe = e;
      sumT[q] += (int64_t)T;
      maxT[q] = max(maxT[q], (int64_t)T);
    }
    a = e;
    pc_a = pc_e;
    pv_a = pv_e;
    pn_a = pn_e;
    pw_a = pw_e;
    pa_a = pa_e;
  }
  int64_t best = kInf;
  int bq = 0;
#pragma unroll
  for (int q = 0; q < NBG; ++q) {
    if (!ok[q]) continue;
    const int64_t ti = sumT[q] + (int64_t)((1ll << lB[q]) - 1) * maxT[q] + maxSync;
    if (ti < best) {
      best = ti;
      bq = q;
    }
  }
  best_p = U.b_mode == 0 ? k : k * U.nB + bg * NBG + bq;
  return best;
}

// ---- NEXT-1: per-stage parallelism assembly ------------------------------
// Terms of stage s (layers [a, e)) run with tp = 2^k, dp = g/tp and mb =
// GB/(B dp) (§N5 evaluated with the stage's own factorisation): T, its inbound
// communication Tc (the term PAPER.md:382-384 overlaps), sync; false if the
// stage does not fit (B dp > GB or memory).
__device__ __forceinline__ bool stage_terms(const UnitCtx &U, int lg, int k, int lB, int s, int a,
                                            int e, int64_t &T, int64_t &Tc, int64_t &sync) {
  const int ldp = lg - k;
  if (lB + ldp > U.lGB) return false;
  const int lmb = U.lGB - lB - ldp;
  const uint64_t tp = 1ull << k, dp = 1ull << ldp;
  const bool tp_in = k <= U.lgpn, dp_in = lg <= U.lgpn;
  const uint64_t a_tp = tp_in ? U.a_in : U.a_x, b_tp = tp_in ? U.b_in : U.b_x;
  const uint64_t a_dp = dp_in ? U.a_in : U.a_x, b_dp = dp_in ? U.b_in : U.b_x;
  const int64_t *PCk = U.PC + k * U.Lp;
  const int64_t W = U.PW[e] - U.PW[a], A = U.PA[e] - U.PA[a];
  const uint64_t mem = ((uint64_t)(U.kst * W + (A << (U.lGB - ldp))) + tp - 1) >> k;
  if (mem > (uint64_t)U.memt) return false;
  uint64_t t = (uint64_t)(PCk[e] - PCk[a]) << lmb;
  if (k) {
    const uint64_t V = (uint64_t)(U.PV[e] - U.PV[a]) << lmb;
    t += (uint64_t)(U.PN[e] - U.PN[a]) * (2 * (tp - 1)) * a_tp + mul_shr_ceil(2 * (tp - 1) * V, b_tp, k + 20);
  }
  uint64_t inb = 0;
  if (s) {
    const int node_mask = lg < U.lgpn ? (1 << (U.lgpn - lg)) - 1 : 0;
    const uint64_t Vb = (uint64_t)U.BND[a - 1] << lmb;
    const bool b_in = (s & node_mask) != 0;
    inb = (b_in ? U.a_in : U.a_x) + mul_shr_ceil((Vb + tp - 1) >> k, b_in ? U.b_in : U.b_x, 20);
    if (k) inb += (tp - 1) * a_tp + mul_shr_ceil((tp - 1) * Vb, b_tp, k + 20);
  }
  T = (int64_t)(t + inb);
  Tc = (int64_t)inb;
  sync = 0;
  if (ldp) {
    const uint64_t Wt = ((uint64_t)W + tp - 1) >> k;
    sync = (int64_t)(2 * (dp - 1) * a_dp + mul_shr_ceil(2 * (dp - 1) * Wt, b_dp, ldp + 20));
  }
  return true;
}

// Exact optimum over the assembled plans of one Cell (AMODE 1: each stage
// DP-only or TP-only, the paper's 2^S plans; AMODE 2: every
// factorisation per stage) without enumerating them.  Enumerate the slowest
// stage s* with its choice (fixing M = T_s*, Tc_s*) and a bound Y on the max
// sync; every other stage then independently takes its cheapest choice with
// T < M (stages before s*: s* is the FIRST slowest) or T <= M (after), sync <= Y.
// F(s*, q*, Y) = sum + (B-1)(M - [form] Tc*) + Y bounds the latency of that
// plan from above and equals it for the optimum's own (s*, q*, max sync), so
// the minimum over all enumerations is the optimum and the plan built at the
// minimiser attains it.  Lanes split the (s*, q*) candidates.
template <int AMODE>
__device__ void assembled_cell(const UnitCtx &U, const EstArgs &A, int G, int S, int lane,
                               int64_t *STT, int64_t *STC, int64_t *STY, uint8_t *STOK,
                               int64_t &bestF, int &bestB, int8_t *kout, const int8_t *fav) {
  const int lS = ilog2_pow2(S), lg = ilog2_pow2(G) - lS;
  const int nq = AMODE == 1 ? (lg ? 2 : 1) : lg + 1;
  CRIUS_CHECK(S * nq <= A.st_cap);
  // half-hybrid point (sqrt(g) x sqrt(g), Fig. pruning); for odd log2 g it
  // falls between two factorisations and both neighbours belong to both halves
  const int kdp_hi = (lg + 1) >> 1, ktp_lo = lg >> 1;
  const int E = S * nq;
  const int16_t *bd = U.BD + (S - 1) + lS;
  bestF = kInf;
  bestB = -1;
  int bestE = -1;
  int64_t bestY = 0;
  const int nBv = U.b_mode == 0 ? 1 : U.nB;
  for (int bi = 0; bi < nBv; ++bi) {
    const int lB = U.b_mode == 0 ? lS + 2 : U.lBv[bi];
    for (int e = lane; e < E; e += 32) {
      const int s = e / nq, q = e - s * nq;
      const int k = AMODE == 1 ? (q ? lg : 0) : q;
      int64_t T = 0, Tc = 0, sy = 0;
      bool ok = stage_terms(U, lg, k, lB, s, bd[s], bd[s + 1], T, Tc, sy);
      if (AMODE == 3) {  // tuner: DP favour keeps k <= khalf, TP favour keeps k >= khalf
        const bool tp_fav = fav[s] > 0;
        ok = ok && (tp_fav ? k >= ktp_lo : k <= kdp_hi);
      }
      STT[e] = T;
      STC[e] = Tc;
      STY[e] = sy;
      STOK[e] = ok;
    }
    __syncwarp();
    const int64_t Bm1 = (1ll << lB) - 1;
    int64_t myF = kInf, myY = 0;
    int myE = -1;
    for (int es = lane; es < E; es += 32) {
      if (!STOK[es]) continue;
      const int ss = es / nq;
      const int64_t M = STT[es], tcs = A.form ? STC[es] : 0, sys = STY[es];
      for (int yi = 0; yi <= E; ++yi) {
        if (yi < E && !STOK[yi]) continue;
        const int64_t Y = yi < E ? STY[yi] : 0;
        if (Y < sys) continue;
        int64_t sum = 0;
        bool ok = true;
        for (int s = 0; s < S && ok; ++s) {
          if (s == ss) continue;
          int64_t bt = kInf;
          for (int q = 0; q < nq; ++q) {
            const int ee = s * nq + q;
            const int64_t T = STT[ee];
            if (STOK[ee] && STY[ee] <= Y && (s < ss ? T < M : T <= M) && T < bt) bt = T;
          }
          ok = bt != kInf;
          sum += bt;
        }
        if (!ok) continue;
        const int64_t F = sum + M + Bm1 * (M - tcs) + Y;
        if (F < myF) {
          myF = F;
          myE = es;
          myY = Y;
        }
      }
    }
    // warp min of F (first lane on ties: any minimiser is a valid plan)
    int64_t wF = myF;
    for (int d = 16; d > 0; d >>= 1) wF = min(wF, __shfl_xor_sync(0xffffffffu, wF, d));
    const unsigned who = __ballot_sync(0xffffffffu, myF == wF && myE >= 0);
    if (wF < bestF && who) {
      const int src = __ffs(who) - 1;
      bestF = wF;
      bestB = bi;
      bestE = __shfl_sync(0xffffffffu, myE, src);
      bestY = __shfl_sync(0xffffffffu, myY, src);
      // rebuild the plan now: the stage table is this B's
      if (kout && lane == 0) {
        const int ss = bestE / nq;
        const int64_t M = STT[bestE];
        for (int s = 0; s < S; ++s) {
          int bq = bestE - ss * nq;
          if (s != ss) {
            int64_t bt = kInf;
            for (int q = 0; q < nq; ++q) {
              const int ee = s * nq + q;
              const int64_t T = STT[ee];
              if (STOK[ee] && STY[ee] <= bestY && (s < ss ? T < M : T <= M) && T < bt) {
                bt = T;
                bq = q;
              }
            }
          }
          kout[s] = (int8_t)(AMODE == 1 ? (bq ? lg : 0) : bq);
        }
      }
    }
    __syncwarp();
  }
}

// ---- NEXT-2: the paper's stage determination ----------
// Cuts (R-8): the S-1 gaps with the smallest boundary bytes; the gaps below the
// (S-1)-th smallest byte count are forced, the rest are taken among the gaps
// equal to it by the min-max of the tp=1 compute with the R0 rule.  One warp,
// lanes over the end position i; f[s][i] = min over allowed k in
// [max(s-1, LF(i)), i-1] of max(f[s-1][k], P[i]-P[k]) (LF(i) = last forced gap
// below i: no forced gap may fall inside a stage), lowest k on ties.
__device__ void paper_cuts_unit(const int64_t *P, const int64_t *BNDr, int L, int S, int Lp,
                                const int64_t *SB, int32_t *LF, int64_t *F0, int64_t *F1,
                                uint8_t *ARG, int16_t *bd, int lane) {
  if (S == 1) {
    if (lane == 0) {
      bd[0] = 0;
      bd[1] = (int16_t)L;
    }
    __syncwarp();
    return;
  }
  const int64_t beta = SB[S - 2];
  // gap q in [1, L-1] carries BNDr[q-1]; allowed = bytes <= beta, forced = bytes < beta
  for (int i = lane; i <= L; i += 32) {
    int lf = 0;
    for (int q = i - 1; q >= 1; --q)
      if (BNDr[q - 1] < beta) {
        lf = q;
        break;
      }
    LF[i] = lf;
    const bool end_ok = i == L || (i >= 1 && BNDr[i - 1] <= beta);
    F0[i] = (i >= 1 && end_ok && lf == 0) ? P[i] : kInf;
  }
  __syncwarp();
  int64_t *fp = F0, *fc = F1;
  for (int s = 2; s <= S; ++s) {
    uint8_t *arow = ARG + s * Lp;
    for (int i = lane; i <= L; i += 32) {
      int64_t best = kInf;
      int a = 0;
      const bool end_ok = i == L || (i >= 1 && BNDr[i - 1] <= beta);
      if (end_ok && i >= s) {
        const int64_t Pi = P[i];
        for (int k = max(s - 1, LF[i]); k <= i - 1; ++k) {
          if (BNDr[k - 1] > beta || fp[k] == kInf) continue;
          const int64_t v = max(fp[k], Pi - P[k]);
          if (v < best) {
            best = v;
            a = k;
          }
        }
      }
      fc[i] = best;
      arow[i] = (uint8_t)a;
    }
    __syncwarp();
    int64_t *tmp = fp;
    fp = fc;
    fc = tmp;
  }
  if (lane == 0) {
    bd[S] = (int16_t)L;
    int b = L;
    for (int s = S; s >= 2; --s) {
      b = ARG[s * Lp + b];
      bd[s - 1] = (int16_t)b;
    }
    bd[0] = 0;
  }
  __syncwarp();
}

// GPUs per stage (R-9): round(G F_s / F) to the nearest power of two (ties up,
// >= 1), then conservation repair (halve the lowest F_s/g_s among g_s >= 2
// while the sum exceeds G; double the highest F_s/g_s that keeps the sum <= G
// while it is below).  One lane; 128-bit products.
__device__ void paper_gpus_lane(const int64_t *P, const int16_t *bd, int S, int G, int32_t *g) {
  const __int128 F = P[bd[S]] - P[bd[0]];
  int64_t sum = 0;
  for (int s = 0; s < S; ++s) {
    const __int128 num = (__int128)G * (P[bd[s + 1]] - P[bd[s]]);
    int v = 1;
    if (num >= F) {  // a = floor(log2(num / F)) from the bit lengths, one correction
      const uint64_t nhi = (uint64_t)(num >> 64), nlo = (uint64_t)num;
      const int lnum = nhi ? 127 - __clzll((long long)nhi) : 63 - __clzll((long long)nlo);
      const int lF = 63 - __clzll((long long)(uint64_t)F);
      int a = lnum - lF;
      if ((F << a) > num) --a;
      v = (2 * num >= 3 * ((__int128)1 << a) * F) ? (2 << a) : (1 << a);
    }
    g[s] = v;
    sum += v;
  }
  while (sum > G) {
    int w = -1;
    for (int s = 0; s < S; ++s) {
      if (g[s] < 2) continue;
      if (w < 0 || (__int128)(P[bd[s + 1]] - P[bd[s]]) * g[w] < (__int128)(P[bd[w + 1]] - P[bd[w]]) * g[s])
        w = s;
    }
    sum -= g[w] / 2;
    g[w] /= 2;
  }
  while (sum < G) {
    int w = -1;
    for (int s = 0; s < S; ++s) {
      if (sum + g[s] > G) continue;
      if (w < 0 || (__int128)(P[bd[s + 1]] - P[bd[s]]) * g[w] > (__int128)(P[bd[w + 1]] - P[bd[w]]) * g[s])
        w = s;
    }
    sum += g[w];
    g[w] *= 2;
  }
}

// The same with lanes = stages (S <= 32): the rounding in parallel, each
// repair step's argmin / argmax of F_s/g_s (exact 128-bit cross products,
// ties to the earliest stage) by a shuffle tournament.
__device__ __forceinline__ int paper_pick(bool elig, int64_t F, int g, bool want_max) {
  const int lane = threadIdx.x & 31;
  int s = lane;
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    const int64_t oF = __shfl_xor_sync(0xffffffffu, F, d);
    const int og = __shfl_xor_sync(0xffffffffu, g, d);
    const int os = __shfl_xor_sync(0xffffffffu, s, d);
    const bool oe = __shfl_xor_sync(0xffffffffu, elig, d);
    bool take = false;
    if (oe) {
      if (!elig) {
        take = true;
      } else {
        const __int128 mine = (__int128)F * og, other = (__int128)oF * g;  // F/g vs oF/og
        take = want_max ? (other > mine || (other == mine && os < s))
                        : (other < mine || (other == mine && os < s));
      }
    }
    if (take) {
      F = oF;
      g = og;
      s = os;
      elig = oe;
    }
  }
  return elig ? s : -1;
}

__device__ void paper_gpus_warp(const int64_t *P, const int16_t *bd, int S, int G, int32_t *gout,
                                int lane) {
  const __int128 Ft = P[bd[S]] - P[bd[0]];
  int64_t F = 0;
  int g = 0;
  if (lane < S) {
    F = P[bd[lane + 1]] - P[bd[lane]];
    const __int128 num = (__int128)G * F;
    g = 1;
    if (num >= Ft) {
      const uint64_t nhi = (uint64_t)(num >> 64), nlo = (uint64_t)num;
      const int lnum = nhi ? 127 - __clzll((long long)nhi) : 63 - __clzll((long long)nlo);
      const int lF = 63 - __clzll((long long)(uint64_t)Ft);
      int a = lnum - lF;
      if ((Ft << a) > num) --a;
      g = (2 * num >= 3 * ((__int128)1 << a) * Ft) ? (2 << a) : (1 << a);
    }
  }
  int sum = __reduce_add_sync(0xffffffffu, (unsigned)g);
  while (sum > G) {
    const int w = paper_pick(lane < S && g >= 2, F, g, false);
    const int gw = __shfl_sync(0xffffffffu, g, w);
    if (lane == w) g /= 2;
    sum -= gw / 2;
  }
  while (sum < G) {
    const int w = paper_pick(lane < S && sum + g <= G, F, g, true);
    const int gw = __shfl_sync(0xffffffffu, g, w);
    if (lane == w) g *= 2;
    sum += gw;
  }
  if (lane < S) gout[lane] = g;
  __syncwarp();
}

// NEXT-2 plan cost (R-10): uniform tp = 2^k (k <= log2 min g_s), dp_s = g_s / tp,
// mb_s = GB/(B dp_s); GPUs packed from a node boundary in stage order (offset
// o): tp intra iff tp <= gpn and tp | o; dp intra iff the stage lies in one
// node; boundary into s intra iff o is not a node boundary.
// NBG microbatch counts at once (the B-independent per-stage work --
// links, memory, sync, the 128-bit alpha-beta products -- done once per stage;
// per B the ceil-shifts are chained as in plan_group_time).  Returns the best
// (T, p) of plan group (k, bg), lowest p on ties.
template <int NBG>
__device__ __forceinline__ int64_t paper_plan_group_time(const UnitCtx &U, const int16_t *bd,
                                                         const int32_t *g, int S, int k, int bg,
                                                         int gpn, int &best_p) {
  const int lS = ilog2_pow2(S);
  int lB[NBG];
  bool ok[NBG];
  bool any = false;
#pragma unroll
  for (int q = 0; q < NBG; ++q) {
    const int b = bg * NBG + q;
    lB[q] = U.b_mode == 0 ? lS + 2 : (b < U.nB ? U.lBv[b] : 0);
    ok[q] = U.b_mode == 0 ? q == 0 : b < U.nB;
    any |= ok[q];
  }
  if (!any) return kInf;
  const uint64_t tp = 1ull << k;
  int64_t sumT[NBG], maxT[NBG];
#pragma unroll
  for (int q = 0; q < NBG; ++q) sumT[q] = maxT[q] = 0;
  int64_t maxSync = 0;
  int64_t o = 0;
  const int64_t *PCk = U.PC + k * U.Lp;
  for (int s = 0; s < S; ++s) {
    const int gs = g[s], a = bd[s], e = bd[s + 1];
    const int ldp = ilog2_pow2((uint32_t)gs) - k;
    if (ldp < 0) return kInf;
    const uint64_t dp = 1ull << ldp;
    const bool tp_in = (int64_t)tp <= gpn && (o & (int64_t)(tp - 1)) == 0;
    const bool dp_in = (o >> U.lgpn) == ((o + gs - 1) >> U.lgpn);  // gpn = 2^lgpn
    const uint64_t a_tp = tp_in ? U.a_in : U.a_x, b_tp = tp_in ? U.b_in : U.b_x;
    const uint64_t a_dp = dp_in ? U.a_in : U.a_x, b_dp = dp_in ? U.b_in : U.b_x;
    const int64_t W = U.PW[e] - U.PW[a], A = U.PA[e] - U.PA[a], C = PCk[e] - PCk[a];
    if (ldp > U.lGB) return kInf;  // dp > GB: no microbatch fits any B
    const uint64_t mem = ((uint64_t)(U.kst * W + (A << (U.lGB - ldp))) + tp - 1) >> k;
    if (mem > (uint64_t)U.memt) return kInf;
    if (ldp) {
      const uint64_t Wt = ((uint64_t)W + tp - 1) >> k;
      const uint64_t sy = 2 * (dp - 1) * a_dp + mul_shr_ceil(2 * (dp - 1) * Wt, b_dp, ldp + 20);
      maxSync = max(maxSync, (int64_t)sy);
    }
    uint64_t Xh = 0, Xl = 0, tpn_alpha = 0;
    if (k) {
      const uint64_t x = 2 * (tp - 1) * (uint64_t)(U.PV[e] - U.PV[a]);
      Xl = x * b_tp;
      Xh = __umul64hi(x, b_tp);
      tpn_alpha = (uint64_t)(U.PN[e] - U.PN[a]) * (2 * (tp - 1)) * a_tp;
    }
    uint64_t Yh = 0, Yl = 0, Zh = 0, Zl = 0, a_b = 0, b_b = 0, bnd = 0;
    if (s) {
      bnd = (uint64_t)U.BND[a - 1];
      const bool b_in = (o & (gpn - 1)) != 0;
      a_b = b_in ? U.a_in : U.a_x;
      b_b = b_in ? U.b_in : U.b_x;
      Yl = bnd * b_b;
      Yh = __umul64hi(bnd, b_b);
      if (k) {
        const uint64_t z = (tp - 1) * bnd;
        Zl = z * b_tp;
        Zh = __umul64hi(z, b_tp);
      }
    }
    uint64_t rX = 0, rY = 0, rZ = 0;
    int pe = 0;
    bool chain = false, chainY = false;
#pragma unroll
    for (int q = 0; q < NBG; ++q) {
      const int lm = U.lGB - lB[q] - ldp;  // mb_s = GB / (B dp_s)
      if (lm < 0) ok[q] = false;           // B dp_s > GB (A-12)
      if (!ok[q]) continue;
      const int ex = k + 20 - lm;
      const int d = ex - pe;
      uint64_t T = (uint64_t)C << lm;
      if (k) {
        rX = chain ? (rX + (1ull << d) - 1) >> d : ceil_shr128(Xh, Xl, ex);
        T += tpn_alpha + rX;
      }
      if (s) {
        if (lm >= k) {
          rY = chainY ? (rY + (1ull << d) - 1) >> d : ceil_shr128(Yh, Yl, ex);
          chainY = true;
          T += a_b + rY;
        } else {
          const int sh = k - lm;
          T += a_b + mul_shr_ceil((bnd + (1ull << sh) - 1) >> sh, b_b, 20);
        }
        if (k) {
          rZ = chain ? (rZ + (1ull << d) - 1) >> d : ceil_shr128(Zh, Zl, ex);
          T += (tp - 1) * a_tp + rZ;
        }
      }
      chain = true;
      pe = ex;
      sumT[q] += (int64_t)T;
      maxT[q] = max(maxT[q], (int64_t)T);
    }
    o += gs;
  }
  int64_t best = kInf;
  int bq = 0;
#pragma unroll
  for (int q = 0; q < NBG; ++q) {
    if (!ok[q]) continue;
    const int64_t ti = sumT[q] + (int64_t)((1ll << lB[q]) - 1) * maxT[q] + maxSync;
    if (ti < best) {
      best = ti;
      bq = q;
    }
  }
  best_p = U.b_mode == 0 ? k : k * U.nB + bg * NBG + bq;
  return best;
}

// ---- cp.async (LDGSTS) staging: global -> shared without registers ---------
__device__ __forceinline__ void cp_async4(void *sdst, const void *gsrc) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async8(void *sdst, const void *gsrc) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

// K2 rows f[2..smax] (lowest-argmin binary search, §N3), in the narrowest
// integer type that holds P[L] (every f value is <= P[L]): exact either way.
// The searched crossing lo(s, i) = first k with f[s-1][k] + P[k] >= P[i] can
// only move right with s (f[s-1][k] <= f[s-2][k]: one more stage never raises
// the min-max), so row s searches [max(s-1, lo(s-1, i)), i] -- the bounds are
// kept in ARG row 0, which the backtrack never reads.
template <typename V>
__device__ __forceinline__ void stage_dp(const V *P0, V *F0, V *F1, uint8_t *ARG, int Lp, int L,
                                         int smax, int lane) {
  uint8_t *LOB = ARG;  // row 0: lo(s-1, i)
  for (int i = lane; i <= L; i += 32) {
    F0[i] = P0[i];
    LOB[i] = 0;
  }
  __syncwarp();
  V *fp = F0, *fc = F1;
  for (int s = 2; s <= smax; ++s) {
    uint8_t *arow = ARG + s * Lp;
    for (int i = s + lane; i <= L; i += 32) {
      const V Pi = P0[i];
      int lo = max(s - 1, (int)LOB[i]), hi = i;  // first k in [lo, i-1] with f[s-1][k] >= P[i]-P[k], else i
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (fp[mid] >= Pi - P0[mid])
          hi = mid;
        else
          lo = mid + 1;
      }
      int a;
      V val;
      if (lo == s - 1) {
        a = lo;
        val = fp[lo];
      } else {
        const V v0 = Pi - P0[lo - 1];  // value at k1-1 (its max is the stage term)
        if (lo == i) {
          a = lo - 1;
          val = v0;
        } else {
          const V v1 = fp[lo];
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
      LOB[i] = (uint8_t)lo;
    }
    __syncwarp();
    V *tmp = fp;
    fp = fc;
    fc = tmp;
  }
}

// Metadata of one unit, loaded one unit ahead (independent loads, one round trip).
struct UnitMeta {
  int64_t u, cb, ce, pb, pe, off;
  int L, ng, gb, kst;
};

__device__ __forceinline__ UnitMeta load_meta(const Params &P, const EstArgs &A, int64_t u) {
  UnitMeta m;
  m.u = u;
  if (u < A.unit_end) {
    const int j = (int)(u / P.T);
    m.cb = A.ucb[u];
    m.ce = A.ucb[u + 1];
    m.pb = A.upb[u];
    m.pe = A.upb[u + 1];
    m.off = P.off[j];
    m.L = P.L[j];
    m.ng = P.ng[j];
    m.gb = P.gb[j];
    m.kst = P.kst[j];
  }
  return m;
}

#ifndef CRIUS_EST_MINB
#define CRIUS_EST_MINB 7  // <= 72 registers: 7 CTAs (28 warps) per SM
#endif
// The B-sweep instantiation (NBG > 1) keeps NBG partial sums per lane and spills
// at 128 registers; its per-warp shared memory already caps it near 3 CTAs per
// SM at large L, so it gets <= 168 registers (measured: cfg5 4.80 -> 4.34 ms,
// cfg3 0.129 -> 0.123 ms).  The NBG = 1 kernel: 80 registers (6 CTAs, 24 warps per SM)
// measured cfg4 0.249 vs 0.257 ms at 128 (per-plan lanes), 0.227 ms with per-stage lanes;
// 72 registers (7 CTAs) 0.220 ms, 64 (8 CTAs) 0.227 ms (spills).
#ifndef CRIUS_EST_MINB_WIDE
#define CRIUS_EST_MINB_WIDE 3
#endif
// NEXT-1 / NEXT-3 (AMODE 1..3) keep <= 128 registers: at 80 the assembly kernel
// spills (cfg4 NEXT-1 estimate 3.05 -> 3.47 ms); NEXT-2 (AMODE 4) runs at 80
// (cfg4 1.44 -> 1.38 ms)
#ifndef CRIUS_EST_MINB_ASM
#define CRIUS_EST_MINB_ASM 4
#endif
#ifndef CRIUS_EST_MINB_PAPER
#define CRIUS_EST_MINB_PAPER 6
#endif
template <int WARPS, int NBG, int AMODE>
__global__ void __launch_bounds__(WARPS * 32,
                                  (NBG > 1 ? CRIUS_EST_MINB_WIDE
                                           : (AMODE == 0 ? CRIUS_EST_MINB
                                                         : (AMODE == 4 ? CRIUS_EST_MINB_PAPER
                                                                       : CRIUS_EST_MINB_ASM))) *
                                      4 / WARPS)
    k_estimate(Params P, EstArgs A) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned char *base = smem + (size_t)wid * A.warp_bytes;
  const int Lp_ = A.Lp;
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
  int32_t *CK = CP + (A.maxCells + 1);  // [maxCells] smallest memory-feasible k per Cell
  int32_t *CRAW = (int32_t *)(base + A.off_CRAW);  // [K1e][Lp] raw compute rows
  int32_t *NRAW = (int32_t *)(base + A.off_NRAW);  // [Lp] raw tp_calls, then the int32 P0
  int64_t *POFF = (int64_t *)(base + A.off_POFF);  // [maxCells] raw plan offsets
  int32_t *ORD = (int32_t *)(base + A.off_ORD);    // [maxCells] processing order (S desc)
  int64_t *STT = (int64_t *)(base + A.off_ST);     // [st_cap] stage table (AMODE > 0)
  int64_t *STC = STT + A.st_cap, *STY = STC + A.st_cap;
  uint8_t *STOK = (uint8_t *)(STY + A.st_cap);
  int64_t *PSB = (int64_t *)(base + A.off_PS);     // NEXT-2: sorted gap bytes [Lp]
  int32_t *PLF = (int32_t *)(PSB + Lp_);           // NEXT-2: last forced gap [Lp]
  int32_t *PGS = PLF + Lp_;                        // NEXT-2: GPUs per stage [Stop]
  const int Lp = A.Lp;
  const int64_t out_cell_base = A.global_out ? 0 : A.ucb[A.unit_begin];

  int64_t un = 0;
  if (lane == 0) un = A.unit_begin + atomicAdd(A.work_counter, 1);
  un = __shfl_sync(0xffffffffu, un, 0);
  UnitMeta nm = load_meta(P, A, un);
  // work tickets run one unit ahead: the ticket drawn now is consumed by the
  // next iteration, so the atomic's round trip hides behind a whole unit
  int ticket = 0;
  if (lane == 0) ticket = atomicAdd(A.work_counter, 1);

  for (;;) {
    const UnitMeta m = nm;
    const int64_t u = m.u;
    if (u >= A.unit_end) break;
    // prefetch the metadata of the next unit (last iteration's ticket) and
    // draw the ticket after it
    un = A.unit_begin + __shfl_sync(0xffffffffu, ticket, 0);
    if (lane == 0) ticket = atomicAdd(A.work_counter, 1);
    nm = load_meta(P, A, un);

    const int t = (int)(u % P.T);
    const int64_t cb = m.cb;
    const int nc = (int)(m.ce - cb);
    int16_t *split_out =
        A.splits ? A.splits + (u - (A.global_out ? 0 : A.unit_begin)) * A.split_stride : nullptr;
    if (nc == 0) {
      if (split_out)
        for (int q = lane; q < A.split_stride; q += 32) split_out[q] = -1;
      continue;
    }
    const int64_t pb = m.pb;
    const int npu = (int)(m.pe - pb);
    const int L = m.L;
    const int64_t off = m.off;
    CRIUS_CHECK(nc <= A.maxCells && L + 1 <= A.Lp);
    // compute planes needed: k <= log2(max g), max g <= min(largest G of the unit, g_max)
    const int cap = P.ty[t].cap;
    const int gtop = P.gpu_set == 1 ? cap : (2 * m.ng <= cap ? 2 * m.ng : (m.ng <= cap ? m.ng : m.ng / 2));
    const int K1s = min(ilog2_pow2(max(1, min(gtop, P.g_max))) + 1, A.K1e);

    // ---- A3: stage every row of the unit with cp.async (one round trip), then scan
    for (int k = 0; k < K1s; ++k) {
      const int32_t *src = P.c + ((int64_t)t * P.K1 + k) * P.TL + off;
      for (int l = lane; l < L; l += 32) cp_async4(CRAW + k * Lp + l, src + l);
    }
    for (int l = lane; l < L; l += 32) {
      cp_async8(PW + l + 1, P.w + off + l);
      cp_async8(PA + l + 1, P.act + off + l);
      cp_async8(PV + l + 1, P.tpv + off + l);
      cp_async8(BND + l, P.bnd + off + l);
      cp_async4(NRAW + l, P.tpn + off + l);
    }
    for (int i = lane; i < nc; i += 32) {
      cp_async4(CG + i, A.cG + cb + i);
      cp_async4(CS + i, A.cS + cb + i);
      cp_async8(POFF + i, A.plan_off + cb + i);
    }
    cp_async_wait_all();
    __syncwarp();
    int smax = 0, gmax = 0;
    for (int i = lane; i < nc; i += 32) {
      CP[i] = (int)(POFF[i] - pb);
      smax = max(smax, CS[i]);
      gmax = max(gmax, CG[i] / CS[i]);
    }
    if (lane == 0) CP[nc] = npu;
    smax = warp_max_int(smax);
    gmax = warp_max_int(gmax);
    const int K1u = ilog2_pow2(gmax) + 1;  // <= K1s
    CRIUS_CHECK(K1u <= K1s && smax <= A.Stop);
    // every row by one lane, a serial scan whose loads do not depend on the
    // running sum (no shuffle rounds): lanes 0..K1u the int32 rows (K1u compute
    // rows + tp_calls) into their int64 prefix rows, lanes 29..31 the int64
    // rows w, act, tpv in place
    if (lane <= K1u) {
      const int32_t *src = lane < K1u ? CRAW + lane * Lp : NRAW;
      int64_t *dst = lane < K1u ? PC + lane * Lp : PN;
      int64_t acc = 0;
      dst[0] = 0;
#pragma unroll 8
      for (int l = 0; l < L; ++l) {
        acc += src[l];
        dst[l + 1] = acc;
      }
    } else if (lane >= 29) {
      int64_t *x = lane == 29 ? PW : (lane == 30 ? PA : PV);
      int64_t acc = 0;
      x[0] = 0;
#pragma unroll 8
      for (int l = 1; l <= L; ++l) {
        acc += x[l];
        x[l] = acc;
      }
    }
    __syncwarp();

    const int nSi = ilog2_pow2(smax) + 1;
    // NEXT-2 with every boundary carrying the same bytes (transformer stacks):
    // every gap ties at beta, none is forced, and the cut rule IS the §N3
    // min-max split with R0 -- take the D1 path below
    bool paper_cuts = false;
    if (AMODE == 4) {
      bool uneq = false;
      for (int q = lane; q < L - 1; q += 32) uneq |= BND[q] != BND[0];
      paper_cuts = __any_sync(0xffffffffu, uneq);
    }
    if (paper_cuts) {  // NEXT-2: the paper's cuts for every S of the unit
      // gap bytes sorted ascending (rank by counting; index breaks ties)
      for (int q = lane; q < L - 1; q += 32) {
        const int64_t v = BND[q];
        int r = 0;
        for (int q2 = 0; q2 < L - 1; ++q2) r += BND[q2] < v || (BND[q2] == v && q2 < q);
        PSB[r] = v;
      }
      __syncwarp();
      for (int si = 0; si < nSi; ++si) {
        const int S = 1 << si;
        paper_cuts_unit(PC, BND, L, S, Lp, PSB, PLF, F0, F1, ARG, BD + (S - 1) + si, lane);
      }
    } else {
    // ---- K2: stage DP rows f[1..smax] over P0 = PC[0]
    if (PC[L] < (int64_t)INT32_MAX) {
      int32_t *P32 = NRAW;
      for (int i = lane; i <= L; i += 32) P32[i] = (int32_t)PC[i];
      __syncwarp();
      stage_dp<int32_t>(P32, (int32_t *)F0, (int32_t *)F0 + Lp, ARG, Lp, L, smax, lane);
    } else {
      stage_dp<int64_t>(PC, F0, F1, ARG, Lp, L, smax, lane);
    }

    // ---- R0 backtrack, one lane per S = 2^si
    if (lane < nSi) {
      const int S = 1 << lane;
      int16_t *bd = BD + (S - 1) + lane;
      bd[S] = (int16_t)L;
      int b = L;
      for (int s = S; s >= 2; --s) {
        b = ARG[s * Lp + b];
        CRIUS_CHECK(b >= s - 1 && b < L);
        bd[s - 1] = (int16_t)b;
      }
      bd[0] = 0;
    }
    }  // AMODE != 4
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
    U.lGB = ilog2_pow2(m.gb);
    U.lgpn = P.ty[t].lgpn;
    U.b_mode = P.b_mode;
    U.nB = P.nB;
    U.kst = m.kst;
    U.memt = P.ty[t].mem;
    U.a_in = P.ty[t].a_in;
    U.b_in = P.ty[t].b_in;
    U.a_x = P.ty[t].a_x;
    U.b_x = P.ty[t].b_x;
    U.lBv = P.lB;

    if (AMODE == 4) {  // NEXT-2: per Cell, the paper's GPUs per stage, then every (k, B)
      const int gpn = P.ty[t].gpn;
      const int nB = P.b_mode == 0 ? 1 : P.nB;
      for (int ci = 0; ci < nc; ++ci) {
        const int G = CG[ci], S = CS[ci], lS = ilog2_pow2(S);
        const int16_t *bd = BD + (S - 1) + lS;
        if (S <= 32) {
          paper_gpus_warp(PC, bd, S, G, PGS, lane);
        } else {
          if (lane == 0) paper_gpus_lane(PC, bd, S, G, PGS);
          __syncwarp();
        }
        int gmin = INT32_MAX, gmx = 0;
        for (int s = lane; s < S; s += 32) {
          gmin = min(gmin, PGS[s]);
          gmx = max(gmx, PGS[s]);
        }
        gmin = (int)__reduce_min_sync(0xffffffffu, (unsigned)gmin);
        gmx = warp_max_int(gmx);
        const int ngrp = (nB + NBG - 1) / NBG;
        const int nitem = gmx > P.g_max ? 0 : (ilog2_pow2((uint32_t)gmin) + 1) * ngrp;
        int64_t bT = kInf;
        int bp = INT32_MAX;
        for (int it = lane; it < nitem; it += 32) {  // item = (k, group of NBG B values)
          const int k = it / ngrp, bgi = it - k * ngrp;
          int p;
          const int64_t T = paper_plan_group_time<NBG>(U, bd, PGS, S, k, bgi, gpn, p);
          if (T < bT) {  // items ascending per lane: ties keep the lower p
            bT = T;
            bp = p;
          }
        }
        int64_t wT = bT;
        for (int d = 16; d > 0; d >>= 1) wT = min(wT, __shfl_xor_sync(0xffffffffu, wT, d));
        const int wp = (int)__reduce_min_sync(0xffffffffu, (unsigned)(bT == wT ? bp : INT32_MAX));
        int8_t *kout = A.stage_tp ? A.stage_tp + (cb + ci - out_cell_base) * A.stage_stride : nullptr;
        if (kout)
          for (int q = lane; q < A.stage_stride; q += 32)
            kout[q] = (int8_t)(q < S ? ilog2_pow2((uint32_t)PGS[q]) : -1);
        if (lane == 0) {
          CellResult res;
          const bool ok = wT != kInf;
          res.t_ns = ok ? wT : kInf;
          res.plan = ok ? wp : -1;
          res.flags = ok ? 1 : 0;
          emit_result(A, cb + ci, out_cell_base, res);
        }
        __syncwarp();
      }
      continue;
    }
    if (AMODE > 0) {  // NEXT-1: per-stage assembly, one Cell at a time
      for (int ci = 0; ci < nc; ++ci) {
        int64_t F;
        int bb;
        int8_t *kout = A.stage_tp ? A.stage_tp + (cb + ci - out_cell_base) * A.stage_stride : nullptr;
        if (kout)
          for (int q = lane; q < A.stage_stride; q += 32) kout[q] = -1;
        __syncwarp();
        const int8_t *fav = A.favor ? A.favor + (cb + ci - out_cell_base) * A.stage_stride : nullptr;
        assembled_cell<AMODE>(U, A, CG[ci], CS[ci], lane, STT, STC, STY, STOK, F, bb, kout, fav);
        if (lane == 0) {
          CellResult res;
          res.t_ns = F;
          res.plan = F == kInf ? -1 : bb;
          res.flags = F == kInf ? 0 : 1;
          emit_result(A, cb + ci, out_cell_base, res);
        }
      }
      __syncwarp();
      continue;
    }
    const int ngrp = P.b_mode == 0 ? 1 : (P.nB + NBG - 1) / NBG;
    // A Cell's memory use is monotone in k (mem = ceil(kst W / tp + GB A / g)
    // shrinks as tp grows, A-13): with a microbatch sweep (NBG > 1: one (Cell,
    // k) spans several lanes' worth of plans) its smallest feasible k, so that
    // the plan items below skip the memory-infeasible plans instead of spending
    // lanes on them (a Cell with none is infeasible: its record right away).
    // With one plan per (Cell, k) the pre-pass costs more than it saves.
    for (int ci = lane; ci < nc && NBG == 1; ci += 32) CK[ci] = 0;
    for (int ci = lane; ci < nc && NBG > 1; ci += 32) {
      const int G = CG[ci], S = CS[ci], lS = ilog2_pow2(S), lg = ilog2_pow2(G) - lS;
      const int K = lg + 1;
      const int16_t *bd = BD + (S - 1) + lS;
      int kmin = 0;
      int64_t pw_a = 0, pa_a = 0;
      for (int s = 0; s < S && kmin < K; ++s) {
        const int e = bd[s + 1];
        const int64_t pw_e = PW[e], pa_e = PA[e];
        const int64_t Wd = pw_e - pw_a, Ad = pa_e - pa_a;
        while (kmin < K) {
          const int sh = U.lGB + kmin - lg;  // GB / dp = 2^sh; dp > GB: no plan of this k
          if (sh >= 0) {
            const uint64_t mem = ((uint64_t)(U.kst * Wd + (Ad << sh)) + (1ull << kmin) - 1) >> kmin;
            if (mem <= (uint64_t)U.memt) break;
          }
          ++kmin;
        }
        pw_a = pw_e;
        pa_a = pa_e;
      }
      CK[ci] = kmin;
      if (kmin == K) {
        CellResult res;
        res.t_ns = kInf;
        res.plan = -1;
        res.flags = 0;
        emit_result(A, cb + ci, out_cell_base, res);
      }
    }
    __syncwarp();
    // Per-stage lanes (below) or per-plan lanes (the loop after it), chosen per
    // launch (A.per_stage): with few plans per unit the per-plan form leaves
    // most lanes of a unit's one chunk idle while its longest plan runs S
    // stages; with many, it packs plans by S and the per-stage form's
    // reductions cost more than they save.  (Chosen per unit, warps of one SM
    // run both forms and the kernel measured slower than either: DESIGN.md §5.)
    if (A.per_stage && smax <= 32) {
      // One (Cell, k, stage) per lane: a plan's S stages are S consecutive
      // lanes.  Cells run by S descending (stable) and a Cell holds K*S items,
      // so every plan's lane group is aligned to S inside one 32-lane chunk:
      // xor butterflies of width S form its sum / max stage time and max sync
      // (integer, so the reduction order is immaterial), the group's first
      // lane holds the plan, and the segmented min-scan below picks the Cell's
      // best plan as in the per-plan path.
      // counting sort by log2 S (0..5): rank = Cells with a larger S + Cells
      // of the same S before it
      const uint32_t lt = (1u << lane) - 1;
      {
        int cnt[6] = {0, 0, 0, 0, 0, 0};
        for (int b0 = 0; b0 < nc; b0 += 32) {
          const int i = b0 + lane;
          const int ls = i < nc ? ilog2_pow2(CS[i]) : -1;
#pragma unroll
          for (int b = 0; b < 6; ++b) cnt[b] += __popc(__ballot_sync(0xffffffffu, ls == b));
        }
        int above[6], seen[6];
        int acc = 0;
#pragma unroll
        for (int b = 5; b >= 0; --b) {
          above[b] = acc;
          acc += cnt[b];
          seen[b] = 0;
        }
        for (int b0 = 0; b0 < nc; b0 += 32) {
          const int i = b0 + lane;
          const int ls = i < nc ? ilog2_pow2(CS[i]) : -1;
          int rk = 0;
#pragma unroll
          for (int b = 0; b < 6; ++b) {
            const uint32_t m = __ballot_sync(0xffffffffu, ls == b);
            if (ls == b) rk = above[b] + seen[b] + __popc(m & lt);
            seen[b] += __popc(m);
          }
          if (i < nc) ORD[rk] = i;
        }
      }
      __syncwarp();
      {
        int carry = 0;
        for (int b0 = 0; b0 < nc; b0 += 32) {
          const int r = b0 + lane;
          int cnt = 0;
          if (r < nc) {
            const int ci = ORD[r];
            cnt = (ilog2_pow2(CG[ci] / CS[ci]) + 1) * CS[ci];
          }
          const int inc = warp_incl_scan32(cnt, lane);
          if (r < nc) CP[r + 1] = carry + inc;
          carry += __shfl_sync(0xffffffffu, inc, 31);
        }
        if (lane == 0) CP[0] = 0;
      }
      __syncwarp();
      const int nitems = CP[nc];
      int carry_r = -1, carry_p = 0;
      int64_t carry_T = kInf;
      int rb = 0;  // the Cell holding the chunk's first item
      for (int f0 = 0; f0 < nitems; f0 += 32) {
        const int f = f0 + lane;
        const bool valid = f < nitems;
        // item -> Cell: the Cells after rb that start inside the chunk (every
        // Cell holds >= 1 item, so at most 31 of them), one per lane
        const int rs = rb + 1 + lane;
        const int st = rs < nc ? CP[rs] - f0 : 32;
        const uint32_t starts = __reduce_or_sync(0xffffffffu, st > 0 && st < 32 ? 1u << st : 0u);
        const int rl = rb + __popc(starts & ((2u << lane) - 1));
        {
          const int r31 = rb + __popc(starts);
          rb = r31 + (r31 + 1 < nc && CP[r31 + 1] == f0 + 32 ? 1 : 0);
        }
        int r = nc, p = 0, S = 1, s = 0, lB = 0;
        bool bad = true;
        int64_t Ts = 0, sy = 0;
        if (valid) {
          r = rl;
          const int ci = ORD[r], local = f - CP[r];
          CRIUS_CHECK(ci >= 0 && ci < nc && local >= 0 && local < CP[r + 1] - CP[r]);
          S = CS[ci];
          const int lS = ilog2_pow2(S), lg = ilog2_pow2(CG[ci]) - lS;
          p = local >> lS;
          s = local & (S - 1);
          lB = lS + 2;  // B = 4S (GPipe)
          const int16_t *bd = BD + (S - 1) + lS;
          int64_t Tc;
          bad = !stage_terms(U, lg, p, lB, s, bd[s], bd[s + 1], Ts, Tc, sy);
        }
        const int Sw = __shfl_sync(0xffffffffu, S, 0);  // the chunk's largest S
        int64_t sumT = Ts, maxT = Ts, maxSync = sy;
        for (int d = 1; d < Sw; d <<= 1) {
          const int64_t o1 = __shfl_xor_sync(0xffffffffu, sumT, d);
          const int64_t o2 = __shfl_xor_sync(0xffffffffu, maxT, d);
          const int64_t o3 = __shfl_xor_sync(0xffffffffu, maxSync, d);
          if (d < S) {
            sumT = (int64_t)((uint64_t)sumT + (uint64_t)o1);
            maxT = max(maxT, o2);
            maxSync = max(maxSync, o3);
          }
        }
        const unsigned badm = __ballot_sync(0xffffffffu, bad);
        const unsigned gmask = S == 32 ? 0xffffffffu : ((1u << S) - 1) << (lane & ~(S - 1));
        int64_t T = kInf;
        if (valid && s == 0 && !(badm & gmask))
          T = (int64_t)((uint64_t)sumT + (uint64_t)((1ll << lB) - 1) * (uint64_t)maxT + (uint64_t)maxSync);
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const int64_t oT = __shfl_up_sync(0xffffffffu, T, d);
          const int op = __shfl_up_sync(0xffffffffu, p, d);
          const int orr = __shfl_up_sync(0xffffffffu, r, d);
          if (lane >= d && orr == r && oT <= T) {
            T = oT;
            p = op;
          }
        }
        const int next_r = __shfl_down_sync(0xffffffffu, r, 1);
        const bool tail = valid && (lane == 31 || next_r != r);
        if (tail && r == carry_r && carry_T <= T) {
          T = carry_T;
          p = carry_p;
        }
        const bool done = valid && (f + 1 == CP[r + 1]);
        if (tail && done) {
          CellResult res;
          res.t_ns = T;
          res.plan = T == kInf ? -1 : p;
          res.flags = T == kInf ? 0 : 1;
          emit_result(A, cb + ORD[r], out_cell_base, res);
        }
        const int r31 = __shfl_sync(0xffffffffu, r, 31);
        const int64_t T31 = __shfl_sync(0xffffffffu, T, 31);
        const int p31 = __shfl_sync(0xffffffffu, p, 31);
        const bool open31 = __shfl_sync(0xffffffffu, (int)(valid && !done), 31);
        if (open31) {
          carry_r = r31;
          carry_T = T31;
          carry_p = p31;
        } else {
          carry_r = -1;
          carry_T = kInf;
        }
      }
      __syncwarp();
      continue;
    }
    // processing order: Cells by S descending (stable) so a 32-lane chunk runs
    // stage loops of one length; item = (Cell, k >= kmin, group of NBG microbatch counts)
    const bool sorted = npu / P.nB * ngrp > 32;  // one chunk: order does not matter
    for (int i = lane; i < nc; i += 32) {
      int r = i;
      if (sorted) {
        const int si = CS[i];
        r = 0;
        for (int q = 0; q < nc; ++q) r += CS[q] > si || (CS[q] == si && q < i);
      }
      ORD[r] = i;
    }
    __syncwarp();
    {
      int carry = 0;  // item counts: <= maxCells * (k_max + 1) * groups, int32
      for (int b0 = 0; b0 < nc; b0 += 32) {
        const int r = b0 + lane;
        int cnt = 0;
        if (r < nc) {
          const int ci = ORD[r];
          cnt = (ilog2_pow2(CG[ci] / CS[ci]) + 1 - CK[ci]) * ngrp;
        }
        const int inc = warp_incl_scan32(cnt, lane);
        if (r < nc) CP[r + 1] = carry + inc;
        carry += __shfl_sync(0xffffffffu, inc, 31);
      }
      if (lane == 0) CP[0] = 0;
    }
    __syncwarp();
    const int nitems = CP[nc];

    int carry_r = -1, carry_p = 0;
    int64_t carry_T = kInf;
    for (int f0 = 0; f0 < nitems; f0 += 32) {
      const int f = f0 + lane;
      const bool valid = f < nitems;
      int r = nc, p = 0;
      int64_t T = kInf;
      if (valid) {
        int lo = 0, hi = nc - 1;  // largest r with CP[r] <= f
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (CP[mid] <= f)
            lo = mid;
          else
            hi = mid - 1;
        }
        r = lo;
        const int ci = ORD[r], local = f - CP[r];
        CRIUS_CHECK(ci >= 0 && ci < nc && local >= 0 && local < CP[r + 1] - CP[r]);
        const int kl = NBG == 1 ? local : local / ngrp, gg = NBG == 1 ? 0 : local - kl * ngrp;
        const int kk = CK[ci] + kl;
        if (NBG == 1) {  // one microbatch count per lane: the per-plan evaluation
          p = P.b_mode == 0 ? kk : kk * P.nB + gg;
          T = plan_time(U, CG[ci], CS[ci], p);
        } else {
          T = plan_group_time<NBG, true>(U, CG[ci], CS[ci], kk, gg, p);
        }
      }
      // segmented inclusive min-scan over (T, p); left lanes have lower p
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int64_t oT = __shfl_up_sync(0xffffffffu, T, d);
        const int op = __shfl_up_sync(0xffffffffu, p, d);
        const int orr = __shfl_up_sync(0xffffffffu, r, d);
        if (lane >= d && orr == r && oT <= T) {
          T = oT;
          p = op;
        }
      }
      const int next_r = __shfl_down_sync(0xffffffffu, r, 1);
      const bool tail = valid && (lane == 31 || next_r != r);
      if (tail && r == carry_r && carry_T <= T) {
        T = carry_T;
        p = carry_p;
      }
      const bool done = valid && (f + 1 == CP[r + 1]);
      if (tail && done) {
        CellResult res;
        res.t_ns = T;
        res.plan = T == kInf ? -1 : p;
        res.flags = T == kInf ? 0 : 1;
        emit_result(A, cb + ORD[r], out_cell_base, res);
      }
      const int r31 = __shfl_sync(0xffffffffu, r, 31);
      const int64_t T31 = __shfl_sync(0xffffffffu, T, 31);
      const int p31 = __shfl_sync(0xffffffffu, p, 31);
      const bool open31 = __shfl_sync(0xffffffffu, (int)(valid && !done), 31);
      if (open31) {
        carry_r = r31;
        carry_T = T31;
        carry_p = p31;
      } else {
        carry_r = -1;
        carry_T = kInf;
      }
    }
    __syncwarp();
  }
  exchange_signal(A);
}

}  // namespace crius
