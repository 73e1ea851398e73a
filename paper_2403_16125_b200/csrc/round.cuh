// round.cuh -- K5/K6: one scheduling round over the job x Cell matrix, on the
// device; K7: compaction of an all-gathered, per-rank-padded result array.
//
// Reading of Alg. 1 fixed by SURVEY §N6 (A-16..A-19):
//   ref_j   = best T at G = N_G (else best overall); score(o) = ref_j / T_o
//   O_j     = per (t, G) the Cell with min (T, S); kappa(o) = (T, G, t)
//   Phase A = SchedArrival: cheapest-kappa option that fits with
//             G <= N_G, else ScaleResource with <= d victim moves
//   Phase B = extra scheduling / reverse scaling, d sweeps
//
// K5 builds O_j for every job in priority order (one warp per job), plus the
// job's arrival options (G <= N_G) in kappa order, transposed [k][J] so that
// one thread per job reads them coalesced.
//
// K6 is ONE CTA (the round is sequential by definition).  It evaluates the
// literal §N6 order with three exact reformulations (DESIGN R-2):
//  * speculative batches -- a job that stays pending changes no state, so the
//    next kRoundThreads jobs are evaluated at once (one THREAD per job, its
//    arrival options in kappa order: the first that fits is its direct choice)
//    against the same state; the first job that is admitted is committed and
//    the next batch starts right after it;
//  * ScaleResource: the victim-move sequence of a trial depends only on the
//    state and on the option's GPU type (G_o only decides where it is cut), so
//    one greedy sequence per type serves every option of every pending job until
//    an admission changes it.  From a type's sequence a table thr[t][log2 G]
//    = the accumulated loss of the shortest prefix that frees G GPUs (or +inf)
//    makes each option's trial one comparison score(o) > thr; the first success
//    in kappa order is the job's ScaleResource outcome;
//  * a type's sequence is computed by ONE warp over the type's admitted jobs
//    (per-type lists): each job's best same-type move (case i) is cached and
//    refreshed only when the job's option changes; its best other-type move
//    (case ii) is computed only when one of its options on another type fits
//    (exact test from per-type smallest-option bytes) and re-evaluated lazily
//    when a move took the GPUs it needed (free' of the other types only
//    decreases along a sequence).  Per move: one warp argmin over the lanes'
//    best candidates, no block barrier.
#pragma once
#include "common.cuh"

namespace crius {

struct OptRec {  // 16 B
  int64_t T;
  int32_t G;
  int32_t t;
};

constexpr int kRT = 8;  // GPU types supported by the round kernel (rejected at load beyond)
#ifndef CRIUS_ROUND_THREADS
#define CRIUS_ROUND_THREADS 256
#endif
constexpr int kRoundThreads = CRIUS_ROUND_THREADS;
constexpr int kRoundWarps = kRoundThreads / 32;
static_assert(kRoundWarps >= kRT && kRoundWarps <= 32, "one warp per GPU type, one ballot word per warp");
constexpr int kLgMax = 31;  // G <= 2^30

// Admitted jobs (SoA; shared memory when they fit, else global).  bi = cached
// best same-type move (case i): option index | log2 G2 << 8; -2 stale (the
// job's option changed), -1 none; bk its key.  ei = best other-type move
// (case ii) under the sequence's current free': index | log2 G2 << 8 | t2 << 16,
// -1 none; ek its key.  slot = position in its type's list tl.
struct AdmView {
  double *bk, *bl, *ek;  // bl = the cached same-type move's loss
  uint64_t *gmb, *tsb;  // the job's gminb / tsb bytes (see RoundBuf)
  int32_t *pos, *cur, *G, *t, *slot, *bi, *ei, *nopt;
  int32_t *po;  // offset of the job's options in the shared-memory pool, -1 = not staged
  int32_t *tl;  // per-type lists of admitted records, type u at tl + toff[u]
  double *psc;  // option pool (shared memory): scores
  int32_t *ppk; //   and log2 G | t << 8 | (index of the entry's rank in score order) << 16
};

struct RoundBuf {
  int32_t J, T, maxopt, depth;
  int32_t policy;        // NEXT-4 ablations (R-11): bit 0 NA (options at G = N_G only),
                         // bit 1 NH (admitted jobs keep their GPU type)
  int64_t smem_bytes;    // dynamic shared memory for the admitted records and type lists
  const int64_t *tmax;   // [J] by job or NULL: deadline bound on an option's T (R-12)
  const int32_t *rank;   // [J] job -> priority position
  const int32_t *pi;     // [J] position -> job
  OptRec *opt;           // [J][maxopt] by position, (t, G) ascending
  double *score;         // [J][maxopt] score(o) = ref / T_o (A-16)
  int64_t *opt_cell;     // [J][maxopt]
  int32_t *nopt;         // [J] by position
  int64_t *ref;          // [J] by position (kInf = unschedulable)
  int32_t *cur;          // [J] by position: option index or -1 (written at the end)
  int64_t *decision;     // [J] by job
  int32_t *free_io;      // [T]
  double *total;
  int64_t *stats;        // [24] counters (see crius_round_stats)
  // arrival options (G <= N_G) in kappa order, transposed: entry k of position
  // p at [k * J + p]; pk = option index | log2 G << 8 | t << 13
  int32_t *ao_pk;
  double *ao_sc;
  int32_t *nao;          // [J] by position
  uint64_t *gminb;       // [J] byte u = log2 of the job's smallest option G on type u (0xff none)
  uint64_t *tsb;         // [J] byte u = index of the job's first option on type u
  uint8_t *operm;        // [J][maxopt] by position: option indices by score descending
                         // (equal scores: lower index first)
  int32_t *opk;          // [J][maxopt] by position: option i's pool word (log2 G | t << 8 |
                         // operm[i] << 16), so staging an option is a plain copy
  // NEXT-4 round state (NULL = every job active, none running)
  const int64_t *run_cell;  // [J] by job: Cell the job runs on, or -1
  const uint8_t *active;    // [J] by job: the job takes part in this round
  int32_t *run_opt;         // [J] by position: option index of the running Cell, or -1
  int8_t *cand;             // [J] by position: 1 = Phase A candidate (active, not running)
  int32_t *err;             // [1] 0 ok; 1 = a running Cell is not one of its job's options;
                            // 2 = free + running GPUs of a type exceed 2^30
  AdmView glob;             // records [J] and type lists [T * J] in global memory
  int32_t *ord;             // [J] scratch: admitted records in priority order
  double *osc;              // [J] scratch: their scores
};

__device__ __forceinline__ double score_of(int64_t ref, int64_t T) {
  return __ddiv_rn((double)ref, (double)T);
}

__device__ __forceinline__ bool kappa_less(const OptRec &a, const OptRec &b) {
  if (a.T != b.T) return a.T < b.T;
  if (a.G != b.G) return a.G < b.G;
  return a.t < b.t;
}

// K5, one warp per job: its options O_j (per (t, G) the Cell with min (T, S),
// A-17), ref and scores from its Cells (contiguous, (t, G, S) order), written
// at the job's priority position; the arrival options (G <= N_G) in kappa
// order, transposed; per-type smallest G and first index; the options in
// score order.  Lanes take the Cells 32 at a time: an option is a run of equal
// (t, G) among the accepted Cells and keeps its smallest T (the earliest Cell,
// i.e. the smallest S, on ties); the rankings are counts over the job's
// options, one option per lane.
__device__ __forceinline__ int64_t warp_min_i64(int64_t v) {
#pragma unroll
  for (int d = 16; d; d >>= 1) v = min(v, (int64_t)__shfl_xor_sync(0xffffffffu, v, d));
  return v;
}
__device__ __forceinline__ uint64_t warp_or_u64(uint64_t v) {
  const uint32_t lo = __reduce_or_sync(0xffffffffu, (uint32_t)v);
  const uint32_t hi = __reduce_or_sync(0xffffffffu, (uint32_t)(v >> 32));
  return ((uint64_t)hi << 32) | lo;
}

__global__ void k_round_options_warp(Params P, const int64_t *__restrict__ ucb,
                                     const int32_t *__restrict__ cType, const int32_t *__restrict__ cG,
                                     const CellResult *__restrict__ res, RoundBuf R) {
  const int lane = threadIdx.x & 31;
  const int j = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  if (j >= R.J) return;  // warp-uniform
  const int pos = R.rank[j];
  const int64_t c0 = ucb[(int64_t)j * R.T], c1 = ucb[(int64_t)(j + 1) * R.T];
  const int ngj = P.ng[j];
  OptRec *og = R.opt + (int64_t)pos * R.maxopt;
  int64_t *ocg = R.opt_cell + (int64_t)pos * R.maxopt;
  double *sc = R.score + (int64_t)pos * R.maxopt;
  const bool act = R.active ? R.active[j] != 0 : true;
  const int64_t rc0 = (act && R.run_cell) ? R.run_cell[j] : -1;
  const int rct = rc0 >= 0 ? cType[rc0] : -1, rcG = rc0 >= 0 ? cG[rc0] : -1;
  const int64_t tmx = R.tmax ? R.tmax[j] : kInf;
  const uint32_t lt = (1u << lane) - 1;
  // ref (A-16): best T at G = N_G, else best overall, over the feasible Cells
  int64_t rng = kInf, rany = kInf;
  for (int64_t c = c0 + lane; c < c1; c += 32) {
    const int64_t T = res[c].t_ns;
    if (T == kInf) continue;
    rany = min(rany, T);
    if (cG[c] == ngj) rng = min(rng, T);
  }
  rng = warp_min_i64(rng);
  rany = warp_min_i64(rany);
  const int64_t ref = rng != kInf ? rng : rany;
  // options: runs of equal (t, G) among the accepted Cells
  int n = 0, kt = -1, kG = -1;  // options so far; (t, G) of the last accepted Cell
  int64_t kT = kInf;            // the best T of the last option so far
  for (int64_t b0 = c0; b0 < c1; b0 += 32) {
    const int64_t c = b0 + lane;
    int64_t T = kInf;
    int t = -1, G = -1;
    if (c < c1) {
      T = res[c].t_ns;
      t = cType[c];
      G = cG[c];
    }
    bool acc = T != kInf;
    if ((R.policy & 1) && G != ngj) acc = false;  // NA: the job stays at N_G GPUs
    if (T > tmx && !(t == rct && G == rcG)) acc = false;  // deadline (R-12)
    const uint32_t am = __ballot_sync(0xffffffffu, acc);
    const uint32_t below = am & lt;
    const int pl = below ? 31 - __clz(below) : -1;  // previous accepted lane
    const int pt = __shfl_sync(0xffffffffu, t, max(pl, 0)), pG = __shfl_sync(0xffffffffu, G, max(pl, 0));
    const bool head = acc && (pl >= 0 ? (t != pt || G != pG) : (t != kt || G != kG));
    const uint32_t hm = __ballot_sync(0xffffffffu, head);
    const int oi = n - 1 + __popc(hm & (lt | (1u << lane)));  // this lane's option
    // per option of the chunk: smallest T, lowest lane (= earliest Cell) on ties
    const uint32_t gm = __match_any_sync(0xffffffffu, acc ? oi : -1 - lane);
    const uint32_t hi = (uint32_t)((uint64_t)T >> 32), lo = (uint32_t)T;
    const uint32_t mhi = __reduce_min_sync(gm, hi);
    const uint32_t mlo = __reduce_min_sync(gm, hi == mhi ? lo : 0xffffffffu);
    const int64_t gmin = (int64_t)(((uint64_t)mhi << 32) | mlo);
    const uint32_t wm = __ballot_sync(0xffffffffu, acc && T == gmin) & gm;
    if (acc && lane == __ffs(wm) - 1) {
      if (oi >= n) {  // a run that starts in this chunk
        og[oi].T = T;
        og[oi].G = G;
        og[oi].t = t;
        ocg[oi] = c;
      } else if (T < kT) {  // the run carried over: strictly better replaces
        og[oi].T = T;
        ocg[oi] = c;
      }
    }
    if (am) {
      const int ll = 31 - __clz(am);  // last accepted lane
      const int loi = __shfl_sync(0xffffffffu, oi, ll);
      const int64_t lmin = __shfl_sync(0xffffffffu, gmin, ll);
      kT = loi == n - 1 ? min(kT, lmin) : lmin;
      kt = __shfl_sync(0xffffffffu, t, ll);
      kG = __shfl_sync(0xffffffffu, G, ll);
      n += __popc(hm);
    }
  }
  __syncwarp();
  // scores, per-type first option, running option
  uint64_t gv = 0, tv = 0, pres = 0;
  int ro = -1;
  for (int i = lane; i < n; i += 32) {
    const OptRec x = og[i];
    sc[i] = score_of(ref, x.T);
    if (i == 0 || og[i - 1].t != x.t) {  // first (smallest G) option of its type
      const int sh = 8 * x.t;
      gv |= (uint64_t)ilog2_pow2((uint32_t)x.G) << sh;
      tv |= (uint64_t)i << sh;
      pres |= 0xffull << sh;
    }
    if (x.t == rct && x.G == rcG) ro = i;
  }
  gv = warp_or_u64(gv);
  tv = warp_or_u64(tv);
  pres = warp_or_u64(pres);
  ro = __reduce_max_sync(0xffffffffu, (unsigned)(ro + 1)) - 1;
  __syncwarp();
  // arrival options (G <= N_G) in kappa order; all options in score order
  uint8_t *pm = R.operm + (int64_t)pos * R.maxopt;
  int na = 0;
  for (int i = lane; i < n; i += 32) {
    const OptRec x = og[i];
    const double si = sc[i];
    int rk = 0, rs = 0;
    for (int i2 = 0; i2 < n; ++i2) {
      const OptRec y = og[i2];
      const double s2 = sc[i2];
      rk += (y.G <= ngj && kappa_less(y, x));
      rs += s2 > si || (s2 == si && i2 < i);
    }
    pm[rs] = (uint8_t)i;
    if (x.G <= ngj) {
      R.ao_pk[(int64_t)rk * R.J + pos] = i | (ilog2_pow2((uint32_t)x.G) << 8) | (x.t << 13);
      R.ao_sc[(int64_t)rk * R.J + pos] = si;
      ++na;
    }
  }
  na = (int)__reduce_add_sync(0xffffffffu, (unsigned)na);
  __syncwarp();
  int32_t *pk = R.opk + (int64_t)pos * R.maxopt;
  for (int i = lane; i < n; i += 32) {
    const OptRec x = og[i];
    pk[i] = ilog2_pow2((uint32_t)x.G) | (x.t << 8) | ((int)pm[i] << 16);
  }
  if (lane == 0) {
    R.gminb[pos] = gv | ~pres;
    R.tsb[pos] = tv | ~pres;
    R.nao[pos] = na;
    R.nopt[pos] = n;
    R.ref[pos] = ref;
    R.cur[pos] = -1;
    if (rc0 >= 0 && ro < 0) atomicExch(R.err, 1);  // the oracle rejects this input (status 2)
    R.run_opt[pos] = rc0 >= 0 ? ro : -1;
    R.cand[pos] = (int8_t)(act && ro < 0 && ref != kInf && na > 0);
  }
}

// ---- warp argmin by lexicographic 3-word keys, one redux.sync per word ------
// Order-preserving u64 image of a double (no NaN; -0.0 normalised to +0.0).
__device__ __forceinline__ uint64_t ord_double(double x) {
  if (x == 0.0) x = 0.0;
  const long long b = __double_as_longlong(x);
  return b < 0 ? ~(uint64_t)b : ((uint64_t)b | 0x8000000000000000ull);
}

// Lane holding the minimum (k, tie) over the lanes with `valid`, or -1.
__device__ __forceinline__ int warp_lex_argmin(bool valid, uint64_t k, uint32_t tie) {
  if (!__ballot_sync(0xffffffffu, valid)) return -1;
  // every lane executes every collective (no short-circuit around redux.sync)
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

// kappa(o) = (T, G, t): G is a power of two, so (log2 G, t) orders like (G, t).
__device__ __forceinline__ uint32_t kappa_tie(const OptRec &x) {
  return ((uint32_t)ilog2_pow2((uint32_t)x.G) << 8) | (uint32_t)x.t;
}

__device__ __forceinline__ OptRec ldg_opt(const OptRec *p) {
  const longlong2 v = __ldg(reinterpret_cast<const longlong2 *>(p));
  OptRec r;
  r.T = v.x;
  r.G = (int32_t)(v.y & 0xffffffff);
  r.t = (int32_t)(v.y >> 32);
  return r;
}

// Cycle stamp that the compiler keeps in program order with memory accesses.
__device__ __forceinline__ long long tstamp() {
  long long c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c)::"memory");
  return c;
}

__device__ __forceinline__ int byte_of(uint64_t v, int u) { return (int)((v >> (8 * u)) & 0xff); }

// One victim-move sequence per GPU type and the ScaleResource thresholds.
constexpr int kTop = 32;      // same-type move candidates kept sorted per type (lane = entry)
constexpr int kTopFill = 16;  // entries a refill selects
constexpr int kQ = 64;        // other-type evaluation queue of a type warp
struct SeqTab {
  int32_t len;
  int32_t mv_a[kMaxDepth];   // victim (admitted record)
  int32_t mv_pk[kMaxDepth];  // its new option: index | log2 G2 << 8 | t2 << 16
  int32_t dfr[kMaxDepth + 1][kRT];  // free-count deltas after m moves
  double cum[kMaxDepth + 1];        // ((0 + loss_1) + loss_2) + ...
  double thr[kLgMax];               // accumulated loss of the shortest prefix freeing 2^lg, or +inf
  int8_t thm[kLgMax];               // that prefix's length
  int32_t f2[kRT];                  // the type warp's working free'
  uint64_t gq;  // byte u <= log2 of the smallest option G on type u over the type's jobs (a lower
                // bound: records only join a type's bound, never leave it -- conservative)
  uint32_t iit;  // types that the sequence's other-type moves go to
  uint32_t plim_lo, plim_hi;  // the fit limits (lim bytes) at the last computation's start
  // top list: the tcnt smallest same-type (case i) candidates of the type's
  // jobs, ascending by (key, priority, option); tall = it holds all of them
  double tk[kTop], tlo[kTop];
  uint32_t tt[kTop];
  int32_t ta[kTop], tp[kTop];
  int32_t tcnt, tall;
  int32_t qd[kQ], ql[kQ];  // work queues of the type warp
};

struct RoundShared {
  int32_t fr[kRT];
  int32_t toff[kRT + 1], tn[kRT];
  unsigned long long tcap[kRT];  // free + GPUs held by running jobs, per type
  int32_t n_adm, advance, any_change, lo;
  int32_t max_adm;           // the round's bound on the admitted records
  int32_t p_used, p_cap;     // option pool entries used / available
  int32_t po_first;          // pool offset of the first record of the current commit
  int32_t dmark;             // records [dmark, n_adm) were admitted since the last recompute
  int32_t n_vic, vic[kMaxDepth];  // records moved by the commit since the last recompute
  uint32_t changed;
  uint32_t stale;            // types whose sequence must be recomputed
  SeqTab sq[kRT];
  uint32_t wk1[kRoundWarps], wnd[kRoundWarps], wk2[kRoundWarps];
  int32_t res[kRoundThreads];  // per job of the batch: option index | log2 G << 8 | t << 13 | m << 16
  uint64_t bs_gmb[kRoundThreads], bs_tsb[kRoundThreads];  // per job of the batch, for its record
  int32_t bs_nopt[kRoundThreads];
  int32_t wsum[kRoundWarps];
  long long prof[8], prof2[8];
  int32_t cnt[12];
};

// ---- type lists -------------------------------------------------------------
__device__ __forceinline__ void list_remove(RoundShared &sh, const AdmView &A, int a) {
  const int u = A.t[a], s = A.slot[a];
  int32_t *tl = A.tl + sh.toff[u];
  const int last = tl[--sh.tn[u]];
  tl[s] = last;
  A.slot[last] = s;
}
__device__ __forceinline__ void list_add(RoundShared &sh, const AdmView &A, int a, int u) {
  CRIUS_CHECK(sh.tn[u] < sh.toff[u + 1] - sh.toff[u]);
  int32_t *tl = A.tl + sh.toff[u];
  const int s = sh.tn[u]++;
  tl[s] = a;
  A.slot[a] = s;
}

// Option i of admitted record a: (log2 G | t << 8) and its score, from the
// shared-memory pool when the record's options were staged there (po >= 0),
// else from the global option table.
__device__ __forceinline__ void opt_get(const RoundBuf &R, const AdmView &A, int po, int p, int i,
                                        int &lg, int &t, double &s) {
  if (po >= 0) {
    const int pk = A.ppk[po + i];
    lg = pk & 0xff;
    t = (pk >> 8) & 0xff;
    s = A.psc[po + i];
  } else {
    const OptRec o = ldg_opt(R.opt + (int64_t)p * R.maxopt + i);
    lg = ilog2_pow2((uint32_t)o.G);
    t = o.t;
    s = __ldg(R.score + (int64_t)p * R.maxopt + i);
  }
}

// One lane: the job's best same-type move (case i): argmin over its options on
// its type with smaller G (indices [first of type, cur) in (t, G) order) of
// key = (score(cur) - score(o')) / (G_cur - G_o'), ties -> lowest index.  The
// core takes the record's fields explicitly (the commit refreshes the records
// it changes while their fields are being written).
__device__ __forceinline__ void refresh_core(const RoundBuf &R, const AdmView &A, int p, int cv, int Gc,
                                             int tt, int po, uint64_t tsb, int &bi, double &bk,
                                             double &bl) {
  const int i0 = byte_of(tsb, tt);
  int lg, t2;
  double sc;
  opt_get(R, A, po, p, cv, lg, t2, sc);
  bi = -1;
  bk = 0.0;
  bl = 0.0;
#pragma unroll 4
  for (int i2 = i0; i2 < cv; ++i2) {  // ascending: strict < keeps the lowest index on ties
    double s2;
    opt_get(R, A, po, p, i2, lg, t2, s2);
    const double l = __dsub_rn(sc, s2);
    const double k = __ddiv_rn(l, (double)(Gc - (1 << lg)));
    if (bi < 0 || k < bk) {
      bi = i2 | (lg << 8);
      bk = k;
      bl = l;
    }
  }
}
__device__ __forceinline__ void refresh_i(const RoundBuf &R, const AdmView &A, int a) {
  int bi;
  double bk, bl;
  refresh_core(R, A, A.pos[a], A.cur[a], A.G[a], A.t[a], A.po[a], A.tsb[a], bi, bk, bl);
  A.bi[a] = bi;
  A.bk[a] = bk;
  A.bl[a] = bl;
}

// One lane: the job's best other-type move (case ii) under free' = f2: argmin
// over its options on other types with G2 <= f2[t2] of loss = score(cur) -
// score(o'), ties -> lowest index; key = loss / G_cur (exact: G_cur is a power
// of two).  Returns the packed move or -1.  At a sequence's start (free' = the
// state's free counts) the cached move is tagged kEiStart: it stays the argmin
// while the job's option is unchanged and no type's free count gains a power-of-
// two level (the options that fit only shrink) as long as it still fits itself.
constexpr int kEiStart = 1 << 30;
__device__ __forceinline__ int compute_ii(const RoundBuf &R, const AdmView &A, int a,
                                          const int32_t *f2, bool at_start = false) {
  const int p = A.pos[a], cv = A.cur[a], tt = A.t[a], Gc = A.G[a], po = A.po[a];
  const int nv = A.nopt[a];
  int lg, t2;
  double sc;
  opt_get(R, A, po, p, cv, lg, t2, sc);
  int bi = -1;
  double bl = 0.0;
  // options by score descending: loss = RN(score(cur) - score(o')) is
  // nondecreasing along them, so the first one that fits has the least loss;
  // later ones of equal loss (rounding) may have a lower index
  // (four entries per step: their loads are independent and issue together)
  const uint8_t *pm = R.operm + (int64_t)p * R.maxopt;
  constexpr int kW = 4;
  for (int r0 = 0; r0 < nv; r0 += kW) {
    int iv[kW], pv[kW];
    double sv[kW];
    bool ok[kW];
#pragma unroll
    for (int q = 0; q < kW; ++q) {
      const int r = min(r0 + q, nv - 1);
      iv[q] = po >= 0 ? (A.ppk[po + r] >> 16) & 0xff : (int)__ldg(pm + r);
    }
#pragma unroll
    for (int q = 0; q < kW; ++q) {
      int lq, tq;
      opt_get(R, A, po, p, iv[q], lq, tq, sv[q]);
      pv[q] = iv[q] | (lq << 8) | (tq << 16);
      ok[q] = r0 + q < nv && tq != tt && (1 << lq) <= f2[tq];
    }
    bool stop = false;
#pragma unroll
    for (int q = 0; q < kW; ++q) {
      if (stop || !ok[q]) continue;
      const double l = __dsub_rn(sc, sv[q]);
      if (bi >= 0 && l != bl) {
        stop = true;
      } else if (bi < 0 || iv[q] < (bi & 0xff)) {
        bi = pv[q];
        bl = l;
      }
    }
    if (stop) break;
  }
  A.ei[a] = bi >= 0 && at_start ? bi | kEiStart : bi;
  // bl / G_cur: G_cur = 2^k, so the quotient is the product with 2^-k (the
  // same real value, rounded once either way)
  if (bi >= 0) A.ek[a] = __dmul_rn(bl, __longlong_as_double((long long)(1023 - ilog2_pow2((uint32_t)Gc)) << 52));
  return bi;
}

// A lane's candidate move.
struct Cand {
  double key;
  uint32_t tie;  // priority position << 8 | option index
  int a, pk;     // record, packed new option (index | log2 G2 << 8 | t2 << 16)
  bool have;
};

__device__ __forceinline__ bool key_less(double k, uint32_t tie, double k2, uint32_t tie2) {
  return k < k2 || (k == k2 && tie < tie2);
}
__device__ __forceinline__ bool cand_less(double k, uint32_t tie, const Cand &b) {
  return !b.have || key_less(k, tie, b.key, b.tie);
}

__device__ __forceinline__ bool ii_fits(int pk, const int32_t *f2) {
  return (1 << ((pk >> 8) & 0xff)) <= f2[(pk >> 16) & 0xff];
}

// Record a's cached other-type move as a candidate (none if ei < 0).
__device__ __forceinline__ Cand ii_cand(const AdmView &A, int a, int ei) {
  Cand c;
  c.have = ei >= 0;
  if (c.have) {
    c.key = A.ek[a];
    c.tie = ((uint32_t)A.pos[a] << 8) | (ei & 0xff);
    c.a = a;
    c.pk = ei & ~kEiStart;
  }
  return c;
}

// Keep the lane's two best candidates (distinct records).
__device__ __forceinline__ void top2_take(Cand &b1, Cand &b2, const Cand &c) {
  if (!c.have) return;
  if (cand_less(c.key, c.tie, b1)) {
    b2 = b1;
    b1 = c;
  } else if (cand_less(c.key, c.tie, b2)) {
    b2 = c;
  }
}

// The type warp's top list in registers: lane i holds entry i.
struct TopLane {
  double k, l;  // key, loss
  uint32_t tie;
  int a, pk;
};

__device__ __forceinline__ TopLane top_shfl(const TopLane &x, int src) {
  TopLane y;
  y.k = __shfl_sync(0xffffffffu, x.k, src);
  y.l = __shfl_sync(0xffffffffu, x.l, src);
  y.tie = __shfl_sync(0xffffffffu, x.tie, src);
  y.a = __shfl_sync(0xffffffffu, x.a, src);
  y.pk = __shfl_sync(0xffffffffu, x.pk, src);
  return y;
}

// Insert candidate c into the sorted top list (cnt entries) if it belongs to
// the prefix the list represents: always when the list holds every candidate,
// else only below its last entry.  A full list drops its last entry.
__device__ __forceinline__ void top_insert(TopLane &x, int &cnt, bool &all, const TopLane &c) {
  const int lane = threadIdx.x & 31;
  if (!all) {
    if (cnt == 0) return;
    const double lk = __shfl_sync(0xffffffffu, x.k, cnt - 1);
    const uint32_t lt = __shfl_sync(0xffffffffu, x.tie, cnt - 1);
    if (!key_less(c.k, c.tie, lk, lt)) return;
  }
  const int p = __popc(__ballot_sync(0xffffffffu, lane < cnt && key_less(x.k, x.tie, c.k, c.tie)));
  const TopLane up = top_shfl(x, max(lane - 1, 0));
  if (lane > p) x = up;
  if (lane == p) x = c;
  if (cnt == kTop) all = false;  // the old last entry dropped out
  cnt = min(cnt + 1, kTop);
}

// Warp t: refill the top list with the kTopFill smallest same-type candidates
// of type t (every record of the type has a fresh cache).  Each lane keeps a
// sorted run of its records' 4 smallest; the warp pops the global minimum.
__device__ __forceinline__ void top_refill(const RoundShared &sh, const AdmView &A, int t, TopLane &x,
                                        int &cnt, bool &all) {
  const int lane = threadIdx.x & 31;
  const int n_t = sh.tn[t];
  const int32_t *tl = A.tl + sh.toff[t];
  constexpr int kL = 4;
  TopLane loc[kL];
  int nloc = 0, nmine = 0;
  // after the first pass a lane only takes candidates above the last one popped from it
  double lk = 0.0;
  uint32_t lt = 0;
  bool first = true;
  auto fill = [&]() {
    nloc = 0;
    for (int k = lane; k < n_t; k += 32) {
      const int a = tl[k], bi = A.bi[a];
      if (bi < 0) continue;
      const TopLane c{A.bk[a], A.bl[a], ((uint32_t)A.pos[a] << 8) | (bi & 0xff), a, bi | (t << 16)};
      if (first) ++nmine;
      else if (!key_less(lk, lt, c.k, c.tie)) continue;
      int pos = 0;
#pragma unroll
      for (int q = 0; q < kL; ++q) pos += (q < nloc && key_less(loc[q].k, loc[q].tie, c.k, c.tie));
      if (pos >= kL) continue;
#pragma unroll
      for (int q = kL - 1; q > 0; --q)
        if (q > pos) loc[q] = loc[q - 1];
#pragma unroll
      for (int q = 0; q < kL; ++q)
        if (q == pos) loc[q] = c;
      nloc = min(nloc + 1, kL);
    }
  };
  fill();
  first = false;
  int left = nmine;  // this lane's candidates not yet popped
  const int total = __reduce_add_sync(0xffffffffu, nmine);
  const int want = min(kTopFill, total);
  for (int i = 0; i < want; ++i) {
    const bool hv = nloc > 0;
    const int src = warp_lex_argmin(hv, ord_double(hv ? loc[0].k : 0.0), hv ? loc[0].tie : 0u);
    const TopLane w = top_shfl(loc[0], src);
    if (lane == i) x = w;
    if (lane == src) {
      lk = loc[0].k;
      lt = loc[0].tie;
#pragma unroll
      for (int q = 0; q < kL - 1; ++q) loc[q] = loc[q + 1];
      --nloc;
      --left;
      if (nloc == 0 && left > 0) fill();
    }
  }
  cnt = want;
  all = total <= want;
}

// Warp t: the greedy victim sequence of GPU type t from the current state (the
// §N6 ScaleResource move loop run for d moves without the G_o stop; an option
// on type t later uses the shortest prefix that frees G_o), its accumulated
// losses and the thresholds.  Per move: the argmin of (key, priority, option)
// over the unmoved type-t jobs' same-type moves (i) -- the first unmoved entry
// of the sorted top list -- and their other-type moves (ii) under free' -- a
// warp argmin over the lanes' best evaluated ones -- with key = loss / freed.
__device__ void type_sequence(RoundShared &sh, const RoundBuf &R, const AdmView &A, int t) {
  const int lane = threadIdx.x & 31, TT = R.T;
  const long long c0 = clock64();
  SeqTab &S = sh.sq[t];
  int32_t *f2 = S.f2;
  if (lane < TT) f2[lane] = sh.fr[lane];
  if (lane < kRT) S.dfr[0][lane] = 0;
  // a job has an other-type move iff on some other type u its smallest option
  // fits: byte_u(gminb) < lim_u = log2(free_u) + 1 (0 for u = t or free_u = 0)
  uint32_t lim_lo = 0, lim_hi = 0;
  if (!(R.policy & 2)) {
    const int f = lane < TT ? sh.fr[lane] : 0;
    const uint32_t l = (lane == t || f <= 0) ? 0u : (uint32_t)(ilog2_pow2((uint32_t)f) + 1);
    const uint32_t sl = lane < 4 ? l << (8 * lane) : 0u, sh_ = lane >= 4 && lane < 8 ? l << (8 * (lane - 4)) : 0u;
    lim_lo = __reduce_or_sync(0xffffffffu, sl);
    lim_hi = __reduce_or_sync(0xffffffffu, sh_);
  }
  // no type's limit grew since the last computation: cached start moves that
  // still fit stay exact (compute_ii)
  const bool mono = (__vcmpgtu4(lim_lo, S.plim_lo) | __vcmpgtu4(lim_hi, S.plim_hi)) == 0;
  // ---- (1) the top list: drop entries whose record changed or left the type
  int cnt = S.tcnt;
  bool all = S.tall != 0;
  TopLane x{S.tk[lane], S.tlo[lane], S.tt[lane], S.ta[lane], S.tp[lane]};
  {
    bool ok = lane < cnt;  // records admitted since the last recompute are in no list
    if (ok) {
      ok = A.t[x.a] == t;
      for (int i = 0; i < sh.n_vic; ++i) ok &= sh.vic[i] != x.a;
    }
    const uint32_t m = __ballot_sync(0xffffffffu, ok);
    if (m != (cnt >= 32 ? 0xffffffffu : (1u << cnt) - 1)) {
      const int nc = __popc(m);
      const int src = lane < nc ? (int)__fns(m, 0, lane + 1) : 0;
      x = top_shfl(x, src);
      cnt = nc;
    }
  }
  // ---- (2) refresh the stale same-type caches of the type's changed records
  // (admitted or moved since the last recompute) and insert them
  int nd = 0, n_ref = 0;
  bool refill = false;
  {
    int32_t *qd = S.qd;
    const int d0 = sh.dmark, d1 = sh.n_adm, nv = sh.n_vic;
    for (int k0 = 0; k0 < (d1 - d0) + nv; k0 += 32) {
      const int k = k0 + lane;
      int a = -1;
      if (k < d1 - d0) a = d0 + k;
      else if (k < d1 - d0 + nv) a = sh.vic[k - (d1 - d0)];
      const bool mine = a >= 0 && A.t[a] == t;
      const uint32_t mm = __ballot_sync(0xffffffffu, mine);
      if (mine && nd + __popc(mm & ((1u << lane) - 1)) < kQ) qd[nd + __popc(mm & ((1u << lane) - 1))] = a;
      nd += __popc(mm);
      if (mine && A.bi[a] == -2) refresh_i(R, A, a);  // lanes in parallel (a commit refreshed the rest)
    }
    __syncwarp();
    n_ref = nd;
    if (nd > 8 || nd > kQ) {
      refill = true;
    } else {
      for (int i = 0; i < nd; ++i) {
        const int a = qd[i], bi = A.bi[a];
        if (bi < 0) continue;
        const TopLane c{A.bk[a], A.bl[a], ((uint32_t)A.pos[a] << 8) | (bi & 0xff), a, bi | (t << 16)};
        top_insert(x, cnt, all, c);
      }
    }
  }
  if (refill || (!all && cnt < R.depth)) {
    top_refill(sh, A, t, x, cnt, all);
    if (lane == 0) atomicAdd(&sh.cnt[5], 1);
  }
  const long long ca = clock64();
  // ---- (3) other-type moves: the type's jobs with an option on another type
  // that fits, evaluated in parallel passes; each lane keeps its two best
  int32_t *ql = S.ql;
  const int n_t = sh.tn[t];
  const int32_t *tl = A.tl + sh.toff[t];
  int nl = 0, n_ii = 0;
  Cand b1, b2;
  b1.have = b2.have = false;
  bool b2_known = true;
  bool own_tl = false;  // more than kQ listed jobs: lane owns tl positions = lane mod 32
  if (lim_lo | lim_hi) {
    for (int k0 = 0; k0 < n_t; k0 += 32) {
      const int k = k0 + lane;
      int a = -1;
      bool listed = false;
      if (k < n_t) {
        a = tl[k];
        const uint64_t gb = A.gmb[a];
        listed = (__vcmpltu4((uint32_t)gb, lim_lo) | __vcmpltu4((uint32_t)(gb >> 32), lim_hi)) != 0;
        if (!listed) A.ei[a] = -1;
      }
      bool fresh = false;  // listed with an exact cached start move
      if (listed && mono) {
        const int ei = A.ei[a];
        fresh = ei >= 0 && (ei & kEiStart) && ii_fits(ei, f2);
      }
      const uint32_t ml = __ballot_sync(0xffffffffu, listed);
      const int slot = nl + __popc(ml & ((1u << lane) - 1));
      if (listed && slot < kQ) ql[slot] = fresh ? ~a : a;
      nl += __popc(ml);
      if (listed && slot >= kQ && !fresh) {  // queue full: evaluate this one in place
        compute_ii(R, A, a, f2, true);
        ++n_ii;
      }
    }
    __syncwarp();
    own_tl = nl > kQ;
    const int nq = min(nl, kQ);
    for (int i = lane; i < nq; i += 32) {
      const int qa = ql[i];
      if (qa >= 0) {
        compute_ii(R, A, qa, f2, true);
        ++n_ii;
      } else {
        ql[i] = ~qa;
      }
    }
    n_ii = __reduce_add_sync(0xffffffffu, n_ii);
    __syncwarp();

    if (!own_tl) {
      for (int i = lane; i < nq; i += 32) {
        const int a = ql[i];
        top2_take(b1, b2, ii_cand(A, a, A.ei[a]));
      }
    } else {
      for (int k = lane; k < n_t; k += 32) {
        const int a = tl[k];
        top2_take(b1, b2, ii_cand(A, a, A.ei[a]));
      }
    }
  } else {
    for (int k = lane; k < n_t; k += 32) A.ei[tl[k]] = -1;
  }
  __syncwarp();
  if (lane == 0) {
    atomicAdd(&sh.cnt[0], n_ref);
    atomicAdd(&sh.cnt[1], n_ii);
    atomicAdd(&sh.cnt[4], n_t);
  }
  const long long c1 = clock64();
  // ---- (4) the moves
  uint32_t iit = 0;   // (lane 0) types of the other-type moves
  bool imov = false;  // this lane's top-list entry was moved
  int m = 0, n_rescan = 0;
  double cacc = 0.0;  // ((0 + loss_1) + loss_2) + ... (fp64, in move order as in the oracle)
  // the lanes' best other-type candidate (argmin over b1), kept while no
  // lane's b1 changes (a same-type move that no other-type entry refers to)
  int src = -1;
  double sk = 0.0;
  uint32_t st = 0;
  bool b1_dirty = true;
  for (; m < R.depth; ++m) {
    const uint32_t im = __ballot_sync(0xffffffffu, lane < cnt && !imov);
    const int h = im ? __ffs(im) - 1 : 0;
    const double hk = __shfl_sync(0xffffffffu, x.k, h);
    const uint32_t ht = __shfl_sync(0xffffffffu, x.tie, h);
    if (b1_dirty) {
      src = warp_lex_argmin(b1.have, ord_double(b1.have ? b1.key : 0.0), b1.tie);
      sk = __shfl_sync(0xffffffffu, b1.key, max(src, 0));
      st = __shfl_sync(0xffffffffu, b1.tie, max(src, 0));
    }
    int wa, wpk;
    bool wii;
    double wl;
    if (im && (src < 0 || key_less(hk, ht, sk, st))) {
      wa = __shfl_sync(0xffffffffu, x.a, h);
      wpk = __shfl_sync(0xffffffffu, x.pk, h);
      wl = __shfl_sync(0xffffffffu, x.l, h);
      wii = false;
    } else if (src >= 0) {
      wa = __shfl_sync(0xffffffffu, b1.a, src);
      wpk = __shfl_sync(0xffffffffu, b1.pk, src);
      wii = true;
    } else {
      break;
    }
    const int Gc = A.G[wa], G2 = 1 << ((wpk >> 8) & 0xff), t2 = (wpk >> 16) & 0xff;
    const int freed = wii ? Gc : Gc - G2;
    if (wii) wl = __dmul_rn(sk, (double)Gc);  // key = loss / G_cur exactly (power of two)
    cacc = __dadd_rn(cacc, wl);
    if (lane == t) f2[t] += freed;
    if (wii && lane == t2) f2[t2] -= G2;
    if (lane == 0) {
      S.mv_a[m] = wa;
      S.mv_pk[m] = wpk;
      S.cum[m + 1] = cacc;
      if (wii) iit |= 1u << t2;
    }
    __syncwarp();
    if (lane < TT) S.dfr[m + 1][lane] = f2[lane] - sh.fr[lane];
    if (lane < cnt && x.a == wa) imov = true;
    bool rs = false, b1_ch = false;
    if (b2.have && b2.a == wa) {  // the moved job's other-type entry leaves the lane's pair
      b2.have = false;
      b2_known = false;
    }
    if (b1.have && b1.a == wa) {  // promote the second best
      b1 = b2;
      b2.have = false;
      rs = !b2_known;
      b2_known = false;
      b1_ch = true;
    }
    if (wii) {  // an other-type move only shrinks free' of type t2
      if (b1.have && !ii_fits(b1.pk, f2)) rs = true;
      if (b2.have && !ii_fits(b2.pk, f2)) {
        b2.have = false;
        b2_known = false;
      }
    }
    if (rs) {  // this lane's own jobs again (moved ones excluded, lost options re-evaluated)
      ++n_rescan;
      b1.have = b2.have = false;
      b2_known = true;
      const int n_own = own_tl ? n_t : min(nl, kQ);
      for (int i = lane; i < n_own; i += 32) {
        const int a = own_tl ? tl[i] : ql[i];
        bool moved = false;
        for (int q = 0; q <= m; ++q) moved |= S.mv_a[q] == a;
        if (moved) continue;
        int ei = A.ei[a];
        if (ei >= 0 && !ii_fits(ei, f2)) ei = compute_ii(R, A, a, f2);
        top2_take(b1, b2, ii_cand(A, a, ei));
      }
    }
    b1_dirty = __any_sync(0xffffffffu, b1_ch || rs);
  }
  n_rescan = __reduce_add_sync(0xffffffffu, n_rescan);
  if (lane == 0) atomicAdd(&sh.cnt[3], n_rescan);
  // the top list persists (the moves were speculative)
  S.tk[lane] = x.k;
  S.tlo[lane] = x.l;
  S.tt[lane] = x.tie;
  S.ta[lane] = x.a;
  S.tp[lane] = x.pk;
  if (lane == 0) {
    S.tcnt = cnt;
    S.tall = all;
  }
  const long long c2 = clock64();
  if (lane == 0) {
    S.cum[0] = 0.0;
    S.len = m;
    S.plim_lo = lim_lo;
    S.plim_hi = lim_hi;
    S.iit = iit;
  }
  __syncwarp();
  // thresholds: lane lg -> the shortest prefix with 2^lg <= free[t] + freed
  if (lane < kLgMax) {
    const int G = 1 << lane;
    double th = __longlong_as_double(0x7ff0000000000000ll);  // +inf: never succeeds
    int mm = -1;
    for (int q = 0; q <= m; ++q)
      if (G <= sh.fr[t] + S.dfr[q][t]) {
        th = S.cum[q];
        mm = q;
        break;
      }
    S.thr[lane] = th;
    S.thm[lane] = (int8_t)mm;
  }
  if (lane == 0) {
    const long long c3 = clock64();
    atomicAdd((unsigned long long *)&sh.prof[3], (unsigned long long)(c1 - c0));
    atomicAdd((unsigned long long *)&sh.prof[4], (unsigned long long)(c2 - c1));
    atomicAdd((unsigned long long *)&sh.prof[5], (unsigned long long)(c3 - c2));
    atomicAdd((unsigned long long *)&sh.prof2[0], (unsigned long long)(ca - c0));
    atomicAdd(&sh.cnt[6], 1);
  }
}

// After a commit (warp 0, lane u checks type u): drop the sequences the commit
// can have changed -- the types whose job set or a job's option changed, and
// the types one of whose jobs has an option on a type whose free count changed
// and that fits under the old or the new count (that changes its other-type
// moves).
__device__ __forceinline__ void invalidate(RoundShared &sh, int TT, uint32_t changed, int o_q, int n_q,
                                           int policy) {
  // lane q holds type q's free count before (o_q) and after (n_q) the commit
  const int u = threadIdx.x & 31;
  bool bad = u < TT && !((sh.stale >> u) & 1) && ((changed >> u) & 1);
  const bool chk = u < TT && !((sh.stale >> u) & 1) && !(policy & 2);
  const uint64_t gq = u < TT ? sh.sq[u].gq : ~0ull;
  const uint32_t iit = u < TT ? sh.sq[u].iit : 0u;
  for (int q = 0; q < TT; ++q) {
    const int o = __shfl_sync(0xffffffffu, o_q, q), n = __shfl_sync(0xffffffffu, n_q, q);
    if (!chk || bad || q == u || o == n) continue;
    if (n < o) {
      // fewer free GPUs on q only removes or worsens other-type moves to q:
      // the argmins of a sequence that made no move to q stand
      bad = (iit >> q) & 1;
    } else {
      const int g = byte_of(gq, q);
      bad = g != 0xff && (1 << g) <= n;
    }
  }
  const uint32_t m = __ballot_sync(0xffffffffu, bad);
  if (u == 0) {
    sh.stale |= m;
    sh.cnt[2] += __popc(m);
  }
}

// Warp-wide argmin of kappa over `nopt` option records passing `pred` -> index or -1.
template <typename Pred>
__device__ __forceinline__ int warp_best_option(const OptRec *o, int nopt, Pred pred) {
  const int lane = threadIdx.x & 31;
  int best = -1;
  OptRec bo{kInf, 0, 0};
  for (int i = lane; i < nopt; i += 32) {
    const OptRec x = ldg_opt(o + i);
    if (pred(i, x) && (best < 0 || kappa_less(x, bo))) {
      best = i;
      bo = x;
    }
  }
  const int src = warp_lex_argmin(best >= 0, (uint64_t)bo.T, kappa_tie(bo));
  return src < 0 ? -1 : __shfl_sync(0xffffffffu, best, src);
}

__device__ __forceinline__ void gq_join(RoundShared &sh, int t, uint64_t gb) {
  uint64_t &g = sh.sq[t].gq;
  g = ((uint64_t)__vminu4((uint32_t)(g >> 32), (uint32_t)(gb >> 32)) << 32) |
      __vminu4((uint32_t)g, (uint32_t)gb);
}

// po: the record's pool offset (allocated by the caller), -1 = none
__device__ __forceinline__ void adm_new(RoundShared &sh, const AdmView &A, int w, int pos, int idx,
                                        int G, int t, int po) {
  const int a = sh.n_adm++;
  CRIUS_CHECK(a < sh.max_adm && idx < sh.bs_nopt[w]);
  CRIUS_CHECK(po < 0 || po + sh.bs_nopt[w] <= sh.p_cap);
  const uint64_t gb = sh.bs_gmb[w];
  A.gmb[a] = gb;
  A.tsb[a] = sh.bs_tsb[w];
  A.nopt[a] = sh.bs_nopt[w];
  gq_join(sh, t, gb);
  A.po[a] = po;
  A.pos[a] = pos;
  A.cur[a] = idx;
  A.G[a] = G;
  A.t[a] = t;
  A.bi[a] = -2;
  A.ei[a] = -1;
  list_add(sh, A, a, t);
}

__device__ __forceinline__ int res_idx(int r) { return r & 0xff; }
__device__ __forceinline__ int res_G(int r) { return 1 << ((r >> 8) & 0x1f); }
__device__ __forceinline__ int res_t(int r) { return (r >> 13) & 0x7; }
__device__ __forceinline__ int res_m(int r) { return (r >> 16) & 0x1f; }

// First set bit over per-warp ballot words (every lane of the calling warp
// gets it); kRoundThreads if none.
__device__ __forceinline__ int first_bit(const uint32_t *w) {
  const int lane = threadIdx.x & 31;
  const uint32_t x = lane < kRoundWarps ? w[lane] : 0u;
  const uint32_t b = __ballot_sync(0xffffffffu, x != 0);
  if (!b) return kRoundThreads;
  const int fw = __ffs(b) - 1;
  return fw * 32 + __ffs(__shfl_sync(0xffffffffu, x, fw)) - 1;
}

// Bytes of dynamic shared memory per admitted record (the AdmView fields; the
// type lists add 4 bytes per entry, bounded per type by its GPU count).
constexpr int kRecBytes = 5 * 8 + 9 * 4;
constexpr int kAO = 8;  // arrival options a batch thread keeps in registers

// Warp: copy the options of records [a0, a1) into the pool (two records per
// pass, 16 lanes each) with cp.async; the copying threads wait before the
// barrier that ends the next direct evaluation (the pool is read only after it).
__device__ __forceinline__ void stage_options(const RoundBuf &R, const AdmView &A, int a0, int a1) {
  const int lane = threadIdx.x & 31;
  for (int a = a0 + (lane >> 4); a < a1; a += 2) {
    const int po = A.po[a];
    if (po < 0) continue;
    const int64_t q = (int64_t)A.pos[a] * R.maxopt;
    const int nv = A.nopt[a];
    for (int i = lane & 15; i < nv; i += 16) {
      cp_async4(A.ppk + po + i, R.opk + q + i);
      cp_async8(A.psc + po + i, R.score + q + i);
    }
  }
}

// Warp: copy job `pos`'s nv options into the pool at po (cp.async, as above).
__device__ __forceinline__ void stage_job(const RoundBuf &R, const AdmView &A, int pos, int nv, int po) {
  const int lane = threadIdx.x & 31;
  const int64_t q = (int64_t)pos * R.maxopt;
  for (int i = lane; i < nv; i += 32) {
    cp_async4(A.ppk + po + i, R.opk + q + i);
    cp_async8(A.psc + po + i, R.score + q + i);
  }
}

__device__ __forceinline__ int pool_alloc(RoundShared &sh, int nv) {
  if (sh.p_used + nv > sh.p_cap) return -1;
  const int po = sh.p_used;
  sh.p_used += nv;
  return po;
}

// K6.
// kSmem: the admitted records live in shared memory (the launch fails with
// err = 3 when the round's bound on them does not fit; the host then relaunches
// the global-memory instantiation).  With the records' address space known at
// compile time every record access is a plain shared-memory instruction.
template <bool kSmem>
__global__ void __launch_bounds__(kRoundThreads, 1) k_round(RoundBuf R) {
  __shared__ RoundShared sh;
  extern __shared__ __align__(16) unsigned char dsm[];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int TT = R.T, J = R.J;
  if (tid < TT) sh.fr[tid] = R.free_io[tid];
  if (tid < 8) {
    sh.prof[tid] = 0;
    sh.prof2[tid] = 0;
    sh.cnt[tid] = 0;
    if (tid < 4) sh.cnt[8 + tid] = 0;
  }
  if (tid == 0) {
    sh.n_adm = 0;
    sh.stale = (1u << TT) - 1;
    sh.dmark = 0;
    sh.n_vic = 0;
  }
  if (tid < kRT) {
    sh.sq[tid].tcnt = 0;
    sh.sq[tid].tall = 1;
    sh.sq[tid].gq = ~0ull;
    sh.sq[tid].plim_lo = sh.sq[tid].plim_hi = 0u;
  }
  __syncthreads();
  long long c_start = clock64();

  // ---- capacity: every admitted job holds >= 1 GPU of its type, and GPUs are
  // conserved per type, so type u never holds more than its free count + the
  // GPUs its running jobs hold; records <= min(J, sum over types)
  if (tid < TT) sh.tcap[tid] = (unsigned long long)sh.fr[tid];
  __syncthreads();
  if (R.run_cell)
    for (int pos = tid; pos < J; pos += kRoundThreads) {
      const int ro = R.run_opt[pos];
      if (ro >= 0) {
        const OptRec x = R.opt[(int64_t)pos * R.maxopt + ro];
        atomicAdd(&sh.tcap[x.t], (unsigned long long)x.G);
      }
    }
  __syncthreads();
  int64_t cap_sum = 0, list_sum = 0;
  for (int u = 0; u < TT; ++u) {
    if (sh.tcap[u] > (1ull << 30)) {  // int32 free counts along a sequence stay exact below 2^31
      if (tid == 0) *R.err = 2;
      return;
    }
    cap_sum += (int64_t)sh.tcap[u];
  }
  const int max_adm = (int)min(cap_sum, (int64_t)J);
  for (int u = 0; u < TT; ++u) list_sum += min((int64_t)sh.tcap[u], (int64_t)max_adm);
  const int64_t rec_bytes = (int64_t)max_adm * kRecBytes + list_sum * 4;
  constexpr bool in_smem = kSmem;
  if (kSmem && rec_bytes > R.smem_bytes) {
    if (tid == 0) *R.err = 3;
    return;
  }
  AdmView A = R.glob;
  int pcap = 0;
  if (kSmem) {
    unsigned char *p = dsm;
    A.bk = (double *)p;
    A.bl = A.bk + max_adm;
    A.ek = A.bl + max_adm;
    A.gmb = (uint64_t *)(A.ek + max_adm);
    A.tsb = A.gmb + max_adm;
    A.pos = (int32_t *)(A.tsb + max_adm);
    A.cur = A.pos + max_adm;
    A.G = A.cur + max_adm;
    A.t = A.G + max_adm;
    A.slot = A.t + max_adm;
    A.bi = A.slot + max_adm;
    A.ei = A.bi + max_adm;
    A.nopt = A.ei + max_adm;
    A.po = A.nopt + max_adm;
    A.tl = A.po + max_adm;
    // the rest is the option pool: 12 bytes per option
    const int64_t pb = (rec_bytes + 15) & ~15ll;
    pcap = (int)max((int64_t)0, min((R.smem_bytes - pb) / 12, (int64_t)INT32_MAX / 2));
    A.psc = (double *)(dsm + pb);
    A.ppk = (int32_t *)(A.psc + pcap);
  }
  if (tid == 0) {
    int o = 0;
    for (int u = 0; u < TT; ++u) {
      sh.toff[u] = o;
      o += in_smem ? (int)min((int64_t)sh.tcap[u], (int64_t)max_adm) : J;
      sh.tn[u] = 0;
    }
    sh.toff[TT] = o;
    sh.max_adm = max_adm;
    sh.p_used = 0;
    sh.p_cap = pcap;
  }
  __syncthreads();

  // ---- running jobs start admitted, in priority order (NEXT-4 round state)
  if (R.run_cell) {
    int base = 0;
    for (int p0 = 0; p0 < J; p0 += kRoundThreads) {
      const int pos = p0 + tid;
      const int ro = pos < J ? R.run_opt[pos] : -1;
      const unsigned b = __ballot_sync(0xffffffffu, ro >= 0);
      if (lane == 0) sh.wsum[wid] = __popc(b);
      __syncthreads();
      int before = base;
      for (int w = 0; w < wid; ++w) before += sh.wsum[w];
      if (ro >= 0) {
        const int a = before + __popc(b & ((1u << lane) - 1));
        const OptRec x = R.opt[(int64_t)pos * R.maxopt + ro];
        A.pos[a] = pos;
        A.cur[a] = ro;
        A.G[a] = x.G;
        A.t[a] = x.t;
        A.bi[a] = -2;
        A.ei[a] = -1;
        A.gmb[a] = R.gminb[pos];
        A.tsb[a] = R.tsb[pos];
        A.nopt[a] = R.nopt[pos];
      }
      for (int w = 0; w < kRoundWarps; ++w) base += sh.wsum[w];
      __syncthreads();
    }
    // type lists: warp u appends its type's records (in record order)
    if (wid < TT) {
      int n = 0;
      int32_t *tl = A.tl + sh.toff[wid];
      for (int a0 = 0; a0 < base; a0 += 32) {
        const int a = a0 + lane;
        const bool mine = a < base && A.t[a] == wid;
        const unsigned b = __ballot_sync(0xffffffffu, mine);
        if (mine) {
          const int s = n + __popc(b & ((1u << lane) - 1));
          tl[s] = a;
          A.slot[a] = s;
        }
        n += __popc(b);
      }
      if (lane == 0) sh.tn[wid] = n;
      uint32_t g_lo = 0xffffffffu, g_hi = 0xffffffffu;
      for (int k = lane; k < n; k += 32) {
        const uint64_t gb = A.gmb[tl[k]];
        g_lo = __vminu4(g_lo, (uint32_t)gb);
        g_hi = __vminu4(g_hi, (uint32_t)(gb >> 32));
      }
#pragma unroll
      for (int d = 16; d >= 1; d >>= 1) {
        g_lo = __vminu4(g_lo, __shfl_xor_sync(0xffffffffu, g_lo, d));
        g_hi = __vminu4(g_hi, __shfl_xor_sync(0xffffffffu, g_hi, d));
      }
      if (lane == 0) sh.sq[wid].gq = ((uint64_t)g_hi << 32) | g_lo;
    }
    // option pool offsets in record order
    if (tid == 0) {
      sh.n_adm = base;
      for (int a = 0; a < base; ++a) {
        const int nv = A.nopt[a];
        int po = -1;
        if (sh.p_used + nv <= sh.p_cap) {
          po = sh.p_used;
          sh.p_used += nv;
        }
        A.po[a] = po;
      }
    }
    __syncthreads();
    for (int a0 = 2 * wid; a0 < base; a0 += 2 * kRoundWarps) stage_options(R, A, a0, min(a0 + 2, base));
    cp_async_wait_all();
    __syncthreads();
  }
  const int n_run = sh.n_adm;

  // ---- Phase A: SchedArrival in priority order.  A window of kRoundThreads
  // jobs (thread = job) stays in registers while its jobs are decided: each
  // iteration evaluates the undecided jobs [lo, kRoundThreads) against the
  // current state and commits the first that changes it.
  long long n_batches = 0, n_seq = 0, n_scale = 0, c_seq = 0;
  long long n_bar = 0;  // CTA-wide barriers on the round's critical chain
  long long tb = clock64();
  for (int w0 = 0; w0 < J; w0 += kRoundThreads) {
    const int q = w0 + tid;
    int na = 0;
    int apk[kAO];
    double asc[kAO];
    if (q < J) {
      const int cq = __ldg(R.cand + q), nq = __ldg(R.nao + q);
#pragma unroll
      for (int u = 0; u < kAO; ++u)
        if (u < R.maxopt) {
          apk[u] = __ldg(R.ao_pk + (int64_t)u * J + q);
          asc[u] = __ldg(R.ao_sc + (int64_t)u * J + q);
        }
      sh.bs_gmb[tid] = __ldg(R.gminb + q);
      sh.bs_tsb[tid] = __ldg(R.tsb + q);
      sh.bs_nopt[tid] = __ldg(R.nopt + q);
      na = cq ? nq : 0;
    }
    int lo = 0;  // jobs [0, lo) of the window are decided
    while (lo < kRoundThreads && w0 + lo < J) {
      // (1) direct choice: the job's first arrival option (kappa order) that fits
      bool k1 = false, need = false;
      int r = 0;
      if (tid >= lo && na > 0) {
#pragma unroll
        for (int u = 0; u < kAO; ++u)
          if (!k1 && u < na && res_G(apk[u]) <= sh.fr[res_t(apk[u])]) {
            k1 = true;
            r = apk[u];
          }
        for (int k = kAO; k < na && !k1; ++k) {
          const int pk = __ldg(R.ao_pk + (int64_t)k * J + q);
          if (res_G(pk) <= sh.fr[res_t(pk)]) {
            k1 = true;
            r = pk;
          }
        }
        need = !k1 && R.depth >= 1;
      }
      sh.res[tid] = r;
      {
        const uint32_t b1 = __ballot_sync(0xffffffffu, k1), bn = __ballot_sync(0xffffffffu, need);
        if (lane == 0) {
          sh.wk1[wid] = b1;
          sh.wnd[wid] = bn;
          sh.wk2[wid] = 0;
        }
      }
      cp_async_wait_all();  // the last commit's option staging (read from here on)
      __syncthreads();
      ++n_bar;
      ++n_batches;
      if (tid == 0) {
        const long long t1 = clock64();
        sh.prof[0] += t1 - tb;
        tb = t1;
      }
      const int fa = first_bit(sh.wk1);
      // any job before fa that needs ScaleResource?
      bool nb;
      {
        const uint32_t x = lane < kRoundWarps ? sh.wnd[lane] : 0u;
        const int w = lane * 32;
        const uint32_t xm = w + 32 <= fa ? x : (w < fa ? x & ((1u << (fa - w)) - 1) : 0u);
        nb = __ballot_sync(0xffffffffu, xm != 0) != 0;
      }
      if (nb) {
        if (sh.stale) {
          const long long c0 = clock64();
          if (tid == 0) sh.cnt[7] += __popc(sh.stale);
          if (wid < TT && ((sh.stale >> wid) & 1)) type_sequence(sh, R, A, wid);
          __syncthreads();
      ++n_bar;
          if (tid == 0) {
            sh.stale = 0;
            sh.dmark = sh.n_adm;  // every changed record's cache is fresh again
            sh.n_vic = 0;
            c_seq += clock64() - c0;
            ++n_seq;
          }
        }
        // (2) ScaleResource(q): the first option in kappa order whose trial succeeds
        bool k2 = false;
        if (need && tid < fa) {
          int r2 = 0;
#pragma unroll
          for (int u = 0; u < kAO; ++u)
            if (!k2 && u < na) {
              const SeqTab &S = sh.sq[res_t(apk[u])];
              const int lg = (apk[u] >> 8) & 0x1f;
              if (asc[u] > S.thr[lg]) {
                k2 = true;
                r2 = apk[u] | ((int)S.thm[lg] << 16);
              }
            }
          for (int k = kAO; k < na && !k2; ++k) {
            const int pk = __ldg(R.ao_pk + (int64_t)k * J + q);
            const SeqTab &S = sh.sq[res_t(pk)];
            const int lg = (pk >> 8) & 0x1f;
            if (__ldg(R.ao_sc + (int64_t)k * J + q) > S.thr[lg]) {
              k2 = true;
              r2 = pk | ((int)S.thm[lg] << 16);
            }
          }
          if (k2) sh.res[tid] = r2;
        }
        const uint32_t b2 = __ballot_sync(0xffffffffu, k2);
        if (lane == 0) sh.wk2[wid] = b2;
        __syncthreads();
      ++n_bar;
        if (tid == 0) {
          const long long t1 = clock64();
          sh.prof[1] += t1 - tb;
          tb = t1;
        }
      }
      // (3) commit the first job f that changes the state: warp 0 updates the
      // records and free counts, warp 1 stages job f's options in the pool, and
      // (ScaleResource) warp 2 invalidates the sequences and warp 3 refreshes
      // the changed records' same-type caches meanwhile -- every input of that
      // is in the sequence and the result word
      if (wid <= 3) {
        const int f2n = nb ? first_bit(sh.wk2) : kRoundThreads;
        const int f = min(fa, f2n);
        const bool scale = f < kRoundThreads && f2n < fa;
        if (wid == 2) {
          const int o = lane < TT ? sh.fr[lane] : 0;  // nobody writes them before bar 1
          asm volatile("bar.sync 1, 128;" ::: "memory");
          if (scale) {
            const int rr = sh.res[f], t = res_t(rr), m = res_m(rr), G = res_G(rr);
            const SeqTab &S = sh.sq[t];
            const int n = lane < TT ? o + S.dfr[m][lane] - (lane == t ? G : 0) : 0;
            // the victims are type-t jobs; the other-type ones land on t2
            const uint32_t ch = lane < m ? 1u << ((S.mv_pk[lane] >> 16) & 0xff) : 0u;
            invalidate(sh, TT, __reduce_or_sync(0xffffffffu, ch) | (1u << t), o, n, R.policy);
          }
        } else if (wid == 1) {
          if (lane == 0) sh.po_first = f < kRoundThreads ? pool_alloc(sh, sh.bs_nopt[f]) : -1;
          asm volatile("bar.sync 1, 128;" ::: "memory");
          if (f < kRoundThreads && sh.po_first >= 0) stage_job(R, A, w0 + f, sh.bs_nopt[f], sh.po_first);
        } else if (wid == 3) {
          const int an = sh.n_adm;  // nobody writes it before bar 1
          asm volatile("bar.sync 1, 128;" ::: "memory");
          if (scale) {
            const int rr = sh.res[f], t = res_t(rr), m = res_m(rr);
            const SeqTab &S = sh.sq[t];
            int a = -1, p = 0, cv = 0, Gc = 0, tt = 0, po = -1;
            uint64_t tsb = 0;
            if (lane < m) {  // victim: its new option; pos, po, tsb do not change
              const int pk = S.mv_pk[lane];
              a = S.mv_a[lane];
              p = A.pos[a];
              po = A.po[a];
              tsb = A.tsb[a];
              cv = pk & 0xff;
              Gc = 1 << ((pk >> 8) & 0xff);
              tt = (pk >> 16) & 0xff;
            } else if (lane == m) {  // the new record (its pool copy is being staged: global path)
              a = an;
              p = w0 + f;
              tsb = sh.bs_tsb[f];
              cv = res_idx(rr);
              Gc = res_G(rr);
              tt = t;
            }
            if (a >= 0) {
              int bi;
              double bk, bl;
              refresh_core(R, A, p, cv, Gc, tt, po, tsb, bi, bk, bl);
              A.bi[a] = bi;
              A.bk[a] = bk;
              A.bl[a] = bl;
            }
          }
        } else {
          asm volatile("bar.sync 1, 128;" ::: "memory");
          const int a_new = sh.n_adm;
          const int old = lane < TT ? sh.fr[lane] : 0;  // free counts before the commit
          if (scale) {
            // ScaleResource: the first m moves of the type's sequence (lane mm
            // updates victim mm), the free counts (lane u), then job f's record
            const int rr = sh.res[f], t = res_t(rr), m = res_m(rr), G = res_G(rr);
            const SeqTab &S = sh.sq[t];
            if (lane < TT) sh.fr[lane] = old + S.dfr[m][lane] - (lane == t ? G : 0);
            bool moved_type = false;
            if (lane < m) {
              const int a = S.mv_a[lane], pk = S.mv_pk[lane];
              moved_type = ((pk >> 16) & 0xff) != t;
              A.cur[a] = pk & 0xff;
              A.G[a] = 1 << ((pk >> 8) & 0xff);  // bi: warp 3 writes the refreshed cache
              A.ei[a] = -1;
              sh.vic[sh.n_vic + lane] = a;
            }
            const uint32_t mt = __ballot_sync(0xffffffffu, moved_type);
            __syncwarp();
            if (lane == 0) {
              ++n_scale;
              const int an = a_new;
              CRIUS_CHECK(an < sh.max_adm && res_idx(rr) < sh.bs_nopt[f] && m <= S.len);
              A.pos[an] = w0 + f;
              A.cur[an] = res_idx(rr);
              A.G[an] = G;
              A.t[an] = t;
              A.ei[an] = -1;
              A.gmb[an] = sh.bs_gmb[f];
              A.tsb[an] = sh.bs_tsb[f];
              A.nopt[an] = sh.bs_nopt[f];
              A.po[an] = sh.po_first;
              // victims that changed type move between the type lists
              for (uint32_t b = mt; b; b &= b - 1) {
                const int mm = __ffs(b) - 1;
                const int a = S.mv_a[mm], t2 = (S.mv_pk[mm] >> 16) & 0xff;
                list_remove(sh, A, a);
                A.t[a] = t2;
                list_add(sh, A, a, t2);
                gq_join(sh, t2, A.gmb[a]);
              }
              sh.n_vic += m;
              sh.n_adm = an + 1;
              list_add(sh, A, an, t);
              gq_join(sh, t, sh.bs_gmb[f]);
              sh.lo = f + 1;
            }
          } else {
            uint32_t changed = 0;
            if (lane == 0) {
              int adv = kRoundThreads;
              if (f < kRoundThreads) {  // direct admissions, chained while later choices provably stand
                int w = f;
                for (;;) {
                  const int rr = sh.res[w], t = res_t(rr);
                  adm_new(sh, A, w, w0 + w, res_idx(rr), res_G(rr), t,
                          w == f ? sh.po_first : pool_alloc(sh, sh.bs_nopt[w]));
                  sh.fr[t] -= res_G(rr);
                  changed |= 1u << t;
                  adv = w + 1;
                  // A direct admission only lowers one free count, so a later job's
                  // direct choice stands iff its option still fits; a job that stays
                  // pending without ScaleResource is unaffected.
                  bool more = false;
                  while (++w < kRoundThreads && w0 + w < J) {
                    const bool wk = (sh.wk1[w >> 5] >> (w & 31)) & 1;
                    const bool wn = (sh.wnd[w >> 5] >> (w & 31)) & 1;
                    if (wk) {
                      const int r2 = sh.res[w];
                      more = res_G(r2) <= sh.fr[res_t(r2)];
                      break;
                    }
                    if (!wn) {
                      adv = w + 1;
                      continue;
                    }
                    break;
                  }
                  if (!more) break;
                }
              }
              sh.lo = adv;
            }
            __syncwarp();
            if (f < kRoundThreads) {
              invalidate(sh, TT, __shfl_sync(0xffffffffu, changed, 0), old, lane < TT ? sh.fr[lane] : 0,
                         R.policy);
              stage_options(R, A, a_new + 1, sh.n_adm);  // the chain's later records
            }
          }
        }
      }
      __syncthreads();
      ++n_bar;
      lo = sh.lo;
      if (tid == 0) {
        const long long t1 = clock64();
        sh.prof[2] += t1 - tb;
        tb = t1;
      }
    }
  }
  cp_async_wait_all();
  __syncthreads();
  const long long c_phaseB = clock64();

  // ---- Phase B: up to d sweeps of reverse scaling over admitted jobs, in
  // priority order.  Records [0, n_run) (running jobs) and [n_run, n_adm)
  // (Phase A) are each in priority order: merge by binary search.
  const int n_adm = sh.n_adm;
  int32_t *ord = R.ord;
  for (int a = tid; a < n_adm; a += kRoundThreads) {
    const int pa = A.pos[a];
    const bool first = a < n_run;
    int lo = first ? n_run : 0, hi = first ? n_adm : n_run;  // count of the other run with pos < pa
    const int base = lo;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (A.pos[mid] < pa) lo = mid + 1;
      else hi = mid;
    }
    ord[(first ? a : a - n_run) + (lo - base)] = a;
  }
  __syncthreads();
      ++n_bar;
  long long n_bb = 0;
  for (int sweep = 0; sweep < R.depth; ++sweep) {
    if (tid == 0) sh.any_change = 0;
    __syncthreads();
      ++n_bar;
    for (int a0 = 0; a0 < n_adm;) {
      const int a = a0 + wid < n_adm ? ord[a0 + wid] : n_adm;
      int opt = -1;
      if (a < n_adm) {
        const int pos = A.pos[a], cv = A.cur[a], Gc = A.G[a], tc = A.t[a];
        const OptRec *o = R.opt + (int64_t)pos * R.maxopt;
        const int64_t Tc = o[cv].T;
        opt = warp_best_option(o, R.nopt[pos], [&](int i, const OptRec &x) {
          const int avail = sh.fr[x.t] + (x.t == tc ? Gc : 0);
          return i != cv && x.G <= avail && x.T < Tc &&
                 (!(R.policy & 2) || x.t == tc);  // NH keeps the type
        });
      }
      if (lane == 0) sh.res[wid] = opt;
      __syncthreads();
      ++n_bar;
      if (tid == 0) {
        int f = 0;
        while (f < kRoundWarps && sh.res[f] < 0) ++f;
        if (f < kRoundWarps) {
          const int aa = ord[a0 + f];
          const OptRec x = R.opt[(int64_t)A.pos[aa] * R.maxopt + sh.res[f]];
          sh.fr[A.t[aa]] += A.G[aa];
          if (A.t[aa] != x.t) {
            list_remove(sh, A, aa);
            list_add(sh, A, aa, x.t);
          }
          A.cur[aa] = sh.res[f];
          A.ei[aa] = -1;
          A.G[aa] = x.G;
          A.t[aa] = x.t;
          sh.fr[x.t] -= x.G;
          sh.any_change = 1;
        }
        sh.advance = f < kRoundWarps ? f + 1 : kRoundWarps;
      }
      __syncthreads();
      ++n_bar;
      a0 += sh.advance;
      ++n_bb;
    }
    if (!sh.any_change) break;
  }
  const long long c_end = clock64();

  // ---- total score in priority order (fp64, sequential: bit-reproducible)
  for (int k = tid; k < n_adm; k += kRoundThreads) {
    const int a = ord[k], pos = A.pos[a];
    R.osc[k] = R.score[(int64_t)pos * R.maxopt + A.cur[a]];
    R.cur[pos] = A.cur[a];
  }
  __syncthreads();
  if (tid == 0) {
    double tot = 0.0;
    for (int k = 0; k < n_adm; ++k) tot = __dadd_rn(tot, R.osc[k]);
    *R.total = tot;
    if (R.stats) {
      R.stats[0] = n_batches;
      R.stats[1] = n_seq;
      R.stats[2] = c_seq;
      R.stats[3] = c_phaseB - c_start;
      R.stats[4] = c_end - c_phaseB;
      R.stats[5] = n_adm;
      R.stats[6] = n_scale;
      R.stats[7] = n_bb;
      R.stats[8] = sh.prof[0];
      R.stats[9] = sh.prof[1];
      R.stats[10] = sh.prof[2];
      R.stats[11] = sh.cnt[0];
      R.stats[12] = sh.cnt[1];
      R.stats[13] = sh.cnt[2];
      R.stats[14] = in_smem;
      R.stats[15] = max_adm;
      R.stats[16] = sh.prof[3];
      R.stats[17] = sh.prof[4];
      R.stats[18] = sh.prof[5];
      R.stats[19] = sh.cnt[3];
      R.stats[20] = sh.cnt[4];
      R.stats[21] = sh.cnt[5];
      R.stats[22] = sh.cnt[6];
      R.stats[23] = sh.prof2[0];
      R.stats[25] = sh.cnt[7];

      R.stats[28] = n_bar;
    }
  }
  if (tid < TT) R.free_io[tid] = sh.fr[tid];
  __syncthreads();
  for (int pos = tid; pos < J; pos += kRoundThreads) {
    const int j = R.pi[pos];
    const int c = R.cur[pos];
    const bool act = R.active ? R.active[j] != 0 : true;
    R.decision[j] = !act ? -3 : R.ref[pos] == kInf ? -2 : (c < 0 ? -1 : R.opt_cell[(int64_t)pos * R.maxopt + c]);
  }
}

// K7: d_all[c] = gathered[r * stride + (c - cell_begin[r])] for the rank r owning c.
struct CompactArgs {
  int64_t cb[9];
  int32_t world;
  int64_t stride, n_cells;
};
__global__ void k_compact(const CellResult *__restrict__ g, CompactArgs A, CellResult *__restrict__ all) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= A.n_cells) return;
  int r = 0;
  while (r + 1 < A.world && A.cb[r + 1] <= c) ++r;
  all[c] = g[r * A.stride + (c - A.cb[r])];
}

}  // namespace crius
