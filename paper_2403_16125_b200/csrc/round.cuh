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
// K5 builds O_j for every job in priority order (one thread per job).
// K6 is ONE CTA of 32 warps (the round is sequential by definition) that
// extracts parallelism without changing the result:
//  * speculative batches -- a job that stays pending changes no state, so 32
//    consecutive jobs are evaluated at once (one per warp) against the same
//    state; the first one that changes the state is committed and the next
//    batch starts right after it: the exact sequential order of §N6;
//  * ScaleResource tries the job's options in kappa order and stops at the
//    first success; each option's success depends only on the state, so the
//    lanes test all options at once and take the kappa-argmin of the successes;
//  * the victim-move sequence of a trial depends only on the state and on the
//    option's GPU type t_o (G_o only decides where it is cut), so the greedy
//    sequence of every type is computed once per state and reused until an
//    admission changes it: per-job caches of the best same-type move and of
//    the best other-type move (staged options in shared memory), then one
//    group of warps per type runs the d moves with one named barrier per move.
#pragma once
#include "common.cuh"

namespace crius {

struct OptRec {  // 16 B
  int64_t T;
  int32_t G;
  int32_t t;
};

// Cached best other-type move (case (ii)) of the listed jobs, entry k of the
// list: the option with t2 != t and G2 <= free'[t2] of minimum loss = sc - s2
// (ties -> lowest index); i = -1 if none.  Shared memory up to kECap entries.
#ifndef CRIUS_ECAP
#define CRIUS_ECAP 256
#endif
constexpr int kECap = CRIUS_ECAP;
struct EView {
  double *loss, *s2, *key;  // key = loss / G_cur (the move's ScaleResource key)
  int64_t *T2;
  int32_t *i, *G2, *t2;
};

struct RoundBuf {
  int32_t J, T, maxopt, depth;
  int32_t policy;        // NEXT-4 ablations (R-11): bit 0 NA (options at G = N_G only),
                         // bit 1 NH (admitted jobs keep their GPU type)
  const int64_t *tmax;   // [J] by job or NULL: deadline bound on an option's T (R-12)
  const int32_t *rank;   // [J] job -> priority position
  const int32_t *pi;     // [J] position -> job
  OptRec *opt;           // [J][maxopt] by position, (t, G) ascending
  double *score;         // [J][maxopt] score(o) = ref / T_o (A-16)
  int64_t *opt_cell;     // [J][maxopt]
  int32_t *nopt;         // [J] by position
  int64_t *ref;          // [J] by position (kInf = unschedulable)
  int32_t *ng;           // [J] by position
  int32_t *cur;          // [J] by position: option index or -1
  int64_t *decision;     // [J] by job
  int32_t *free_io;      // [T]
  double *total;
  int64_t *stats;        // [16] counters (see crius_round_stats)
  int32_t *list;         // [J] scratch list (used when admitted records live in global memory)
  // NEXT-4 round state (NULL = every job active, none running)
  const int64_t *run_cell;  // [J] by job: Cell the job runs on, or -1
  const uint8_t *active;    // [J] by job: the job takes part in this round
  int32_t *run_opt;         // [J] by position: option index of the running Cell, or -1
  int8_t *cand;             // [J] by position: 1 = Phase A candidate (active, not running)
  EView eg;                 // [J] (ii) caches when more than kECap jobs are listed
};

__device__ __forceinline__ double score_of(int64_t ref, int64_t T) {
  return __ddiv_rn((double)ref, (double)T);
}

// K5: per job (thread), options, ref and scores from its Cells (contiguous,
// (t, G, S) order), written at the job's priority position.
__global__ void k_round_options(Params P, const int64_t *__restrict__ ucb,
                                const int32_t *__restrict__ cType, const int32_t *__restrict__ cG,
                                const CellResult *__restrict__ res, RoundBuf R) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= R.J) return;
  const int pos = R.rank[j];
  const int64_t c0 = ucb[(int64_t)j * R.T], c1 = ucb[(int64_t)(j + 1) * R.T];
  const int ngj = P.ng[j];
  OptRec *o = R.opt + (int64_t)pos * R.maxopt;
  int64_t *oc = R.opt_cell + (int64_t)pos * R.maxopt;
  int n = 0;
  int64_t ref_ng = kInf, ref_any = kInf;
  int lastT = -1, lastG = -1;
  const bool act0 = R.active ? R.active[j] != 0 : true;
  const int64_t rc0 = (act0 && R.run_cell) ? R.run_cell[j] : -1;
  const int64_t tmx = R.tmax ? R.tmax[j] : kInf;
  for (int64_t c = c0; c < c1; ++c) {
    const int64_t T = res[c].t_ns;
    const int t = cType[c], G = cG[c];
    if (T == kInf) continue;
    ref_any = min(ref_any, T);
    if (G == ngj) ref_ng = min(ref_ng, T);
    if ((R.policy & 1) && G != ngj) continue;  // NA: the job stays at N_G GPUs
    // deadline: a Cell slower than the job's bound is no option, except the
    // (type, G) the job runs on (its completion was guaranteed at placement)
    if (T > tmx && !(rc0 >= 0 && t == cType[rc0] && G == cG[rc0])) continue;
    if (t == lastT && G == lastG) {
      if (T < o[n - 1].T) {  // equal T keeps the earlier (smaller S) Cell
        o[n - 1].T = T;
        oc[n - 1] = c;
      }
    } else {
      o[n].T = T;
      o[n].G = G;
      o[n].t = t;
      oc[n] = c;
      ++n;
      lastT = t;
      lastG = G;
    }
  }
  const int64_t ref = ref_ng != kInf ? ref_ng : ref_any;
  double *sc = R.score + (int64_t)pos * R.maxopt;
  for (int i = 0; i < n; ++i) sc[i] = score_of(ref, o[i].T);
  R.nopt[pos] = n;
  R.ref[pos] = ref;
  R.ng[pos] = ngj;
  R.cur[pos] = -1;
  // round state: a running job keeps the option of its Cell's (type, G)
  const bool act = R.active ? R.active[j] != 0 : true;
  int ro = -1;
  if (act && R.run_cell && R.run_cell[j] >= 0) {
    const int64_t rc = R.run_cell[j];
    for (int i = 0; i < n; ++i)
      if (o[i].t == cType[rc] && o[i].G == cG[rc]) ro = i;
    CRIUS_CHECK(ro >= 0);
  }
  R.run_opt[pos] = ro;
  R.cand[pos] = (int8_t)(act && ro < 0 && ref != kInf);
}

// Option records are read-only inside K6: load them through the non-coherent
// (L1-cached) path so repeated scans of the same admitted jobs hit L1.
__device__ __forceinline__ OptRec ldg_opt(const OptRec *p) {
  const longlong2 v = __ldg(reinterpret_cast<const longlong2 *>(p));
  OptRec r;
  r.T = v.x;
  r.G = (int32_t)(v.y & 0xffffffff);
  r.t = (int32_t)(v.y >> 32);
  return r;
}

__device__ __forceinline__ bool kappa_less(const OptRec &a, const OptRec &b) {
  if (a.T != b.T) return a.T < b.T;
  if (a.G != b.G) return a.G < b.G;
  return a.t < b.t;
}

constexpr int kRoundThreads = 1024;
constexpr int kRT = 8;  // GPU types supported by the round kernel (shared-memory tables)
constexpr int kRoundWarps = kRoundThreads / 32;
#ifndef CRIUS_ADM_SMEM
#define CRIUS_ADM_SMEM 2048
#endif
constexpr int kAdmSmem = CRIUS_ADM_SMEM;  // admitted-job records kept in shared memory up to this many
constexpr int kAdmBytes = 76;   // bytes per admitted-job record (incl. scratch list)

// Other-type options of the listed jobs, staged in shared memory by the warp
// that fills their entry (po[k] = offset, pn[k] = count, -1 = not staged:
// refills then re-read the options from global memory).
#ifndef CRIUS_POOL
#define CRIUS_POOL 512
#endif
constexpr int kPool = CRIUS_POOL;
struct OptPool {
  int64_t *T2;
  double *s2;
  int32_t *G2, *ti;  // ti = t2 << 8 | option index
  int32_t *po, *pn;
  int32_t *used;
};

// Admitted jobs, in priority order (SoA; shared memory when they fit, else global).
// bi_* caches the job's best same-type victim move (case (i) of ScaleResource),
// which depends only on its current option: bi_opt = -2 marks a stale cache
// (set whenever the option changes), -1 = no such move.  gmin = the job's
// smallest option G (an other-type move (ii) needs G_o' <= free'[t_o']).
struct AdmView {
  int64_t *T, *bi_T;
  double *sc, *bi_key, *bi_s;
  int32_t *pos, *cur, *G, *t, *nopt, *bi_opt, *bi_G2, *gmin;
};

// Window of upcoming jobs (priority positions [w0, w0 + wn)) staged in shared memory.
struct JobWin {
  int64_t *ref;
  int32_t *nopt, *ng;
  int8_t *cand;
  OptRec *opt;
  double *score;
  int cap, w0, wn;
};

struct RoundShared {
  int32_t fr[kRT];
  int32_t n_adm, advance, any_change, n_dirty, n_list, n_invalid;
  // per-type sequence validity: a sequence is reused until a job of its type
  // changes or a changed free count could admit an other-type move of one of its
  // jobs (gmin_type = smallest option G over its jobs, a conservative bound)
  int32_t seq_ok[kRT], comp[kRT], gmin_type[kRT];
  int32_t fr_base[kRT][kRT];  // free counts the sequence was computed from
  int32_t old_fr[kRT];        // free counts before the current commit (thread 0)
  uint32_t changed;           // types changed by the current commit; 0 = no commit
  long long prof[12];  // cycles: [0] setup+dirty, [1] listing, [2] (ii) caches, [3] sequences; [4] dirty jobs, [5] listed jobs
  // victim-move sequences, one per GPU type, cut at <= d moves
  int32_t len[kRT];
  int32_t mv_a[kRT][kMaxDepth], mv_opt[kRT][kMaxDepth];
  int32_t mv_G[kRT][kMaxDepth], mv_t[kRT][kMaxDepth];  // the victim's new option
  int64_t mv_T[kRT][kMaxDepth];
  double mv_sc[kRT][kMaxDepth];
  double cum[kRT][kMaxDepth + 1];                 // ((0 + loss_1) + loss_2) + ...
  int32_t frs[kRT][kMaxDepth + 1][kRT];      // free' after m moves
  int32_t fmax_other[kRT];                         // max_{t2 != t} free'[t2]
  // per-warp outcome of one speculative batch
  int32_t res_kind[kRoundWarps], res_opt[kRoundWarps], res_m[kRoundWarps], need[kRoundWarps];
  int32_t res_G[kRoundWarps], res_t[kRoundWarps];
  int64_t res_T[kRoundWarps];
  double res_sc[kRoundWarps];
  // per-warp best move of the current sequence step (type groups of warps,
  // double-buffered by move parity), each warp's free' and moved jobs
  double g_key[2][kRoundWarps];
  uint32_t g_tie[2][kRoundWarps];
  int32_t g_a[2][kRoundWarps], g_idx[2][kRoundWarps], g_G2[2][kRoundWarps];
  int32_t g_t2o[2][kRoundWarps], g_freed[2][kRoundWarps];
  int32_t wf2[kRoundWarps][kRT], wmv[kRoundWarps][kMaxDepth];
  // cached best other-type moves of the listed jobs (EView, up to kECap)
  double e_loss[kECap], e_s2[kECap], e_key[kECap];
  int64_t e_T2[kECap];
  int32_t e_i[kECap], e_G2[kECap], e_t2[kECap], e_po[kECap], e_pn[kECap];
  // their other-type options (OptPool)
  int64_t p_T2[kPool];
  double p_s2[kPool];
  int32_t p_G2[kPool], p_ti[kPool], p_used;
};

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

// Warp: refresh the same-type move cache (case (i)) and gmin of admitted job a.
// The cached move is the job's argmin of key = loss / freed over its same-type
// options with smaller G, ties -> lowest option index.  Lanes cover the job's
// options (coalesced 16-byte records and their scores, one round trip).
__device__ __forceinline__ void refresh_victim_cache(const RoundBuf &R, const AdmView &A, int a) {
  const int lane = threadIdx.x & 31;
  const int v = A.pos[a], cv = A.cur[a], Gc = A.G[a], t = A.t[a], nv = A.nopt[a];
  const double sc = A.sc[a];
  bool have = false;
  double bk = 0.0, bs = 0.0;
  int bi = 0, bG = 0;
  int64_t bT = 0;
  int gmin = INT32_MAX;
  for (int i2 = lane; i2 < nv; i2 += 32) {
    const OptRec o2 = ldg_opt(R.opt + (int64_t)v * R.maxopt + i2);
    const double s2 = __ldg(R.score + (int64_t)v * R.maxopt + i2);
    gmin = min(gmin, o2.G);
    if (i2 == cv || o2.t != t || o2.G >= Gc) continue;
    const double k = __ddiv_rn(sc - s2, (double)(Gc - o2.G));
    if (!have || k < bk) {  // i2 ascending per lane: ties keep the lower index
      have = true;
      bk = k;
      bs = s2;
      bi = i2;
      bG = o2.G;
      bT = o2.T;
    }
  }
  gmin = (int)__reduce_min_sync(0xffffffffu, (unsigned)gmin);
  const int src = warp_lex_argmin(have, ord_double(bk), (uint32_t)bi);
  if (src < 0) {
    if (lane == 0) A.bi_opt[a] = -1;
  } else if (lane == src) {
    A.bi_opt[a] = bi;
    A.bi_key[a] = bk;
    A.bi_G2[a] = bG;
    A.bi_T[a] = bT;
    A.bi_s[a] = bs;
  }
  if (lane == 0) A.gmin[a] = gmin;
}

// Warp: fill entry k for admitted job a under free' = f2 (lanes over options)
// and stage the job's other-type options in the pool when it has room.
__device__ __forceinline__ void other_type_best_warp(const RoundBuf &R, const AdmView &A, int a,
                                                     const int32_t *f2, const EView &E, int k,
                                                     const OptPool *pool) {
  const int lane = threadIdx.x & 31;
  const int v = A.pos[a], t = A.t[a], nv = A.nopt[a];
  const double sc = A.sc[a];
  int off = -1;
  if (pool) {
    if (lane == 0) {
      off = atomicAdd(pool->used, nv);
      if (off + nv > kPool) off = -1;
    }
    off = __shfl_sync(0xffffffffu, off, 0);
  }
  int cnt = 0;
  bool have = false;
  double bl = 0.0, bs = 0.0;
  int bi = 0, bG = 0, bt = 0;
  int64_t bT = 0;
  for (int i0 = 0; i0 < nv; i0 += 32) {
    const int i2 = i0 + lane;
    OptRec o2{0, 0, t};
    double s2 = 0.0;
    if (i2 < nv) {
      o2 = ldg_opt(R.opt + (int64_t)v * R.maxopt + i2);
      s2 = __ldg(R.score + (int64_t)v * R.maxopt + i2);
    }
    const bool oth = i2 < nv && o2.t != t;
    if (off >= 0) {
      const unsigned bm = __ballot_sync(0xffffffffu, oth);
      if (oth) {
        const int q = off + cnt + __popc(bm & ((1u << lane) - 1));
        pool->T2[q] = o2.T;
        pool->s2[q] = s2;
        pool->G2[q] = o2.G;
        pool->ti[q] = (o2.t << 8) | i2;
      }
      cnt += __popc(bm);
    }
    if (!oth || o2.G > f2[o2.t]) continue;
    const double l = sc - s2;
    if (!have || l < bl) {
      have = true;
      bl = l;
      bs = s2;
      bi = i2;
      bG = o2.G;
      bt = o2.t;
      bT = o2.T;
    }
  }
  if (pool && lane == 0) {
    pool->po[k] = off;
    pool->pn[k] = cnt;
  }
  const int src = warp_lex_argmin(have, ord_double(bl), (uint32_t)bi);
  if (src < 0) {
    if (lane == 0) E.i[k] = -1;
  } else if (lane == src) {
    E.i[k] = bi;
    E.loss[k] = bl;
    E.key[k] = __ddiv_rn(bl, (double)A.G[a]);
    E.s2[k] = bs;
    E.G2[k] = bG;
    E.t2[k] = bt;
    E.T2[k] = bT;
  }
}

// One lane: recompute entry k after a (ii) move took GPUs its option needed
// (free' only decreases for the other types along a sequence); options from
// the pool (shared memory) when staged, else from global memory.
__device__ __forceinline__ int other_type_best_lane(const RoundBuf &R, const AdmView &A, int a,
                                                    const int32_t *f2, const EView &E, int k,
                                                    const OptPool *pool) {
  const double sc = A.sc[a];
  int bi = -1;
  double bl = 0.0;
  const int off = pool ? pool->po[k] : -1;
  if (off >= 0) {  // other-type options in index order
    const int n = pool->pn[k];
    int bq = -1;
    for (int q = off; q < off + n; ++q) {
      const int ti = pool->ti[q], G2 = pool->G2[q];
      if (G2 > f2[ti >> 8]) continue;
      const double l = sc - pool->s2[q];
      if (bi < 0 || l < bl) {
        bi = ti & 0xff;
        bl = l;
        bq = q;
      }
    }
    if (bq >= 0) {
      E.loss[k] = bl;
      E.key[k] = __ddiv_rn(bl, (double)A.G[a]);
      E.s2[k] = pool->s2[bq];
      E.G2[k] = pool->G2[bq];
      E.t2[k] = pool->ti[bq] >> 8;
      E.T2[k] = pool->T2[bq];
    }
    E.i[k] = bi;
    return bi;
  }
  const int v = A.pos[a], t = A.t[a], nv = A.nopt[a];
#pragma unroll 4
  for (int i2 = 0; i2 < nv; ++i2) {
    const OptRec o2 = ldg_opt(R.opt + (int64_t)v * R.maxopt + i2);
    const double s2 = __ldg(R.score + (int64_t)v * R.maxopt + i2);
    if (o2.t == t || o2.G > f2[o2.t]) continue;
    const double l = sc - s2;
    if (bi < 0 || l < bl) {
      bi = i2;
      bl = l;
      E.loss[k] = l;
      E.s2[k] = s2;
      E.G2[k] = o2.G;
      E.t2[k] = o2.t;
      E.T2[k] = o2.T;
    }
  }
  if (bi >= 0) E.key[k] = __ddiv_rn(bl, (double)A.G[a]);
  E.i[k] = bi;
  return bi;
}

__device__ __forceinline__ void group_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Warps [t*gw, (t+1)*gw): the greedy victim sequence of GPU type t (the §N6
// ScaleResource move loop run for d moves without the G_o stop; an option on
// type t later uses the shortest prefix that frees G_o).  Per move, the argmin
// of (key, priority position, option) over the unmoved type-t jobs' cached
// same-type moves (i) and the listed jobs' cached other-type moves (ii),
// key = loss / freed.  One named barrier (1 + t) per move: every warp reduces
// the group's per-warp winners itself (slots double-buffered by move parity)
// and keeps its own copy of free' and of the moved jobs; the group's first
// warp records the sequence.
__device__ void type_sequence(RoundShared &sh, const RoundBuf &R, const AdmView &A,
                              const int32_t *list, int nE, const EView &E, const OptPool *pool,
                              int t, int gw) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int gwid = wid - t * gw, gt = gwid * 32 + lane, gn = gw * 32, w0 = t * gw;
  const int n_adm = sh.n_adm, TT = R.T;
  int32_t *f2 = sh.wf2[wid];
  int32_t *mv = sh.wmv[wid];
  if (lane < TT) f2[lane] = sh.frs[t][0][lane];
  __syncwarp();
  // each thread's best cached same-type move (i) over its strided jobs only
  // changes when that job is moved: rescan only then
  bool hv1 = false;
  double bk1 = 0.0;
  int bp1 = 0, bi1 = 0, ba1 = -1;
  bool rescan = true;
  for (int m = 0; m < R.depth; ++m) {
    if (rescan) {
      hv1 = false;
      ba1 = -1;
      for (int a = gt; a < n_adm; a += gn) {  // (i): loads issued together
        const int ta = A.t[a], bo = A.bi_opt[a], p = A.pos[a];
        const double k = A.bi_key[a];
        bool moved = false;
        for (int q = 0; q < m; ++q) moved |= mv[q] == a;
        if (ta != t || bo < 0 || moved) continue;
        if (!hv1 || k < bk1 || (k == bk1 && (p < bp1 || (p == bp1 && bo < bi1)))) {
          hv1 = true;
          bk1 = k;
          bp1 = p;
          bi1 = bo;
          ba1 = a;
        }
      }
    }
    bool have = hv1;
    double bk = bk1;
    int bp = bp1, bi = bi1, ba = ba1, bidx = -1;
    for (int k = gt; k < nE; k += gn) {  // (ii)
      const int a = list[k];
      const int ta = A.t[a], p = A.pos[a], G2 = E.G2[k], t2 = E.t2[k];
      int ei = E.i[k];
      double key = E.key[k];
      bool moved = false;
      for (int q = 0; q < m; ++q) moved |= mv[q] == a;
      if (ta != t || moved) continue;
      if (ei >= 0 && G2 > f2[t2]) {
        ei = other_type_best_lane(R, A, a, f2, E, k, pool);
        key = E.key[k];
      }
      if (ei < 0) continue;
      if (!have || key < bk || (key == bk && (p < bp || (p == bp && ei < bi)))) {
        have = true;
        bk = key;
        bp = p;
        bi = ei;
        ba = a;
        bidx = k;
      }
    }
    const uint32_t tie = ((uint32_t)bp << 8) | (uint32_t)bi;
    const int src = warp_lex_argmin(have, ord_double(bk), tie);
    const int par = m & 1;
    if (lane == 0) sh.g_a[par][wid] = -1;
    __syncwarp();
    if (lane == src) {
      int G2, t2o, freed;
      if (bidx < 0) {
        G2 = A.bi_G2[ba];
        t2o = t;
        freed = A.G[ba] - G2;
      } else {
        G2 = E.G2[bidx];
        t2o = E.t2[bidx] | 0x100;
        freed = A.G[ba];
      }
      sh.g_key[par][wid] = bk;
      sh.g_tie[par][wid] = tie;
      sh.g_a[par][wid] = ba;
      sh.g_idx[par][wid] = bidx;
      sh.g_G2[par][wid] = G2;
      sh.g_t2o[par][wid] = t2o;
      sh.g_freed[par][wid] = freed;
    }
    group_bar(1 + t, gn);
    // every warp: the group's winner (lanes < gw hold the per-warp winners)
    const int w = w0 + lane;
    const bool in = lane < gw && sh.g_a[par][w] >= 0;
    const int wl = warp_lex_argmin(in, ord_double(in ? sh.g_key[par][w] : 0.0),
                                   in ? sh.g_tie[par][w] : 0u);
    if (wl < 0) break;
    const int ws = w0 + wl;
    const int ca = sh.g_a[par][ws], t2o = sh.g_t2o[par][ws], G2 = sh.g_G2[par][ws];
    const int t2 = t2o & 0xff, other = t2o >> 8;
    if (lane < TT) {
      int f = f2[lane];
      if (lane == t) f += sh.g_freed[par][ws];
      if (lane == t2 && other) f -= G2;
      f2[lane] = f;
      if (gwid == 0) sh.frs[t][m + 1][lane] = f;
    }
    if (lane == 0) mv[m] = ca;
    rescan = ba1 == ca;  // this thread's (i) candidate was moved
    if (gwid == 0 && lane == 0) {  // record move m
      const int idx = sh.g_idx[par][ws];
      const double s2 = idx < 0 ? A.bi_s[ca] : E.s2[idx];
      sh.mv_a[t][m] = ca;
      sh.mv_opt[t][m] = (int)(sh.g_tie[par][ws] & 0xff);
      sh.mv_G[t][m] = G2;
      sh.mv_t[t][m] = t2;
      sh.mv_T[t][m] = idx < 0 ? A.bi_T[ca] : E.T2[idx];
      sh.mv_sc[t][m] = s2;
      sh.cum[t][m + 1] = __dadd_rn(sh.cum[t][m], A.sc[ca] - s2);
      sh.len[t] = m + 1;
    }
    __syncwarp();
  }
}

// All threads: the victim sequences of every stale GPU type from the current
// state.  (1) refresh the stale same-type caches (one warp per job); (2) list
// the jobs that may have an other-type move (smallest option G <= the largest
// free count of another type -- free' of the other types only decreases along
// a sequence, so this superset holds for every move); (3) their best
// other-type move under the current free counts (one warp per job); (4) one
// warp per stale type runs its d moves from shared-memory caches only.
__device__ void compute_all_seqs(RoundShared &sh, const RoundBuf &R, const AdmView &A,
                                 int32_t *list, const EView &Es) {
  const int tid = threadIdx.x, wid = tid >> 5;
  const int TT = R.T, n_adm = sh.n_adm;
  if (tid < TT) {
    const int c = !sh.seq_ok[tid];
    sh.comp[tid] = c;
    if (c) {
      sh.len[tid] = 0;
      sh.cum[tid][0] = 0.0;
      sh.gmin_type[tid] = INT32_MAX;
      int fm = -1;
      for (int q = 0; q < TT; ++q)
        if (q != tid) fm = max(fm, sh.fr[q]);
      sh.fmax_other[tid] = (R.policy & 2) ? -1 : fm;  // NH: no other-type victim move
    }
  }
  if (tid < TT * TT && !sh.seq_ok[tid / TT]) {
    sh.frs[tid / TT][0][tid % TT] = sh.fr[tid % TT];
    sh.fr_base[tid / TT][tid % TT] = sh.fr[tid % TT];
  }
  if (tid == 0) {
    sh.n_dirty = 0;
    sh.p_used = 0;
  }
  long long t0 = clock64();
  __syncthreads();
  // (1) stale same-type caches -> list -> one warp per job
  for (int a = tid; a < n_adm; a += kRoundThreads)
    if (A.bi_opt[a] == -2) list[atomicAdd(&sh.n_dirty, 1)] = a;
  CRIUS_CHECK(n_adm <= R.J);
  __syncthreads();
  for (int k = wid; k < sh.n_dirty; k += kRoundWarps) refresh_victim_cache(R, A, list[k]);
  if (tid == 0) sh.n_list = 0;
  __syncthreads();
  if (tid == 0) {
    const long long t1 = clock64();
    sh.prof[0] += t1 - t0;
    sh.prof[4] += sh.n_dirty;
    t0 = t1;
  }
  // (2) gmin per type; listed jobs
  for (int a = tid; a < n_adm; a += kRoundThreads) {
    const int myt = A.t[a];
    if (!sh.comp[myt]) continue;
    const int g = A.gmin[a];
    atomicMin(&sh.gmin_type[myt], g);
    if (g <= sh.fmax_other[myt]) list[atomicAdd(&sh.n_list, 1)] = a;
  }
  __syncthreads();
  const int nE = sh.n_list;
  const EView E = nE <= kECap ? Es : R.eg;
  if (tid == 0) {
    const long long t1 = clock64();
    sh.prof[1] += t1 - t0;
    sh.prof[5] += nE;
    t0 = t1;
  }
  // (3) best other-type move of each listed job under the current free counts
  OptPool pl{sh.p_T2, sh.p_s2, sh.p_G2, sh.p_ti, sh.e_po, sh.e_pn, &sh.p_used};
  const OptPool *pool = nE <= kECap ? &pl : nullptr;
  for (int k = wid; k < nE; k += kRoundWarps) other_type_best_warp(R, A, list[k], sh.fr, E, k, pool);
  __syncthreads();
  if (tid == 0) {
    const long long t1 = clock64();
    sh.prof[2] += t1 - t0;
    t0 = t1;
  }
  // (4) one warp per stale type
  {
#ifndef CRIUS_SEQ_WARPS
#define CRIUS_SEQ_WARPS 32
#endif
    const int gw = min(CRIUS_SEQ_WARPS, kRoundWarps / TT), t = wid / gw;  // warps per type
    if (t < TT && sh.comp[t]) type_sequence(sh, R, A, list, nE, E, pool, t, gw);
  }
  __syncthreads();
  if (tid == 0) {
    const long long t1 = clock64();
    sh.prof[3] += t1 - t0;
  }
  if (tid < TT && sh.comp[tid]) sh.seq_ok[tid] = 1;
  __syncthreads();
}

// Warp 0 after a commit (lane t checks type t): drop the sequences the commit
// can have changed.  sh.changed = types whose job set or a job's option changed;
// sh.old_fr = free counts before the commit.
__device__ __forceinline__ void invalidate_seqs(RoundShared &sh, int TT) {
  const int t = threadIdx.x & 31;
  if (t >= TT || !sh.seq_ok[t]) return;
  bool bad = (sh.changed >> t) & 1;
  for (int q = 0; q < TT && !bad; ++q)
    if (q != t && sh.old_fr[q] != sh.fr[q] && sh.gmin_type[t] <= max(sh.old_fr[q], sh.fr[q]))
      bad = true;
  if (bad) {
    sh.seq_ok[t] = 0;
    atomicAdd(&sh.n_invalid, 1);
  }
}

// Warp-wide argmin of kappa over `nopt` option records passing `pred` -> index or -1.
template <typename Pred>
__device__ __forceinline__ int warp_best_option(const OptRec *o, int nopt, Pred pred) {
  const int lane = threadIdx.x & 31;
  int best = -1;
  OptRec bo{kInf, 0, 0};
  for (int i = lane; i < nopt; i += 32) {
    const OptRec x = o[i];
    if (pred(i, x) && (best < 0 || kappa_less(x, bo))) {
      best = i;
      bo = x;
    }
  }
  const int src = warp_lex_argmin(best >= 0, (uint64_t)bo.T, kappa_tie(bo));
  return src < 0 ? -1 : __shfl_sync(0xffffffffu, best, src);
}

// (Re)point admitted record a at option `opt` (G, t, T, score) of job `pos`.
__device__ __forceinline__ void adm_set(const AdmView &A, const RoundBuf &R, int a, int pos, int opt,
                                        int G, int t, int64_t T, double sc) {
  A.pos[a] = pos;
  A.cur[a] = opt;
  A.G[a] = G;
  A.t[a] = t;
  A.T[a] = T;
  A.sc[a] = sc;
  A.bi_opt[a] = -2;
  R.cur[pos] = opt;
}

// All threads: stage positions [w0, w0 + cap) into the shared window.
__device__ void load_window(JobWin &W, const RoundBuf &R, int w0) {
  const int tid = threadIdx.x;
  const int wn = min(W.cap, R.J - w0);
  for (int i = tid; i < wn; i += kRoundThreads) {
    W.ref[i] = R.ref[w0 + i];
    W.nopt[i] = R.nopt[w0 + i];
    W.ng[i] = R.ng[w0 + i];
    W.cand[i] = R.cand[w0 + i];
  }
  const int n = wn * R.maxopt;
  const longlong2 *so = reinterpret_cast<const longlong2 *>(R.opt + (int64_t)w0 * R.maxopt);
  longlong2 *d = reinterpret_cast<longlong2 *>(W.opt);
  for (int i = tid; i < n; i += kRoundThreads) {
    d[i] = so[i];
    W.score[i] = R.score[(int64_t)w0 * R.maxopt + i];
  }
  W.w0 = w0;
  W.wn = wn;
  __syncthreads();
}

// K6.  Speculative batches: warp w evaluates job pos0 + w against the current
// state.  A job that stays pending changes nothing, so the first job of the
// batch that is admitted (directly or through ScaleResource) is committed and
// the next batch starts right after it -- exactly the sequential §N6 order.
__global__ void __launch_bounds__(kRoundThreads, 1) k_round_greedy(RoundBuf R, int adm_in_smem,
                                                                   AdmView Aglob, int win_cap) {
  __shared__ RoundShared sh;
  extern __shared__ __align__(16) unsigned char dsm[];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int TT = R.T;
  // dynamic shared memory: [window][admitted records]
  unsigned char *p = dsm;
  JobWin W;
  W.cap = win_cap;
  W.opt = (OptRec *)p;
  p += (size_t)win_cap * R.maxopt * sizeof(OptRec);
  W.score = (double *)p;
  p += (size_t)win_cap * R.maxopt * sizeof(double);
  W.ref = (int64_t *)p;
  p += (size_t)win_cap * 8;
  W.nopt = (int32_t *)p;
  p += (size_t)win_cap * 4;
  W.ng = (int32_t *)p;
  p += (size_t)win_cap * 4;
  W.cand = (int8_t *)p;
  p += (size_t)win_cap * 8;
  AdmView A = Aglob;
  if (adm_in_smem) {
    A.T = (int64_t *)p;
    A.bi_T = A.T + kAdmSmem;
    A.sc = (double *)(A.bi_T + kAdmSmem);
    A.bi_key = A.sc + kAdmSmem;
    A.bi_s = A.bi_key + kAdmSmem;
    A.pos = (int32_t *)(A.bi_s + kAdmSmem);
    A.cur = A.pos + kAdmSmem;
    A.G = A.cur + kAdmSmem;
    A.t = A.G + kAdmSmem;
    A.nopt = A.t + kAdmSmem;
    A.bi_opt = A.nopt + kAdmSmem;
    A.bi_G2 = A.bi_opt + kAdmSmem;
    A.gmin = A.bi_G2 + kAdmSmem;
  }
  int32_t *list = adm_in_smem ? (int32_t *)(A.gmin + kAdmSmem) : R.list;
  if (tid < TT) sh.fr[tid] = R.free_io[tid];
  if (tid == 0) {
    sh.n_adm = 0;
    sh.n_invalid = 0;
  }
  if (tid < kRT) sh.seq_ok[tid] = 0;
  if (tid == 0) sh.changed = 0;
  if (tid < 12) sh.prof[tid] = 0;
  __syncthreads();
  long long c_start = clock64(), c_seq = 0, n_batches = 0, n_seq = 0, n_scale = 0, n_bb = 0;
  load_window(W, R, 0);
  // running jobs start admitted, in priority order (NEXT-4 round state)
  if (R.run_cell) {
    __shared__ int32_t wsum[kRoundWarps];
    int base = 0;
    for (int p0 = 0; p0 < R.J; p0 += kRoundThreads) {
      const int pos = p0 + tid;
      const int ro = pos < R.J ? R.run_opt[pos] : -1;
      const unsigned b = __ballot_sync(0xffffffffu, ro >= 0);
      if (lane == 0) wsum[wid] = __popc(b);
      __syncthreads();
      int before = base;
      for (int w = 0; w < wid; ++w) before += wsum[w];
      if (ro >= 0) {
        const int a = before + __popc(b & ((1u << lane) - 1));
        const OptRec x = R.opt[(int64_t)pos * R.maxopt + ro];
        adm_set(A, R, a, pos, ro, x.G, x.t, x.T, R.score[(int64_t)pos * R.maxopt + ro]);
        A.nopt[a] = R.nopt[pos];
      }
      for (int w = 0; w < kRoundWarps; ++w) base += wsum[w];
      __syncthreads();
    }
    if (tid == 0) sh.n_adm = base;
    __syncthreads();
  }

  // ---- Phase A: SchedArrival in priority order
  long long tb = clock64();
  for (int pos0 = 0; pos0 < R.J;) {
    if (pos0 + kRoundWarps > W.w0 + W.wn && W.w0 + W.wn < R.J) load_window(W, R, pos0);
    if (tid == 0) {
      const long long t1 = clock64();
      sh.prof[8] += t1 - tb;
      tb = t1;
    }
    const int q = pos0 + wid, wq = q - W.w0;
    CRIUS_CHECK(q >= R.J || (wq >= 0 && wq < W.wn));
    int kind = 0, opt = -1, need = 0;
    if (q < R.J && W.cand[wq]) {
      const int nopt = W.nopt[wq], ngj = W.ng[wq];
      const int best = warp_best_option(W.opt + (size_t)wq * R.maxopt, nopt,
                                        [&](int, const OptRec &x) {
                                          return x.G <= ngj && x.G <= sh.fr[x.t];
                                        });
      if (best >= 0) {
        kind = 1;
        opt = best;
      } else if (R.depth >= 1) {
        need = 1;
      }
    }
    if (lane == 0) {
      sh.res_kind[wid] = kind;
      sh.res_opt[wid] = opt;
      sh.need[wid] = need;
    }
    __syncthreads();
    ++n_batches;
    if (tid == 0) {
      const long long t1 = clock64();
      sh.prof[9] += t1 - tb;
      tb = t1;
    }
    const unsigned kmask = __ballot_sync(0xffffffffu, lane < kRoundWarps && sh.res_kind[lane] != 0);
    const int fa = kmask ? __ffs(kmask) - 1 : kRoundWarps;
    const unsigned nmask = __ballot_sync(0xffffffffu, lane < fa && sh.need[lane]);
    if (nmask) {
      bool stale = false;
      for (int q = 0; q < TT; ++q) stale |= !sh.seq_ok[q];
      if (stale) {
        const long long c0 = clock64();
        compute_all_seqs(sh, R, A, list,
                         EView{sh.e_loss, sh.e_s2, sh.e_key, sh.e_T2, sh.e_i, sh.e_G2, sh.e_t2});
        c_seq += clock64() - c0;
        ++n_seq;
      }
      if (wid < fa && need) {  // ScaleResource(q): first success in kappa order
        const int nopt = W.nopt[wq], ngj = W.ng[wq];
        const OptRec *o = W.opt + (size_t)wq * R.maxopt;
        const double *so = W.score + (size_t)wq * R.maxopt;
        int best = -1, bm = 0;
        OptRec bo{kInf, 0, 0};
        for (int i = lane; i < nopt; i += 32) {
          const OptRec x = o[i];
          if (x.G > ngj) continue;
          const int len = sh.len[x.t];
          int m = -1;
          for (int mm = 0; mm <= len; ++mm)
            if (x.G <= sh.frs[x.t][mm][x.t] - sh.fr_base[x.t][x.t] + sh.fr[x.t]) {
              m = mm;
              break;
            }
          if (m < 0 || !(so[i] > sh.cum[x.t][m])) continue;
          if (best < 0 || kappa_less(x, bo)) {
            best = i;
            bo = x;
            bm = m;
          }
        }
        const int src = warp_lex_argmin(best >= 0, (uint64_t)bo.T, kappa_tie(bo));
        best = src < 0 ? -1 : __shfl_sync(0xffffffffu, best, src);
        bm = src < 0 ? 0 : __shfl_sync(0xffffffffu, bm, src);
        if (lane == 0 && best >= 0) {
          sh.res_kind[wid] = 2;
          sh.res_opt[wid] = best;
          sh.res_m[wid] = bm;
        }
      }
      __syncthreads();
    }
    if (tid == 0) {
      const long long t1 = clock64();
      sh.prof[10] += t1 - tb;
      tb = t1;
    }
    if (tid < 32) {
      const unsigned fmask = __ballot_sync(0xffffffffu, lane < kRoundWarps && sh.res_kind[lane] != 0);
      const int f = fmask ? __ffs(fmask) - 1 : kRoundWarps;
      if (tid == 0) {
        int adv = kRoundWarps;
        if (f < kRoundWarps) {
          const int pos = pos0 + f, oi = sh.res_opt[f];
          const OptRec x = W.opt[(size_t)(pos - W.w0) * R.maxopt + oi];
          int32_t *old_fr = sh.old_fr;
          for (int qq = 0; qq < TT; ++qq) old_fr[qq] = sh.fr[qq];
          unsigned changed = 1u << 31;  // bit 31: a commit happened
          if (sh.res_kind[f] == 2) {
            ++n_scale;
            const int m = sh.res_m[f], t = x.t;
            CRIUS_CHECK(m >= 0 && m <= sh.len[t] && sh.seq_ok[t]);
            for (int mm = 0; mm < m; ++mm) {
              const int a = sh.mv_a[t][mm];
              changed |= (1u << A.t[a]) | (1u << sh.mv_t[t][mm]);
              adm_set(A, R, a, A.pos[a], sh.mv_opt[t][mm], sh.mv_G[t][mm], sh.mv_t[t][mm],
                      sh.mv_T[t][mm], sh.mv_sc[t][mm]);
            }
            for (int qq = 0; qq < TT; ++qq)
              sh.fr[qq] = sh.frs[t][m][qq] - sh.fr_base[t][qq] + old_fr[qq];
          }
          const int kind0 = sh.res_kind[f];
          int w = f;
          for (;;) {  // commit job w (admitted directly, or the first job's scale result)
            const int wq0 = pos0 + w - W.w0, o = sh.res_opt[w];
            CRIUS_CHECK(wq0 >= 0 && wq0 < W.wn && o >= 0 && o < W.nopt[wq0]);
            const OptRec y = W.opt[(size_t)wq0 * R.maxopt + o];
            sh.fr[y.t] -= y.G;
            changed |= 1u << y.t;
            const int na = sh.n_adm;
        CRIUS_CHECK(na < R.J);
            adm_set(A, R, na, pos0 + w, o, y.G, y.t, y.T, W.score[(size_t)wq0 * R.maxopt + o]);
            A.nopt[na] = W.nopt[wq0];
            sh.n_adm += 1;
            adv = w + 1;
            if (kind0 != 1) break;
            // A direct admission only lowers one free count, so a later job's
            // direct choice stands iff its option still fits; a job that stays
            // pending/unschedulable without ScaleResource is unaffected.
            bool more = false;
            while (++w < kRoundWarps && pos0 + w < R.J) {
              const int kw = sh.res_kind[w];
              if (kw == 1) {
                const OptRec z = W.opt[(size_t)(pos0 + w - W.w0) * R.maxopt + sh.res_opt[w]];
                more = z.G <= sh.fr[z.t];
                break;
              }
              if (kw == 0 && !sh.need[w]) {
                adv = w + 1;
                continue;
              }
              break;
            }
            if (!more) break;
          }
          sh.changed = changed;
        }
        sh.advance = adv;
      }
      __syncwarp();
      if (sh.changed) invalidate_seqs(sh, TT);
      __syncwarp();
      if (tid == 0) sh.changed = 0;
    }
    __syncthreads();
    pos0 += sh.advance;
    if (tid == 0) {
      const long long t1 = clock64();
      sh.prof[11] += t1 - tb;
      tb = t1;
    }
  }

  // ---- Phase B: up to d sweeps of reverse scaling over admitted jobs, in
  // priority order (running jobs were admitted first: sort by position)
  const long long c_phaseB = clock64();
  const int n_adm = sh.n_adm;
  int32_t *ord = list;
  for (int a = tid; a < n_adm; a += kRoundThreads) {
    const int pa = A.pos[a];
    int r = 0;
    for (int b = 0; b < n_adm; ++b) r += A.pos[b] < pa;
    ord[r] = a;
  }
  __syncthreads();
  for (int sweep = 0; sweep < R.depth; ++sweep) {
    if (tid == 0) sh.any_change = 0;
    __syncthreads();
    for (int a0 = 0; a0 < n_adm;) {
      const int a = a0 + wid < n_adm ? ord[a0 + wid] : n_adm;
      int opt = -1;
      if (a < n_adm) {
        const int pos = A.pos[a], cv = A.cur[a], Gc = A.G[a], tc = A.t[a];
        const int64_t Tc = A.T[a];
        opt = warp_best_option(R.opt + (int64_t)pos * R.maxopt, A.nopt[a],
                               [&](int i, const OptRec &x) {
                                 const int avail = sh.fr[x.t] + (x.t == tc ? Gc : 0);
                                 return i != cv && x.G <= avail && x.T < Tc &&
                                        (!(R.policy & 2) || x.t == tc);  // NH keeps the type
                               });
      }
      if (lane == 0) {
        sh.res_opt[wid] = opt;
        if (opt >= 0) {
          const int pos = A.pos[a];
          const OptRec x = R.opt[(int64_t)pos * R.maxopt + opt];
          sh.res_G[wid] = x.G;
          sh.res_t[wid] = x.t;
          sh.res_T[wid] = x.T;
          sh.res_sc[wid] = R.score[(int64_t)pos * R.maxopt + opt];
        }
      }
      __syncthreads();
      if (tid < 32) {
        const unsigned fmask = __ballot_sync(0xffffffffu, lane < kRoundWarps && sh.res_opt[lane] >= 0);
        const int f = fmask ? __ffs(fmask) - 1 : kRoundWarps;
        if (tid == 0 && f < kRoundWarps) {
          const int aa = ord[a0 + f];
          sh.fr[A.t[aa]] += A.G[aa];
          adm_set(A, R, aa, A.pos[aa], sh.res_opt[f], sh.res_G[f], sh.res_t[f], sh.res_T[f],
                  sh.res_sc[f]);
          sh.fr[A.t[aa]] -= A.G[aa];
          sh.any_change = 1;
        }
        if (tid == 0) sh.advance = f < kRoundWarps ? f + 1 : kRoundWarps;
      }
      __syncthreads();
      a0 += sh.advance;
      ++n_bb;
    }
    if (!sh.any_change) break;
  }
  const long long c_end = clock64();

  // ---- total score in priority order (fp64, sequential: bit-reproducible)
  if (tid == 0) {
    double tot = 0.0;
    for (int k = 0; k < n_adm; ++k) tot = __dadd_rn(tot, A.sc[ord[k]]);
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
      for (int q = 0; q < 6; ++q) R.stats[8 + q] = sh.prof[q];
      R.stats[14] = sh.n_invalid;
      for (int q = 8; q < 12; ++q) R.stats[7 + q] = sh.prof[q];
    }
  }
  __syncthreads();
  if (tid < TT) R.free_io[tid] = sh.fr[tid];
  for (int pos = tid; pos < R.J; pos += kRoundThreads) {
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
