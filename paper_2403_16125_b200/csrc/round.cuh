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
//    sequence of every type is computed once per state, in parallel over all
//    admitted jobs, and reused until an admission changes the state.
#pragma once
#include "common.cuh"

namespace crius {

struct OptRec {  // 16 B
  int64_t T;
  int32_t G;
  int32_t t;
};

struct RoundBuf {
  int32_t J, T, maxopt, depth;
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
  for (int64_t c = c0; c < c1; ++c) {
    const int64_t T = res[c].t_ns;
    const int t = cType[c], G = cG[c];
    if (T == kInf) continue;
    ref_any = min(ref_any, T);
    if (G == ngj) ref_ng = min(ref_ng, T);
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
constexpr int kAdmSmem = 2048;  // admitted-job records kept in shared memory up to this many
constexpr int kAdmBytes = 76;   // bytes per admitted-job record (incl. scratch list)

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
  long long prof[12];  // cycles: [0] setup+dirty, [1] (i) pass, [2] (ii) pass, [3] reduce+apply; [4] dirty jobs, [5] listed jobs
  // victim-move sequences, one per GPU type, cut at <= d moves
  int32_t len[kRT], active[kRT];
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
  // per-(type, warp) best move of the current step, with the move's option data
  double r_key[kRT][kRoundWarps], r_s2[kRT][kRoundWarps];
  int64_t r_T2[kRT][kRoundWarps];
  int32_t r_a[kRT][kRoundWarps], r_i[kRT][kRoundWarps], r_p[kRT][kRoundWarps];
  int32_t r_freed[kRT][kRoundWarps], r_other[kRT][kRoundWarps];
  int32_t r_G2[kRT][kRoundWarps], r_t2[kRT][kRoundWarps];
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

// A victim move: key = loss / freed, ordered by (key, admitted index a, option i).
struct Cand {
  int have;
  double key;
  int a, i, freed, other, G2, t2;
  int64_t T2;
  double s2;
  int p;  // the victim's priority position: ties go to the earlier job (§N6)
};

__device__ __forceinline__ bool cand_less(const Cand &x, const Cand &y) {
  if (!x.have) return false;
  if (!y.have) return true;
  if (x.key != y.key) return x.key < y.key;
  if (x.p != y.p) return x.p < y.p;
  return x.i < y.i;
}

// Warp-wide argmin of Cands (one per lane) -> winning lane or -1.
__device__ __forceinline__ int warp_cand_argmin(const Cand &c) {
  return warp_lex_argmin(c.have, ord_double(c.key), ((uint32_t)c.p << 8) | (uint32_t)c.i);
}

// Per-(type, warp) best-move slot: written only by the winning lane of its warp.
__device__ __forceinline__ bool slot_take(RoundShared &sh, int t, int w, const Cand &c) {
  const int sa = sh.r_a[t][w], sp = sh.r_p[t][w];
  if (!c.have) return false;
  if (sa >= 0) {
    const double sk = sh.r_key[t][w];
    if (!(c.key < sk || (c.key == sk && (c.p < sp || (c.p == sp && c.i < sh.r_i[t][w])))))
      return false;
  }
  sh.r_key[t][w] = c.key;
  sh.r_a[t][w] = c.a;
  sh.r_p[t][w] = c.p;
  sh.r_i[t][w] = c.i;
  sh.r_freed[t][w] = c.freed;
  sh.r_other[t][w] = c.other;
  sh.r_G2[t][w] = c.G2;
  sh.r_t2[t][w] = c.t2;
  sh.r_T2[t][w] = c.T2;
  sh.r_s2[t][w] = c.s2;
  return true;
}

// Warp: refresh the same-type move cache (case (i)) and gmin of admitted job a.
// Lanes cover the job's options (coalesced 16-byte records, one round trip).
__device__ __forceinline__ void refresh_victim_cache(const RoundBuf &R, const AdmView &A, int a) {
  const int lane = threadIdx.x & 31;
  const int v = A.pos[a], cv = A.cur[a], Gc = A.G[a], t = A.t[a], nv = A.nopt[a];
  const double sc = A.sc[a];
  Cand best{0, 0.0, a, 0, 0, 0, 0, 0, 0, 0.0, v};
  int gmin = INT32_MAX;
  for (int i2 = lane; i2 < nv; i2 += 32) {
    const OptRec o2 = ldg_opt(R.opt + (int64_t)v * R.maxopt + i2);
    gmin = min(gmin, o2.G);
    if (i2 == cv || o2.t != t || o2.G >= Gc) continue;
    const double s2 = __ldg(R.score + (int64_t)v * R.maxopt + i2);
    Cand c{1, __ddiv_rn(sc - s2, (double)(Gc - o2.G)), a, i2, Gc - o2.G, 0, o2.G, o2.t, o2.T, s2, v};
    if (cand_less(c, best)) best = c;
  }
  gmin = (int)__reduce_min_sync(0xffffffffu, (unsigned)gmin);
  const int src = warp_cand_argmin(best);
  if (src < 0) {
    if (lane == 0) A.bi_opt[a] = -1;
  } else if (lane == src) {
    A.bi_opt[a] = best.i;
    A.bi_key[a] = best.key;
    A.bi_G2[a] = best.G2;
    A.bi_T[a] = best.T2;
    A.bi_s[a] = best.s2;
  }
  if (lane == 0) A.gmin[a] = gmin;
}

// Warp: best other-type move (case (ii)) of admitted job a under free' = f2;
// the winning lane offers it to the (type, warp) slot.  freed = G_cur is a
// power of two, so key = loss * 2^-log2(G_cur) exactly: the minimum key is the
// minimum rounded loss (ties -> lowest option index), one division.
__device__ __forceinline__ void other_type_move(RoundShared &sh, const RoundBuf &R,
                                                const AdmView &A, int a, const int32_t *f2) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int v = A.pos[a], Gc = A.G[a], t = A.t[a], nv = A.nopt[a];
  const double sc = A.sc[a];
  Cand best{0, 0.0, a, 0, 0, 0, 0, 0, 0, 0.0, v};
  for (int i2 = lane; i2 < nv; i2 += 32) {
    const OptRec o2 = ldg_opt(R.opt + (int64_t)v * R.maxopt + i2);
    if (o2.t == t || o2.G > f2[o2.t]) continue;
    const double s2 = __ldg(R.score + (int64_t)v * R.maxopt + i2);
    Cand c{1, sc - s2, a, i2, Gc, 1, o2.G, o2.t, o2.T, s2, v};  // key holds the loss here
    if (cand_less(c, best)) best = c;
  }
  const int src = warp_cand_argmin(best);
  if (lane == src) {
    best.key = __ddiv_rn(best.key, (double)Gc);
    slot_take(sh, t, wid, best);
  }
  __syncwarp();
}

// All threads: the greedy victim sequence of every GPU type t from the current
// state (the §N6 ScaleResource move loop run for d moves without the G_o stop;
// an option on type t uses the shortest prefix that frees G_o).  Each admitted
// job is a candidate only for the sequence of its own current type.  Per move,
// in one pass: cached same-type moves of every job (shared memory only), and
// other-type moves of the few jobs whose smallest option could fit free'[t2].
__device__ void compute_all_seqs(RoundShared &sh, const RoundBuf &R, const AdmView &A,
                                 int32_t *list) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int TT = R.T, n_adm = sh.n_adm;
  if (tid < TT) {
    const int c = !sh.seq_ok[tid];
    sh.comp[tid] = c;
    sh.active[tid] = c;
    if (c) {
      sh.len[tid] = 0;
      sh.cum[tid][0] = 0.0;
      sh.gmin_type[tid] = INT32_MAX;
      int fm = -1;
      for (int q = 0; q < TT; ++q)
        if (q != tid) fm = max(fm, sh.fr[q]);
      sh.fmax_other[tid] = fm;
    }
  }
  if (tid < TT * TT && !sh.seq_ok[tid / TT]) {
    sh.frs[tid / TT][0][tid % TT] = sh.fr[tid % TT];
    sh.fr_base[tid / TT][tid % TT] = sh.fr[tid % TT];
  }
  if (lane < TT) sh.r_a[lane][wid] = -1;
  if (tid == 0) sh.n_dirty = 0;
  long long t0 = clock64();
  __syncthreads();
  // stale same-type caches -> list -> one warp per job
  for (int a = tid; a < n_adm; a += kRoundThreads)
    if (A.bi_opt[a] == -2) list[atomicAdd(&sh.n_dirty, 1)] = a;
  CRIUS_CHECK(n_adm <= R.J);
  __syncthreads();
  for (int k = wid; k < sh.n_dirty; k += kRoundWarps) refresh_victim_cache(R, A, list[k]);
  __syncthreads();
  if (tid == 0) {
    const long long t1 = clock64();
    sh.prof[0] += t1 - t0;
    sh.prof[4] += sh.n_dirty;
    t0 = t1;
  }

  for (int m = 0; m < R.depth; ++m) {
    if (tid == 0) sh.n_list = 0;
    __syncthreads();
    for (int a0 = 0; a0 < n_adm; a0 += kRoundThreads) {
      const int a = a0 + tid;
      Cand mine{0, 0.0, 0, 0, 0, 0, 0, 0, 0, 0.0, 0};
      int myt = -1;
      if (a < n_adm) {
        myt = A.t[a];
        if (m == 0 && sh.comp[myt]) atomicMin(&sh.gmin_type[myt], A.gmin[a]);
        bool moved = !sh.active[myt];
        for (int q = 0; q < m; ++q) moved |= sh.mv_a[myt][q] == a;
        if (!moved) {
          const int bo = A.bi_opt[a];
          if (bo >= 0)
            mine = Cand{1, A.bi_key[a], a, bo, A.G[a] - A.bi_G2[a], 0, A.bi_G2[a], myt, A.bi_T[a],
                        A.bi_s[a], A.pos[a]};
          if (A.gmin[a] <= sh.fmax_other[myt]) list[atomicAdd(&sh.n_list, 1)] = a;
        }
      }
      // (i) cached same-type moves: per type, the warp's winner offers itself
      for (int t = 0; t < TT; ++t) {
        const bool v = myt == t && mine.have;
        const int src = warp_lex_argmin(v, ord_double(mine.key), ((uint32_t)mine.p << 8) | (uint32_t)mine.i);
        if (lane == src) slot_take(sh, t, wid, mine);
        __syncwarp();
      }
    }
    __syncthreads();
    // (ii) other-type moves of the listed jobs, one warp per job (balanced)
    for (int k = wid; k < sh.n_list; k += kRoundWarps) {
      const int aa = list[k];
      other_type_move(sh, R, A, aa, sh.frs[A.t[aa]][m]);
    }
    if (tid == 0) sh.prof[5] += sh.n_list;
    __syncthreads();
    if (tid == 0) {
      const long long t1 = clock64();
      sh.prof[1] += t1 - t0;
      t0 = t1;
    }
    if (wid < TT && sh.active[wid]) {  // warp t reduces type t, applies its move, preps m+1
      const int t = wid;
      const bool in = lane < kRoundWarps;
      const int ra = in ? sh.r_a[t][lane] : -1;
      const int rp = in ? sh.r_p[t][lane] : 0;
      const int src = warp_lex_argmin(ra >= 0, ord_double(in ? sh.r_key[t][lane] : 0.0),
                                      ((uint32_t)rp << 8) | (uint32_t)(in ? sh.r_i[t][lane] : 0));
      if (src < 0) {
        if (lane == 0) sh.active[t] = 0;
      } else {
        if (lane == 0) {
          const int ca = sh.r_a[t][src];
          sh.mv_a[t][m] = ca;
          sh.mv_opt[t][m] = sh.r_i[t][src];
          sh.mv_G[t][m] = sh.r_G2[t][src];
          sh.mv_t[t][m] = sh.r_t2[t][src];
          sh.mv_T[t][m] = sh.r_T2[t][src];
          sh.mv_sc[t][m] = sh.r_s2[t][src];
          const double loss = A.sc[ca] - sh.r_s2[t][src];
          sh.cum[t][m + 1] = __dadd_rn(sh.cum[t][m], loss);
          int fm = -1;
          for (int q = 0; q < TT; ++q) {
            int f = sh.frs[t][m][q];
            if (q == t) f += sh.r_freed[t][src];
            if (q == sh.r_t2[t][src] && sh.r_other[t][src]) f -= sh.r_G2[t][src];
            sh.frs[t][m + 1][q] = f;
            if (q != t) fm = max(fm, f);
          }
          sh.fmax_other[t] = fm;
          sh.len[t] = m + 1;
        }
        __syncwarp();
        if (lane < kRoundWarps) sh.r_a[t][lane] = -1;  // reset this type's slots for move m + 1
      }
    }
    __syncthreads();
    if (tid == 0) {
      const long long t1 = clock64();
      sh.prof[3] += t1 - t0;
      t0 = t1;
    }
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
        compute_all_seqs(sh, R, A, list);
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
                                 return i != cv && x.G <= avail && x.T < Tc;
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
