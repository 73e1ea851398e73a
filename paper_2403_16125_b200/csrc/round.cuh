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
  int64_t *stats;        // [8] counters (see crius_round_stats)
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
}

__device__ __forceinline__ bool kappa_less(const OptRec &a, const OptRec &b) {
  if (a.T != b.T) return a.T < b.T;
  if (a.G != b.G) return a.G < b.G;
  return a.t < b.t;
}

constexpr int kRoundThreads = 1024;
constexpr int kRoundWarps = kRoundThreads / 32;
constexpr int kAdmSmem = 2048;  // admitted-job records kept in shared memory up to this many
constexpr int kAdmBytes = 60;   // bytes per admitted-job record

// Admitted jobs, in priority order (SoA; shared memory when they fit, else global).
// bi_* caches the job's best same-type victim move (case (i)), which depends
// only on its current option; bi_valid = 0 after every change of that option.
struct AdmView {
  int64_t *T;
  double *sc, *bi_key;
  int32_t *pos, *cur, *G, *t, *nopt, *bi_opt, *bi_freed, *bi_valid, *gmin;
};

// Window of upcoming jobs (priority positions [w0, w0 + wn)) staged in shared memory.
struct JobWin {
  int64_t *ref;
  int32_t *nopt, *ng;
  OptRec *opt;
  double *score;
  int cap, w0, wn;
};

struct RoundShared {
  int32_t fr[kMaxTypes];
  int32_t n_adm, seq_valid, advance, any_change, win0;
  // victim-move sequences, one per GPU type, cut at <= d moves
  int32_t len[kMaxTypes], active[kMaxTypes];
  int32_t mv_a[kMaxTypes][kMaxDepth], mv_opt[kMaxTypes][kMaxDepth];
  int32_t mv_G[kMaxTypes][kMaxDepth], mv_t[kMaxTypes][kMaxDepth];   // the victim's new option
  int64_t mv_T[kMaxTypes][kMaxDepth];
  double mv_sc[kMaxTypes][kMaxDepth];
  int32_t fmax_other[kMaxTypes];  // max_{t2 != t} free'[t2] of the current move
  double cum[kMaxTypes][kMaxDepth + 1];                 // ((0 + loss_1) + loss_2) + ...
  int32_t frs[kMaxTypes][kMaxDepth + 1][kMaxTypes];      // free' after m moves
  // per-warp outcome of one speculative batch
  int32_t res_kind[kRoundWarps], res_opt[kRoundWarps], res_m[kRoundWarps], need[kRoundWarps];
  int32_t res_G[kRoundWarps], res_t[kRoundWarps];
  int64_t res_T[kRoundWarps];
  double res_sc[kRoundWarps];
  // per-(type, warp) argmin scratch
  double r_key[kMaxTypes][kRoundWarps];
  int32_t r_a[kMaxTypes][kRoundWarps], r_i[kMaxTypes][kRoundWarps];
  int32_t r_freed[kMaxTypes][kRoundWarps], r_other[kMaxTypes][kRoundWarps];
};

struct Cand {
  int have;
  double key;
  int a, i, freed, other;
};

// (key, admitted index = priority order, option index = (t, G) order) ascending
__device__ __forceinline__ bool cand_less(const Cand &x, const Cand &y) {
  if (!x.have) return false;
  if (!y.have) return true;
  if (x.key != y.key) return x.key < y.key;
  if (x.a != y.a) return x.a < y.a;
  return x.i < y.i;
}

__device__ __forceinline__ Cand warp_min_cand(Cand c) {
  for (int d = 16; d > 0; d >>= 1) {
    Cand o;
    o.have = __shfl_xor_sync(0xffffffffu, c.have, d);
    o.key = __shfl_xor_sync(0xffffffffu, c.key, d);
    o.a = __shfl_xor_sync(0xffffffffu, c.a, d);
    o.i = __shfl_xor_sync(0xffffffffu, c.i, d);
    o.freed = __shfl_xor_sync(0xffffffffu, c.freed, d);
    o.other = __shfl_xor_sync(0xffffffffu, c.other, d);
    if (cand_less(o, c)) c = o;
  }
  return c;
}

// Best victim move of admitted job a for the sequence of its own type t under
// free' = f2 (§N6 ScaleResource candidates; key = loss / freed, loss =
// score(cur) - score(o')).  Exact shortcuts:
//  (i)  same type, smaller G: independent of free' -> cached per current option;
//  (ii) other type with G_o' <= free'[t_o']: impossible when the job's smallest
//       option G exceeds every other type's free' (fmax); otherwise freed =
//       G_cur, a power of two, so key = loss * 2^-log2(G_cur) exactly (no
//       rounding): min key <=> min rounded loss (ties -> lowest option index),
//       one division for the winner.
// Option records are fetched 4 at a time with all loads in flight.
__device__ __forceinline__ Cand eval_victim(const RoundBuf &R, const AdmView &A, int a, int t,
                                            const int32_t *f2, int fmax) {
  const int v = A.pos[a], cv = A.cur[a], Gc = A.G[a], nv = A.nopt[a];
  const double sc = A.sc[a];
  const longlong2 *ov = reinterpret_cast<const longlong2 *>(R.opt + (int64_t)v * R.maxopt);
  const double *so = R.score + (int64_t)v * R.maxopt;
  Cand best{0, 0.0, a, 0, 0, 0};
  if (!A.bi_valid[a]) {
    int bi = -1, bf = 0, gmin = INT32_MAX;
    double bk = 0.0;
    for (int i0 = 0; i0 < nv; i0 += 4) {
      longlong2 buf[4];
      double sb[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (i0 + u < nv) {
          buf[u] = ov[i0 + u];
          sb[u] = so[i0 + u];
        }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i2 = i0 + u;
        if (i2 >= nv) continue;
        const int G2 = (int)(buf[u].y & 0xffffffff), t2 = (int)(buf[u].y >> 32);
        gmin = min(gmin, G2);
        if (i2 == cv || t2 != t || G2 >= Gc) continue;
        const double key = __ddiv_rn(sc - sb[u], (double)(Gc - G2));
        if (bi < 0 || key < bk) {
          bi = i2;
          bk = key;
          bf = Gc - G2;
        }
      }
    }
    A.bi_opt[a] = bi;
    A.bi_key[a] = bk;
    A.bi_freed[a] = bf;
    A.gmin[a] = gmin;
    A.bi_valid[a] = 1;
  }
  if (A.bi_opt[a] >= 0) {
    best.have = 1;
    best.key = A.bi_key[a];
    best.i = A.bi_opt[a];
    best.freed = A.bi_freed[a];
    best.other = 0;
  }
  if (A.gmin[a] > fmax) return best;
  int ii = -1;
  double lmin = 0.0;
  for (int i0 = 0; i0 < nv; i0 += 4) {
    longlong2 buf[4];
    double sb[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (i0 + u < nv) {
        buf[u] = ov[i0 + u];
        sb[u] = so[i0 + u];
      }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i2 = i0 + u;
      if (i2 >= nv) continue;
      const int G2 = (int)(buf[u].y & 0xffffffff), t2 = (int)(buf[u].y >> 32);
      if (t2 == t || G2 > f2[t2]) continue;
      const double loss = sc - sb[u];
      if (ii < 0 || loss < lmin) {
        ii = i2;
        lmin = loss;
      }
    }
  }
  if (ii >= 0) {
    Cand c{1, __ddiv_rn(lmin, (double)Gc), a, ii, Gc, 1};
    if (cand_less(c, best)) best = c;
  }
  return best;
}

// All threads: the greedy victim sequence of every GPU type t from the current
// state (the §N6 ScaleResource move loop run for d moves without the G_o stop;
// an option on type t uses the shortest prefix that frees G_o).  Each admitted
// job is a candidate only for the sequence of its own current type, so one
// pass over the admitted jobs serves every type's next move.
__device__ void compute_all_seqs(RoundShared &sh, const RoundBuf &R, const AdmView &A) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int TT = R.T, n_adm = sh.n_adm;
  if (tid < TT) {
    sh.len[tid] = 0;
    sh.active[tid] = 1;
    sh.cum[tid][0] = 0.0;
  }
  if (tid < TT * TT) sh.frs[tid / TT][0][tid % TT] = sh.fr[tid % TT];
  __syncthreads();
  for (int m = 0; m < R.depth; ++m) {
    if (tid < TT) {
      int fm = -1;
      for (int q = 0; q < TT; ++q)
        if (q != tid) fm = max(fm, sh.frs[tid][m][q]);
      sh.fmax_other[tid] = fm;
    }
    __syncthreads();
    Cand run{0, 0.0, 0, 0, 0, 0};  // lane t < TT: this warp's best for type t
    for (int a0 = 0; a0 < n_adm; a0 += kRoundThreads) {
      const int a = a0 + tid;
      Cand mine{0, 0.0, 0, 0, 0, 0};
      int myt = -1;
      if (a < n_adm) {
        myt = A.t[a];
        bool moved = !sh.active[myt];
        for (int q = 0; q < m; ++q) moved |= sh.mv_a[myt][q] == a;
        if (!moved) mine = eval_victim(R, A, a, myt, sh.frs[myt][m], sh.fmax_other[myt]);
      }
      for (int t = 0; t < TT; ++t) {
        if (!__ballot_sync(0xffffffffu, myt == t && mine.have)) continue;
        Cand c = mine;
        if (myt != t) c.have = 0;
        c = warp_min_cand(c);
        if (lane == t && cand_less(c, run)) run = c;
      }
    }
    if (lane < TT) {
      sh.r_key[lane][wid] = run.key;
      sh.r_a[lane][wid] = run.have ? run.a : -1;
      sh.r_i[lane][wid] = run.i;
      sh.r_freed[lane][wid] = run.freed;
      sh.r_other[lane][wid] = run.other;
    }
    __syncthreads();
    if (wid < TT && sh.active[wid]) {  // warp t reduces type t and applies its move
      const int t = wid;
      Cand c;
      c.have = sh.r_a[t][lane] >= 0;
      c.key = sh.r_key[t][lane];
      c.a = sh.r_a[t][lane];
      c.i = sh.r_i[t][lane];
      c.freed = sh.r_freed[t][lane];
      c.other = sh.r_other[t][lane];
      c = warp_min_cand(c);
      if (lane == 0) {
        if (!c.have) {
          sh.active[t] = 0;
        } else {
          const int v = A.pos[c.a];
          const OptRec o2 = R.opt[(int64_t)v * R.maxopt + c.i];
          const double loss = A.sc[c.a] - R.score[(int64_t)v * R.maxopt + c.i];
          sh.mv_a[t][m] = c.a;
          sh.mv_opt[t][m] = c.i;
          sh.mv_G[t][m] = o2.G;
          sh.mv_t[t][m] = o2.t;
          sh.mv_T[t][m] = o2.T;
          sh.mv_sc[t][m] = R.score[(int64_t)v * R.maxopt + c.i];
          sh.cum[t][m + 1] = __dadd_rn(sh.cum[t][m], loss);
          for (int q = 0; q < TT; ++q) sh.frs[t][m + 1][q] = sh.frs[t][m][q];
          sh.frs[t][m + 1][t] += c.freed;
          if (c.other) sh.frs[t][m + 1][o2.t] -= o2.G;
          sh.len[t] = m + 1;
        }
      }
    }
    __syncthreads();
  }
  if (tid == 0) sh.seq_valid = 1;
  __syncthreads();
}

// Warp-wide argmin of kappa over `nopt` option records passing `pred`.
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
  for (int d = 16; d > 0; d >>= 1) {
    const int ob = __shfl_xor_sync(0xffffffffu, best, d);
    const int64_t oT = __shfl_xor_sync(0xffffffffu, bo.T, d);
    const int oG = __shfl_xor_sync(0xffffffffu, bo.G, d);
    const int ot = __shfl_xor_sync(0xffffffffu, bo.t, d);
    const OptRec ox{oT, oG, ot};
    if (ob >= 0 && (best < 0 || kappa_less(ox, bo))) {
      best = ob;
      bo = ox;
    }
  }
  return best;
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
  A.bi_valid[a] = 0;
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
  AdmView A = Aglob;
  if (adm_in_smem) {
    A.T = (int64_t *)p;
    A.sc = (double *)(A.T + kAdmSmem);
    A.bi_key = A.sc + kAdmSmem;
    A.pos = (int32_t *)(A.bi_key + kAdmSmem);
    A.cur = A.pos + kAdmSmem;
    A.G = A.cur + kAdmSmem;
    A.t = A.G + kAdmSmem;
    A.nopt = A.t + kAdmSmem;
    A.bi_opt = A.nopt + kAdmSmem;
    A.bi_freed = A.bi_opt + kAdmSmem;
    A.bi_valid = A.bi_freed + kAdmSmem;
    A.gmin = A.bi_valid + kAdmSmem;
  }
  if (tid < TT) sh.fr[tid] = R.free_io[tid];
  if (tid == 0) {
    sh.n_adm = 0;
    sh.seq_valid = 0;
  }
  __syncthreads();
  long long c_start = clock64(), c_seq = 0, n_batches = 0, n_seq = 0, n_scale = 0, n_bb = 0;
  load_window(W, R, 0);

  // ---- Phase A: SchedArrival in priority order
  for (int pos0 = 0; pos0 < R.J;) {
    if (pos0 + kRoundWarps > W.w0 + W.wn && W.w0 + W.wn < R.J) load_window(W, R, pos0);
    const int q = pos0 + wid, wq = q - W.w0;
    int kind = 0, opt = -1, need = 0;
    if (q < R.J && W.ref[wq] != kInf) {
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
    const unsigned kmask = __ballot_sync(0xffffffffu, sh.res_kind[lane] != 0);
    const int fa = kmask ? __ffs(kmask) - 1 : kRoundWarps;
    const unsigned nmask = __ballot_sync(0xffffffffu, lane < fa && sh.need[lane]);
    if (nmask) {
      if (!sh.seq_valid) {
        const long long c0 = clock64();
        compute_all_seqs(sh, R, A);
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
            if (x.G <= sh.frs[x.t][mm][x.t]) {
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
        for (int d = 16; d > 0; d >>= 1) {
          const int ob = __shfl_xor_sync(0xffffffffu, best, d);
          const int om = __shfl_xor_sync(0xffffffffu, bm, d);
          const int64_t oT = __shfl_xor_sync(0xffffffffu, bo.T, d);
          const int oG = __shfl_xor_sync(0xffffffffu, bo.G, d);
          const int ot = __shfl_xor_sync(0xffffffffu, bo.t, d);
          const OptRec ox{oT, oG, ot};
          if (ob >= 0 && (best < 0 || kappa_less(ox, bo))) {
            best = ob;
            bo = ox;
            bm = om;
          }
        }
        if (lane == 0 && best >= 0) {
          sh.res_kind[wid] = 2;
          sh.res_opt[wid] = best;
          sh.res_m[wid] = bm;
        }
      }
      __syncthreads();
    }
    if (tid < 32) {
      const unsigned fmask = __ballot_sync(0xffffffffu, sh.res_kind[lane] != 0);
      const int f = fmask ? __ffs(fmask) - 1 : kRoundWarps;
      if (tid == 0 && f < kRoundWarps) {
        const int pos = pos0 + f, oi = sh.res_opt[f];
        const OptRec x = W.opt[(size_t)(pos - W.w0) * R.maxopt + oi];
        if (sh.res_kind[f] == 2) {
          ++n_scale;
          const int m = sh.res_m[f], t = x.t;
          for (int mm = 0; mm < m; ++mm) {
            const int a = sh.mv_a[t][mm];
            adm_set(A, R, a, A.pos[a], sh.mv_opt[t][mm], sh.mv_G[t][mm], sh.mv_t[t][mm],
                    sh.mv_T[t][mm], sh.mv_sc[t][mm]);
          }
          for (int qq = 0; qq < TT; ++qq) sh.fr[qq] = sh.frs[t][m][qq];
        }
        sh.fr[x.t] -= x.G;
        const int wq0 = pos - W.w0;
        const int na = sh.n_adm;
        adm_set(A, R, na, pos, oi, x.G, x.t, x.T, W.score[(size_t)wq0 * R.maxopt + oi]);
        A.nopt[na] = W.nopt[wq0];
        sh.n_adm += 1;
        sh.seq_valid = 0;
      }
      if (tid == 0) sh.advance = f < kRoundWarps ? f + 1 : kRoundWarps;
    }
    __syncthreads();
    pos0 += sh.advance;
  }

  // ---- Phase B: up to d sweeps of reverse scaling over admitted jobs
  const long long c_phaseB = clock64();
  const int n_adm = sh.n_adm;
  for (int sweep = 0; sweep < R.depth; ++sweep) {
    if (tid == 0) sh.any_change = 0;
    __syncthreads();
    for (int a0 = 0; a0 < n_adm;) {
      const int a = a0 + wid;
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
        const unsigned fmask = __ballot_sync(0xffffffffu, sh.res_opt[lane] >= 0);
        const int f = fmask ? __ffs(fmask) - 1 : kRoundWarps;
        if (tid == 0 && f < kRoundWarps) {
          const int aa = a0 + f;
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
    for (int a = 0; a < n_adm; ++a) tot = __dadd_rn(tot, A.sc[a]);
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
    }
  }
  __syncthreads();
  if (tid < TT) R.free_io[tid] = sh.fr[tid];
  for (int pos = tid; pos < R.J; pos += kRoundThreads) {
    const int j = R.pi[pos];
    const int c = R.cur[pos];
    R.decision[j] = R.ref[pos] == kInf ? -2 : (c < 0 ? -1 : R.opt_cell[(int64_t)pos * R.maxopt + c]);
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
