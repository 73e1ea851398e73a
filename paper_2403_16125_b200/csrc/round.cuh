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
// K6 is ONE CTA: warp 0 walks the jobs in priority order (the round is
// sequential by definition); the other 31 warps sleep on a named barrier and
// are woken only to compute a victim-move sequence, a parallel argmin over
// (admitted job, option) pairs.
//
// Exact equivalence used by K6 (not an approximation): within one trial the
// victim sequence depends only on the state (free counts, admitted jobs and
// their options) and on the option's GPU type t_o -- not on the pending job or
// on G_o, which only decides where the sequence is cut.  K6 therefore computes
// the greedy sequence once per (state, t) and reuses it for every option and
// every pending job until an admission changes the state.
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
  const int32_t *ng_job; // [J] by job
  OptRec *opt;           // [J][maxopt] by position, (t, G) ascending
  int64_t *opt_cell;     // [J][maxopt]
  int32_t *nopt;         // [J] by position
  int64_t *ref;          // [J] by position (kInf = unschedulable)
  int32_t *ng;           // [J] by position
  int32_t *cur;          // [J] by position: option index or -1
  int32_t *adm;          // [J] admitted positions, in priority order
  int64_t *decision;     // [J] by job
  int32_t *free_io;      // [T]
  double *total;
};

// K5: per job (thread), options and ref from its Cells (contiguous, (t, G, S) order).
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
  R.nopt[pos] = n;
  R.ref[pos] = ref_ng != kInf ? ref_ng : ref_any;
  R.ng[pos] = ngj;
  R.cur[pos] = -1;
}

__device__ __forceinline__ bool kappa_less(const OptRec &a, const OptRec &b) {
  if (a.T != b.T) return a.T < b.T;
  if (a.G != b.G) return a.G < b.G;
  return a.t < b.t;
}

__device__ __forceinline__ double score_of(int64_t ref, int64_t T) {
  return __ddiv_rn((double)ref, (double)T);
}

__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

constexpr int kRoundThreads = 1024;
constexpr int kMaxOptLanes = 2;  // options per lane in warp-level option scans (maxopt <= 64)

struct RoundShared {
  int32_t fr[kMaxTypes];
  int32_t req;           // sequence request: type, or -1 = exit
  int32_t n_adm;
  int32_t seq_valid[kMaxTypes];
  int32_t seq_len[kMaxTypes];
  int32_t mv_pos[kMaxTypes][kMaxDepth];
  int32_t mv_opt[kMaxTypes][kMaxDepth];
  double mv_loss[kMaxTypes][kMaxDepth];
  int32_t frs[kMaxTypes][kMaxDepth + 1][kMaxTypes];  // free' after m moves
  // block argmin scratch
  double r_key[32];
  int32_t r_a[32], r_i[32], r_freed[32], r_other[32];
  int32_t cont;
  int32_t sorted[64];
};

// Parallel (all 1024 threads): greedy victim sequence for type t from the
// current state (SURVEY §N6 ScaleResource loop body, executed for up to d
// moves without the G_o stop condition).
__device__ void compute_seq(RoundShared &sh, const RoundBuf &R, int t) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int TT = R.T;
  if (tid < TT) sh.frs[t][0][tid] = sh.fr[tid];
  named_bar(2, kRoundThreads);
  int len = 0;
  const int n_adm = sh.n_adm;
  for (int m = 0; m < R.depth; ++m) {
    const int32_t *f2 = sh.frs[t][m];
    bool have = false;
    double bkey = 0.0;
    int ba = 0, bi = 0, bfreed = 0, bother = 0;
    for (int a = tid; a < n_adm; a += kRoundThreads) {
      const int v = R.adm[a];
      const int cv = R.cur[v];
      const OptRec *ov = R.opt + (int64_t)v * R.maxopt;
      const OptRec cur = ov[cv];
      if (cur.t != t) continue;
      bool moved = false;
      for (int q = 0; q < m; ++q) moved |= sh.mv_pos[t][q] == v;
      if (moved) continue;
      const int64_t ref = R.ref[v];
      const double sc = score_of(ref, cur.T);
      const int nv = R.nopt[v];
      for (int i2 = 0; i2 < nv; ++i2) {
        if (i2 == cv) continue;
        const OptRec o2 = ov[i2];
        int freed, other;
        if (o2.t == t && o2.G < cur.G) {
          freed = cur.G - o2.G;
          other = 0;
        } else if (o2.t != t && o2.G <= f2[o2.t]) {
          freed = cur.G;
          other = 1;
        } else {
          continue;
        }
        const double loss = sc - score_of(ref, o2.T);
        const double key = __ddiv_rn(loss, (double)freed);
        // order: key, then earlier priority position (a), then (t, G) order (i2)
        if (!have || key < bkey) {
          have = true;
          bkey = key;
          ba = a;
          bi = i2;
          bfreed = freed;
          bother = other;
        }
      }
    }
    // warp argmin
    for (int d = 16; d > 0; d >>= 1) {
      const int oh = __shfl_xor_sync(0xffffffffu, (int)have, d);
      const double ok = __shfl_xor_sync(0xffffffffu, bkey, d);
      const int oa = __shfl_xor_sync(0xffffffffu, ba, d);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, d);
      const int of = __shfl_xor_sync(0xffffffffu, bfreed, d);
      const int oo = __shfl_xor_sync(0xffffffffu, bother, d);
      const bool take = oh && (!have || ok < bkey || (ok == bkey && (oa < ba || (oa == ba && oi < bi))));
      if (take) {
        have = true;
        bkey = ok;
        ba = oa;
        bi = oi;
        bfreed = of;
        bother = oo;
      }
    }
    if (lane == 0) {
      sh.r_key[wid] = bkey;
      sh.r_a[wid] = have ? ba : -1;
      sh.r_i[wid] = bi;
      sh.r_freed[wid] = bfreed;
      sh.r_other[wid] = bother;
    }
    named_bar(2, kRoundThreads);
    if (wid == 0) {
      have = sh.r_a[lane] >= 0;
      bkey = sh.r_key[lane];
      ba = sh.r_a[lane];
      bi = sh.r_i[lane];
      bfreed = sh.r_freed[lane];
      bother = sh.r_other[lane];
      for (int d = 16; d > 0; d >>= 1) {
        const int oh = __shfl_xor_sync(0xffffffffu, (int)have, d);
        const double ok = __shfl_xor_sync(0xffffffffu, bkey, d);
        const int oa = __shfl_xor_sync(0xffffffffu, ba, d);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, d);
        const int of = __shfl_xor_sync(0xffffffffu, bfreed, d);
        const int oo = __shfl_xor_sync(0xffffffffu, bother, d);
        const bool take =
            oh && (!have || ok < bkey || (ok == bkey && (oa < ba || (oa == ba && oi < bi))));
        if (take) {
          have = true;
          bkey = ok;
          ba = oa;
          bi = oi;
          bfreed = of;
          bother = oo;
        }
      }
      if (lane == 0) {
        sh.cont = have ? 1 : 0;
        if (have) {
          const int v = R.adm[ba];
          const OptRec *ov = R.opt + (int64_t)v * R.maxopt;
          const OptRec cur = ov[R.cur[v]], o2 = ov[bi];
          sh.mv_pos[t][m] = v;
          sh.mv_opt[t][m] = bi;
          sh.mv_loss[t][m] = score_of(R.ref[v], cur.T) - score_of(R.ref[v], o2.T);
          for (int q = 0; q < TT; ++q) sh.frs[t][m + 1][q] = sh.frs[t][m][q];
          sh.frs[t][m + 1][t] += bfreed;
          if (bother) sh.frs[t][m + 1][o2.t] -= o2.G;
        }
      }
    }
    named_bar(2, kRoundThreads);
    if (!sh.cont) break;
    ++len;
  }
  if (tid == 0) {
    sh.seq_len[t] = len;
    sh.seq_valid[t] = 1;
  }
  named_bar(2, kRoundThreads);
}

// Warp 0 only: argmin over the options of position `pos` under a predicate.
template <typename Pred>
__device__ __forceinline__ int warp_best_option(const RoundBuf &R, int pos, int nopt, Pred pred) {
  const int lane = threadIdx.x & 31;
  const OptRec *o = R.opt + (int64_t)pos * R.maxopt;
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

__device__ __forceinline__ void invalidate_seqs(RoundShared &sh, int TT) {
  for (int q = 0; q < TT; ++q) sh.seq_valid[q] = 0;
}

// Warp 0: ScaleResource(pos) using (and lazily computing) the type sequences.
__device__ bool scale_resource(RoundShared &sh, const RoundBuf &R, int pos) {
  const int lane = threadIdx.x & 31;
  const int TT = R.T;
  const int nopt = R.nopt[pos], ngj = R.ng[pos];
  const OptRec *o = R.opt + (int64_t)pos * R.maxopt;
  const int64_t ref = R.ref[pos];
  // eligible options (G <= N_G) sorted by kappa: rank sort
  int n_el = 0;
  for (int i = lane; i < nopt; i += 32) {
    const OptRec x = o[i];
    if (x.G > ngj) continue;
    int r = 0;
    for (int q = 0; q < nopt; ++q) {
      const OptRec y = o[q];
      r += (y.G <= ngj) && kappa_less(y, x);
    }
    sh.sorted[r] = i;
  }
  for (int i = lane; i < nopt; i += 32) n_el += o[i].G <= ngj;
  for (int d = 16; d > 0; d >>= 1) n_el += __shfl_xor_sync(0xffffffffu, n_el, d);
  __syncwarp();
  for (int r = 0; r < n_el; ++r) {
    const int oi = sh.sorted[r];
    const OptRec x = o[oi];
    const int t = x.t;
    if (!sh.seq_valid[t]) {
      if (lane == 0) sh.req = t;
      __syncwarp();
      named_bar(1, kRoundThreads);  // wake the helper warps
      compute_seq(sh, R, t);
    }
    // shortest prefix m of the sequence with G_o <= free'_m[t]
    const int len = sh.seq_len[t];
    int m = -1;
    for (int q = 0; q <= len; ++q)
      if (x.G <= sh.frs[t][q][t]) {
        m = q;
        break;
      }
    if (m < 0) continue;
    double acc = 0.0;
    for (int q = 0; q < m; ++q) acc = __dadd_rn(acc, sh.mv_loss[t][q]);
    if (score_of(ref, x.T) > acc) {
      if (lane == 0) {
        for (int q = 0; q < m; ++q) R.cur[sh.mv_pos[t][q]] = sh.mv_opt[t][q];
        for (int q = 0; q < TT; ++q) sh.fr[q] = sh.frs[t][m][q];
        sh.fr[t] -= x.G;
        R.cur[pos] = oi;
        R.adm[sh.n_adm] = pos;
        sh.n_adm += 1;
        invalidate_seqs(sh, TT);
      }
      __syncwarp();
      return true;
    }
  }
  return false;
}

__global__ void __launch_bounds__(kRoundThreads, 1) k_round_greedy(RoundBuf R) {
  __shared__ RoundShared sh;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int TT = R.T;
  if (tid < TT) {
    sh.fr[tid] = R.free_io[tid];
    sh.seq_valid[tid] = 0;
  }
  if (tid == 0) sh.n_adm = 0;
  __syncthreads();

  if (wid != 0) {  // helper warps: wait for sequence requests
    for (;;) {
      named_bar(1, kRoundThreads);
      const int t = sh.req;
      if (t < 0) break;
      compute_seq(sh, R, t);
    }
  } else {
    // ---- Phase A: SchedArrival in priority order
    for (int pos = 0; pos < R.J; ++pos) {
      const int64_t ref = R.ref[pos];
      if (ref == kInf) continue;  // unschedulable
      const int nopt = R.nopt[pos], ngj = R.ng[pos];
      const int best = warp_best_option(R, pos, nopt, [&](int, const OptRec &x) {
        return x.G <= ngj && x.G <= sh.fr[x.t];
      });
      if (best >= 0) {
        if (lane == 0) {
          const OptRec x = R.opt[(int64_t)pos * R.maxopt + best];
          R.cur[pos] = best;
          sh.fr[x.t] -= x.G;
          R.adm[sh.n_adm] = pos;
          sh.n_adm += 1;
          invalidate_seqs(sh, TT);
        }
        __syncwarp();
      } else if (R.depth >= 1) {
        scale_resource(sh, R, pos);
      }
    }
    // ---- Phase B: up to d sweeps of reverse scaling
    for (int sweep = 0; sweep < R.depth; ++sweep) {
      bool changed = false;
      const int n_adm = sh.n_adm;
      for (int a = 0; a < n_adm; ++a) {
        const int pos = R.adm[a];
        const int cv = R.cur[pos];
        const OptRec cur = R.opt[(int64_t)pos * R.maxopt + cv];
        const int best = warp_best_option(R, pos, R.nopt[pos], [&](int i, const OptRec &x) {
          const int avail = sh.fr[x.t] + (x.t == cur.t ? cur.G : 0);
          return i != cv && x.G <= avail && x.T < cur.T;
        });
        if (best >= 0) {
          if (lane == 0) {
            const OptRec x = R.opt[(int64_t)pos * R.maxopt + best];
            sh.fr[cur.t] += cur.G;
            sh.fr[x.t] -= x.G;
            R.cur[pos] = best;
          }
          __syncwarp();
          changed = true;
        }
      }
      if (!changed) break;
    }
    // ---- total score in priority order (fp64, sequential: bit-reproducible)
    if (lane == 0) {
      double tot = 0.0;
      for (int a = 0; a < sh.n_adm; ++a) {
        const int pos = R.adm[a];
        tot = __dadd_rn(tot, score_of(R.ref[pos], R.opt[(int64_t)pos * R.maxopt + R.cur[pos]].T));
      }
      *R.total = tot;
      sh.req = -1;
    }
    __syncwarp();
    named_bar(1, kRoundThreads);  // release helpers
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
