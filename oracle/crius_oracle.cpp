// crius_oracle.cpp -- TEST INFRASTRUCTURE ONLY (see crius_oracle.h).
//
// A plain, slow, single-threaded CPU implementation of what the Crius hot path
// computes, written from the paper (arXiv 2403.16125, /root/reference/PAPER.md,
// cited as P:<line>) and the normative readings of SURVEY.md §8(c) / §N0-§N6
// (cited as §Nx, A-n).  Every sum is taken directly over its layers, every
// argmin is a first-minimum scan, the round is executed literally.  No prefix
// sums, no binary search, no caching beyond what the definitions state.
//
// Arithmetic: all decision-path quantities are integers (A-1); intermediate
// products use signed/unsigned 128-bit so nothing can wrap; any result that
// would leave the documented range (T_iter < 2^62, §N0) returns code 7.
// fp64 appears only in the round's scores (§N6), with no FMA contraction
// (built with -ffp-contract=off).
//
// Parity pins for every function live in tests/test_oracle_pins.py.
#include "crius_oracle.h"

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <vector>

typedef __int128 i128;
typedef unsigned __int128 u128;

static const int64_t INF = INT64_MAX;
static const int64_t MIB = 1 << 20;
static const i128 LIMIT = (i128)1 << 62;

namespace {

struct Overflow {};

int64_t narrow(i128 v) {
  if (v < 0 || v >= LIMIT) throw Overflow();
  return (int64_t)v;
}

// cdiv(a, b) = ceil(a / b) for a >= 0, b > 0 (§N0).
i128 cdiv(i128 a, i128 b) { return (a + b - 1) / b; }

int ilog2(int64_t x) {
  int e = 0;
  while ((int64_t(1) << e) < x) ++e;
  return e;
}

// ---- §N4 communication (A-14: ring alpha-beta; beta in ns per MiB) --------
// AR(p, l, V, n) = 0 if p == 1 else n*2(p-1)*alpha + cdiv(2(p-1)*V*beta, p*2^20)
i128 AR(i128 p, i128 alpha, i128 beta, i128 V, i128 n) {
  if (p == 1) return 0;
  return n * 2 * (p - 1) * alpha + cdiv(2 * (p - 1) * V * beta, p * MIB);
}
// AG(p, l, V) = 0 if p == 1 else (p-1)*alpha + cdiv((p-1)*V*beta, p*2^20)
i128 AG(i128 p, i128 alpha, i128 beta, i128 V) {
  if (p == 1) return 0;
  return (p - 1) * alpha + cdiv((p - 1) * V * beta, p * MIB);
}
// P2P(l, V) = alpha + cdiv(V*beta, 2^20)
i128 P2P(i128 alpha, i128 beta, i128 V) { return alpha + cdiv(V * beta, MIB); }

struct Cell {
  int32_t job, type, G, S, nplans;
};

// ---- §N2 enumeration ("Initializing Cells"; A-6) ---------------
std::vector<int32_t> gpu_counts(const oracle_problem *pr, int j, int t) {
  std::vector<int32_t> Gs;
  int32_t cap = pr->cap[t], ng = pr->ng[j];
  if (pr->gpu_set == 0) {  // paper: N_G/2, N_G, 2N_G
    if (ng >= 2 && ng / 2 <= cap) Gs.push_back(ng / 2);
    if (ng <= cap) Gs.push_back(ng);
    if (2 * ng <= cap) Gs.push_back(2 * ng);
  } else {  // all powers of two <= capacity
    for (int32_t G = 1; G <= cap; G *= 2) Gs.push_back(G);
  }
  return Gs;
}

int32_t n_bvalues(const oracle_problem *pr) { return pr->b_mode == 0 ? 1 : pr->b_count; }

// Bset[b]: {4S} (GPipe) or the configured list (A-11).
int32_t b_value(const oracle_problem *pr, int32_t S, int32_t b) {
  return pr->b_mode == 0 ? 4 * S : pr->b_values[b];
}

std::vector<Cell> enumerate(const oracle_problem *pr) {
  std::vector<Cell> cells;
  for (int32_t j = 0; j < pr->n_jobs; ++j)
    for (int32_t t = 0; t < pr->n_types; ++t)
      for (int32_t G : gpu_counts(pr, j, t))
        for (int32_t S = 1; S <= std::min(std::min(G, pr->n_layers[j]), pr->s_max); S *= 2)
          if (G / S <= pr->g_max) {
            int32_t g = G / S;
            int32_t K = ilog2(g) + 1;  // k = 0..log2 g
            cells.push_back({j, t, G, S, K * n_bvalues(pr)});
          }
  return cells;
}

// ---- §N3 stage split: min-max DP over tp=1 per-layer compute (A-2..A-4) ---
// f[1][i] = P[i];  f[s][i] = min_{k in [s-1, i-1]} max(f[s-1][k], P[i]-P[k]);
// a[s][i] = smallest k attaining it (strict < while scanning k ascending);
// b_S = L, b_{s-1} = a[s][b_s].
std::vector<int32_t> split(const oracle_problem *pr, int32_t j, int32_t t, int32_t S) {
  const int32_t L = pr->n_layers[j];
  const int64_t off = pr->layer_off[j];
  const int64_t TL = pr->layer_off[pr->n_jobs];
  const int32_t *c0 = pr->c + ((int64_t)t * (pr->k_max + 1) + 0) * TL + off;
  std::vector<std::vector<int64_t>> f(S + 1, std::vector<int64_t>(L + 1, INF));
  std::vector<std::vector<int32_t>> arg(S + 1, std::vector<int32_t>(L + 1, -1));
  std::vector<int64_t> last(L + 1, 0);  // last[k] = cost of the stage [k, i)
  for (int32_t i = 1; i <= L; ++i) {
    f[1][i] = 0;
    for (int32_t l = 0; l < i; ++l) f[1][i] += c0[l];
  }
  for (int32_t s = 2; s <= S; ++s)
    for (int32_t i = s; i <= L; ++i) {
      // the stage [k, i) summed directly over its layers, k = i-1 down to 0
      last[i] = 0;
      for (int32_t k = i - 1; k >= 0; --k) last[k] = last[k + 1] + c0[k];
      for (int32_t k = s - 1; k <= i - 1; ++k) {
        int64_t v = std::max(f[s - 1][k], last[k]);
        if (v < f[s][i]) {
          f[s][i] = v;
          arg[s][i] = k;
        }
      }
    }
  std::vector<int32_t> b(S + 1);
  b[S] = L;
  for (int32_t s = S; s >= 2; --s) b[s - 1] = arg[s][b[s]];
  b[0] = 0;
  return b;
}

// ---- §N5 plan cost, every stage sum taken directly over its layers -------
struct PlanOut {
  bool feasible;
  int64_t t_iter;
};

PlanOut plan_cost(const oracle_problem *pr, const Cell &cell, const std::vector<int32_t> &b,
                  int32_t p, int64_t *T_out, int64_t *sync_out, int64_t *mem_out) {
  const int32_t j = cell.job, t = cell.type, S = cell.S;
  const int64_t off = pr->layer_off[j];
  const int64_t TL = pr->layer_off[pr->n_jobs];
  const int32_t nB = n_bvalues(pr);
  const int32_t k = p / nB;                      // plan p = k*nB + b (A-9)
  const int32_t B = b_value(pr, S, p % nB);
  const i128 g = cell.G / S;                     // uniform GPUs per stage (A-5)
  const i128 tp = (i128)1 << k, dp = g / tp;
  const i128 GB = pr->gb[j];
  if (B * dp > GB) return {false, 0};            // A-12
  const i128 mb = GB / (B * dp);
  const int64_t gpn = pr->gpn[t];
  const int32_t *ck = pr->c + ((int64_t)t * (pr->k_max + 1) + k) * TL + off;
  // link classes (A-15)
  const bool tp_in = tp <= gpn, dp_in = g <= gpn;
  const i128 a_tp = tp_in ? pr->alpha_in[t] : pr->alpha_x[t];
  const i128 b_tp = tp_in ? pr->beta_in[t] : pr->beta_x[t];
  const i128 a_dp = dp_in ? pr->alpha_in[t] : pr->alpha_x[t];
  const i128 b_dp = dp_in ? pr->beta_in[t] : pr->beta_x[t];
  bool feasible = true;
  i128 sumT = 0, maxT = 0, maxSync = 0;
  for (int32_t s = 0; s < S; ++s) {
    const int32_t a = b[s], e = b[s + 1];
    i128 C = 0, TPV = 0, TPN = 0, W = 0, A = 0;
    for (int32_t l = a; l < e; ++l) {
      C += ck[l];
      TPV += pr->tpv[off + l];
      TPN += pr->tpn[off + l];
      W += pr->w[off + l];
      A += pr->act[off + l];
    }
    const i128 comp = mb * C;
    const i128 tpc = AR(tp, a_tp, b_tp, mb * TPV, TPN);
    i128 inb = 0;
    if (s > 0) {
      const bool b_in = (g < gpn) && ((int64_t)s % (gpn / (int64_t)g) != 0);
      const i128 a_b = b_in ? pr->alpha_in[t] : pr->alpha_x[t];
      const i128 b_b = b_in ? pr->beta_in[t] : pr->beta_x[t];
      const i128 V = mb * pr->bnd[off + a - 1];
      inb = P2P(a_b, b_b, cdiv(V, tp)) + AG(tp, a_tp, b_tp, V);
    }
    const i128 T = comp + tpc + inb;
    const i128 sync = AR(dp, a_dp, b_dp, cdiv(W, tp), 1);
    const i128 mem = cdiv((i128)pr->kst[j] * W + (GB / dp) * A, tp);
    if (mem > pr->mem[t]) feasible = false;       // memory filter (A-13)
    if (T_out) T_out[s] = narrow(T);
    if (sync_out) sync_out[s] = narrow(sync);
    if (mem_out) mem_out[s] = narrow(mem);
    sumT += T;
    maxT = std::max(maxT, T);
    maxSync = std::max(maxSync, sync);
  }
  // T_iter = sum_s T_s + (B-1) max_s T_s + max_s sync_s   (north_star; D4, A-7)
  const i128 t_iter = sumT + (i128)(B - 1) * maxT + maxSync;
  return {feasible, narrow(t_iter)};
}

// ---- NEXT-1: per-stage parallelism assembly ------
// Each stage independently takes a DP x TP factorisation of its g = G/S GPUs:
// mode 1 = the paper's assembled set, every stage DP-only or TP-only (2^S
// plans); mode 2 = every factorisation per stage.  A stage's costs
// are the §N5 terms evaluated with its own tp, dp and mb = GB/(B dp).
struct StageCost {
  bool ok;
  i128 T, Tc, sync;  // Tc = the stage's inbound communication
};

std::vector<int32_t> stage_choices(int32_t mode, int32_t g) {
  const int32_t K = ilog2(g);
  std::vector<int32_t> ks;
  if (mode == 1) {
    ks.push_back(0);              // data-parallelism-only
    if (K > 0) ks.push_back(K);   // tensor-parallelism-only
  } else {
    for (int32_t k = 0; k <= K; ++k) ks.push_back(k);
  }
  return ks;
}

StageCost stage_cost(const oracle_problem *pr, int32_t j, int32_t t, int32_t g, int32_t B,
                     const std::vector<int32_t> &b, int32_t s, int32_t k) {
  const int64_t off = pr->layer_off[j];
  const int64_t TL = pr->layer_off[pr->n_jobs];
  const i128 tp = (i128)1 << k, dp = (i128)g / tp, GB = pr->gb[j];
  if (B * dp > GB) return {false, 0, 0, 0};
  const i128 mb = GB / (B * dp);
  const int64_t gpn = pr->gpn[t];
  const int32_t *ck = pr->c + ((int64_t)t * (pr->k_max + 1) + k) * TL + off;
  const bool tp_in = tp <= gpn, dp_in = (i128)g <= gpn;
  const i128 a_tp = tp_in ? pr->alpha_in[t] : pr->alpha_x[t];
  const i128 b_tp = tp_in ? pr->beta_in[t] : pr->beta_x[t];
  const i128 a_dp = dp_in ? pr->alpha_in[t] : pr->alpha_x[t];
  const i128 b_dp = dp_in ? pr->beta_in[t] : pr->beta_x[t];
  i128 C = 0, TPV = 0, TPN = 0, W = 0, A = 0;
  for (int32_t l = b[s]; l < b[s + 1]; ++l) {
    C += ck[l];
    TPV += pr->tpv[off + l];
    TPN += pr->tpn[off + l];
    W += pr->w[off + l];
    A += pr->act[off + l];
  }
  const i128 mem = cdiv((i128)pr->kst[j] * W + (GB / dp) * A, tp);
  if (mem > pr->mem[t]) return {false, 0, 0, 0};
  i128 inb = 0;
  if (s > 0) {
    const bool b_in = ((i128)g < gpn) && ((int64_t)s % (gpn / (int64_t)g) != 0);
    const i128 a_b = b_in ? pr->alpha_in[t] : pr->alpha_x[t];
    const i128 b_b = b_in ? pr->beta_in[t] : pr->beta_x[t];
    const i128 V = mb * pr->bnd[off + b[s] - 1];
    inb = P2P(a_b, b_b, cdiv(V, tp)) + AG(tp, a_tp, b_tp, V);
  }
  const i128 T = mb * C + AR(tp, a_tp, b_tp, mb * TPV, TPN) + inb;
  return {true, T, inb, AR(dp, a_dp, b_dp, cdiv(W, tp), 1)};
}

// Pipeline latency of one assembled plan: sum_s T_s + (B-1) * (T_s* - [form 1] Tc_s*)
// + max_s sync_s, s* = the first slowest stage (north_star form 0; paper form 1).
i128 assembled_latency(const std::vector<StageCost> &st, int32_t B, int32_t form) {
  i128 sum = 0, mx = -1, tc = 0, sy = 0;
  for (const StageCost &c : st) {
    sum += c.T;
    if (c.T > mx) {
      mx = c.T;
      tc = c.Tc;
    }
    sy = std::max(sy, c.sync);
  }
  return sum + (i128)(B - 1) * (mx - (form == 1 ? tc : 0)) + sy;
}

// ---- NEXT-2: the paper's stage determination (Fig. stage_partition)
// Reading R-8 (cuts): the model is cut at the S-1 inter-layer gaps with the
// smallest boundary bytes ("selects the smallest 3 inter-operator
// communication as the clustering boundaries").  With beta = the
// (S-1)-th smallest gap byte count, every gap below beta is a cut and the rest
// are chosen among the gaps equal to beta; among those cut sets, the one that
// keeps the stages' computation most similar: min-max of the tp=1
// per-sample compute, lowest argmin at every step (the R0 rule of §N3).
// Gap q (1 <= q <= L-1) lies between layers q-1 and q and carries bnd[q-1].
std::vector<int32_t> paper_cuts(const oracle_problem *pr, int32_t j, int32_t t, int32_t S) {
  const int32_t L = pr->n_layers[j];
  const int64_t off = pr->layer_off[j];
  const int64_t TL = pr->layer_off[pr->n_jobs];
  const int32_t *c0 = pr->c + ((int64_t)t * (pr->k_max + 1) + 0) * TL + off;
  std::vector<int32_t> b(S + 1);
  b[0] = 0;
  b[S] = L;
  if (S == 1) return b;
  std::vector<int64_t> bytes;
  for (int32_t q = 1; q < L; ++q) bytes.push_back(pr->bnd[off + q - 1]);
  std::vector<int64_t> sorted = bytes;
  std::sort(sorted.begin(), sorted.end());
  const int64_t beta = sorted[S - 2];
  auto forced = [&](int32_t q) { return q >= 1 && q < L && bytes[q - 1] < beta; };
  auto allowed = [&](int32_t q) { return q >= 1 && q < L && bytes[q - 1] <= beta; };
  // no forced gap strictly inside (k, i)
  auto clear = [&](int32_t k, int32_t i) {
    for (int32_t q = k + 1; q < i; ++q)
      if (forced(q)) return false;
    return true;
  };
  auto stage = [&](int32_t k, int32_t i) {  // tp=1 compute of layers [k, i), summed directly
    int64_t v = 0;
    for (int32_t l = k; l < i; ++l) v += c0[l];
    return v;
  };
  std::vector<std::vector<int64_t>> f(S + 1, std::vector<int64_t>(L + 1, INF));
  std::vector<std::vector<int32_t>> arg(S + 1, std::vector<int32_t>(L + 1, -1));
  for (int32_t i = 1; i <= L; ++i)
    if ((allowed(i) || i == L) && clear(0, i)) f[1][i] = stage(0, i);
  for (int32_t s = 2; s <= S; ++s)
    for (int32_t i = s; i <= L; ++i) {
      if (!(allowed(i) || i == L)) continue;
      for (int32_t k = s - 1; k <= i - 1; ++k) {
        if (!allowed(k) || f[s - 1][k] == INF || !clear(k, i)) continue;
        const int64_t v = std::max(f[s - 1][k], stage(k, i));
        if (v < f[s][i]) {
          f[s][i] = v;
          arg[s][i] = k;
        }
      }
    }
  for (int32_t s = S; s >= 2; --s) b[s - 1] = arg[s][b[s]];
  return b;
}

// Reading R-9 (GPUs per stage): stage s maps G * F_s / F GPUs (F = tp=1
// compute, the FLOP proxy of A-3; "T_elapsed = FLOPs / Number_GPU"),
// rounded to the nearest power of two (linear distance, ties up, at least 1;
// "approximates a power of 2"); conservation repair: while the sum
// exceeds G halve the stage with the lowest F_s/g_s among g_s >= 2, then while
// it is below G double the stage with the highest F_s/g_s among those that
// keep the sum <= G (ties: earliest stage).
// Nearest power of two to x = num / den (linear distance, ties up), at least 1.
int32_t round_pow2(i128 num, i128 den) {
  if (num < den) return 1;
  int32_t a = 0;
  while (((i128)2 << a) * den <= num) ++a;  // 2^a <= x < 2^(a+1)
  return (2 * num >= 3 * ((i128)1 << a) * den) ? (2 << a) : (1 << a);
}

std::vector<int32_t> paper_gpus(const oracle_problem *pr, int32_t j, int32_t t, int32_t G,
                                const std::vector<int32_t> &b) {
  const int32_t S = (int32_t)b.size() - 1;
  const int64_t off = pr->layer_off[j];
  const int64_t TL = pr->layer_off[pr->n_jobs];
  const int32_t *c0 = pr->c + ((int64_t)t * (pr->k_max + 1) + 0) * TL + off;
  std::vector<i128> F(S, 0);
  i128 Ftot = 0;
  for (int32_t s = 0; s < S; ++s) {
    for (int32_t l = b[s]; l < b[s + 1]; ++l) F[s] += c0[l];
    Ftot += F[s];
  }
  std::vector<int32_t> g(S);
  for (int32_t s = 0; s < S; ++s) g[s] = round_pow2((i128)G * F[s], Ftot);  // x = G F_s / F
  auto sum = [&]() {
    int64_t v = 0;
    for (int32_t x : g) v += x;
    return v;
  };
  while (sum() > G) {
    int32_t w = -1;
    for (int32_t s = 0; s < S; ++s)
      if (g[s] >= 2 && (w < 0 || F[s] * g[w] < F[w] * g[s])) w = s;
    g[w] /= 2;
  }
  while (sum() < G) {
    int32_t w = -1;
    const int64_t sm = sum();
    for (int32_t s = 0; s < S; ++s)
      if (sm + g[s] <= G && (w < 0 || F[s] * g[w] > F[w] * g[s])) w = s;
    g[w] *= 2;
  }
  return g;
}

// Reading R-10 (cost with per-stage GPU counts): plan p = k*nB + b runs every
// stage with tp = 2^k (k <= log2 min g_s) and dp_s = g_s / tp; stage s is
// costed with the §N5 terms at its own dp_s and mb_s = GB/(B dp_s) (as NEXT-1,
// R-5).  GPUs are packed from a node boundary in stage order (offset o_s =
// sum of the earlier g): tp groups are intra-node iff tp <= gpn and tp | o_s;
// the dp all-reduce is intra iff the stage lies within one node; the boundary
// into s is intra iff o_s is not a node boundary -- for uniform g these are
// exactly A-15.  A Cell whose stages exceed g_max is infeasible.
PlanOut paper_plan_cost(const oracle_problem *pr, int32_t j, int32_t t, int32_t S,
                        const std::vector<int32_t> &b, const std::vector<int32_t> &g, int32_t p) {
  const int64_t off = pr->layer_off[j];
  const int64_t TL = pr->layer_off[pr->n_jobs];
  const int32_t nB = n_bvalues(pr);
  const int32_t k = p / nB;
  const int32_t B = b_value(pr, S, p % nB);
  const i128 tp = (i128)1 << k, GB = pr->gb[j];
  const int64_t gpn = pr->gpn[t];
  const int32_t *ck = pr->c + ((int64_t)t * (pr->k_max + 1) + k) * TL + off;
  bool feasible = true;
  i128 sumT = 0, maxT = 0, maxSync = 0;
  int64_t o = 0;
  for (int32_t s = 0; s < S; ++s) {
    if (g[s] > pr->g_max || (i128)g[s] < tp) return {false, 0};
    const i128 dp = (i128)g[s] / tp;
    if (B * dp > GB) return {false, 0};
    const i128 mb = GB / (B * dp);
    const bool tp_in = tp <= gpn && o % (int64_t)tp == 0;
    const bool dp_in = o / gpn == (o + g[s] - 1) / gpn;
    const i128 a_tp = tp_in ? pr->alpha_in[t] : pr->alpha_x[t];
    const i128 b_tp = tp_in ? pr->beta_in[t] : pr->beta_x[t];
    const i128 a_dp = dp_in ? pr->alpha_in[t] : pr->alpha_x[t];
    const i128 b_dp = dp_in ? pr->beta_in[t] : pr->beta_x[t];
    i128 C = 0, TPV = 0, TPN = 0, W = 0, A = 0;
    for (int32_t l = b[s]; l < b[s + 1]; ++l) {
      C += ck[l];
      TPV += pr->tpv[off + l];
      TPN += pr->tpn[off + l];
      W += pr->w[off + l];
      A += pr->act[off + l];
    }
    i128 inb = 0;
    if (s > 0) {
      const bool b_in = o % gpn != 0;
      const i128 a_b = b_in ? pr->alpha_in[t] : pr->alpha_x[t];
      const i128 b_b = b_in ? pr->beta_in[t] : pr->beta_x[t];
      const i128 V = mb * pr->bnd[off + b[s] - 1];
      inb = P2P(a_b, b_b, cdiv(V, tp)) + AG(tp, a_tp, b_tp, V);
    }
    const i128 T = mb * C + AR(tp, a_tp, b_tp, mb * TPV, TPN) + inb;
    const i128 sync = AR(dp, a_dp, b_dp, cdiv(W, tp), 1);
    const i128 mem = cdiv((i128)pr->kst[j] * W + (GB / dp) * A, tp);
    if (mem > pr->mem[t]) feasible = false;
    sumT += T;
    maxT = std::max(maxT, T);
    maxSync = std::max(maxSync, sync);
    o += g[s];
  }
  return {feasible, narrow(sumT + (i128)(B - 1) * maxT + maxSync)};
}

bool valid_problem(const oracle_problem *pr) {
  if (!pr || pr->n_types < 1 || pr->n_jobs < 0 || pr->k_max < 0) return false;
  if (pr->s_max < 1 || pr->g_max < 1 || pr->g_max > (1 << pr->k_max) || pr->depth < 0) return false;
  if (pr->b_mode == 1 && pr->b_count < 1) return false;
  return true;
}

}  // namespace

extern "C" {

int64_t oracle_comm(int32_t kind, int64_t p, int64_t alpha, int64_t beta, int64_t V, int64_t n) {
  if (kind == 0) return (int64_t)AR(p, alpha, beta, V, n);
  if (kind == 1) return (int64_t)AG(p, alpha, beta, V);
  return (int64_t)P2P(alpha, beta, V);
}

int oracle_count(const oracle_problem *pr, int64_t *n_cells, int64_t *n_plans) {
  if (!valid_problem(pr)) return 2;
  std::vector<Cell> cells = enumerate(pr);
  int64_t np = 0;
  for (const Cell &c : cells) np += c.nplans;
  *n_cells = (int64_t)cells.size();
  *n_plans = np;
  return 0;
}

int oracle_enumerate(const oracle_problem *pr, int32_t *cell_job, int32_t *cell_type,
                     int32_t *cell_G, int32_t *cell_S, int32_t *cell_nplans) {
  if (!valid_problem(pr)) return 2;
  std::vector<Cell> cells = enumerate(pr);
  for (size_t i = 0; i < cells.size(); ++i) {
    cell_job[i] = cells[i].job;
    cell_type[i] = cells[i].type;
    cell_G[i] = cells[i].G;
    cell_S[i] = cells[i].S;
    cell_nplans[i] = cells[i].nplans;
  }
  return 0;
}

int oracle_split(const oracle_problem *pr, int32_t j, int32_t t, int32_t S, int32_t *bounds) {
  if (!valid_problem(pr) || j < 0 || j >= pr->n_jobs || t < 0 || t >= pr->n_types) return 2;
  if (S < 1 || S > pr->n_layers[j]) return 2;
  std::vector<int32_t> b = split(pr, j, t, S);
  for (int32_t s = 0; s <= S; ++s) bounds[s] = b[s];
  return 0;
}

int oracle_plan_cost(const oracle_problem *pr, int32_t j, int32_t t, int32_t G, int32_t S,
                     int32_t p, int64_t *T_stage, int64_t *sync_stage, int64_t *mem_stage,
                     int64_t *t_iter, int32_t *feasible) {
  if (!valid_problem(pr) || j < 0 || j >= pr->n_jobs || t < 0 || t >= pr->n_types) return 2;
  if (S < 1 || S > pr->n_layers[j] || G < S || G % S) return 2;
  Cell cell{j, t, G, S, (ilog2(G / S) + 1) * n_bvalues(pr)};
  if (p < 0 || p >= cell.nplans) return 2;
  try {
    std::vector<int32_t> b = split(pr, j, t, S);
    PlanOut o = plan_cost(pr, cell, b, p, T_stage, sync_stage, mem_stage);
    *feasible = o.feasible ? 1 : 0;
    *t_iter = o.feasible ? o.t_iter : INF;
  } catch (Overflow &) {
    return 7;
  }
  return 0;
}

int oracle_estimate(const oracle_problem *pr, const int32_t *cell_job, const int32_t *cell_type,
                    const int32_t *cell_G, const int32_t *cell_S, const int32_t *cell_nplans,
                    int64_t c0, int64_t c1, int64_t *t_ns, int32_t *plan) {
  if (!valid_problem(pr) || c0 < 0 || c1 < c0) return 2;
  try {
    // memo of O2 results for the current (job, type): splits do not depend on G
    int32_t memo_j = -1, memo_t = -1;
    std::vector<std::vector<int32_t>> memo;
    for (int64_t i = c0; i < c1; ++i) {
      Cell cell{cell_job[i], cell_type[i], cell_G[i], cell_S[i], cell_nplans[i]};
      if (cell.job != memo_j || cell.type != memo_t) {
        memo_j = cell.job;
        memo_t = cell.type;
        memo.assign(pr->n_layers[cell.job] + 1, std::vector<int32_t>());
      }
      if (memo[cell.S].empty()) memo[cell.S] = split(pr, cell.job, cell.type, cell.S);
      const std::vector<int32_t> &b = memo[cell.S];
      // O4: first minimum over p ascending, strict < (lowest p wins ties, A-10)
      int64_t best = INF;
      int32_t best_p = -1;
      for (int32_t p = 0; p < cell.nplans; ++p) {
        PlanOut o = plan_cost(pr, cell, b, p, nullptr, nullptr, nullptr);
        if (o.feasible && o.t_iter < best) {
          best = o.t_iter;
          best_p = p;
        }
      }
      t_ns[i - c0] = best;
      plan[i - c0] = best_p;
    }
  } catch (Overflow &) {
    return 7;
  }
  return 0;
}

// NEXT-2: cuts (bounds[S+1]) and per-stage GPU counts (g[S]) of (j, t, G, S).
int oracle_paper_stages(const oracle_problem *pr, int32_t j, int32_t t, int32_t G, int32_t S,
                        int32_t *bounds, int32_t *g) {
  if (!valid_problem(pr) || j < 0 || j >= pr->n_jobs || S < 1 || S > pr->n_layers[j] || G < S)
    return 2;
  const std::vector<int32_t> b = paper_cuts(pr, j, t, S);
  for (int32_t s = 0; s <= S; ++s) bounds[s] = b[s];
  if (g) {
    const std::vector<int32_t> gg = paper_gpus(pr, j, t, G, b);
    for (int32_t s = 0; s < S; ++s) g[s] = gg[s];
  }
  return 0;
}

// NEXT-2 pieces for the pins: x = num/den rounded (R-9), and the fractional
// GPUs G F_s / F of the stages of given bounds (num[s] over den).
int32_t oracle_paper_round_pow2(int64_t num, int64_t den) { return round_pow2(num, den); }

int oracle_paper_fractional(const oracle_problem *pr, int32_t j, int32_t t, int32_t G, int32_t S,
                            const int32_t *bounds, int64_t *num, int64_t *den) {
  if (!valid_problem(pr)) return 2;
  const int64_t off = pr->layer_off[j];
  const int64_t TL = pr->layer_off[pr->n_jobs];
  const int32_t *c0 = pr->c + ((int64_t)t * (pr->k_max + 1) + 0) * TL + off;
  i128 F = 0;
  for (int32_t s = 0; s < S; ++s) {
    i128 Fs = 0;
    for (int32_t l = bounds[s]; l < bounds[s + 1]; ++l) Fs += c0[l];
    num[s] = narrow((i128)G * Fs);
    F += Fs;
  }
  *den = narrow(F);
  return 0;
}

// NEXT-2 plan cost of plan p given explicit bounds and per-stage GPU counts.
int oracle_paper_plan_cost(const oracle_problem *pr, int32_t j, int32_t t, int32_t S,
                           const int32_t *bounds, const int32_t *g, int32_t p, int64_t *t_iter,
                           int32_t *feasible) {
  if (!valid_problem(pr)) return 2;
  try {
    const PlanOut r = paper_plan_cost(pr, j, t, S, std::vector<int32_t>(bounds, bounds + S + 1),
                                      std::vector<int32_t>(g, g + S), p);
    *t_iter = r.feasible ? r.t_iter : INF;
    *feasible = r.feasible;
  } catch (const Overflow &) {
    return 7;
  }
  return 0;
}

// NEXT-2 estimate for Cells [c0, c1): the paper's stages and GPU counts, then
// the first-minimum plan over k <= log2 min g_s and every B (p = k*nB + b).
// stage_lg[(i-c0)*kstride + s] = log2 g_s (-1 padding).
int oracle_estimate_paper(const oracle_problem *pr, const int32_t *cell_job,
                          const int32_t *cell_type, const int32_t *cell_G, const int32_t *cell_S,
                          int64_t c0, int64_t c1, int64_t *t_ns, int32_t *plan, int8_t *stage_lg,
                          int32_t kstride) {
  if (!valid_problem(pr)) return 2;
  try {
    for (int64_t i = c0; i < c1; ++i) {
      const int32_t j = cell_job[i], t = cell_type[i], G = cell_G[i], S = cell_S[i];
      const std::vector<int32_t> b = paper_cuts(pr, j, t, S);
      const std::vector<int32_t> g = paper_gpus(pr, j, t, G, b);
      int32_t gmin = g[0];
      for (int32_t x : g) gmin = std::min(gmin, x);
      int64_t best = INF;
      int32_t bp = -1;
      const int32_t np = (ilog2(gmin) + 1) * n_bvalues(pr);
      for (int32_t p = 0; p < np; ++p) {
        const PlanOut r = paper_plan_cost(pr, j, t, S, b, g, p);
        if (r.feasible && r.t_iter < best) {
          best = r.t_iter;
          bp = p;
        }
      }
      t_ns[i - c0] = best;
      plan[i - c0] = bp;
      if (stage_lg)
        for (int32_t s = 0; s < kstride; ++s)
          stage_lg[(i - c0) * kstride + s] = (int8_t)(s < S ? ilog2(g[s]) : -1);
    }
  } catch (const Overflow &) {
    return 7;
  }
  return 0;
}

// NEXT-1 estimate: for Cells [c0, c1), every microbatch count and every
// assembled plan (brute force over the product of the per-stage choices).
// t_ns = best latency, bidx = its B index (lowest on ties), stage_k[(i-c0)*kstride + s]
// = log2 tp of stage s in the first best plan found (-1 padding).
int oracle_estimate_assembled(const oracle_problem *pr, int32_t mode, int32_t form,
                              const int32_t *cell_job, const int32_t *cell_type,
                              const int32_t *cell_G, const int32_t *cell_S, int64_t c0,
                              int64_t c1, int64_t *t_ns, int32_t *bidx, int8_t *stage_k,
                              int32_t kstride) {
  if (!valid_problem(pr) || c0 < 0 || c1 < c0 || (mode != 1 && mode != 2) ||
      (form != 0 && form != 1))
    return 2;
  try {
    for (int64_t i = c0; i < c1; ++i) {
      const int32_t j = cell_job[i], t = cell_type[i], G = cell_G[i], S = cell_S[i];
      if (S > kstride) return 2;
      const int32_t g = G / S;
      const std::vector<int32_t> b = split(pr, j, t, S);
      const std::vector<int32_t> ks = stage_choices(mode, g);
      i128 best = -1;
      int32_t best_b = -1;
      std::vector<int32_t> best_k(S, -1);
      for (int32_t bi = 0; bi < n_bvalues(pr); ++bi) {
        const int32_t B = b_value(pr, S, bi);
        // per-stage cost of every choice
        std::vector<std::vector<StageCost>> tab(S, std::vector<StageCost>(ks.size()));
        for (int32_t s = 0; s < S; ++s)
          for (size_t q = 0; q < ks.size(); ++q) tab[s][q] = stage_cost(pr, j, t, g, B, b, s, ks[q]);
        std::vector<size_t> digit(S, 0);  // mixed-radix counter, stage 0 least significant
        for (;;) {
          bool ok = true;
          std::vector<StageCost> st(S);
          for (int32_t s = 0; s < S; ++s) {
            st[s] = tab[s][digit[s]];
            ok = ok && st[s].ok;
          }
          if (ok) {
            const i128 F = assembled_latency(st, B, form);
            if (best < 0 || F < best) {
              best = F;
              best_b = bi;
              for (int32_t s = 0; s < S; ++s) best_k[s] = ks[digit[s]];
            }
          }
          int32_t s = 0;
          while (s < S && ++digit[s] == ks.size()) digit[s++] = 0;
          if (s == S) break;
        }
      }
      t_ns[i - c0] = best < 0 ? INF : narrow(best);
      bidx[i - c0] = best_b;
      for (int32_t s = 0; s < kstride; ++s)
        stage_k[(i - c0) * kstride + s] = (int8_t)(s < S ? best_k[s] : -1);
    }
  } catch (Overflow &) {
    return 7;
  }
  return 0;
}

// NEXT-3: the factorisations a stage keeps under its favour
// (tp_favour = the estimated plan ran the stage tensor-parallel).  The axis
// runs dp-only (k = 0) .. tp-only (k = K = log2 g); half-hybrid = sqrt(g) x
// sqrt(g) (Fig. pruning); for odd K both neighbours of the half point
// are kept on both sides.
std::vector<int32_t> tuned_choices(int32_t g, bool tp_favour) {
  const int32_t K = ilog2(g);
  std::vector<int32_t> ks;
  for (int32_t k = 0; k <= K; ++k) {
    const bool dp_half = 2 * k <= K + 1;  // k <= ceil(K/2)
    const bool tp_half = k >= K / 2;      // k >= floor(K/2)
    if (tp_favour ? tp_half : dp_half) ks.push_back(k);
  }
  return ks;
}

int oracle_tune_choices(int32_t g, int32_t tp_favour, int32_t *ks) {
  std::vector<int32_t> v = tuned_choices(g, tp_favour != 0);
  for (size_t i = 0; i < v.size(); ++i) ks[i] = v[i];
  return (int)v.size();
}

// NEXT-3: best plan over the product of the pruned per-stage sets (brute
// force), every B of the set.  favor[(i-c0)*kstride + s] = log2 tp of stage s
// in the estimated plan (> 0 = TP favour).
int oracle_tune_assembled(const oracle_problem *pr, int32_t form, const int32_t *cell_job,
                          const int32_t *cell_type, const int32_t *cell_G, const int32_t *cell_S,
                          int64_t c0, int64_t c1, const int8_t *favor, int32_t kstride,
                          int64_t *t_ns, int32_t *bidx, int8_t *stage_k) {
  if (!valid_problem(pr) || c0 < 0 || c1 < c0 || (form != 0 && form != 1)) return 2;
  try {
    for (int64_t i = c0; i < c1; ++i) {
      const int32_t j = cell_job[i], t = cell_type[i], G = cell_G[i], S = cell_S[i];
      if (S > kstride) return 2;
      const int32_t g = G / S;
      const std::vector<int32_t> b = split(pr, j, t, S);
      std::vector<std::vector<int32_t>> ch(S);
      for (int32_t s = 0; s < S; ++s) ch[s] = tuned_choices(g, favor[(i - c0) * kstride + s] > 0);
      i128 best = -1;
      int32_t best_b = -1;
      std::vector<int32_t> best_k(S, -1);
      for (int32_t bi = 0; bi < n_bvalues(pr); ++bi) {
        const int32_t B = b_value(pr, S, bi);
        std::vector<size_t> digit(S, 0);
        for (;;) {
          std::vector<StageCost> st(S);
          bool ok = true;
          for (int32_t s = 0; s < S; ++s) {
            st[s] = stage_cost(pr, j, t, g, B, b, s, ch[s][digit[s]]);
            ok = ok && st[s].ok;
          }
          if (ok) {
            const i128 F = assembled_latency(st, B, form);
            if (best < 0 || F < best) {
              best = F;
              best_b = bi;
              for (int32_t s = 0; s < S; ++s) best_k[s] = ch[s][digit[s]];
            }
          }
          int32_t s = 0;
          while (s < S && ++digit[s] == ch[s].size()) digit[s++] = 0;
          if (s == S) break;
        }
      }
      t_ns[i - c0] = best < 0 ? INF : narrow(best);
      bidx[i - c0] = best_b;
      for (int32_t s = 0; s < kstride; ++s)
        stage_k[(i - c0) * kstride + s] = (int8_t)(s < S ? best_k[s] : -1);
    }
  } catch (Overflow &) {
    return 7;
  }
  return 0;
}

// NEXT-1: latency of one given assembled plan (stage_k[s] = log2 tp of stage s).
int oracle_assembled_cost(const oracle_problem *pr, int32_t form, int32_t j, int32_t t, int32_t G,
                          int32_t S, int32_t bi, const int8_t *stage_k, int64_t *latency,
                          int32_t *feasible) {
  if (!valid_problem(pr) || S < 1 || G % S || bi < 0 || bi >= n_bvalues(pr)) return 2;
  try {
    const int32_t g = G / S, B = b_value(pr, S, bi);
    const std::vector<int32_t> b = split(pr, j, t, S);
    std::vector<StageCost> st(S);
    bool ok = true;
    for (int32_t s = 0; s < S; ++s) {
      if (stage_k[s] < 0 || (1 << stage_k[s]) > g) return 2;
      st[s] = stage_cost(pr, j, t, g, B, b, s, stage_k[s]);
      ok = ok && st[s].ok;
    }
    *feasible = ok ? 1 : 0;
    *latency = ok ? narrow(assembled_latency(st, B, form)) : INF;
  } catch (Overflow &) {
    return 7;
  }
  return 0;
}

// ---- §N6 scheduling round (Alg. 1; policy P:466-507) ----------
int oracle_round(const oracle_problem *pr, int64_t n_cells, const int32_t *cell_job,
                 const int32_t *cell_type, const int32_t *cell_G, const int32_t *cell_S,
                 const int64_t *t_ns, const int32_t *free_in, int64_t *decision,
                 int32_t *free_after, double *total_score) {
  return oracle_round_state(pr, n_cells, cell_job, cell_type, cell_G, cell_S, t_ns, free_in,
                            nullptr, nullptr, decision, free_after, total_score);
}

// NEXT-4: the round from a cluster state -- running jobs (run_cell >= 0) start
// admitted on the option of their Cell's (type, G); inactive jobs are skipped
// (decision -3).  With run_cell = active = NULL this is oracle_round.
int oracle_round_state(const oracle_problem *pr, int64_t n_cells, const int32_t *cell_job,
                       const int32_t *cell_type, const int32_t *cell_G, const int32_t *cell_S,
                       const int64_t *t_ns, const int32_t *free_in, const int64_t *run_cell,
                       const uint8_t *active, int64_t *decision, int32_t *free_after,
                       double *total_score) {
  return oracle_round_policy(pr, n_cells, cell_job, cell_type, cell_G, cell_S, t_ns, free_in,
                             run_cell, active, 0, nullptr, decision, free_after, total_score);
}

/* NEXT-4 ablations ("adaptivity scaling as changing the
 * allocated number of GPUs, heterogeneity scaling as changing the allocated GPU
 * type"), reading R-11: policy bit 0 (NA) keeps every job at its requested N_G
 * -- O_j holds only the options with G = N_G (ref_j is unchanged); bit 1 (NH)
 * keeps every admitted job on its GPU type -- no other-type victim move (case
 * ii) and Phase B only considers options of the job's current type; a job's
 * first placement may use any type.
 * Deadline-aware variant ("strict deadline guarantees for
 * each scheduled job"), reading R-12: t_max (per job, NULL = none) bounds the
 * iteration time of the job's options -- a Cell with T > t_max[j] is not an
 * option, except the (type, G) a running job currently uses (its completion
 * was guaranteed when it was placed). */
int oracle_round_policy(const oracle_problem *pr, int64_t n_cells, const int32_t *cell_job,
                        const int32_t *cell_type, const int32_t *cell_G, const int32_t *cell_S,
                        const int64_t *t_ns, const int32_t *free_in, const int64_t *run_cell,
                        const uint8_t *active, int32_t policy, const int64_t *t_max,
                        int64_t *decision, int32_t *free_after, double *total_score) {
  if (!valid_problem(pr) || n_cells < 0 || policy < 0 || policy > 3) return 2;
  const bool no_adapt = (policy & 1) != 0, no_hetero = (policy & 2) != 0;
  const int32_t J = pr->n_jobs, TT = pr->n_types, d = pr->depth;

  // Options O_j: for each (t, G) with a feasible Cell, the Cell with min (T_c, S_c),
  // listed in (t, G) ascending order.
  struct Opt {
    int32_t t, G;
    int64_t T, cell;
    int32_t S;
  };
  std::vector<std::vector<Opt>> O(J);
  std::vector<int64_t> ref(J, INF);
  std::vector<int64_t> ref_any(J, INF);
  for (int64_t c = 0; c < n_cells; ++c) {
    const int32_t j = cell_job[c];
    if (t_ns[c] == INF) continue;
    ref_any[j] = std::min(ref_any[j], t_ns[c]);
    if (cell_G[c] == pr->ng[j]) ref[j] = std::min(ref[j], t_ns[c]);
    if (no_adapt && cell_G[c] != pr->ng[j]) continue;  // NA: only G = N_G is an option
    if (t_max && t_ns[c] > t_max[j]) {  // deadline: too slow, unless the running (type, G)
      const bool running = run_cell && run_cell[j] >= 0 && (active == nullptr || active[j] != 0);
      if (!running || cell_type[c] != cell_type[run_cell[j]] || cell_G[c] != cell_G[run_cell[j]])
        continue;
    }
    bool found = false;
    for (Opt &o : O[j])
      if (o.t == cell_type[c] && o.G == cell_G[c]) {
        found = true;
        if (t_ns[c] < o.T || (t_ns[c] == o.T && cell_S[c] < o.S)) o = {o.t, o.G, t_ns[c], c, cell_S[c]};
      }
    if (!found) O[j].push_back({cell_type[c], cell_G[c], t_ns[c], c, cell_S[c]});
  }
  for (int32_t j = 0; j < J; ++j) {
    std::sort(O[j].begin(), O[j].end(),
              [](const Opt &a, const Opt &b) { return a.t != b.t ? a.t < b.t : a.G < b.G; });
    if (ref[j] == INF) ref[j] = ref_any[j];  // else best overall; INF -> unschedulable
  }
  auto score = [&](int32_t j, const Opt &o) { return (double)ref[j] / (double)o.T; };
  // kappa(o) = (T_o, G_o, t_o) ascending
  auto kappa_less = [](const Opt &a, const Opt &b) {
    if (a.T != b.T) return a.T < b.T;
    if (a.G != b.G) return a.G < b.G;
    return a.t < b.t;
  };

  // pi = jobs by (submit, id) ascending (A-18)
  std::vector<int32_t> pi(J);
  for (int32_t j = 0; j < J; ++j) pi[j] = j;
  std::sort(pi.begin(), pi.end(), [&](int32_t a, int32_t b) {
    if (pr->submit[a] != pr->submit[b]) return pr->submit[a] < pr->submit[b];
    return pr->job_id[a] < pr->job_id[b];
  });

  std::vector<int32_t> fr(TT);
  for (int32_t t = 0; t < TT; ++t) fr[t] = free_in ? free_in[t] : pr->cap[t];
  std::vector<int32_t> cur(J, -1);  // index into O[j]; -1 = not admitted
  auto is_active = [&](int32_t j) { return active == nullptr || active[j] != 0; };
  for (int32_t j = 0; j < J; ++j)
    if (is_active(j) && run_cell && run_cell[j] >= 0) {
      const int64_t rc = run_cell[j];
      for (int32_t i = 0; i < (int32_t)O[j].size(); ++i)
        if (O[j][i].t == cell_type[rc] && O[j][i].G == cell_G[rc]) cur[j] = i;
      if (cur[j] < 0) return 2;  // a running Cell must be one of the job's options
    }

  // ScaleResource(j) (A-17): at most d victim moves per option trial.
  struct Move {
    int32_t v, o2;
    double loss;
  };
  auto scale_resource = [&](int32_t j) -> bool {
    std::vector<int32_t> opts;
    for (int32_t i = 0; i < (int32_t)O[j].size(); ++i)
      if (O[j][i].G <= pr->ng[j]) opts.push_back(i);
    std::sort(opts.begin(), opts.end(),
              [&](int32_t a, int32_t b) { return kappa_less(O[j][a], O[j][b]); });
    for (int32_t oi : opts) {
      const Opt &o = O[j][oi];
      std::vector<int32_t> fr2 = fr;
      std::vector<Move> moves;
      while (o.G > fr2[o.t] && (int32_t)moves.size() < d) {
        bool have = false;
        double best_key = 0;
        int32_t bv = -1, bo = -1, b_freed = 0;
        bool b_other = false;
        for (int32_t v : pi) {  // candidates in pi order, then o' in (t, G) order
          if (cur[v] < 0) continue;
          bool moved = false;
          for (const Move &m : moves) moved = moved || m.v == v;
          if (moved) continue;
          const Opt &cv = O[v][cur[v]];
          if (cv.t != o.t) continue;
          for (int32_t i2 = 0; i2 < (int32_t)O[v].size(); ++i2) {
            if (i2 == cur[v]) continue;
            const Opt &o2 = O[v][i2];
            int32_t freed;
            bool other;
            if (o2.t == o.t && o2.G < cv.G) {
              freed = cv.G - o2.G;
              other = false;
            } else if (!no_hetero && o2.t != o.t && o2.G <= fr2[o2.t]) {
              freed = cv.G;
              other = true;
            } else {
              continue;
            }
            const double loss = score(v, cv) - score(v, o2);
            const double key = loss / (double)freed;
            if (!have || key < best_key) {  // first minimum: earlier pi, then (t, G)
              have = true;
              best_key = key;
              bv = v;
              bo = i2;
              b_freed = freed;
              b_other = other;
            }
          }
        }
        if (!have) break;
        fr2[o.t] += b_freed;
        if (b_other) fr2[O[bv][bo].t] -= O[bv][bo].G;
        moves.push_back({bv, bo, score(bv, O[bv][cur[bv]]) - score(bv, O[bv][bo])});
      }
      if (o.G <= fr2[o.t]) {
        double acc = 0.0;
        for (const Move &m : moves) acc = acc + m.loss;
        if (score(j, o) > acc) {
          for (const Move &m : moves) cur[m.v] = m.o2;
          cur[j] = oi;
          fr = fr2;
          fr[o.t] -= o.G;
          return true;
        }
      }
    }
    return false;
  };

  // Phase A: SchedArrival
  for (int32_t j : pi) {
    if (ref[j] == INF || !is_active(j) || cur[j] >= 0) continue;  // unschedulable / not a candidate
    int32_t best = -1;
    for (int32_t i = 0; i < (int32_t)O[j].size(); ++i) {
      const Opt &o = O[j][i];
      if (o.G <= pr->ng[j] && o.G <= fr[o.t] && (best < 0 || kappa_less(o, O[j][best]))) best = i;
    }
    if (best >= 0) {
      cur[j] = best;
      fr[O[j][best].t] -= O[j][best].G;
    } else if (d >= 1 && scale_resource(j)) {
      // admitted by resource scaling
    }
  }

  // Phase B: extra scheduling / reverse scaling, <= d sweeps
  for (int32_t sweep = 0; sweep < d; ++sweep) {
    bool changed = false;
    for (int32_t j : pi) {
      if (cur[j] < 0) continue;
      const Opt cj = O[j][cur[j]];
      int32_t best = -1;
      for (int32_t i = 0; i < (int32_t)O[j].size(); ++i) {
        if (i == cur[j]) continue;
        const Opt &o = O[j][i];
        if (no_hetero && o.t != cj.t) continue;  // NH: an admitted job keeps its type
        const int32_t avail = fr[o.t] + (o.t == cj.t ? cj.G : 0);
        if (o.G <= avail && o.T < cj.T && (best < 0 || kappa_less(o, O[j][best]))) best = i;
      }
      if (best >= 0) {
        fr[cj.t] += cj.G;
        fr[O[j][best].t] -= O[j][best].G;
        cur[j] = best;
        changed = true;
      }
    }
    if (!changed) break;
  }

  double total = 0.0;
  for (int32_t j : pi)
    if (cur[j] >= 0) total = total + score(j, O[j][cur[j]]);
  for (int32_t j = 0; j < J; ++j)
    decision[j] = !is_active(j) ? -3 : ref[j] == INF ? -2 : (cur[j] < 0 ? -1 : O[j][cur[j]].cell);
  for (int32_t t = 0; t < TT; ++t) free_after[t] = fr[t];
  *total_score = total;
  return 0;
}

}  // extern "C"
