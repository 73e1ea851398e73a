// crius_lib.cu -- libcrius: C-ABI host side (include/crius.h) + kernel launches.
//
// Host code here only validates, allocates, copies and launches; every step of
// the hot path runs in the kernels of enumerate.cuh, estimate.cuh, round.cuh.
// There is no CPU fallback: without a CUDA device every call fails loudly.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/crius.h"
#include "common.cuh"
#include "enumerate.cuh"
#include "estimate.cuh"
#include "round.cuh"
#include "exchange.cuh"

using namespace crius;

namespace {

thread_local std::string g_err;

crius_status fail(crius_status s, const std::string &msg) {
  g_err = msg;
  return s;
}

#define CK(call)                                                                        \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      return fail(e_ == cudaErrorMemoryAllocation ? CRIUS_ENOMEM : CRIUS_ECUDA,         \
                  std::string(#call) + ": " + cudaGetErrorString(e_));                  \
  } while (0)

#define CKL()                                                                           \
  do {                                                                                  \
    cudaError_t e_ = cudaGetLastError();                                                \
    if (e_ != cudaSuccess) return fail(CRIUS_ECUDA, std::string("launch: ") + cudaGetErrorString(e_)); \
  } while (0)

bool pow2(int64_t x) { return x >= 1 && (x & (x - 1)) == 0; }

// One NVTX range per C-ABI call (SURVEY §5 tracing): nsys / ncu --nvtx show
// the boundary calls around their kernels; a no-op without an attached tool.
struct AbiRange {
  explicit AbiRange(const char *name) { nvtxRangePushA(name); }
  ~AbiRange() { nvtxRangePop(); }
};
#define CRIUS_ABI_RANGE() AbiRange abi_range_(__func__)
int ilog2_host(int64_t x) {
  int e = 0;
  while ((int64_t(1) << e) < x) ++e;
  return e;
}

template <typename T>
cudaError_t dalloc(T **p, size_t n) {
  return cudaMalloc((void **)p, (n ? n : 1) * sizeof(T));
}

}  // namespace

struct crius_ctx {
  int device = 0;
  int n_sm = 148;
  Params P{};                 // host copy holding device pointers
  int32_t k_max = 0;
  int64_t TL = 0;
  int32_t Lmax = 0;
  int64_t launches = 0;
  // inputs (device)
  int32_t *d_ng = nullptr, *d_gb = nullptr, *d_kst = nullptr, *d_L = nullptr;
  int64_t *d_off = nullptr, *d_submit = nullptr, *d_id = nullptr;
  int32_t *d_c = nullptr, *d_tpn = nullptr;
  int64_t *d_w = nullptr, *d_act = nullptr, *d_bnd = nullptr, *d_tpv = nullptr;
  int32_t *d_rank = nullptr, *d_pi = nullptr;
  int64_t *d_pkeys = nullptr;     // [4J] priority sort keys: (submit, id), double buffered
  int32_t *d_pvals = nullptr;     // [2J] priority sort job indices, double buffered
  std::vector<int64_t> h_submit, h_id;  // the (submit, id) pi was computed from
  int32_t *d_scratch = nullptr;  // [J + 8] stats
  // host copies needed later
  std::vector<int32_t> cap;
  // enumeration
  bool enumerated = false;
  int64_t n_units = 0, n_cells = 0, n_plans = 0, cells_capacity = 0;
  int32_t stat_maxcells = 0, stat_smax = 0, stat_gmax = 0;
  Cells C{};
  int64_t *d_scan_sums[3] = {nullptr, nullptr, nullptr};
  int64_t scan_sums_cap = 0;
  int64_t *d_part = nullptr;  // partition outputs
  int32_t *d_counter = nullptr;
  // round
  int32_t maxopt = 0;
  OptRec *d_opt = nullptr;
  double *d_score = nullptr;
  int64_t *d_opt_cell = nullptr, *d_ref = nullptr, *d_decision = nullptr;
  int32_t *d_nopt = nullptr, *d_rng = nullptr, *d_cur = nullptr, *d_free = nullptr;
  int32_t *d_run_opt = nullptr;
  int8_t *d_cand = nullptr;
  int64_t *d_run_cell = nullptr;
  uint8_t *d_active = nullptr;
  double *d_total = nullptr;
  int64_t *d_round_stats = nullptr;
  int32_t *d_ao_pk = nullptr, *d_nao = nullptr, *d_rerr = nullptr, *d_ord = nullptr;
  double *d_ao_sc = nullptr, *d_osc = nullptr;
  uint64_t *d_gminb = nullptr, *d_tsb = nullptr;
  uint8_t *d_operm = nullptr;
  int32_t *d_opk = nullptr;
  // crius_update_estimate: the row upload runs on its own stream, one event per chunk
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_start = nullptr;
  std::vector<cudaEvent_t> ev_chunk;
  AdmView adm_glob{};  // admitted-job records and type lists in global memory (beyond shared)
  int32_t round_policy = 0;  // crius_set_round_policy (NEXT-4 ablations)
  int64_t *d_tmax = nullptr;  // crius_set_deadline_bounds: [J] or unset
  bool has_tmax = false;
  // fused exchange (crius_exchange_*): own window = [flags int64[kMaxRanks] | pad to
  // kXchHdr][2][x_cap] records; x_peer[r] = rank r's window mapped over CUDA IPC
  int32_t x_rank = -1, x_world = 0;
  int64_t x_cap = 0, x_epoch = 0;
  int64_t x_min_cap = 0;  // smallest window capacity over the ranks (read from their headers)
  // jobs whose per-layer rows the last load / update uploaded (estimates of
  // units outside them would read stale rows)
  int32_t rows_j0 = 0, rows_j1 = 0;
  bool x_open = false;
  unsigned char *x_base = nullptr;
  unsigned char *x_peer[kMaxRanks] = {};
  uint32_t *x_done = nullptr;
};

namespace {

constexpr int kMaxChunks = 64;  // crius_update_estimate row chunks

void free_all(crius_ctx *c) {
  void *ptrs[] = {c->d_ng, c->d_gb, c->d_kst, c->d_L, c->d_off, c->d_submit, c->d_id, c->d_c,
                  c->d_tpn, c->d_w, c->d_act, c->d_bnd, c->d_tpv, c->d_rank, c->d_pi,
                  c->d_pkeys, c->d_pvals,
                  c->d_scratch, c->d_tmax, c->C.job, c->C.type, c->C.G, c->C.S, c->C.nplans, c->C.plan_off,
                  c->C.unit_cell_begin, c->C.unit_plan_begin, c->C.unit_weight,
                  c->d_scan_sums[0], c->d_scan_sums[1], c->d_scan_sums[2], c->d_part,
                  c->d_counter, c->d_opt, c->d_opt_cell, c->d_ref, c->d_decision, c->d_nopt,
                  c->d_rng, c->d_cur, c->d_free, c->d_total, c->d_round_stats, c->d_score,
                  c->d_ao_pk, c->d_nao, c->d_rerr, c->d_ord, c->d_ao_sc, c->d_osc, c->d_gminb, c->d_tsb,
                  c->d_operm, c->d_opk, c->adm_glob.bk, c->adm_glob.bl, c->adm_glob.ek, c->adm_glob.pos, c->adm_glob.cur, c->adm_glob.G,
                  c->adm_glob.t, c->adm_glob.slot, c->adm_glob.bi, c->adm_glob.ei, c->adm_glob.tl,
                  c->adm_glob.gmb, c->adm_glob.tsb, c->adm_glob.nopt, c->adm_glob.po,
                  c->d_run_opt, c->d_cand, c->d_run_cell, c->d_active};
  for (void *p : ptrs)
    if (p) cudaFree(p);
}

// ---- validation (host): shapes, powers of two, §N0 bounds -----------------
struct JobSums {
  std::vector<__int128> W, A, TPV, TPN, BNDmax;
};

crius_status validate_static(const crius_cluster *cl, const crius_jobs *jb, const crius_config *cf,
                             int64_t *TL_out, int32_t *Lmax_out) {
  if (!cl || !jb || !cf) return fail(CRIUS_EINVAL, "null argument");
  if (cl->n_types < 1 || cl->n_types > kRT)
    return fail(CRIUS_EINVAL, "n_types must be 1..8 (the scheduling round's tables)");
  if (!cl->capacity || !cl->gpus_per_node || !cl->mem_bytes || !cl->alpha_intra_ns ||
      !cl->beta_intra_ns_per_mib || !cl->alpha_inter_ns || !cl->beta_inter_ns_per_mib)
    return fail(CRIUS_EINVAL, "null cluster array");
  for (int t = 0; t < cl->n_types; ++t) {
    if (!pow2(cl->capacity[t]) || cl->capacity[t] > (1 << 30))
      return fail(CRIUS_EINVAL, "capacity[" + std::to_string(t) + "] must be a power of two");
    if (!pow2(cl->gpus_per_node[t]) || cl->gpus_per_node[t] > (1 << 30))
      return fail(CRIUS_EINVAL, "gpus_per_node[" + std::to_string(t) + "] must be a power of two");
    if (cl->mem_bytes[t] < 0 || cl->alpha_intra_ns[t] < 0 || cl->alpha_inter_ns[t] < 0 ||
        cl->alpha_intra_ns[t] >= (int64_t(1) << 40) || cl->alpha_inter_ns[t] >= (int64_t(1) << 40))
      return fail(CRIUS_EINVAL, "mem/alpha out of range for type " + std::to_string(t));
    if (cl->beta_intra_ns_per_mib[t] < 0 || cl->beta_inter_ns_per_mib[t] < 0 ||
        cl->beta_intra_ns_per_mib[t] >= (int64_t(1) << 40) ||
        cl->beta_inter_ns_per_mib[t] >= (int64_t(1) << 40))
      return fail(CRIUS_EINVAL, "beta out of range [0, 2^40) for type " + std::to_string(t));
  }
  if (jb->n_jobs < 1 || jb->n_jobs >= (1 << 24))
    return fail(CRIUS_EINVAL, "n_jobs must be in [1, 2^24) (the round's 24-bit priority tie keys)");
  if (jb->k_max < 0 || jb->k_max > kMaxKmax) return fail(CRIUS_EINVAL, "k_max must be 0..6");
  if (!jb->job_id || !jb->submit_time || !jb->n_gpus_req || !jb->global_batch || !jb->k_state ||
      !jb->n_layers || !jb->layer_off || !jb->compute_ns || !jb->param_bytes || !jb->act_bytes ||
      !jb->boundary_bytes || !jb->tp_bytes || !jb->tp_calls)
    return fail(CRIUS_EINVAL, "null jobs array");
  if (jb->layer_off[0] != 0) return fail(CRIUS_EINVAL, "layer_off[0] must be 0");
  int32_t Lmax = 0;
  for (int j = 0; j < jb->n_jobs; ++j) {
    auto js = [j] { return "job " + std::to_string(j); };  // built only on failure
    if (!pow2(jb->n_gpus_req[j]) || jb->n_gpus_req[j] > (1 << 29))
      return fail(CRIUS_EINVAL, js() + ": N_G must be a power of two");
    if (!pow2(jb->global_batch[j]) || jb->global_batch[j] > (1 << 30))
      return fail(CRIUS_EINVAL, js() + ": global batch must be a power of two");
    if (jb->k_state[j] < 1) return fail(CRIUS_EINVAL, js() + ": k_state must be >= 1");
    if (jb->n_layers[j] < 1 || jb->n_layers[j] > 255)
      return fail(CRIUS_EINVAL, js() + ": n_layers must be 1..255");
    if (jb->layer_off[j + 1] != jb->layer_off[j] + jb->n_layers[j])
      return fail(CRIUS_EINVAL, js() + ": layer_off is not the prefix of n_layers");
    Lmax = std::max(Lmax, jb->n_layers[j]);
  }
  if (!(cf->gpu_set == 0 || cf->gpu_set == 1)) return fail(CRIUS_EINVAL, "gpu_set must be 0 or 1");
  if (cf->s_max < 1) return fail(CRIUS_EINVAL, "s_max must be >= 1");
  if (!pow2(cf->g_max) || cf->g_max > (1 << jb->k_max))
    return fail(CRIUS_EINVAL, "g_max must be a power of two <= 2^k_max");
  if (cf->b_mode == 1) {
    if (cf->b_count < 1 || cf->b_count > kMaxB || !cf->b_values)
      return fail(CRIUS_EINVAL, "b_count must be 1..16");
    for (int b = 0; b < cf->b_count; ++b)
      if (!pow2(cf->b_values[b]) || cf->b_values[b] > (1 << 30) ||
          (b && cf->b_values[b] <= cf->b_values[b - 1]))
        return fail(CRIUS_EINVAL, "b_values must be ascending powers of two");
  } else if (cf->b_mode != 0) {
    return fail(CRIUS_EINVAL, "b_mode must be 0 or 1");
  }
  if (cf->search_depth < 0 || cf->search_depth > kMaxDepth)
    return fail(CRIUS_EINVAL, "search_depth must be 0..16");
  *TL_out = jb->layer_off[jb->n_jobs];
  *Lmax_out = Lmax;
  return CRIUS_OK;
}

crius_status copy_rows(crius_ctx *c, const crius_jobs *jb, int T, cudaStream_t st, int j0, int j1);
crius_status copy_inputs(crius_ctx *c, const crius_cluster *cl, const crius_jobs *jb,
                         cudaStream_t st, int j0, int j1) {
  const int J = jb->n_jobs, T = cl->n_types;
  CK(cudaMemcpyAsync(c->d_ng, jb->n_gpus_req, J * 4, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(c->d_gb, jb->global_batch, J * 4, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(c->d_kst, jb->k_state, J * 4, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(c->d_L, jb->n_layers, J * 4, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(c->d_off, jb->layer_off, (J + 1) * 8, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(c->d_submit, jb->submit_time, J * 8, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(c->d_id, jb->job_id, J * 8, cudaMemcpyHostToDevice, st));
  return copy_rows(c, jb, T, st, j0, j1);
}

// Per-layer rows of jobs [j0, j1): layers [l0, l1), one strided 2-D copy for c.
crius_status copy_rows(crius_ctx *c, const crius_jobs *jb, int T, cudaStream_t st, int j0, int j1) {
  if (j1 <= j0) return CRIUS_OK;
  const size_t TL = (size_t)c->TL;
  const size_t l0 = (size_t)jb->layer_off[j0], nl = (size_t)jb->layer_off[j1] - l0;
  const size_t planes = (size_t)T * (jb->k_max + 1);
  if (nl == TL) {
    CK(cudaMemcpyAsync(c->d_c, jb->compute_ns, planes * TL * 4, cudaMemcpyHostToDevice, st));
  } else {
    CK(cudaMemcpy2DAsync(c->d_c + l0, TL * 4, jb->compute_ns + l0, TL * 4, nl * 4, planes,
                         cudaMemcpyHostToDevice, st));
  }
  CK(cudaMemcpyAsync(c->d_w + l0, jb->param_bytes + l0, nl * 8, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(c->d_act + l0, jb->act_bytes + l0, nl * 8, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(c->d_bnd + l0, jb->boundary_bytes + l0, nl * 8, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(c->d_tpv + l0, jb->tp_bytes + l0, nl * 8, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(c->d_tpn + l0, jb->tp_calls + l0, nl * 4, cudaMemcpyHostToDevice, st));
  return CRIUS_OK;
}

void fill_types(crius_ctx *c, const crius_cluster *cl) {
  c->cap.assign(cl->capacity, cl->capacity + cl->n_types);
  for (int t = 0; t < cl->n_types; ++t) {
    TypeParams &tp = c->P.ty[t];
    tp.cap = cl->capacity[t];
    tp.gpn = cl->gpus_per_node[t];
    tp.lgpn = ilog2_host(cl->gpus_per_node[t]);
    tp.mem = cl->mem_bytes[t];
    tp.a_in = cl->alpha_intra_ns[t];
    tp.b_in = cl->beta_intra_ns_per_mib[t];
    tp.a_x = cl->alpha_inter_ns[t];
    tp.b_x = cl->beta_inter_ns_per_mib[t];
  }
}

// Scratch for the checks: per-job status words and the smallest compute value.
crius_status check_init(crius_ctx *c, int J, cudaStream_t st) {
  CK(cudaMemsetAsync(c->d_scratch, 0, (J + 8) * 4, st));
  static const int32_t big = INT32_MAX;
  CK(cudaMemcpyAsync(c->d_scratch + J, &big, 4, cudaMemcpyHostToDevice, st));
  return CRIUS_OK;
}
// Device bound checks of the rows of jobs [j0, j1) (per-job status in scratch).
crius_status check_rows(crius_ctx *c, const crius_cluster *cl, const crius_config *cf, int J,
                        cudaStream_t st, int j0, int j1) {
  if (j1 > j0) {
    BoundArgs BA{};
    for (int t = 0; t < cl->n_types; ++t) {
      BA.amax = std::max<int64_t>(BA.amax, std::max(cl->alpha_intra_ns[t], cl->alpha_inter_ns[t]));
      BA.bmax = std::max<int64_t>(BA.bmax, std::max(cl->beta_intra_ns_per_mib[t],
                                                    cl->beta_inter_ns_per_mib[t]));
    }
    BA.p = cf->g_max;
    BA.bmax_list = cf->b_mode == 1 ? cf->b_values[cf->b_count - 1] : 0;
    k_profile_check<<<j1 - j0, 64, 0, st>>>(c->P, j0, BA, c->d_scratch, c->d_scratch + J);
    CKL();
    c->launches += 1;
  }
  return CRIUS_OK;
}
// Priority order pi (launches only when submit/id changed).
crius_status sort_priority(crius_ctx *c, const crius_jobs *jb, cudaStream_t st) {
  const int J = jb->n_jobs;
  // priority order pi by (submit, id) (A-18): recomputed only when they changed
  const bool same = c->h_submit.size() == (size_t)J &&
                    std::equal(c->h_submit.begin(), c->h_submit.end(), jb->submit_time) &&
                    std::equal(c->h_id.begin(), c->h_id.end(), jb->job_id);
  int n_sort = 0;
  if (!same) {
    c->h_submit.assign(jb->submit_time, jb->submit_time + J);
    c->h_id.assign(jb->job_id, jb->job_id + J);
    int64_t *sa = c->d_pkeys, *ia = c->d_pkeys + J, *sb = c->d_pkeys + 2 * (size_t)J,
            *ib = c->d_pkeys + 3 * (size_t)J;
    int32_t *ja = c->d_pvals, *jb2 = c->d_pvals + J;
    k_prio_tiles<<<(J + kPrioTile - 1) / kPrioTile, 1024, 0, st>>>(c->d_submit, c->d_id, J, sa, ia, ja);
    CKL();
    n_sort = 2;
    for (int W = kPrioTile; W < J; W <<= 1) {
      k_prio_merge<<<(J + 255) / 256, 256, 0, st>>>(sa, ia, ja, J, W, sb, ib, jb2);
      CKL();
      std::swap(sa, sb);
      std::swap(ia, ib);
      std::swap(ja, jb2);
      ++n_sort;
    }
    k_priority_scatter<<<(unsigned)((J + 255) / 256), 256, 0, st>>>(ja, J, c->d_pi, c->d_rank);
    CKL();
  }
  c->launches += n_sort;
  return CRIUS_OK;
}
// The checks' verdict (synchronises).
crius_status check_result(crius_ctx *c, int J, cudaStream_t st, int j0, int j1) {
  std::vector<int32_t> stats(J + 1);
  CK(cudaMemcpyAsync(stats.data(), c->d_scratch, (J + 1) * 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (j1 > j0 && stats[J] < 1) return fail(CRIUS_EINVAL, "compute_ns must be >= 1 everywhere");
  static const char *why[] = {"", "negative per-layer value", "L*max(c)*GB >= 2^52",
                              "alpha-beta numerator >= 2^63", "kst*sum(w) + GB*sum(act) >= 2^62",
                              "T_iter bound >= 2^62"};
  for (int j = j0; j < j1; ++j)
    if (stats[j] != 0)
      return fail(CRIUS_EINVAL, "job " + std::to_string(j) + ": " + why[std::min(stats[j], 5)]);
  return CRIUS_OK;
}

// Device stats of c -> §N0 bounds; then priority ranks.  Synchronises.
crius_status finish_load(crius_ctx *c, const crius_cluster *cl, const crius_jobs *jb,
                         const crius_config *cf, cudaStream_t st, int j0, int j1) {
  const int J = jb->n_jobs;
  crius_status s = check_init(c, J, st);
  if (s == CRIUS_OK) s = check_rows(c, cl, cf, J, st, j0, j1);
  if (s == CRIUS_OK) s = sort_priority(c, jb, st);
  if (s == CRIUS_OK) s = check_result(c, J, st, j0, j1);
  return s;
}

}  // namespace

extern "C" {

const char *crius_last_error(void) { return g_err.c_str(); }

int64_t crius_kernel_launches(const crius_ctx *ctx) { return ctx ? ctx->launches : 0; }

crius_status crius_load_profiles(crius_ctx **out, const crius_cluster *cl, const crius_jobs *jb,
                                 const crius_config *cf, int32_t device, void *stream) {
  CRIUS_ABI_RANGE();
  if (!out) return fail(CRIUS_EINVAL, "null out");
  *out = nullptr;
  int64_t TL = 0;
  int32_t Lmax = 0;
  crius_status s = validate_static(cl, jb, cf, &TL, &Lmax);
  if (s != CRIUS_OK) return s;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0)
    return fail(CRIUS_ECUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
  if (device < 0 || device >= ndev) return fail(CRIUS_EINVAL, "bad device ordinal");
  CK(cudaSetDevice(device));
  cudaStream_t st = (cudaStream_t)stream;

  crius_ctx *c = new crius_ctx();
  c->device = device;
  cudaDeviceGetAttribute(&c->n_sm, cudaDevAttrMultiProcessorCount, device);
  c->k_max = jb->k_max;
  c->TL = TL;
  c->Lmax = Lmax;
  const int J = jb->n_jobs, T = cl->n_types;
  Params &P = c->P;
  P.T = T;
  P.J = J;
  P.K1 = jb->k_max + 1;
  P.TL = TL;
  P.gpu_set = cf->gpu_set;
  P.s_max = cf->s_max;
  P.g_max = cf->g_max;
  P.b_mode = cf->b_mode;
  P.nB = cf->b_mode == 0 ? 1 : cf->b_count;
  P.depth = cf->search_depth;
  for (int b = 0; b < (cf->b_mode == 1 ? cf->b_count : 0); ++b) P.lB[b] = ilog2_host(cf->b_values[b]);
  fill_types(c, cl);
  int nG = 3;
  if (cf->gpu_set == 1) {
    nG = 0;
    for (int t = 0; t < T; ++t) nG = std::max(nG, ilog2_host(cl->capacity[t]) + 1);
  }
  c->maxopt = T * nG;
  if (c->maxopt > 256) {
    delete c;
    return fail(CRIUS_EINVAL, "n_types x GPU-count choices must be <= 256");
  }

  auto cleanup = [&](crius_status st_) {
    free_all(c);
    delete c;
    return st_;
  };
#define CKA(call)                                                                       \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      return cleanup(fail(e_ == cudaErrorMemoryAllocation ? CRIUS_ENOMEM : CRIUS_ECUDA, \
                          std::string(#call) + ": " + cudaGetErrorString(e_)));        \
  } while (0)
  CKA(dalloc(&c->d_ng, J));
  CKA(dalloc(&c->d_gb, J));
  CKA(dalloc(&c->d_kst, J));
  CKA(dalloc(&c->d_L, J));
  CKA(dalloc(&c->d_off, J + 1));
  CKA(dalloc(&c->d_submit, J));
  CKA(dalloc(&c->d_id, J));
  CKA(dalloc(&c->d_c, (size_t)T * P.K1 * TL));
  CKA(dalloc(&c->d_w, TL));
  CKA(dalloc(&c->d_act, TL));
  CKA(dalloc(&c->d_bnd, TL));
  CKA(dalloc(&c->d_tpv, TL));
  CKA(dalloc(&c->d_tpn, TL));
  CKA(dalloc(&c->d_rank, J));
  CKA(dalloc(&c->d_pi, J));
  CKA(dalloc(&c->d_pkeys, 4 * (size_t)J));
  CKA(dalloc(&c->d_pvals, 2 * (size_t)J));
  CKA(dalloc(&c->d_scratch, J + 8));
  CKA(dalloc(&c->d_counter, 4));
  CKA(dalloc(&c->d_part, 2 * 9 + 2));
  P.ng = c->d_ng;
  P.gb = c->d_gb;
  P.kst = c->d_kst;
  P.L = c->d_L;
  P.off = c->d_off;
  P.c = c->d_c;
  P.w = c->d_w;
  P.act = c->d_act;
  P.bnd = c->d_bnd;
  P.tpv = c->d_tpv;
  P.tpn = c->d_tpn;
  s = copy_inputs(c, cl, jb, st, 0, jb->n_jobs);
  if (s != CRIUS_OK) return cleanup(s);
  c->rows_j0 = 0;
  c->rows_j1 = jb->n_jobs;
  s = finish_load(c, cl, jb, cf, st, 0, jb->n_jobs);
  if (s != CRIUS_OK) return cleanup(s);
#undef CKA
  *out = c;
  return CRIUS_OK;
}

crius_status crius_update_profiles(crius_ctx *c, const crius_cluster *cl, const crius_jobs *jb,
                                   void *stream) {
  if (!c) return fail(CRIUS_EINVAL, "null ctx");
  return crius_update_profiles_range(c, cl, jb, 0, c->P.J, stream);
}

crius_status crius_update_profiles_range(crius_ctx *c, const crius_cluster *cl,
                                         const crius_jobs *jb, int32_t job_begin,
                                         int32_t job_end, void *stream) {
  CRIUS_ABI_RANGE();
  if (!c) return fail(CRIUS_EINVAL, "null ctx");
  if (job_begin < 0 || job_end > c->P.J || job_begin > job_end)
    return fail(CRIUS_EINVAL, "update_profiles_range: bad job range");
  if (!cl || !jb || cl->n_types != c->P.T || jb->n_jobs != c->P.J || jb->k_max != c->k_max)
    return fail(CRIUS_EINVAL, "update_profiles: shape differs from the loaded problem");
  crius_config cf{};
  cf.gpu_set = c->P.gpu_set;
  cf.s_max = c->P.s_max;
  cf.g_max = c->P.g_max;
  cf.b_mode = c->P.b_mode;
  std::vector<int32_t> bv;
  for (int b = 0; b < (c->P.b_mode ? c->P.nB : 0); ++b) bv.push_back(1 << c->P.lB[b]);
  cf.b_count = (int32_t)bv.size();
  cf.b_values = bv.data();
  cf.search_depth = c->P.depth;
  int64_t TL = 0;
  int32_t Lmax = 0;
  crius_status s = validate_static(cl, jb, &cf, &TL, &Lmax);
  if (s != CRIUS_OK) return s;
  if (TL != c->TL) return fail(CRIUS_EINVAL, "update_profiles: total layers differ");
  for (int t = 0; t < cl->n_types; ++t)
    if (cl->capacity[t] != c->cap[t]) return fail(CRIUS_EINVAL, "update_profiles: capacity differs");
  CK(cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  fill_types(c, cl);
  c->Lmax = Lmax;
  s = copy_inputs(c, cl, jb, st, job_begin, job_end);
  if (s != CRIUS_OK) return s;
  c->enumerated = false;
  c->rows_j0 = job_begin;
  c->rows_j1 = job_end;
  return finish_load(c, cl, jb, &cf, st, job_begin, job_end);
}

crius_status crius_enumerate_cells(crius_ctx *c, int64_t *n_cells, int64_t *n_plans,
                                   int64_t *n_units, void *stream) {
  CRIUS_ABI_RANGE();
  if (!c) return fail(CRIUS_EINVAL, "null ctx");
  CK(cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t U = (int64_t)c->P.J * c->P.T;
  if (c->n_units != U || !c->C.unit_cell_begin) {
    if (c->C.unit_cell_begin) cudaFree(c->C.unit_cell_begin);
    if (c->C.unit_plan_begin) cudaFree(c->C.unit_plan_begin);
    if (c->C.unit_weight) cudaFree(c->C.unit_weight);
    CK(dalloc(&c->C.unit_cell_begin, U + 1));
    CK(dalloc(&c->C.unit_plan_begin, U + 1));
    CK(dalloc(&c->C.unit_weight, U + 1));
    const int64_t tiles = (U + kScanTile - 1) / kScanTile;
    for (int q = 0; q < 3; ++q) {
      if (c->d_scan_sums[q]) cudaFree(c->d_scan_sums[q]);
      CK(dalloc(&c->d_scan_sums[q], tiles + 1));
    }
    c->n_units = U;
  }
  int32_t *stats = c->d_scratch + c->P.J + 1;  // 3 ints
  CK(cudaMemsetAsync(stats, 0, 3 * 4, st));
  UnitCounts UC{c->C.unit_cell_begin, c->C.unit_plan_begin, c->C.unit_weight, stats};
  k_unit_count<<<(unsigned)((U + 255) / 256), 256, 0, st>>>(c->P, UC, U);
  CKL();
  const int64_t tiles = (U + kScanTile - 1) / kScanTile;
  Scan3 X{{c->C.unit_cell_begin, c->C.unit_plan_begin, c->C.unit_weight}};
  Scan3 S{{c->d_scan_sums[0], c->d_scan_sums[1], c->d_scan_sums[2]}};
  k_scan_tiles<<<(unsigned)tiles, kScanThreads, 0, st>>>(X, U, S);
  CKL();
  k_scan_sums<<<1, kScanThreads, 0, st>>>(S, tiles);
  CKL();
  k_scan_add<<<(unsigned)((U + 255) / 256), 256, 0, st>>>(X, U, S, tiles);
  CKL();
  c->launches += 4;
  int64_t tot[2];
  int32_t hs[3];
  CK(cudaMemcpyAsync(&tot[0], c->C.unit_cell_begin + U, 8, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&tot[1], c->C.unit_plan_begin + U, 8, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(hs, stats, 12, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  c->n_cells = tot[0];
  c->n_plans = tot[1];
  c->stat_maxcells = hs[0];
  c->stat_smax = hs[1];
  c->stat_gmax = hs[2];
  if (c->n_cells > c->cells_capacity) {
    int32_t **i32s[] = {&c->C.job, &c->C.type, &c->C.G, &c->C.S, &c->C.nplans};
    for (int32_t **p : i32s) {
      if (*p) cudaFree(*p);
      CK(dalloc(p, c->n_cells));
    }
    if (c->C.plan_off) cudaFree(c->C.plan_off);
    CK(dalloc(&c->C.plan_off, c->n_cells));
    c->cells_capacity = c->n_cells;
  }
  if (c->n_cells > 0) {
    k_unit_fill<<<(unsigned)((U + 255) / 256), 256, 0, st>>>(c->P, c->C, U);
    CKL();
    c->launches += 1;  // stream-ordered: no second host round trip
  }
  if (n_cells) *n_cells = c->n_cells;
  if (n_plans) *n_plans = c->n_plans;
  if (n_units) *n_units = U;
  c->enumerated = true;
  if (c->n_cells == 0) return fail(CRIUS_EINFEASIBLE, "enumeration produced zero Cells");
  return CRIUS_OK;
}

crius_status crius_cells(crius_ctx *c, crius_cell_view *v) {
  if (!c || !v) return fail(CRIUS_EINVAL, "null argument");
  if (!c->enumerated) return fail(CRIUS_ESTATE, "crius_cells before crius_enumerate_cells");
  v->n_cells = c->n_cells;
  v->n_cell_plans = c->n_plans;
  v->n_units = c->n_units;
  v->job = c->C.job;
  v->type = c->C.type;
  v->G = c->C.G;
  v->S = c->C.S;
  v->nplans = c->C.nplans;
  v->plan_off = c->C.plan_off;
  v->unit_cell_begin = c->C.unit_cell_begin;
  v->unit_plan_begin = c->C.unit_plan_begin;
  return CRIUS_OK;
}

int32_t crius_max_stages(const crius_ctx *c) { return c ? std::max(1, c->stat_smax) : 0; }

int32_t crius_split_stride(const crius_ctx *c) {
  if (!c) return 0;
  int nsi = 0;
  while ((1 << nsi) <= std::max(1, c->stat_smax)) ++nsi;  // S = 1 .. stat_smax
  return (1 << nsi) - 1 + nsi;
}

}  // extern "C"

namespace {

__global__ void k_partition(const int64_t *__restrict__ wprefix, const int64_t *__restrict__ ucb,
                            int64_t n_units, int32_t world, int64_t *out) {
  const int r = threadIdx.x;
  if (r > world) return;
  const int64_t W = wprefix[n_units];
  int64_t ub;
  if (r == world) {
    ub = n_units;
  } else {
    const int64_t target = (int64_t)((__int128)W * r / world);
    int64_t lo = 0, hi = n_units;  // first u with prefix[u] >= target
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (wprefix[mid] >= target)
        hi = mid;
      else
        lo = mid + 1;
    }
    ub = r == 0 ? 0 : lo;
  }
  out[r] = ub;
  out[world + 1 + r] = ucb[ub];
}

}  // namespace

extern "C" {

crius_status crius_partition_units(crius_ctx *c, int32_t world, int64_t *unit_begin,
                                   int64_t *cell_begin, void *stream) {
  CRIUS_ABI_RANGE();
  if (!c || !unit_begin || !cell_begin) return fail(CRIUS_EINVAL, "null argument");
  if (!c->enumerated) return fail(CRIUS_ESTATE, "partition before enumerate");
  if (world < 1 || world > 8) return fail(CRIUS_EINVAL, "world must be 1..8");
  CK(cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  k_partition<<<1, 32, 0, st>>>(c->C.unit_weight, c->C.unit_cell_begin, c->n_units, world, c->d_part);
  CKL();
  c->launches += 1;
  std::vector<int64_t> h(2 * (world + 1));
  CK(cudaMemcpyAsync(h.data(), c->d_part, h.size() * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  for (int r = 0; r <= world; ++r) {
    unit_begin[r] = h[r];
    cell_begin[r] = h[world + 1 + r];
  }
  return CRIUS_OK;
}

}  // extern "C"

namespace {

// Shared launcher of k_estimate: amode 0 = uniform plans (§N5), 1/2 = NEXT-1
// per-stage assembly (paper DP-only/TP-only per stage; every factorisation).
constexpr int64_t kXchHdr = 256;     // header bytes at the head of a window: flags int64[8], ...
constexpr int64_t kXchCapOff = 128;  // ... and the window's capacity (int64)

crius_status launch_estimate(crius_ctx *c, int amode, int form, int64_t unit_begin,
                             int64_t unit_end, crius_cell_result *d_out, int16_t *d_splits,
                             int8_t *d_stage_tp, const int8_t *d_favor, cudaStream_t st,
                             bool exchange = false, bool global_out = false) {
  if (!c->enumerated) return fail(CRIUS_ESTATE, "estimate before enumerate");
  if (unit_begin < 0 || unit_end > c->n_units || unit_begin > unit_end)
    return fail(CRIUS_EINVAL, "bad unit range");
  if (unit_begin < unit_end &&
      (unit_begin / c->P.T < c->rows_j0 || (unit_end - 1) / c->P.T >= c->rows_j1))
    return fail(CRIUS_EINVAL, "unit range reaches jobs whose profile rows the last update did not upload");
  if (!d_out && !exchange) return fail(CRIUS_EINVAL, "null d_out");
  CK(cudaSetDevice(c->device));
  EstArgs A{};
  if (exchange) {
    A.nx = c->x_world;
    A.x_rank = c->x_rank;
    A.x_epoch = c->x_epoch;
    A.x_done = c->x_done;
    const int64_t half = (c->x_epoch & 1) * c->x_cap * (int64_t)sizeof(CellResult);
    for (int r = 0; r < c->x_world; ++r) {
      A.xflag[r] = (int64_t *)c->x_peer[r];
      A.xout[r] = (CellResult *)(c->x_peer[r] + kXchHdr + half);
    }
  }
  if (unit_begin == unit_end) {
    if (!exchange) return CRIUS_OK;
    // nothing to estimate: still tell every rank this rank's (empty) range is done
    k_xch_signal_only<<<1, 32, 0, st>>>(A);
    CKL();
    c->launches += 1;
    return CRIUS_OK;
  }
  A.cG = c->C.G;
  A.cS = c->C.S;
  A.plan_off = c->C.plan_off;
  A.ucb = c->C.unit_cell_begin;
  A.upb = c->C.unit_plan_begin;
  A.unit_begin = unit_begin;
  A.unit_end = unit_end;
  A.out = (CellResult *)d_out;
  A.splits = d_splits;
  A.global_out = global_out;
  A.split_stride = crius_split_stride(c);
  A.work_counter = c->d_counter;
  A.form = form;
  A.stage_tp = d_stage_tp;
  A.favor = d_favor;
  A.stage_stride = std::max(1, c->stat_smax);
  // per-warp shared-memory layout
  const int Lp = c->Lmax + 1;
  const int K1e = ilog2_host(std::max(1, c->stat_gmax)) + 1;
  const int Stop = std::max(1, c->stat_smax);
  const int maxCells = std::max(1, c->stat_maxcells);
  int o = 0;
  auto take = [&](int bytes) {
    const int at = o;
    o += (bytes + 15) & ~15;
    return at;
  };
  A.Lp = Lp;
  A.K1e = K1e;
  A.Stop = Stop;
  A.maxCells = maxCells;
  A.off_PC = take(K1e * Lp * 8);
  A.off_PW = take(Lp * 8);
  A.off_PA = take(Lp * 8);
  A.off_PV = take(Lp * 8);
  A.off_PN = take(Lp * 8);
  A.off_BND = take(Lp * 8);
  A.off_F = take(2 * Lp * 8);
  A.off_ARG = take((Stop + 1) * Lp);
  // the raw int32 compute rows are dead once their prefix sums are in PC, before
  // the DP first writes F / ARG: share those bytes when they are large enough
  const bool craw_alias = K1e * Lp * 4 <= o - A.off_F;
  A.off_CRAW = craw_alias ? A.off_F : 0;
  A.off_BD = take(A.split_stride * 2);
  A.off_CELL = take(4 * (maxCells + 1) * 4);
  if (!craw_alias) A.off_CRAW = take(K1e * Lp * 4);
  A.off_NRAW = take(Lp * 4);
  A.off_POFF = take(maxCells * 8);
  A.off_ORD = take((maxCells + 1) * 4);
  A.st_cap = (amode == 0 || amode == 4) ? 0 : Stop * (amode == 1 ? 2 : K1e);  // modes 2, 3: every k
  A.off_ST = take(A.st_cap * 25);
  A.off_PS = take(amode == 4 ? Lp * 12 + Stop * 4 : 0);
  A.warp_bytes = o;
  const int64_t nunits = unit_end - unit_begin;
  // per-stage plan lanes when units hold few plans (cfg4: 21 per unit, 0.25 ->
  // 0.23 ms; the all-pow2 variant's 132 per unit: 0.65 -> 0.85 ms, so per plan)
  A.per_stage = c->P.b_mode == 0 && c->n_plans <= 48 * c->n_units;
  if (const char *e = getenv("CRIUS_EST_PER_STAGE")) A.per_stage = c->P.b_mode == 0 && atoi(e) != 0;
  CK(cudaMemsetAsync(c->d_counter, 0, 4, st));
  int warps = 4;
  if (4 * A.warp_bytes > 200 * 1024) warps = 1;
#ifdef CRIUS_EST_FORCE_W1
  warps = 1;  // experiment: one warp per CTA (finer shared-memory granularity)
#endif
  if (A.warp_bytes > 220 * 1024) return fail(CRIUS_EINVAL, "unit too large for shared memory");
  const size_t smem = (size_t)warps * A.warp_bytes;
#ifndef CRIUS_NBG_WIDE
#define CRIUS_NBG_WIDE 4  // microbatch counts per lane in b_mode 1 (measured best)
#endif
  // one lane per (Cell, k, group of microbatch counts): 1 B per lane (B = 4S)
  // or up to CRIUS_NBG_WIDE of the configured B values per lane
  const bool wide = c->P.b_mode == 1;
  void (*kern)(Params, EstArgs) = nullptr;
  if (amode == 0)
    kern = warps == 4 ? (wide ? k_estimate<4, CRIUS_NBG_WIDE, 0> : k_estimate<4, 1, 0>)
                      : (wide ? k_estimate<1, CRIUS_NBG_WIDE, 0> : k_estimate<1, 1, 0>);
  else if (amode == 1)
    kern = warps == 4 ? k_estimate<4, 1, 1> : k_estimate<1, 1, 1>;
  else if (amode == 2)
    kern = warps == 4 ? k_estimate<4, 1, 2> : k_estimate<1, 1, 2>;
  else if (amode == 3)
    kern = warps == 4 ? k_estimate<4, 1, 3> : k_estimate<1, 1, 3>;
  else
    kern = warps == 4 ? (wide ? k_estimate<4, CRIUS_NBG_WIDE, 4> : k_estimate<4, 1, 4>)
                      : (wide ? k_estimate<1, CRIUS_NBG_WIDE, 4> : k_estimate<1, 1, 4>);
  int per_sm = 1;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * warps, smem));
  per_sm = std::max(per_sm, 1);
  const int64_t want = (nunits + warps - 1) / warps;
  const unsigned grid = (unsigned)std::min<int64_t>(want, (int64_t)c->n_sm * per_sm);
  kern<<<grid, 32 * warps, smem, st>>>(c->P, A);
  CKL();
  c->launches += 1;
  return CRIUS_OK;
}

}  // namespace

extern "C" {

crius_status crius_estimate_cells(crius_ctx *c, int64_t unit_begin, int64_t unit_end,
                                  crius_cell_result *d_out, int16_t *d_splits, void *stream) {
  CRIUS_ABI_RANGE();
  if (!c) return fail(CRIUS_EINVAL, "null ctx");
  return launch_estimate(c, 0, 0, unit_begin, unit_end, d_out, d_splits, nullptr, nullptr,
                         (cudaStream_t)stream);
}

crius_status crius_update_estimate(crius_ctx *c, const crius_cluster *cl, const crius_jobs *jb,
                                   int32_t n_chunks, crius_cell_result *d_out, int64_t out_capacity,
                                   int16_t *d_splits, int64_t *n_cells, int64_t *n_cell_plans,
                                   int64_t *n_units, void *stream) {
  CRIUS_ABI_RANGE();
  if (!c) return fail(CRIUS_EINVAL, "null ctx");
  if (!d_out) return fail(CRIUS_EINVAL, "null d_out");
  if (n_chunks < 1 || n_chunks > kMaxChunks)
    return fail(CRIUS_EINVAL, "update_estimate: n_chunks outside [1, 64]");
  if (!cl || !jb || cl->n_types != c->P.T || jb->n_jobs != c->P.J || jb->k_max != c->k_max)
    return fail(CRIUS_EINVAL, "update_profiles: shape differs from the loaded problem");
  crius_config cf{};
  cf.gpu_set = c->P.gpu_set;
  cf.s_max = c->P.s_max;
  cf.g_max = c->P.g_max;
  cf.b_mode = c->P.b_mode;
  std::vector<int32_t> bv;
  for (int b = 0; b < (c->P.b_mode ? c->P.nB : 0); ++b) bv.push_back(1 << c->P.lB[b]);
  cf.b_count = (int32_t)bv.size();
  cf.b_values = bv.data();
  cf.search_depth = c->P.depth;
  int64_t TL = 0;
  int32_t Lmax = 0;
  crius_status s = validate_static(cl, jb, &cf, &TL, &Lmax);
  if (s != CRIUS_OK) return s;
  if (TL != c->TL) return fail(CRIUS_EINVAL, "update_profiles: total layers differ");
  for (int t = 0; t < cl->n_types; ++t)
    if (cl->capacity[t] != c->cap[t]) return fail(CRIUS_EINVAL, "update_profiles: capacity differs");
  CK(cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  const int J = c->P.J, T = c->P.T;
  n_chunks = std::min(n_chunks, J);
  if (!c->copy_stream) {
    CK(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&c->ev_start, cudaEventDisableTiming));
    c->ev_chunk.resize(kMaxChunks);
    for (cudaEvent_t &e : c->ev_chunk) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  fill_types(c, cl);
  c->Lmax = Lmax;
  c->enumerated = false;
  // per-job arrays on `stream`; the rows on the copy stream, which first waits
  // for the work already queued on `stream` (it may still read the old rows)
  s = copy_inputs(c, cl, jb, st, 0, 0);
  if (s != CRIUS_OK) return s;
  CK(cudaEventRecord(c->ev_start, st));
  CK(cudaStreamWaitEvent(c->copy_stream, c->ev_start, 0));
  // chunk q = jobs [jq[q], jq[q+1]), cut at equal layer counts (equal bytes)
  std::vector<int> jq(n_chunks + 1, J);
  jq[0] = 0;
  for (int q = 1, j = 0; q < n_chunks; ++q) {
    const int64_t want = TL * q / n_chunks;
    while (j < J && jb->layer_off[j] < want) ++j;
    jq[q] = std::max(jq[q - 1], j);
  }
  // on any failure from here the caller's host rows must outlive the copies
  auto bail = [&](crius_status e) {
    cudaStreamSynchronize(c->copy_stream);
    return e;
  };
  for (int q = 0; q < n_chunks; ++q) {
    s = copy_rows(c, jb, T, c->copy_stream, jq[q], jq[q + 1]);
    if (s != CRIUS_OK) return bail(s);
    CK(cudaEventRecord(c->ev_chunk[q], c->copy_stream));
  }
  c->rows_j0 = 0;
  c->rows_j1 = J;
  s = check_init(c, J, st);
  if (s == CRIUS_OK) s = sort_priority(c, jb, st);
  if (s != CRIUS_OK) return bail(s);
  // enumeration needs only the per-job arrays: it runs while the rows go up
  int64_t nc = 0, np = 0, nu = 0;
  s = crius_enumerate_cells(c, &nc, &np, &nu, stream);
  if (n_cells) *n_cells = nc;
  if (n_cell_plans) *n_cell_plans = np;
  if (n_units) *n_units = nu;
  if (s != CRIUS_OK) return bail(s);
  if (nc > out_capacity)
    return bail(fail(CRIUS_EINVAL, "update_estimate: d_out holds fewer records than n_cells (returned)"));
  // chunk q's checks and estimate as soon as its rows are resident; records
  // and splits at their global Cell / unit index
  for (int q = 0; q < n_chunks; ++q) {
    CK(cudaStreamWaitEvent(st, c->ev_chunk[q], 0));
    s = check_rows(c, cl, &cf, J, st, jq[q], jq[q + 1]);
    if (s == CRIUS_OK)
      s = launch_estimate(c, 0, 0, (int64_t)jq[q] * T, (int64_t)jq[q + 1] * T, d_out, d_splits,
                          nullptr, nullptr, st, false, true);
    if (s != CRIUS_OK) return bail(s);
  }
  s = check_result(c, J, st, 0, J);
  if (s != CRIUS_OK) c->enumerated = false;  // the estimates read rows that failed the checks
  return s;
}

// ---- fused exchange (SURVEY §8(e) fused-collective option) -------------------
crius_status crius_exchange_init(crius_ctx *c, int32_t rank, int32_t world, int64_t capacity_cells,
                                 uint8_t *handle_out) {
  CRIUS_ABI_RANGE();
  if (!c || !handle_out) return fail(CRIUS_EINVAL, "null argument");
  if (world < 1 || world > kMaxRanks || rank < 0 || rank >= world)
    return fail(CRIUS_EINVAL, "rank/world out of range (world <= 8)");
  if (capacity_cells < 1) return fail(CRIUS_EINVAL, "capacity_cells must be >= 1");
  if (c->x_base) return fail(CRIUS_ESTATE, "exchange already initialised");
  CK(cudaSetDevice(c->device));
  const size_t bytes = (size_t)kXchHdr + 2 * (size_t)capacity_cells * sizeof(CellResult);
  CK(cudaMalloc((void **)&c->x_base, bytes));
  CK(cudaMalloc((void **)&c->x_done, sizeof(uint32_t)));
  CK(cudaMemset(c->x_base, 0, kXchHdr));
  // the window's capacity sits in its header (offset kXchCapOff) for the peers to check
  CK(cudaMemcpy(c->x_base + kXchCapOff, &capacity_cells, sizeof(int64_t), cudaMemcpyHostToDevice));
  CK(cudaMemset(c->x_done, 0, sizeof(uint32_t)));
  CK(cudaDeviceSynchronize());  // flags are zero before any peer can signal
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, c->x_base));
  std::memcpy(handle_out, &h, sizeof(h));
  c->x_rank = rank;
  c->x_world = world;
  c->x_cap = capacity_cells;
  c->x_epoch = 0;
  c->x_open = false;
  return CRIUS_OK;
}

crius_status crius_exchange_open(crius_ctx *c, const uint8_t *handles) {
  CRIUS_ABI_RANGE();
  if (!c || !handles) return fail(CRIUS_EINVAL, "null argument");
  if (!c->x_base || c->x_open) return fail(CRIUS_ESTATE, "exchange not initialised or already open");
  CK(cudaSetDevice(c->device));
  for (int r = 0; r < c->x_world; ++r) {
    if (r == c->x_rank) {
      c->x_peer[r] = c->x_base;
      continue;
    }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handles + (size_t)r * sizeof(h), sizeof(h));
    void *p = nullptr;
    CK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    c->x_peer[r] = (unsigned char *)p;
  }
  // every rank stores its records into every window: the smallest capacity bounds n_cells
  c->x_min_cap = c->x_cap;
  for (int r = 0; r < c->x_world; ++r) {
    int64_t cap = 0;
    CK(cudaMemcpy(&cap, c->x_peer[r] + kXchCapOff, sizeof(int64_t), cudaMemcpyDeviceToHost));
    c->x_min_cap = std::min(c->x_min_cap, cap);
  }
  c->x_open = true;
  return CRIUS_OK;
}

crius_status crius_estimate_exchange(crius_ctx *c, int64_t unit_begin, int64_t unit_end, void *stream) {
  CRIUS_ABI_RANGE();
  if (!c) return fail(CRIUS_EINVAL, "null ctx");
  if (!c->x_open) return fail(CRIUS_ESTATE, "exchange not open");
  if (!c->enumerated) return fail(CRIUS_ESTATE, "estimate before enumerate");
  if (c->n_cells > c->x_min_cap)
    return fail(CRIUS_EINVAL, "more Cells than the smallest exchange window (over the ranks)");
  c->x_epoch += 1;
  const crius_status s = launch_estimate(c, 0, 0, unit_begin, unit_end, nullptr, nullptr, nullptr,
                                         nullptr, (cudaStream_t)stream, true);
  if (s != CRIUS_OK) c->x_epoch -= 1;
  return s;
}

crius_status crius_exchange_wait(crius_ctx *c, crius_cell_result **d_all, void *stream) {
  CRIUS_ABI_RANGE();
  if (!c || !d_all) return fail(CRIUS_EINVAL, "null argument");
  if (!c->x_open || c->x_epoch < 1) return fail(CRIUS_ESTATE, "no exchange step to wait for");
  CK(cudaSetDevice(c->device));
  k_xch_wait<<<1, 32, 0, (cudaStream_t)stream>>>((const int64_t *)c->x_base, c->x_world, c->x_epoch);
  CKL();
  c->launches += 1;
  *d_all = (crius_cell_result *)(c->x_base + kXchHdr +
                                 (c->x_epoch & 1) * c->x_cap * (int64_t)sizeof(CellResult));
  return CRIUS_OK;
}

crius_status crius_exchange_close(crius_ctx *c) {
  CRIUS_ABI_RANGE();
  if (!c) return fail(CRIUS_EINVAL, "null ctx");
  if (!c->x_base) return CRIUS_OK;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  for (int r = 0; r < c->x_world; ++r)
    if (c->x_peer[r] && r != c->x_rank) cudaIpcCloseMemHandle(c->x_peer[r]);
  cudaFree(c->x_base);
  cudaFree(c->x_done);
  for (int r = 0; r < kMaxRanks; ++r) c->x_peer[r] = nullptr;
  c->x_base = nullptr;
  c->x_done = nullptr;
  c->x_open = false;
  c->x_world = 0;
  c->x_rank = -1;
  return CRIUS_OK;
}

crius_status crius_estimate_assembled(crius_ctx *c, const crius_assembly *asm_cfg,
                                      int64_t unit_begin, int64_t unit_end,
                                      crius_cell_result *d_out, int8_t *d_stage_tp, void *stream) {
  CRIUS_ABI_RANGE();
  if (!c || !asm_cfg) return fail(CRIUS_EINVAL, "null argument");
  if (asm_cfg->mode != 1 && asm_cfg->mode != 2) return fail(CRIUS_EINVAL, "assembly mode must be 1 or 2");
  if (asm_cfg->pipeline_form != 0 && asm_cfg->pipeline_form != 1)
    return fail(CRIUS_EINVAL, "pipeline_form must be 0 or 1");
  return launch_estimate(c, asm_cfg->mode, asm_cfg->pipeline_form, unit_begin, unit_end, d_out,
                         nullptr, d_stage_tp, nullptr, (cudaStream_t)stream);
}

crius_status crius_estimate_paper_stages(crius_ctx *c, int64_t unit_begin, int64_t unit_end,
                                        crius_cell_result *d_out, int16_t *d_splits,
                                        int8_t *d_stage_lg, void *stream) {
  CRIUS_ABI_RANGE();
  if (!c) return fail(CRIUS_EINVAL, "null ctx");
  return launch_estimate(c, 4, 0, unit_begin, unit_end, d_out, d_splits, d_stage_lg, nullptr,
                         (cudaStream_t)stream);
}

crius_status crius_tune_assembled(crius_ctx *c, int32_t pipeline_form, int64_t unit_begin,
                                  int64_t unit_end, const int8_t *d_favor,
                                  crius_cell_result *d_out, int8_t *d_stage_tp, void *stream) {
  CRIUS_ABI_RANGE();
  if (!c || !d_favor) return fail(CRIUS_EINVAL, "null argument");
  if (pipeline_form != 0 && pipeline_form != 1)
    return fail(CRIUS_EINVAL, "pipeline_form must be 0 or 1");
  return launch_estimate(c, 3, pipeline_form, unit_begin, unit_end, d_out, nullptr, d_stage_tp,
                         d_favor, (cudaStream_t)stream);
}

crius_status crius_compact_gathered(crius_ctx *c, const crius_cell_result *d_gathered,
                                    int64_t chunk_stride, int32_t world, const int64_t *cell_begin,
                                    crius_cell_result *d_all, void *stream) {
  CRIUS_ABI_RANGE();
  if (!c || !d_gathered || !cell_begin || !d_all) return fail(CRIUS_EINVAL, "null argument");
  if (!c->enumerated) return fail(CRIUS_ESTATE, "compact before enumerate");
  if (world < 1 || world > 8) return fail(CRIUS_EINVAL, "world must be 1..8");
  CompactArgs A{};
  for (int r = 0; r <= world; ++r) A.cb[r] = cell_begin[r];
  A.world = world;
  A.stride = chunk_stride;
  A.n_cells = c->n_cells;
  for (int r = 0; r < world; ++r)
    if (A.cb[r + 1] - A.cb[r] > chunk_stride || A.cb[r + 1] < A.cb[r])
      return fail(CRIUS_EINVAL, "chunk larger than chunk_stride");
  if (A.cb[0] != 0 || A.cb[world] != c->n_cells) return fail(CRIUS_EINVAL, "cell_begin must span all Cells");
  CK(cudaSetDevice(c->device));
  k_compact<<<(unsigned)((c->n_cells + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      (const CellResult *)d_gathered, A, (CellResult *)d_all);
  CKL();
  c->launches += 1;
  return CRIUS_OK;
}

crius_status crius_schedule_round(crius_ctx *c, const crius_cell_result *d_all,
                                  const int32_t *free_gpus, int64_t *decision, int32_t *free_after,
                                  double *total_score, void *stream) {
  return crius_schedule_round_state(c, d_all, free_gpus, nullptr, nullptr, decision, free_after,
                                    total_score, stream);
}

crius_status crius_schedule_round_state(crius_ctx *c, const crius_cell_result *d_all,
                                        const int32_t *free_gpus, const int64_t *run_cell,
                                        const uint8_t *active, int64_t *decision,
                                        int32_t *free_after, double *total_score, void *stream) {
  CRIUS_ABI_RANGE();
  if (!c || !d_all || !decision || !free_after || !total_score)
    return fail(CRIUS_EINVAL, "null argument");
  if (!c->enumerated) return fail(CRIUS_ESTATE, "round before enumerate");
  CK(cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  const int J = c->P.J, T = c->P.T;
  if (!c->d_opt) {
    const size_t JO = (size_t)J * c->maxopt;
    CK(dalloc(&c->d_opt, JO));
    CK(dalloc(&c->d_score, JO));
    CK(dalloc(&c->d_opt_cell, JO));
    CK(dalloc(&c->d_ao_pk, JO));
    CK(dalloc(&c->d_ao_sc, JO));
    CK(dalloc(&c->d_operm, JO));
    CK(dalloc(&c->d_opk, JO));
    CK(dalloc(&c->d_ref, J));
    CK(dalloc(&c->d_decision, J));
    CK(dalloc(&c->d_nopt, J));
    CK(dalloc(&c->d_nao, J));
    CK(dalloc(&c->d_gminb, J));
    CK(dalloc(&c->d_tsb, J));
    CK(dalloc(&c->d_rng, J));
    CK(dalloc(&c->d_cur, J));
    CK(dalloc(&c->d_free, 16));
    CK(dalloc(&c->d_total, 1));
    CK(dalloc(&c->d_round_stats, 32));
    CK(cudaMemset(c->d_round_stats, 0, 32 * 8));
    CK(dalloc(&c->d_run_opt, J));
    CK(dalloc(&c->d_cand, J));
    CK(dalloc(&c->d_run_cell, J));
    CK(dalloc(&c->d_active, J));
    CK(dalloc(&c->d_rerr, 1));
    CK(dalloc(&c->d_ord, J));
    CK(dalloc(&c->d_osc, J));
    // admitted records in global memory (used when they exceed shared memory)
    CK(dalloc(&c->adm_glob.bk, J));
    CK(dalloc(&c->adm_glob.bl, J));
    CK(dalloc(&c->adm_glob.ek, J));
    CK(dalloc(&c->adm_glob.pos, J));
    CK(dalloc(&c->adm_glob.cur, J));
    CK(dalloc(&c->adm_glob.G, J));
    CK(dalloc(&c->adm_glob.t, J));
    CK(dalloc(&c->adm_glob.slot, J));
    CK(dalloc(&c->adm_glob.bi, J));
    CK(dalloc(&c->adm_glob.ei, J));
    CK(dalloc(&c->adm_glob.gmb, J));
    CK(dalloc(&c->adm_glob.tsb, J));
    CK(dalloc(&c->adm_glob.nopt, J));
    CK(dalloc(&c->adm_glob.po, J));
    CK(dalloc(&c->adm_glob.tl, (size_t)T * J));
  }
  std::vector<int32_t> fr(T);
  for (int t = 0; t < T; ++t) {
    fr[t] = free_gpus ? free_gpus[t] : c->cap[t];
    if (fr[t] < 0 || fr[t] > (1 << 30)) return fail(CRIUS_EINVAL, "free_gpus must be in [0, 2^30]");
  }
  CK(cudaMemcpyAsync(c->d_free, fr.data(), T * 4, cudaMemcpyHostToDevice, st));
  CK(cudaMemsetAsync(c->d_rerr, 0, 4, st));
  if (run_cell) {
    for (int j = 0; j < J; ++j)
      if (run_cell[j] < -1 || run_cell[j] >= c->n_cells)
        return fail(CRIUS_EINVAL, "run_cell out of range");
    CK(cudaMemcpyAsync(c->d_run_cell, run_cell, (size_t)J * 8, cudaMemcpyHostToDevice, st));
  }
  if (active) CK(cudaMemcpyAsync(c->d_active, active, (size_t)J, cudaMemcpyHostToDevice, st));
  RoundBuf R{};
  R.J = J;
  R.T = T;
  R.maxopt = c->maxopt;
  R.depth = c->P.depth;
  R.policy = c->round_policy;
  R.tmax = c->has_tmax ? c->d_tmax : nullptr;
  R.rank = c->d_rank;
  R.pi = c->d_pi;
  R.opt = c->d_opt;
  R.score = c->d_score;
  R.opt_cell = c->d_opt_cell;
  R.nopt = c->d_nopt;
  R.ref = c->d_ref;
  R.cur = c->d_cur;
  R.decision = c->d_decision;
  R.free_io = c->d_free;
  R.total = c->d_total;
  R.stats = c->d_round_stats;
  R.ao_pk = c->d_ao_pk;
  R.ao_sc = c->d_ao_sc;
  R.nao = c->d_nao;
  R.gminb = c->d_gminb;
  R.tsb = c->d_tsb;
  R.operm = c->d_operm;
  R.opk = c->d_opk;
  R.run_cell = run_cell ? c->d_run_cell : nullptr;
  R.active = active ? c->d_active : nullptr;
  R.run_opt = c->d_run_opt;
  R.cand = c->d_cand;
  R.err = c->d_rerr;
  R.glob = c->adm_glob;
  R.ord = c->d_ord;
  R.osc = c->d_osc;
  k_round_options_warp<<<(unsigned)(((int64_t)J * 32 + 127) / 128), 128, 0, st>>>(c->P, c->C.unit_cell_begin, c->C.type, c->C.G,
                                                   (const CellResult *)d_all, R);
  CKL();
  // K6 keeps the admitted records in dynamic shared memory when its own bound
  // on their number fits (else global memory), and stages the admitted jobs'
  // options in the rest (an option pool; jobs that find no room read the global
  // table).  It gets the whole budget.
  cudaFuncAttributes fa{};
  CK(cudaFuncGetAttributes(&fa, k_round<true>));
  int optin = 0;
  CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device));
  size_t dsm = (size_t)optin - fa.sharedSizeBytes - 1024;
  if (const char *cap = getenv("CRIUS_ROUND_SMEM")) dsm = std::min<size_t>(dsm, (size_t)atoll(cap));
  R.smem_bytes = (int64_t)dsm;
  // shared-memory records when they can fit (exactly known without running jobs)
  bool smem = true;
  if (!run_cell) {
    int64_t nb = 0, lists = 0;
    for (int t = 0; t < T; ++t) nb += fr[t];
    nb = std::min<int64_t>(nb, J);
    for (int t = 0; t < T; ++t) lists += std::min<int64_t>(fr[t], nb);
    smem = nb * kRecBytes + lists * 4 <= (int64_t)dsm;
  }
  if (smem) {
    CK(cudaFuncSetAttribute(k_round<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm));
    k_round<true><<<1, kRoundThreads, dsm, st>>>(R);
  } else {
    k_round<false><<<1, kRoundThreads, 0, st>>>(R);
  }
  CKL();
  c->launches += 2;
  int32_t rerr = 0;
  CK(cudaMemcpyAsync(decision, c->d_decision, (size_t)J * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(free_after, c->d_free, T * 4, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(total_score, c->d_total, 8, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&rerr, c->d_rerr, 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (rerr == 3) {  // the records did not fit in shared memory: the global-memory kernel
    CK(cudaMemsetAsync(c->d_rerr, 0, 4, st));
    k_round<false><<<1, kRoundThreads, 0, st>>>(R);
    CKL();
    c->launches += 1;
    CK(cudaMemcpyAsync(decision, c->d_decision, (size_t)J * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(free_after, c->d_free, T * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(total_score, c->d_total, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&rerr, c->d_rerr, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  }
  if (rerr == 1) return fail(CRIUS_EINVAL, "run_cell: a running Cell's (type, G) is not one of its job's options");
  if (rerr == 2) return fail(CRIUS_EINVAL, "free + running GPUs of a type exceed 2^30");
  return CRIUS_OK;
}

crius_status crius_set_round_policy(crius_ctx *c, int32_t policy) {
  if (!c) return fail(CRIUS_EINVAL, "null ctx");
  if (policy < 0 || policy > 3) return fail(CRIUS_EINVAL, "round policy must be 0..3 (bit 0 NA, bit 1 NH)");
  c->round_policy = policy;
  return CRIUS_OK;
}

crius_status crius_set_deadline_bounds(crius_ctx *c, const int64_t *t_max, void *stream) {
  if (!c) return fail(CRIUS_EINVAL, "null ctx");
  if (!t_max) {
    c->has_tmax = false;
    return CRIUS_OK;
  }
  CK(cudaSetDevice(c->device));
  if (!c->d_tmax) CK(dalloc(&c->d_tmax, c->P.J));
  CK(cudaMemcpyAsync(c->d_tmax, t_max, (size_t)c->P.J * 8, cudaMemcpyHostToDevice,
                     (cudaStream_t)stream));
  c->has_tmax = true;
  return CRIUS_OK;
}

crius_status crius_round_stats(crius_ctx *c, int64_t *out16, void *stream) {
  CRIUS_ABI_RANGE();
  int64_t *out8 = out16;
  if (!c || !out16) return fail(CRIUS_EINVAL, "null argument");
  if (!c->d_round_stats) return fail(CRIUS_ESTATE, "no round has run");
  CK(cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  CK(cudaMemcpyAsync(out8, c->d_round_stats, 32 * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return CRIUS_OK;
}

void crius_destroy(crius_ctx *c) {
  if (!c) return;
  crius_exchange_close(c);
  cudaSetDevice(c->device);
  for (cudaEvent_t e : c->ev_chunk) cudaEventDestroy(e);
  if (c->ev_start) cudaEventDestroy(c->ev_start);
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  free_all(c);
  delete c;
}

}  // extern "C"
