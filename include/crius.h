/* crius.h -- C-ABI of libcrius, the B200-native Crius Cell estimator.
 *
 * Crius (arXiv 2403.16125, /root/reference/PAPER.md, cited P:<line>) shards a
 * cluster's scheduling space into Cells: a job with a fixed GPU type, GPU
 * count and pipeline-stage count ("Cell"), estimates every Cell
 * ("Agile Cell Estimation") and schedules jobs on Cells (Alg. 1,
 * P:432-464).  This library computes that hot path on one GPU:
 *
 *   crius_load_profiles    profiles -> device (decoupled compute/comm)
 *   crius_enumerate_cells  Cells of every job
 *   crius_estimate_cells   stage split (P:266-283 read as a min-max DP, §N3),
 *                          every DP x TP x microbatch plan (§N5),
 *                          best plan per Cell
 *   crius_schedule_round   one scheduling round (Alg. 1)
 *
 * The normative formulas are SURVEY.md §N0-§N6 (part of the contract), the
 * readings of the paper are listed in DESIGN.md.  Everything here is plain C:
 * fixed-width integers, host or device pointers, sizes.  Streams are passed as
 * `void *` holding a cudaStream_t (NULL = legacy default stream).
 *
 * Arithmetic.  Every decision-path quantity is an integer: int64 ns, int64
 * bytes, alpha in ns, beta in ns per MiB (2^20 B).  Every degree (G, S, g, tp,
 * dp, B, GB, cap, gpn, g_max) is a power of two.  fp64 appears only in the
 * round's scores (IEEE, no FMA contraction).  Results are bit-reproducible
 * and independent of the number of GPUs the Cell space is sharded over.
 *
 * Errors.  Every call returns a crius_status; crius_last_error() gives a
 * thread-local message for the last failing call.  A Cell with no feasible
 * plan is data (plan = -1, t_ns = INT64_MAX), not an error.  Asynchronous
 * CUDA faults surface as CRIUS_ECUDA at the next synchronising call.
 *
 * Threads.  One context per device; calls on one context are not thread-safe.
 */
#ifndef CRIUS_H
#define CRIUS_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct crius_ctx crius_ctx; /* opaque, owned by the library */

typedef enum {
  CRIUS_OK = 0,
  CRIUS_EINVAL = 2,      /* bad argument, non-power-of-two degree, bound violated */
  CRIUS_EINFEASIBLE = 3, /* the enumeration produced zero Cells */
  CRIUS_ECUDA = 4,       /* CUDA runtime error (message has the CUDA string) */
  CRIUS_ENOMEM = 5,      /* device allocation failed */
  CRIUS_ESTATE = 6       /* call out of order (e.g. estimate before enumerate) */
} crius_status;

/* GPU types (Table sim_cluster).  Host pointers, read during the
 * call only.  capacity and gpus_per_node are powers of two (A-19, A-20). */
typedef struct {
  int32_t n_types;                 /* 1..8 (the round's shared-memory tables) */
  const int32_t *capacity;         /* [n_types] GPUs of this type in the cluster */
  const int32_t *gpus_per_node;    /* [n_types] node size: link class boundary (A-15) */
  const int64_t *mem_bytes;        /* [n_types] per-GPU memory (memory filter) */
  const int64_t *alpha_intra_ns;   /* [n_types] alpha-beta of the intra-node link (D3) */
  const int64_t *beta_intra_ns_per_mib;
  const int64_t *alpha_inter_ns;   /* [n_types] inter-node link */
  const int64_t *beta_inter_ns_per_mib;
} crius_cluster;

/* Jobs and their profiles (decoupled computation/communication).
 * Host pointers, read during the call only. */
typedef struct {
  int32_t n_jobs;                  /* 1 .. 2^24 - 1 (the round's tie keys hold a
                                      priority position in 24 bits) */
  int32_t k_max;                   /* compute profiled for tp = 2^0 .. 2^k_max, k_max <= 6 */
  const int64_t *job_id;           /* [n_jobs] unique; priority = (submit, id) ascending (A-18) */
  const int64_t *submit_time;      /* [n_jobs] */
  const int32_t *n_gpus_req;       /* [n_jobs] N_G given by the user, power of two */
  const int32_t *global_batch;     /* [n_jobs] GB, power of two */
  const int32_t *k_state;          /* [n_jobs] bytes of state per param byte (A-13), >= 1 */
  const int32_t *n_layers;         /* [n_jobs] L >= 1 (operator chain) */
  const int64_t *layer_off;        /* [n_jobs+1] exclusive prefix of n_layers */
  const int32_t *compute_ns;       /* [n_types][k_max+1][total_layers] ns per sample, fwd+bwd,
                                      at tp = 2^k; every entry >= 1 */
  const int64_t *param_bytes;      /* [total_layers] w */
  const int64_t *act_bytes;        /* [total_layers] stored activation bytes per sample */
  const int64_t *boundary_bytes;   /* [total_layers] bytes per sample sent to the next stage */
  const int64_t *tp_bytes;         /* [total_layers] TP all-reduce bytes per sample */
  const int32_t *tp_calls;         /* [total_layers] TP all-reduce calls per microbatch */
} crius_jobs;

typedef struct {
  int32_t gpu_set;     /* 0 = paper {N_G/2, N_G, 2N_G}; 1 = all powers of two <= capacity */
  int32_t s_max;       /* stage-count cap (S in {1,2,4,..} <= min(G, L, s_max), A-6) */
  int32_t g_max;       /* per-stage GPU cap: G/S <= g_max <= 2^k_max */
  int32_t b_mode;      /* 0 = B = 4*S microbatches (GPipe); 1 = the list below */
  int32_t b_count;     /* b_mode 1: 1..16 ascending powers of two */
  const int32_t *b_values;
  int32_t search_depth; /* d in [0, 16]: victim moves per trial and reverse-scaling sweeps
                           (default 3 at P:737; A-17) */
} crius_config;

/* One per Cell, 16 bytes.  t_ns = best T_iter (int64 ns) or INT64_MAX;
 * plan = p = k*nB + b (tp = 2^k, B = Bset[b]) or -1; flags bit 0 = feasible.
 * The estimate in seconds is (double)t_ns / 1e9. */
typedef struct {
  int64_t t_ns;
  int32_t plan;
  int32_t flags;
} crius_cell_result;

/* Read-only DEVICE view of the Cell table (SoA, §N2 order: job, type, G asc,
 * S asc).  Cell ids are positions in this order.  Valid until crius_destroy. */
typedef struct {
  int64_t n_cells, n_cell_plans, n_units; /* unit = (job, type) = j*n_types + t */
  const int32_t *job, *type, *G, *S, *nplans;   /* [n_cells] */
  const int64_t *plan_off;                      /* [n_cells] global plan offset */
  const int64_t *unit_cell_begin;               /* [n_units+1] */
  const int64_t *unit_plan_begin;               /* [n_units+1] */
} crius_cell_view;

/* Validate inputs (SURVEY §N0 bounds: L*max(c)*GB < 2^52, every T_iter < 2^62,
 * kst*sum(w) + GB*sum(act) < 2^62, ...), copy them H2D into library-owned
 * SoA buffers on `device` (enqueued on `stream`, synchronised before return),
 * and compute the round's priority order.  On success *out owns the context.
 * EINVAL names the first violated rule. */
crius_status crius_load_profiles(crius_ctx **out, const crius_cluster *cluster,
                                 const crius_jobs *jobs, const crius_config *config,
                                 int32_t device, void *stream);

/* Re-copy new profile VALUES of the same shape (same n_types, n_jobs,
 * n_layers, k_max, config) into the existing buffers; validates like load.
 * Invalidates previous enumeration/estimates (call enumerate again). */
crius_status crius_update_profiles(crius_ctx *ctx, const crius_cluster *cluster,
                                   const crius_jobs *jobs, void *stream);

/* As crius_update_profiles, but the per-layer rows (compute_ns of every
 * (type, k) plane, param/act/boundary/tp bytes, tp_calls) are copied and
 * bound-checked only for jobs [job_begin, job_end); the per-job arrays and
 * the cluster parameters are copied for every job.  A rank of a sharded run
 * ("each rank needs H2D only for its jobs' profile rows") uploads
 * the jobs of its unit range (crius_partition_units, units = (job, type) in job
 * order) and must then estimate only Cells of those jobs; rows of the other
 * jobs keep whatever values they had.  [0, n_jobs) == crius_update_profiles.
 * EINVAL on a range outside [0, n_jobs]. */
crius_status crius_update_profiles_range(crius_ctx *ctx, const crius_cluster *cluster,
                                         const crius_jobs *jobs, int32_t job_begin,
                                         int32_t job_end, void *stream);

/* Enumerate every Cell (§N2) on the device: per-unit counts, scan,
 * fill.  Synchronises `stream` once, for the counts it returns; the fill of the
 * Cell table is then queued on `stream` (work queued after it on `stream`, or
 * anything after a synchronisation of `stream`, sees the complete table).
 * EINFEASIBLE if 0 Cells. */
crius_status crius_enumerate_cells(crius_ctx *ctx, int64_t *n_cells, int64_t *n_cell_plans,
                                   int64_t *n_units, void *stream);

/* Device view of the Cell table (after enumerate). */
crius_status crius_cells(crius_ctx *ctx, crius_cell_view *view);

/* int16 entries per unit in the optional d_splits output of estimate; the
 * split of S = 2^si for unit u is at (u - unit_begin)*stride + (2^si - 1) + si,
 * S+1 boundaries b_0=0 < b_1 < .. < b_S = L (stage s covers layers [b_s, b_{s+1}));
 * entries of S values the unit does not use are -1. */
int32_t crius_split_stride(const crius_ctx *ctx);

/* Contiguous unit ranges for `world` ranks, balanced by per-unit work weight
 * (SURVEY §8(e)); host outputs unit_begin[world+1], cell_begin[world+1].
 * Synchronous (small D2H). */
crius_status crius_partition_units(crius_ctx *ctx, int32_t world, int64_t *unit_begin,
                                   int64_t *cell_begin, void *stream);

/* Estimate every Cell of units [unit_begin, unit_end): one fused kernel does
 * the per-unit prefix staging, the min-max stage DP with the lowest-argmin tie
 * rule R0 (A-4), the cost of every plan (§N5) and the per-Cell argmin (lowest
 * plan index wins ties, A-10).  d_out (caller-owned DEVICE buffer) receives one
 * record per Cell: d_out[i] = Cell (unit_cell_begin[unit_begin] + i).
 * d_splits (optional DEVICE int16 buffer or NULL) receives the splits.
 * Asynchronous on `stream`. */
crius_status crius_estimate_cells(crius_ctx *ctx, int64_t unit_begin, int64_t unit_end,
                                  crius_cell_result *d_out, int16_t *d_splits, void *stream);

/* One call per new batch of profiles (the same shapes as loaded): the effect of
 * crius_update_profiles + crius_enumerate_cells + crius_estimate_cells over
 * every unit, with the per-layer row upload (the bulk of the input bytes)
 * pipelined against the work that needs it.  The per-job arrays go up on
 * `stream` and the Cells are enumerated from them while the rows go up in
 * n_chunks (1..64) job ranges of equal layer count on a stream of the context;
 * each range's rows are bound-checked and its units estimated on `stream` as
 * soon as they are resident.  Host arrays as crius_update_profiles (pinned host
 * memory lets the copies overlap; pageable memory still works, without
 * overlap).  d_out: caller-owned DEVICE buffer of out_capacity records; record
 * of Cell i at d_out[i] (GLOBAL Cell order); d_splits (optional DEVICE buffer
 * of n_units * crius_split_stride entries) at unit u's row u * stride.
 * Synchronises `stream`; returns the counts as crius_enumerate_cells (also on
 * failure once enumerated).  EINVAL as crius_update_profiles (the records are
 * then not valid and the context needs a new enumeration) or when n_cells >
 * out_capacity (nothing estimated: grow d_out to the returned n_cells and call
 * again); EINFEASIBLE if 0 Cells.  The default single-GPU estimator only. */
crius_status crius_update_estimate(crius_ctx *ctx, const crius_cluster *cluster,
                                   const crius_jobs *jobs, int32_t n_chunks,
                                   crius_cell_result *d_out, int64_t out_capacity,
                                   int16_t *d_splits, int64_t *n_cells, int64_t *n_cell_plans,
                                   int64_t *n_units, void *stream);

/* NEXT-1: per-stage parallelism assembly -- the paper's own
 * sampling, where each stage picks its parallelism independently ("assemble
 * 2^{N_S} distinct parallelism plans") -- with either pipeline
 * latency form.  Same Cells, splits and B set as crius_estimate_cells. */
typedef struct {
  int32_t mode;          /* 1 = each stage DP-only or TP-only (2^S plans);
                            2 = every DP x TP factorisation per stage */
  int32_t pipeline_form; /* 0 = sum + (B-1) max T (north_star);
                            1 = sum + (B-1)(T_s* - T_comm,s*), s* = first slowest stage,
                                T_comm its inbound communication */
} crius_assembly;

/* Exact best assembled plan of every Cell of units [unit_begin, unit_end)
 * (no enumeration of the 2^S / K^S plans: threshold search over the slowest
 * stage and the sync bound).  d_out[i]: t_ns = best latency, plan = index of
 * the best microbatch count (B = 4S: 0), flags bit 0 = feasible.  d_stage_tp
 * (optional DEVICE int8 buffer): per Cell crius_split_stride-independent row of
 * max_S entries = log2 tp of each stage in one optimal plan, -1 padding
 * (several plans can be optimal; any returned one attains t_ns).  max_S is the
 * largest S of the enumeration (crius_max_stages).  Asynchronous. */
crius_status crius_estimate_assembled(crius_ctx *ctx, const crius_assembly *assembly,
                                      int64_t unit_begin, int64_t unit_end,
                                      crius_cell_result *d_out, int8_t *d_stage_tp, void *stream);

/* NEXT-3: Cell-guided parallelism tuning.  Each
 * stage's parallelism in the estimated plan is its favour; the stage is tuned
 * only within its half of the factorisation axis -- DP favour: dp-only ..
 * half-hybrid (k <= ceil(log2 g / 2)), TP favour: half-hybrid .. tp-only
 * (k >= floor(log2 g / 2)); half-hybrid = sqrt(g) replicas x sqrt(g) tensor
 * shards (Fig. pruning); for odd log2 g both neighbouring
 * factorisations belong to both halves (matches SPEC.md's g=8 and g=16 examples).  The best plan of the pruned product (every B of the set) is
 * returned like crius_estimate_assembled.  d_favor (DEVICE int8, same layout as
 * d_stage_tp): log2 tp of each stage of the estimated plan; a stage favours TP
 * iff its entry is > 0.  Asynchronous. */
crius_status crius_tune_assembled(crius_ctx *ctx, int32_t pipeline_form, int64_t unit_begin,
                                  int64_t unit_end, const int8_t *d_favor,
                                  crius_cell_result *d_out, int8_t *d_stage_tp, void *stream);

/* NEXT-2: the paper's stage determination (PAPER.md:266-283,
 * "Stage determination of a Cell"), readings R-8..R-10 of DESIGN.md §13.
 * Per (job, type, S) the model is cut at the S-1 inter-layer gaps with the
 * smallest boundary bytes; gaps tied at the (S-1)-th smallest byte
 * count are chosen by the min-max of the tp=1 compute with the R0 rule.
 * Per Cell, stage s gets G * F_s / F GPUs (F = tp=1 compute, the FLOP proxy;
 * "T_elapsed = FLOPs / Number_GPU") rounded to the nearest power of
 * two (ties up, >= 1) with a conservation repair to sum G.  Plans
 * p = k * nB + b run tp = 2^k in every stage (k <= log2 min g_s) and
 * dp_s = g_s / tp; GPUs are packed from a node boundary in stage order, which
 * fixes the intra/inter link of every term.  A Cell with a stage above g_max
 * is infeasible.  d_out[i] as crius_estimate_cells (t_ns, plan = p, flags);
 * d_splits (optional DEVICE int16) receives the cuts in the split layout;
 * d_stage_lg (optional DEVICE int8, rows of crius_max_stages entries) receives
 * log2 g_s per stage, -1 padding.  Asynchronous on `stream`. */
crius_status crius_estimate_paper_stages(crius_ctx *ctx, int64_t unit_begin, int64_t unit_end,
                                         crius_cell_result *d_out, int16_t *d_splits,
                                         int8_t *d_stage_lg, void *stream);

/* Largest stage count S of the enumerated Cells (row length of d_stage_tp). */
int32_t crius_max_stages(const crius_ctx *ctx);

/* Undo per-rank padding after an all-gather: d_gathered holds `world` chunks of
 * `chunk_stride` records, chunk r = Cells [cell_begin[r], cell_begin[r+1]) (host
 * array from crius_partition_units); writes d_all[n_cells].  Asynchronous. */
crius_status crius_compact_gathered(crius_ctx *ctx, const crius_cell_result *d_gathered,
                                    int64_t chunk_stride, int32_t world,
                                    const int64_t *cell_begin, crius_cell_result *d_all,
                                    void *stream);

/* Fused exchange: the all-gather of A7 done by the estimate kernel itself over
 * NVLink / NVSwitch peer memory ("fused-collective option": the
 * north_star exchange -- every rank gets every Cell's best plan before the
 * round -- without a separate collective or compaction).  One process per GPU,
 * all on one node, world <= 8.  Sequence per rank:
 *   crius_exchange_init  -> 64-byte CUDA IPC handle of this rank's window
 *   (the caller all-gathers the handles, e.g. over the process group)
 *   crius_exchange_open  with every rank's handle (rank order)
 *   per step: crius_estimate_exchange(this rank's unit range)
 *             crius_exchange_wait -> device pointer to all n_cells records
 *             crius_schedule_round(that pointer)
 * Every rank must call crius_estimate_exchange once per step (also with an
 * empty range) or the others' waits never complete (they trap after 30 s).
 * Window (library-owned device memory): arrival flags int64[8] (256 B) +
 * 2 x capacity_cells records, used alternately by step parity, so a fast rank's
 * next step never overwrites records a slow rank's round is still reading. */

/* Allocate this rank's window for up to capacity_cells Cells and write its
 * CUDA IPC handle (64 bytes) to handle_out (HOST).  Synchronous.
 * EINVAL: world not in 1..8, rank not in [0, world); ESTATE: already initialised. */
crius_status crius_exchange_init(crius_ctx *ctx, int32_t rank, int32_t world,
                                 int64_t capacity_cells, uint8_t *handle_out);

/* Map every other rank's window: handles (HOST) = world x 64 bytes, rank order
 * (this rank's own entry is ignored).  Synchronous.  ECUDA if a handle cannot
 * be opened (e.g. the GPUs are not peers). */
crius_status crius_exchange_open(crius_ctx *ctx, const uint8_t *handles);

/* As crius_estimate_cells for units [unit_begin, unit_end), but each Cell's
 * record is stored at its GLOBAL Cell index into every rank's window (16-byte
 * P2P stores from the kernel's epilogue); the kernel's last CTA then
 * release-stores the step number into every rank's arrival flag for this rank.
 * Asynchronous on `stream`.  EINVAL if n_cells exceeds capacity_cells. */
crius_status crius_estimate_exchange(crius_ctx *ctx, int64_t unit_begin, int64_t unit_end,
                                     void *stream);

/* Enqueue on `stream` a wait until every rank's flag for this step has arrived;
 * *d_all = this rank's window half of the step (DEVICE, n_cells records in
 * global Cell order, valid until the step after next).  Asynchronous. */
crius_status crius_exchange_wait(crius_ctx *ctx, crius_cell_result **d_all, void *stream);

/* Unmap the peers' windows and free this rank's (also done by crius_destroy).
 * Synchronises the device. */
crius_status crius_exchange_close(crius_ctx *ctx);

/* One scheduling round (§N6: Phase A SchedArrival P:436-445 with ScaleResource
 * P:491-497 at search depth d, Phase B extra scheduling / reverse scaling
 * P:449-450) over all Cells, on the device.  d_all: DEVICE results of
 * every Cell.  free_gpus: HOST [n_types] or NULL (= capacity).  Outputs (HOST):
 * decision[n_jobs] = Cell id | -1 pending | -2 unschedulable; free_after[n_types];
 * *total_score = sum of normalised throughputs (A-16) in priority order.
 * Synchronises `stream`. */
crius_status crius_schedule_round(crius_ctx *ctx, const crius_cell_result *d_all,
                                  const int32_t *free_gpus, int64_t *decision,
                                  int32_t *free_after, double *total_score, void *stream);

/* NEXT-4: one round from a cluster state, for multi-event
 * simulation (Alg. 1: SchedArrival P:436-445 and SchedDeparture = retry the
 * pending jobs then extra scheduling).  run_cell (HOST int64
 * [n_jobs] or NULL): Cell a job currently runs on (-1 = not running); running
 * jobs start admitted on the option of that Cell's (type, G), may be moved as
 * victims or reverse-scaled, never evicted.  active (HOST uint8 [n_jobs] or
 * NULL = all): jobs that take part (arrived, not finished); inactive jobs get
 * decision -3.  free_gpus = free counts with the running jobs' GPUs taken.
 * Ties between victims go to the earlier job in (submit, id) order.
 * crius_schedule_round(..) == this call with run_cell = active = NULL. */
crius_status crius_schedule_round_state(crius_ctx *ctx, const crius_cell_result *d_all,
                                        const int32_t *free_gpus, const int64_t *run_cell,
                                        const uint8_t *active, int64_t *decision,
                                        int32_t *free_after, double *total_score, void *stream);

/* NEXT-4 ablations of the round (Fig. `ablation`; reading
 * R-11 in DESIGN.md): policy bit 0 = NA, no adaptivity scaling -- every job's
 * options are restricted to G = N_G, so no GPU count ever changes; bit 1 = NH,
 * no heterogeneity scaling -- an admitted job never changes its GPU type (no
 * other-type victim move in ScaleResource, Phase B only within the type; a
 * job's first placement may use any type).  0 = the full round (default).
 * Applies to every later crius_schedule_round(_state) call of this context.
 * EINVAL unless 0 <= policy <= 3. */
crius_status crius_set_round_policy(crius_ctx *ctx, int32_t policy);

/* Deadline-aware rounds ("strict deadline guarantees for
 * each scheduled job"; reading R-12 in DESIGN.md).  t_max (HOST int64
 * [n_jobs], read during the call; NULL = no deadlines): per job, the largest
 * iteration time an option may have (the caller derives it from the deadline,
 * the remaining iterations and any restart penalty); a Cell with T > t_max[j]
 * is not an option of job j, except the (type, G) a running job uses.  Applies
 * to every later round of this context until reset with NULL.  Asynchronous
 * upload on `stream`. */
crius_status crius_set_deadline_bounds(crius_ctx *ctx, const int64_t *t_max, void *stream);

/* Counters of the last round (HOST int64 out[32]): [0] Phase A iterations
 * (batches), [1] victim-sequence recomputations, [2] SM cycles in them, [3] SM
 * cycles of Phase A, [4] SM cycles of Phase B, [5] admitted jobs, [6]
 * admissions through ScaleResource, [7] Phase B batches, [8..10] SM cycles of
 * the Phase A batches (direct evaluation; sequences + ScaleResource
 * evaluation; commit), [11] stale same-type move caches refreshed, [12]
 * other-type move evaluations, [13] per-type sequence invalidations, [14] 1 if
 * the admitted records lived in shared memory, [15] the round's bound on the
 * number of admitted records, [16..18] SM cycles of the per-type sequence
 * computations summed over types (preparation, moves, thresholds), [19]
 * candidate rescans, [20] type-list entries scanned, [21] top-list refills,
 * [22] per-type sequence computations, [23] SM cycles of their top-list and
 * cache refresh, [25] stale types summed over the recomputations, [28]
 * CTA-wide barriers on the round's critical chain.
 * Other entries are reserved (0).  Synchronises `stream`. */
crius_status crius_round_stats(crius_ctx *ctx, int64_t *out16, void *stream);

/* Number of kernels this context has launched so far (for launch accounting). */
int64_t crius_kernel_launches(const crius_ctx *ctx);

const char *crius_last_error(void);
void crius_destroy(crius_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* CRIUS_H */
