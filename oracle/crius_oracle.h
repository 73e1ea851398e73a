/* crius_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, single-threaded CPU oracle of the Crius Cell-estimation hot
 * path (arXiv 2403.16125) as fixed by SURVEY.md §8(c) and §N0-§N6.  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference arm
 * may load it.  It shares no code, header, table or helper with the CUDA
 * library (paper_2403_16125_b200/csrc, include/crius.h).
 *
 * All integers are fixed width; every array is caller-owned and read only.
 * Return codes: 0 ok, 2 bad argument, 7 arithmetic bound exceeded.
 */
#ifndef CRIUS_ORACLE_H
#define CRIUS_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  /* GPU types (Table sim_cluster) */
  int32_t n_types;
  const int32_t *cap, *gpn;
  const int64_t *mem, *alpha_in, *beta_in, *alpha_x, *beta_x; /* ns, ns per MiB */
  /* jobs (N_G given by the user) */
  int32_t n_jobs, k_max;
  const int64_t *job_id, *submit;
  const int32_t *ng, *gb, *kst, *n_layers;
  const int64_t *layer_off;           /* [n_jobs+1] */
  const int32_t *c;                   /* [n_types][k_max+1][total_layers] */
  const int64_t *w, *act, *bnd, *tpv; /* [total_layers] */
  const int32_t *tpn;                 /* [total_layers] */
  /* config */
  int32_t gpu_set, s_max, g_max, b_mode, b_count;
  const int32_t *b_values;
  int32_t depth;
} oracle_problem;

/* Π6 helpers: kind 0 = AR(p, V, n), 1 = AG(p, V), 2 = P2P(V). */
int64_t oracle_comm(int32_t kind, int64_t p, int64_t alpha, int64_t beta, int64_t V, int64_t n);

/* O1: count, then list the Cells in §N2 order. */
int oracle_count(const oracle_problem *pr, int64_t *n_cells, int64_t *n_plans);
int oracle_enumerate(const oracle_problem *pr, int32_t *cell_job, int32_t *cell_type,
                     int32_t *cell_G, int32_t *cell_S, int32_t *cell_nplans);

/* O2: R0 min-max split of job j on type t into S stages; bounds[0..S]. */
int oracle_split(const oracle_problem *pr, int32_t j, int32_t t, int32_t S, int32_t *bounds);

/* O3 for one plan: per-stage T, sync, mem (arrays of length S), T_iter.
 * *feasible = 0 when B*dp > GB or some mem > mem_t (T_iter then undefined). */
int oracle_plan_cost(const oracle_problem *pr, int32_t j, int32_t t, int32_t G, int32_t S,
                     int32_t p, int64_t *T_stage, int64_t *sync_stage, int64_t *mem_stage,
                     int64_t *t_iter, int32_t *feasible);

/* O3+O4 for Cells [c0, c1) of the enumerated list: best (t_ns, plan) per Cell;
 * plan = -1, t_ns = INT64_MAX if no plan is feasible. */
int oracle_estimate(const oracle_problem *pr, const int32_t *cell_job, const int32_t *cell_type,
                    const int32_t *cell_G, const int32_t *cell_S, const int32_t *cell_nplans,
                    int64_t c0, int64_t c1, int64_t *t_ns, int32_t *plan);

/* NEXT-1: per-stage parallelism assembly.  mode 1 = each
 * stage DP-only or TP-only (the paper's 2^S assembled plans),
 * mode 2 = every DP x TP factorisation per stage; form 0 = sum + (B-1) max,
 * form 1 = sum + (B-1)(T_s* - T_comm,s*).  Brute force over
 * every assembled plan and microbatch count.  stage_k: [c1-c0][kstride]. */
int oracle_estimate_assembled(const oracle_problem *pr, int32_t mode, int32_t form,
                              const int32_t *cell_job, const int32_t *cell_type,
                              const int32_t *cell_G, const int32_t *cell_S, int64_t c0,
                              int64_t c1, int64_t *t_ns, int32_t *bidx, int8_t *stage_k,
                              int32_t kstride);
int oracle_assembled_cost(const oracle_problem *pr, int32_t form, int32_t j, int32_t t, int32_t G,
                          int32_t S, int32_t bi, const int8_t *stage_k, int64_t *latency,
                          int32_t *feasible);

/* NEXT-3: Cell-guided tuning.  Choices of a
 * stage of g GPUs under its favour (ks[] receives them, returns the count), and
 * the brute-force best plan over the pruned product given each Cell's favour
 * row (log2 tp of the estimated plan per stage, > 0 = tensor-parallel favour). */
int oracle_tune_choices(int32_t g, int32_t tp_favour, int32_t *ks);
int oracle_tune_assembled(const oracle_problem *pr, int32_t form, const int32_t *cell_job,
                          const int32_t *cell_type, const int32_t *cell_G, const int32_t *cell_S,
                          int64_t c0, int64_t c1, const int8_t *favor, int32_t kstride,
                          int64_t *t_ns, int32_t *bidx, int8_t *stage_k);

/* NEXT-2: the paper's stage determination:
 * cuts at the S-1 smallest boundary bytes (ties: min-max tp=1 compute, R0),
 * FLOP-proportional GPUs per stage rounded to powers of two with conservation
 * repair, plans with uniform tp and per-stage dp (R-8..R-10). */
int oracle_paper_stages(const oracle_problem *pr, int32_t j, int32_t t, int32_t G, int32_t S,
                        int32_t *bounds, int32_t *g);
int32_t oracle_paper_round_pow2(int64_t num, int64_t den);
int oracle_paper_fractional(const oracle_problem *pr, int32_t j, int32_t t, int32_t G, int32_t S,
                            const int32_t *bounds, int64_t *num, int64_t *den);
int oracle_paper_plan_cost(const oracle_problem *pr, int32_t j, int32_t t, int32_t S,
                           const int32_t *bounds, const int32_t *g, int32_t p, int64_t *t_iter,
                           int32_t *feasible);
int oracle_estimate_paper(const oracle_problem *pr, const int32_t *cell_job,
                          const int32_t *cell_type, const int32_t *cell_G, const int32_t *cell_S,
                          int64_t c0, int64_t c1, int64_t *t_ns, int32_t *plan, int8_t *stage_lg,
                          int32_t kstride);

/* O5: the §N6 round over all Cells.  free_in may be NULL (= capacity).
 * decision[j] = Cell id | -1 pending | -2 unschedulable. */
int oracle_round(const oracle_problem *pr, int64_t n_cells, const int32_t *cell_job,
                 const int32_t *cell_type, const int32_t *cell_G, const int32_t *cell_S,
                 const int64_t *t_ns, const int32_t *free_in, int64_t *decision,
                 int32_t *free_after, double *total_score);

/* NEXT-4: the round from a cluster state (running jobs start admitted on
 * the option of their Cell's (type, G); inactive jobs get decision -3). */
/* NEXT-4 ablations: as oracle_round_state with policy bit 0 = NA (options only
 * at G = N_G), bit 1 = NH (admitted jobs keep their GPU type); t_max (per job
 * or NULL): deadline bound on an option's T (a running job's (type, G) exempt). */
int oracle_round_policy(const oracle_problem *pr, int64_t n_cells, const int32_t *cell_job,
                        const int32_t *cell_type, const int32_t *cell_G, const int32_t *cell_S,
                        const int64_t *t_ns, const int32_t *free_in, const int64_t *run_cell,
                        const uint8_t *active, int32_t policy, const int64_t *t_max,
                        int64_t *decision, int32_t *free_after, double *total_score);
int oracle_round_state(const oracle_problem *pr, int64_t n_cells, const int32_t *cell_job,
                       const int32_t *cell_type, const int32_t *cell_G, const int32_t *cell_S,
                       const int64_t *t_ns, const int32_t *free_in, const int64_t *run_cell,
                       const uint8_t *active, int64_t *decision, int32_t *free_after,
                       double *total_score);

#ifdef __cplusplus
}
#endif
#endif
