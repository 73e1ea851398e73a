"""NEXT-4: multi-event trace simulation around the round.

Crius schedules on events: a job's arrival triggers
SchedArrival, a completion triggers SchedDeparture -- retry the pending jobs,
then extra scheduling of the released resources (Alg. 1).  Every
scheduling decision here is one `crius_schedule_round_state` call on the GPU
(running jobs keep their Cells unless downscaled/moved as victims or scaled up
in Phase B); this module only keeps the event clock and job states.

Event semantics (reading R-13), all integer nanoseconds:
  * a job with N iterations started on Cell c at time s finishes at
    s + penalty + N * T(c) (T = the Cell's estimated iteration time); the
    penalty is paid on every restart (Cell change), not on the first start;
  * at an event time t: completions (finish <= t) leave and free their GPUs,
    arrivals (submit <= t) join the pending set, then ONE round runs over the
    pending + running jobs;
  * a restarted job keeps the iterations completed in its segment:
    done = floor((t - s - penalty) / T(c_old)) (>= 0);
  * decision -2 (no feasible Cell) drops the job; the run ends when nothing is
    running and no arrival is left (jobs still pending then are "starved").
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

NS = 1_000_000_000
FUTURE, PENDING, RUNNING, DONE, DROPPED, STARVED = range(6)


@dataclass
class SimResult:
    first_start: np.ndarray   # int64 ns (-1 never started)
    finish: np.ndarray        # int64 ns (-1 never finished)
    restarts: np.ndarray      # int32
    state: np.ndarray         # int8 final state
    rounds: int
    events: list              # (t, n_started, n_restarted, n_finished) per round

    def summary(self, submit_ns):
        done = self.state == DONE
        jct = (self.finish[done] - submit_ns[done]) / NS
        q = (self.first_start[done] - submit_ns[done]) / NS
        return {"jobs_done": int(done.sum()), "dropped": int((self.state == DROPPED).sum()),
                "starved": int((self.state == STARVED).sum()), "rounds": self.rounds,
                "avg_jct_s": float(jct.mean()) if done.any() else None,
                "avg_queue_s": float(q.mean()) if done.any() else None,
                "makespan_s": float(self.finish[done].max() / NS) if done.any() else None,
                "avg_restarts": float(self.restarts[done].mean()) if done.any() else None}


def simulate(cr, pr, iterations, penalty_s=30, results=None, policy=0, deadlines=None,
             opportunistic=False):
    """Replay the Problem's trace through GPU rounds; `cr` is a Crius context.
    policy: the round's ablation flags (bit 0 NA: no GPU-count scaling, bit 1 NH:
    no GPU-type scaling), set for this run and reset after.
    deadlines: absolute ns per job, or None -- the deadline-aware variant
    (reading R-12): before each round a pending job that no
    Cell can finish in time is dropped, and every job's options are bounded by
    t_max = floor((D - t - penalty) / remaining) (penalty only for a running
    job, which would restart), so every placement meets its deadline.
    opportunistic: opportunistic execution (reading R-14): a
    running job is opportunistic while a job of earlier priority is pending;
    before a round, a pending job that fits nowhere directly but would fit on a
    type once the opportunistic jobs of later priority there are suspended gets
    them suspended (latest priority first, until its smallest option on that
    type fits; the type with the smallest such option, lowest index on ties).
    A suspended job keeps its completed iterations and pays the restart
    penalty when it resumes."""
    cr.set_round_policy(policy)
    try:
        return _simulate(cr, pr, iterations, penalty_s, results, deadlines, opportunistic)
    finally:
        cr.set_round_policy(0)
        cr.set_deadline_bounds(None)


def deadline_bound(D, t, pen, rem):
    """Largest iteration time that finishes `rem` iterations by D after a start
    (or restart, pen > 0) at t; -1 if none does."""
    if rem <= 0 or D - t - pen <= 0:
        return -1
    return (D - t - pen) // rem


def _suspend_for_pending(state, run, rank, opp, gmin_t, free, cells, suspend):
    """Opportunistic execution (R-14): suspend later-priority opportunistic jobs
    for each pending job, in priority order; returns the suspended jobs."""
    BIG = np.iinfo(np.int64).max
    out = []
    for p in np.argsort(rank):
        if state[p] != PENDING:
            continue
        g_row = gmin_t[p]
        if np.any((g_row < BIG) & (g_row <= free)):
            continue  # fits directly: the round places it
        best = None
        for tt in range(len(free)):
            if g_row[tt] >= BIG:
                continue
            cand = [j for j in np.where((state == RUNNING) & opp)[0]
                    if cells["type"][run[j]] == tt and rank[j] > rank[p]]
            room = int(free[tt]) + sum(int(cells["G"][run[j]]) for j in cand)
            if room >= g_row[tt] and (best is None or (int(g_row[tt]), tt) < best[:2]):
                best = (int(g_row[tt]), tt, cand)
        if best is None:
            continue
        g, tt, cand = best
        for v in sorted(cand, key=lambda j: -rank[j]):
            if free[tt] >= g:
                break
            free[tt] += int(cells["G"][run[v]])
            suspend(v)
            out.append(v)
    return out


def _simulate(cr, pr, iterations, penalty_s, results, deadlines, opportunistic):
    J = pr.n_jobs
    if cr.n_cells is None:
        cr.enumerate()
    if results is None:
        results = cr.estimate()
    cells = {k: v.cpu().numpy() for k, v in cr.cells().items() if k in ("job", "type", "G")}
    t_cell = results[:cr.n_cells, 0].cpu().numpy()
    INF = np.iinfo(np.int64).max
    t_best = np.full(J, INF, np.int64)  # fastest feasible Cell per job (early drop)
    np.minimum.at(t_best, cells["job"], t_cell)
    submit = np.asarray(pr.submit, np.int64) * NS
    iters = np.asarray(iterations, np.int64)
    pen = int(penalty_s) * NS
    state = np.full(J, FUTURE, np.int8)
    run = np.full(J, -1, np.int64)
    remaining = iters.copy()
    seg_start = np.zeros(J, np.int64)
    seg_pen = np.zeros(J, np.int64)
    finish = np.full(J, -1, np.int64)
    first = np.full(J, -1, np.int64)
    restarts = np.zeros(J, np.int32)
    events = []
    # priority (submit, id) and, per job and type, its smallest option G (<= N_G)
    rank = np.empty(J, np.int64)
    rank[np.lexsort((np.asarray(pr.job_id), np.asarray(pr.submit)))] = np.arange(J)
    opp = np.zeros(J, bool)
    resumed = np.zeros(J, bool)
    gmin_t = np.full((J, pr.n_types), INF, np.int64)
    okc = (t_cell != INF) & (cells["G"] <= np.asarray(pr.ng)[cells["job"]])
    np.minimum.at(gmin_t, (cells["job"][okc], cells["type"][okc]), cells["G"][okc])

    def suspend(v):
        ran = t - seg_start[v] - seg_pen[v]
        done_it = ran // int(t_cell[run[v]]) if ran > 0 else 0
        remaining[v] -= min(done_it, remaining[v])
        state[v], run[v], opp[v], resumed[v] = PENDING, -1, False, True

    order = np.argsort(submit, kind="stable")
    nxt = 0
    t = 0
    while True:
        running = np.where(state == RUNNING)[0]
        t_fin = finish[running].min() if running.size else None
        t_arr = submit[order[nxt]] if nxt < J else None
        if t_fin is None and t_arr is None:
            break
        t = min(x for x in (t_fin, t_arr) if x is not None)
        ended = running[finish[running] <= t]
        state[ended] = DONE
        run[ended] = -1
        while nxt < J and submit[order[nxt]] <= t:
            state[order[nxt]] = PENDING
            nxt += 1
        if opportunistic:
            used = np.zeros(pr.n_types, np.int64)
            for j in np.where(state == RUNNING)[0]:
                used[cells["type"][run[j]]] += cells["G"][run[j]]
            _suspend_for_pending(state, run, rank, opp, gmin_t,
                                 np.asarray(pr.cap, np.int64) - used, cells, suspend)
        if deadlines is not None:
            tmax = np.full(J, -1, np.int64)
            for j in np.where((state == PENDING) | (state == RUNNING))[0]:
                if state[j] == RUNNING:
                    ran = t - seg_start[j] - seg_pen[j]
                    done_it = ran // int(t_cell[run[j]]) if ran > 0 else 0
                    tmax[j] = deadline_bound(int(deadlines[j]), int(t), pen,
                                             int(remaining[j]) - min(done_it, int(remaining[j])))
                else:
                    tmax[j] = deadline_bound(int(deadlines[j]), int(t), pen if resumed[j] else 0,
                                             int(remaining[j]))
                    if t_best[j] > tmax[j]:
                        state[j] = DROPPED  # early drop: no Cell finishes in time
            cr.set_deadline_bounds(tmax)
        active = ((state == PENDING) | (state == RUNNING)).astype(np.uint8)
        used = np.zeros(pr.n_types, np.int64)
        for j in np.where(state == RUNNING)[0]:
            used[cells["type"][run[j]]] += cells["G"][run[j]]
        free = (np.asarray(pr.cap, np.int64) - used).astype(np.int32)
        dec, _, _ = cr.schedule_round_state(results, free, run_cell=run, active=active)
        n_start = n_restart = 0
        for j in np.where(active == 1)[0]:
            d = int(dec[j])
            if d == -2:
                state[j] = DROPPED
            elif d >= 0:
                if state[j] == PENDING:
                    p0 = pen if resumed[j] else 0  # a suspended job resumes with a restart
                    state[j] = RUNNING
                    run[j], seg_start[j], seg_pen[j] = d, t, p0
                    if first[j] < 0:
                        first[j] = t
                    finish[j] = t + p0 + int(remaining[j]) * int(t_cell[d])
                    if resumed[j]:
                        restarts[j] += 1
                        resumed[j] = False
                    n_start += 1
                elif d != run[j]:
                    ran = t - seg_start[j] - seg_pen[j]
                    done_it = max(0, ran // int(t_cell[run[j]])) if ran > 0 else 0
                    remaining[j] -= min(done_it, remaining[j])
                    run[j], seg_start[j], seg_pen[j] = d, t, pen
                    finish[j] = t + pen + int(remaining[j]) * int(t_cell[d])
                    restarts[j] += 1
                    n_restart += 1
        if opportunistic:  # opportunistic = running while an earlier job waits
            pend = np.where(state == PENDING)[0]
            first_wait = rank[pend].min() if pend.size else J
            opp[:] = (state == RUNNING) & (rank > first_wait)
        events.append((int(t), n_start, n_restart, int(ended.size)))
    state[state == PENDING] = STARVED
    return SimResult(first, finish, restarts, state, len(events), events)
