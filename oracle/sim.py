"""Oracle trace simulator for NEXT-4 -- TEST INFRASTRUCTURE ONLY.

A plain, literal event loop over the oracle's round (oracle_round_state),
written independently of paper_2403_16125_b200/sim.py; the two share no code.
Semantics (reading R-13), integer nanoseconds:
  - first start on Cell c at time s: finish = s + N * T(c)      (N iterations)
  - restart (Cell change) at time t: the segment's completed iterations
    floor((t - s - pen_seg) / T(c_old)) are kept; finish = t + P + N' * T(c_new)
  - at each event time: completions leave, arrivals join, one round runs
    over pending + running jobs; -2 drops a job; leftover pending = starved.
"""
import numpy as np

NS = 10 ** 9


def simulate(o, cells, t_ns, iterations, penalty_s=30, policy=0, deadlines=None,
             opportunistic=False):
    """policy: the round's NEXT-4 ablation flags (bit 0 NA, bit 1 NH; R-11).
    deadlines: absolute ns per job or None (deadline-aware variant, R-12): a
    pending job no Cell can finish by its deadline is dropped before the round;
    an option's T must satisfy start + penalty + remaining * T <= deadline.
    opportunistic (R-14): before the round, each pending job
    in priority order that fits nowhere directly, but would fit on some type if
    the running jobs of later priority there that were opportunistic (running
    while an earlier job waited, judged after the previous round) were
    suspended, gets them suspended, latest priority first, until its smallest
    option (G <= N_G) on that type fits -- the type with the smallest such
    option, lowest type on ties.  Suspended jobs keep their completed
    iterations and pay the penalty when they resume."""
    pr = o.pr
    J = pr.n_jobs
    submit = [int(x) * NS for x in pr.submit]
    iters = [int(x) for x in iterations]
    P = int(penalty_s) * NS
    status = ["future"] * J
    run = [-1] * J
    left = list(iters)
    seg = [(0, 0)] * J          # (segment start, segment penalty)
    fin = [-1] * J
    first = [-1] * J
    restarts = [0] * J
    rounds = 0
    INF = np.iinfo(np.int64).max
    TT = int(pr.n_types)
    prio = sorted(range(J), key=lambda j: (int(pr.submit[j]), int(pr.job_id[j])))
    rank = [0] * J
    for r, j in enumerate(prio):
        rank[j] = r
    small = [[None] * TT for _ in range(J)]  # smallest option G <= N_G per (job, type)
    for c in range(len(t_ns)):
        j, tt, g = int(cells["job"][c]), int(cells["type"][c]), int(cells["G"][c])
        if int(t_ns[c]) != INF and g <= int(pr.ng[j]) and (small[j][tt] is None or g < small[j][tt]):
            small[j][tt] = g
    opp = [False] * J
    resumed = [False] * J
    best_T = [None] * J  # fastest feasible Cell of each job
    for c in range(len(t_ns)):
        j, T = int(cells["job"][c]), int(t_ns[c])
        if T != np.iinfo(np.int64).max and (best_T[j] is None or T < best_T[j]):
            best_T[j] = T
    while True:
        t_next = [fin[j] for j in range(J) if status[j] == "running"]
        t_next += [submit[j] for j in range(J) if status[j] == "future"]
        if not t_next:
            break
        t = min(t_next)
        for j in range(J):
            if status[j] == "running" and fin[j] <= t:
                status[j] = "done"
                run[j] = -1
        for j in range(J):
            if status[j] == "future" and submit[j] <= t:
                status[j] = "pending"
        if opportunistic:
            free_now = [int(c) for c in pr.cap]
            for j in range(J):
                if status[j] == "running":
                    free_now[int(cells["type"][run[j]])] -= int(cells["G"][run[j]])
            for p in prio:
                if status[p] != "pending":
                    continue
                if any(small[p][tt] is not None and small[p][tt] <= free_now[tt] for tt in range(TT)):
                    continue
                pick = None
                for tt in range(TT):
                    if small[p][tt] is None:
                        continue
                    later = [v for v in range(J) if status[v] == "running" and opp[v]
                             and int(cells["type"][run[v]]) == tt and rank[v] > rank[p]]
                    room = free_now[tt] + sum(int(cells["G"][run[v]]) for v in later)
                    if room >= small[p][tt] and (pick is None or (small[p][tt], tt) < (pick[0], pick[1])):
                        pick = (small[p][tt], tt, later)
                if pick is None:
                    continue
                need, tt, later = pick
                for v in sorted(later, key=lambda x: rank[x], reverse=True):
                    if free_now[tt] >= need:
                        break
                    free_now[tt] += int(cells["G"][run[v]])
                    s0, p0 = seg[v]
                    ran = t - s0 - p0
                    done_it = ran // int(t_ns[run[v]]) if ran > 0 else 0
                    left[v] -= min(done_it, left[v])
                    status[v], run[v], opp[v], resumed[v] = "pending", -1, False, True
        t_max = None
        if deadlines is not None:
            t_max = [-1] * J
            for j in range(J):
                if status[j] not in ("pending", "running"):
                    continue
                pen_j, rem = (P if resumed[j] else 0), left[j]
                if status[j] == "running":
                    s0, p0 = seg[j]
                    ran = t - s0 - p0
                    done_it = ran // int(t_ns[run[j]]) if ran > 0 else 0
                    rem = left[j] - min(done_it, left[j])
                    pen_j = P
                slack = int(deadlines[j]) - t - pen_j
                t_max[j] = slack // rem if rem > 0 and slack > 0 else -1
                if status[j] == "pending" and (best_T[j] is None or best_T[j] > t_max[j]):
                    status[j] = "dropped"  # no Cell finishes before the deadline
        active = np.array([s in ("pending", "running") for s in status], np.uint8)
        free = [int(c) for c in pr.cap]
        for j in range(J):
            if status[j] == "running":
                free[int(cells["type"][run[j]])] -= int(cells["G"][run[j]])
        dec, _, _ = o.round_state(cells, t_ns, free, run_cell=np.array(run, np.int64),
                                  active=active, policy=policy,
                                  t_max=None if t_max is None else np.array(t_max, np.int64))
        rounds += 1
        for j in range(J):
            if not active[j]:
                continue
            d = int(dec[j])
            if d == -2:
                status[j] = "dropped"
            elif d >= 0 and status[j] == "pending":
                pj = P if resumed[j] else 0  # a suspended job resumes with a restart
                status[j] = "running"
                run[j] = d
                seg[j] = (t, pj)
                if first[j] < 0:
                    first[j] = t
                fin[j] = t + pj + left[j] * int(t_ns[d])
                if resumed[j]:
                    restarts[j] += 1
                    resumed[j] = False
            elif d >= 0 and d != run[j]:
                s0, p0 = seg[j]
                ran = t - s0 - p0
                done_it = ran // int(t_ns[run[j]]) if ran > 0 else 0
                left[j] -= min(done_it, left[j])
                run[j] = d
                seg[j] = (t, P)
                fin[j] = t + P + left[j] * int(t_ns[d])
                restarts[j] += 1
        if opportunistic:  # running while a job of earlier priority waits
            waiting = [rank[j] for j in range(J) if status[j] == "pending"]
            first_wait = min(waiting) if waiting else J
            for j in range(J):
                opp[j] = status[j] == "running" and rank[j] > first_wait
    state = np.array([{"done": 3, "dropped": 4, "pending": 5, "future": 0}[s] for s in status],
                     np.int8)
    return dict(first_start=np.array(first, np.int64), finish=np.array(fin, np.int64),
                restarts=np.array(restarts, np.int32), state=state, rounds=rounds)
