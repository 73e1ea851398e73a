"""Shared test helpers: small hand-built Problems and brute-force references.

Nothing here imports the CUDA path; the brute-force routines are independent
re-derivations used to PIN the oracle (SURVEY §8(c) pins Π1-Π9), not copies of
its code: they enumerate instead of optimise.
"""
from __future__ import annotations

import itertools
import json
import os

import numpy as np

from paper_2403_16125_b200.workload import MiB, Problem

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def problem_from(types, jobs, *, k_max=2, gpu_set=1, s_max=64, g_max=4, b_mode=0, b_values=(),
                 depth=3, c_planes=None):
    """types: list of dicts (cap, gpn, mem, alpha_in, beta_in, alpha_x, beta_x);
    jobs: list of dicts (c: [K+1][L] or [L], ng, gb, kst, w, act, bnd, tpv, tpn,
    submit, id).  Layers default to zeros; compute for k>0 defaults to k=0's."""
    T = len(types)
    nl = np.array([len(np.atleast_2d(j["c"])[0]) for j in jobs], np.int32)
    off = np.zeros(len(jobs) + 1, np.int64)
    off[1:] = np.cumsum(nl)
    L = int(off[-1])
    K1 = k_max + 1
    c = np.zeros((T, K1, L), np.int32)
    for ji, j in enumerate(jobs):
        cj = np.atleast_2d(np.asarray(j["c"], np.int64))
        for t in range(T):
            for k in range(K1):
                row = cj[min(k, cj.shape[0] - 1)]
                if c_planes is not None:
                    row = c_planes(ji, t, k, row)
                c[t, k, off[ji]:off[ji + 1]] = row

    def lay(key, dtype):
        out = np.zeros(L, dtype)
        for ji, j in enumerate(jobs):
            if key in j:
                out[off[ji]:off[ji + 1]] = j[key]
        return out

    def typ(key, default, dtype):
        return np.array([t.get(key, default) for t in types], dtype)

    return Problem(
        name="hand", type_names=[f"T{i}" for i in range(T)], cap=typ("cap", 4, np.int32),
        gpn=typ("gpn", 4, np.int32), mem=typ("mem", 1 << 40, np.int64),
        alpha_in=typ("alpha_in", 1, np.int64), beta_in=typ("beta_in", MiB, np.int64),
        alpha_x=typ("alpha_x", 1, np.int64), beta_x=typ("beta_x", MiB, np.int64),
        job_id=np.array([j.get("id", i) for i, j in enumerate(jobs)], np.int64),
        submit=np.array([j.get("submit", 0) for j in jobs], np.int64),
        ng=np.array([j.get("ng", 1) for j in jobs], np.int32),
        gb=np.array([j.get("gb", 1) for j in jobs], np.int32),
        kst=np.array([j.get("kst", 1) for j in jobs], np.int32), n_layers=nl, layer_off=off, c=c,
        w=lay("w", np.int64), act=lay("act", np.int64), bnd=lay("bnd", np.int64),
        tpv=lay("tpv", np.int64), tpn=lay("tpn", np.int32), k_max=k_max, gpu_set=gpu_set,
        s_max=s_max, g_max=g_max, b_mode=b_mode, b_values=np.array(b_values, np.int32),
        depth=depth)


def split_problem(c0, cap=None):
    """One job, one type, compute row c0; cap large enough for S = L."""
    L = len(c0)
    cap = cap or 1 << int(np.ceil(np.log2(max(L, 1))) + 1)
    return problem_from([dict(cap=cap, gpn=cap)], [dict(c=list(c0), ng=1, gb=1)], k_max=0, g_max=1)


# ---------------------------------------------------------------------------
# Brute force (Π2): characterise the R0 split without a DP.
# ---------------------------------------------------------------------------

def all_splits(L, S):
    """Every boundary vector 0 = b0 < b1 < .. < bS = L."""
    for mid in itertools.combinations(range(1, L), S - 1):
        yield (0,) + mid + (L,)


def stage_costs(c, b):
    return [sum(c[b[s]:b[s + 1]]) for s in range(len(b) - 1)]


def brute_prefix_opt(c):
    """F[s][i] = min over splits of the first i layers into s stages of the max stage cost."""
    L = len(c)
    F = {}
    for i in range(1, L + 1):
        for s in range(1, i + 1):
            F[s, i] = min(max(stage_costs(c[:i], b)) for b in all_splits(i, s))
    return F


def brute_r0_split(c, S, F=None):
    """R0 (SURVEY A-4): among optimal splits whose every prefix split is itself
    optimal, the reverse-lexicographically smallest boundary vector."""
    L = len(c)
    F = F or brute_prefix_opt(c)
    good = []
    for b in all_splits(L, S):
        costs = stage_costs(c, b)
        if all(max(costs[:s]) == F[s, b[s]] for s in range(1, S + 1)):
            good.append(b)
    return min(good, key=lambda b: tuple(reversed(b))), F[S, L]


def painter_opt(c, S):
    """Textbook linear-partition optimum by binary search on the answer with a
    greedy feasibility check (Π9 iii) -- an algorithm unrelated to the DP."""
    lo, hi = max(c), sum(c)
    while lo < hi:
        mid = (lo + hi) // 2
        parts, acc = 1, 0
        for x in c:
            if acc + x > mid:
                parts, acc = parts + 1, x
            else:
                acc += x
        if parts <= S:
            hi = mid
        else:
            lo = mid + 1
    return lo


def flow_shop_makespan(T, B):
    """B identical jobs through len(T) machines in order, unbounded buffers:
    C[m][s] = max(C[m-1][s], C[m][s-1]) + T[s]  (Π5)."""
    S = len(T)
    prev = [0] * S
    for _ in range(B):
        cur = [0] * S
        for s in range(S):
            cur[s] = max(prev[s], cur[s - 1] if s else 0) + T[s]
        prev = cur
    return prev[-1]


def enumerate_cells_ref(pr):
    """§N2 written as set comprehensions (independent of the oracle's loops)."""
    out = []
    for j in range(pr.n_jobs):
        for t in range(pr.n_types):
            ng, cap = int(pr.ng[j]), int(pr.cap[t])
            if pr.gpu_set == 0:
                Gs = sorted({g for g in (ng // 2 if ng >= 2 else 0, ng, 2 * ng) if 1 <= g <= cap})
            else:
                Gs = [1 << e for e in range(0, 31) if (1 << e) <= cap]
            for G in Gs:
                for e in range(0, 31):
                    S = 1 << e
                    if S > min(G, int(pr.n_layers[j]), pr.s_max):
                        break
                    if G // S <= pr.g_max:
                        nB = 1 if pr.b_mode == 0 else len(pr.b_values)
                        out.append((j, t, G, S, (int(np.log2(G // S)) + 1) * nB))
    return out
