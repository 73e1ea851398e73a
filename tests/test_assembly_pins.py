"""Pins of the NEXT-1 oracle (per-stage parallelism assembly, PAPER.md:344-361,
pipeline latency with the slowest stage's overlapped inbound communication
subtracted) against a hand vector and against the already
pinned uniform-plan oracle."""
import itertools

import numpy as np
import pytest

from helpers import flow_shop_makespan, golden, problem_from
from paper_2403_16125_b200 import workload as W
from test_oracle_pins import _hcost_problem

INF = np.iinfo(np.int64).max


def test_assembly_hand_vector(oracle_mod):
    h, fx = golden("h_cost.json"), golden("assembly_hcost.json")
    o = oracle_mod.Oracle(_hcost_problem(h))
    G, S = h["cell"]["G"], h["cell"]["S"]
    for pl in fx["plans"]:
        for form in (0, 1):
            lat, ok = o.assembled_cost(form, 0, 0, G, S, 0, np.array(pl["k"], np.int8))
            assert ok and lat == pl[f"form{form}"], (pl, form)
    cells = o.enumerate()
    i = [q for q in range(len(cells["G"])) if cells["G"][q] == G and cells["S"][q] == S][0]
    for form in (0, 1):
        t, b, sk = o.estimate_assembled(cells, 1, form, i, i + 1)
        assert t[0] == fx["best"][f"form{form}"] and b[0] == 0 and list(sk[0][:S]) == [0, 0]


def test_uniform_assignment_equals_uniform_plan(oracle_mod):
    """Every stage on the same factorisation is the north_star uniform plan."""
    for seed in range(40):
        pr = W.random_tiny(seed, max_layers=8)
        o = oracle_mod.Oracle(pr)
        cells = o.enumerate()
        nB = 1 if pr.b_mode == 0 else len(pr.b_values)
        for i in range(len(cells["G"])):
            j, t, G, S = (int(cells[k][i]) for k in ("job", "type", "G", "S"))
            for p in range(int(cells["nplans"][i])):
                k, bi = divmod(p, nB)
                r = o.plan_cost(j, t, G, S, p)
                lat, ok = o.assembled_cost(0, j, t, G, S, bi, np.full(S, k, np.int8))
                assert ok == r["feasible"]
                if ok:
                    assert lat == r["t_iter"]
                    assert lat == flow_shop_makespan(list(r["T"]), 4 * S if pr.b_mode == 0 else
                                                     int(pr.b_values[bi])) + max(r["sync"])


def test_single_stage_assembly_equals_uniform_estimate(oracle_mod):
    """S = 1: the assembled space (mode 2) is the uniform space; forms agree
    (the only stage has no inbound communication)."""
    for seed in range(60):
        pr = W.random_tiny(seed, max_layers=6)
        o = oracle_mod.Oracle(pr)
        cells = o.enumerate()
        idx = np.where(cells["S"] == 1)[0]
        if len(idx) == 0:
            continue
        sub = {k: np.ascontiguousarray(v[idx]) for k, v in cells.items()}
        t_u, p_u = o.estimate(sub)
        for form in (0, 1):
            t_a, b_a, _ = o.estimate_assembled(sub, 2, form, kstride=1)
            assert np.array_equal(t_a, t_u)


def test_assembly_bounds_and_bruteforce(oracle_mod):
    """mode 2 <= uniform optimum (superset); mode 2 <= mode 1; form 1 <= form 0;
    the reported best is the minimum of assembled_cost over every plan."""
    checked = 0
    for seed in range(25):
        pr = W.random_tiny(500 + seed, max_layers=6, n_types=1, n_jobs=2)
        o = oracle_mod.Oracle(pr)
        cells = o.enumerate()
        t_u, _ = o.estimate(cells)
        res = {(m, f): o.estimate_assembled(cells, m, f) for m in (1, 2) for f in (0, 1)}
        nB = 1 if pr.b_mode == 0 else len(pr.b_values)
        for i in range(len(cells["G"])):
            j, t, G, S = (int(cells[k][i]) for k in ("job", "type", "G", "S"))
            assert res[2, 0][0][i] <= t_u[i]
            for f in (0, 1):
                assert res[2, f][0][i] <= res[1, f][0][i]
            for m in (1, 2):
                assert res[m, 1][0][i] <= res[m, 0][0][i]
            g = G // S
            K = int(np.log2(g))
            choices = [0, K] if (K and True) else [0]
            for m in (1, 2):
                ch = sorted(set(choices)) if m == 1 else list(range(K + 1))
                for f in (0, 1):
                    best = INF
                    for bi in range(nB):
                        for ks in itertools.product(ch, repeat=S):
                            lat, ok = o.assembled_cost(f, j, t, G, S, bi, np.array(ks, np.int8))
                            if ok:
                                best = min(best, lat)
                    assert res[m, f][0][i] == best
                    if best < INF:
                        lat, ok = o.assembled_cost(f, j, t, G, S, int(res[m, f][1][i]),
                                                   res[m, f][2][i])
                        assert ok and lat == best
                    checked += 1
    assert checked > 100
