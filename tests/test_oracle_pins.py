"""Pins of the CPU oracle against things other than itself (SURVEY §8(c) Π1-Π9).

Every test here is CPU-only.  A plausible slip anywhere in the oracle (a dropped
term, a wrong sign or index, a transposed operand, a wrong tie rule) should
fail at least one of them:
  * hand vectors and closed forms from tests/golden (cited in each fixture);
  * brute force over every split / every plan on tiny inputs;
  * an unrelated algorithm (painter's-partition parametric search) for the OPT;
  * a flow-shop event simulation for the pipeline formula;
  * special cases that reduce to textbook results and invariants.
"""
import math

import numpy as np
import pytest

from helpers import (all_splits, brute_prefix_opt, brute_r0_split, enumerate_cells_ref,
                     flow_shop_makespan, golden, painter_opt, problem_from, split_problem,
                     stage_costs)
from paper_2403_16125_b200 import workload as W

INF = np.iinfo(np.int64).max
MiB = 1 << 20


# ---------------------------------------------------------------- Π1 / Π3 splits
def test_split_hand_vectors(oracle_mod):
    for case in golden("split_vectors.json")["cases"]:
        o = oracle_mod.Oracle(split_problem(case["c"]))
        b = o.split(0, 0, case["S"])
        assert list(b) == case["bounds"], case
        assert max(stage_costs(case["c"], b)) == case["opt"]


def test_split_closed_forms(oracle_mod):
    rng = np.random.default_rng(0)
    for _ in range(50):
        L = int(rng.integers(1, 40))
        c = rng.integers(1, 100, size=L).tolist()
        o = oracle_mod.Oracle(split_problem(c))
        assert list(o.split(0, 0, 1)) == [0, L]                  # S=1 -> OPT = sum c
        assert list(o.split(0, 0, L)) == list(range(L + 1))      # S=L -> OPT = max c
    for L, S in ((8, 2), (16, 4), (32, 8), (96, 32), (64, 16)):
        o = oracle_mod.Oracle(split_problem([7] * L))
        assert list(o.split(0, 0, S)) == list(range(0, L + 1, L // S))  # uniform, S | L


# ---------------------------------------------------------------- Π2 brute force
def test_split_matches_bruteforce_r0(oracle_mod):
    rng = np.random.default_rng(1)
    n = 0
    for case in range(1500):
        L = int(rng.integers(1, 9))
        hi = int(rng.choice([2, 3, 5, 20]))  # small ranges -> many ties
        c = rng.integers(1, hi + 1, size=L).tolist()
        o = oracle_mod.Oracle(split_problem(c))
        F = brute_prefix_opt(c)
        for S in range(1, L + 1):
            want, opt = brute_r0_split(c, S, F)
            got = tuple(int(x) for x in o.split(0, 0, S))
            assert got == want, (c, S, got, want)
            assert max(stage_costs(c, got)) == opt
            n += 1
    assert n > 4000


def test_split_r0_differs_from_threshold_backtrack(oracle_mod):
    # SURVEY A-4: R0 -> (2,3) on c=[2,2,3,3,2], S=3; a threshold backtrack gives (1,3).
    o = oracle_mod.Oracle(split_problem([2, 2, 3, 3, 2]))
    assert list(o.split(0, 0, 3)) == [0, 2, 3, 5]


# ---------------------------------------------------------------- Π9(iii) OPT
def test_split_opt_equals_painter_partition(oracle_mod):
    rng = np.random.default_rng(2)
    for _ in range(300):
        L = int(rng.integers(1, 97))
        c = rng.integers(1, int(rng.choice([3, 1000, 10 ** 7])), size=L).tolist()
        o = oracle_mod.Oracle(split_problem(c))
        for S in (1, 2, 4, 8, 16, 32):
            if S > L:
                break
            b = o.split(0, 0, S)
            assert b[0] == 0 and b[-1] == L and all(b[i] < b[i + 1] for i in range(S))
            assert max(stage_costs(c, b)) == painter_opt(c, S)


# ---------------------------------------------------------------- Π6 comm
def test_comm_closed_forms(oracle_mod):
    comm = oracle_mod.comm
    rng = np.random.default_rng(3)
    for _ in range(200):
        a = int(rng.integers(0, 10 ** 5))
        b = int(rng.integers(1, 10 ** 7))
        V = int(rng.integers(0, 10 ** 9))
        n = int(rng.integers(0, 9))
        assert comm(0, 1, a, b, V, n) == 0 and comm(1, 1, a, b, V, 1) == 0
        assert comm(0, 2, a, b, V, 1) == 2 * a + -(-V * b // MiB)
        assert comm(2, 0, a, b, 0, 0) == a                       # P2P(V=0) = alpha
        assert comm(2, 0, a, b, V, 0) == a + -(-V * b // MiB)
        for p in (2, 4, 8, 64):
            if a >= 1:
                assert comm(1, p, a, b, V, 1) < comm(0, p, a, b, V, 1)   # AG < AR
    # hand: AR(4, 10, 2^20 (1 ns/B), 1000 B, 3 calls) = 3*2*3*10 + 6*1000/4 = 180 + 1500
    assert comm(0, 4, 10, MiB, 1000, 3) == 1680
    # hand: AG(8, 5, 2^20, 7 B) = 7*5 + ceil(7*7/8) = 35 + 7
    assert comm(1, 8, 5, MiB, 7, 1) == 42
    # ceil, not floor: 1 byte at 1 ns/MiB
    assert comm(2, 0, 0, 1, 1, 0) == 1


# ---------------------------------------------------------------- Π4 H-cost
def _hcost_problem(h, mem=None, gpn=None):
    ty, jb = dict(h["type"]), h["job"]
    if mem is not None:
        ty["mem"] = mem
    if gpn is not None:
        ty["gpn"] = gpn
    return problem_from([ty], [dict(c=jb["c"], ng=jb["ng"], gb=jb["GB"], kst=jb["kst"], w=jb["w"],
                                    act=jb["act"], bnd=jb["bnd"], tpv=jb["tpv"], tpn=jb["tpn"])],
                        k_max=2, g_max=4, gpu_set=1)


def test_hcost_hand_vector(oracle_mod):
    h = golden("h_cost.json")
    e = h["expect"]
    G, S = h["cell"]["G"], h["cell"]["S"]
    o = oracle_mod.Oracle(_hcost_problem(h))
    assert list(o.split(0, 0, S)) == e["split"]
    r0 = o.plan_cost(0, 0, G, S, 0)
    assert r0["feasible"] and list(r0["T"]) == e["k0"]["T"] and list(r0["sync"]) == e["k0"]["sync"]
    assert list(r0["mem"]) == e["k0"]["mem"] and r0["t_iter"] == e["k0"]["t_iter"]
    r1 = o.plan_cost(0, 0, G, S, 1)
    assert list(r1["T"]) == e["k1"]["T"] and list(r1["sync"]) == e["k1"]["sync"]
    assert r1["t_iter"] == e["k1"]["t_iter"]
    cells = o.enumerate()
    idx = [i for i in range(len(cells["G"])) if cells["G"][i] == G and cells["S"][i] == S][0]
    t, p = o.estimate(cells, idx, idx + 1)
    assert (p[0], t[0]) == (e["best_plan"], e["best_t"])
    # memory forces tensor parallelism
    om = oracle_mod.Oracle(_hcost_problem(h, mem=150))
    assert not om.plan_cost(0, 0, G, S, 0)["feasible"]
    t, p = om.estimate(cells, idx, idx + 1)
    assert (p[0], t[0]) == (e["mem150"]["best_plan"], e["mem150"]["best_t"])
    # boundary crosses nodes when gpn = 2
    og = oracle_mod.Oracle(_hcost_problem(h, gpn=2))
    assert og.plan_cost(0, 0, G, S, 0)["t_iter"] == e["gpn2"]["k0"]
    assert og.plan_cost(0, 0, G, S, 1)["t_iter"] == e["gpn2"]["k1"]


def test_memory_hand_vector(oracle_mod):
    m = golden("mem_vector.json")
    pr = problem_from([dict(cap=4, gpn=4)], [m["job"]], k_max=2, g_max=4, gpu_set=1)
    o = oracle_mod.Oracle(pr)
    for k, want in enumerate(m["mem"]):
        r = o.plan_cost(0, 0, m["cell"]["G"], m["cell"]["S"], k)
        assert list(r["mem"]) == [want]
        pr2 = problem_from([dict(cap=4, gpn=4, mem=want - 1)], [m["job"]], k_max=2, g_max=4)
        assert not oracle_mod.Oracle(pr2).plan_cost(0, 0, 4, 1, k)["feasible"]
        pr3 = problem_from([dict(cap=4, gpn=4, mem=want)], [m["job"]], k_max=2, g_max=4)
        assert oracle_mod.Oracle(pr3).plan_cost(0, 0, 4, 1, k)["feasible"]


# ---------------------------------------------------------------- Π5 pipeline
def test_flow_shop_reference_itself():
    sp = golden("pipeline_spec.json")
    assert flow_shop_makespan(sp["T"], sp["B"]) == sp["north_star"]
    assert sum(sp["T"]) + (sp["B"] - 1) * (max(sp["T"]) - sp["paper_form_T_comm"]) == sp["paper_form"]
    assert flow_shop_makespan([3] * 5, 7) == (5 + 7 - 1) * 3      # (S+B-1) T


def test_pipeline_formula_is_flow_shop_makespan(oracle_mod):
    checked = 0
    for seed in range(60):
        pr = W.random_tiny(seed, max_layers=8)
        o = oracle_mod.Oracle(pr)
        cells = o.enumerate()
        nB = 1 if pr.b_mode == 0 else len(pr.b_values)
        for i in range(len(cells["G"])):
            j, t, G, S = (int(cells[k][i]) for k in ("job", "type", "G", "S"))
            for p in range(int(cells["nplans"][i])):
                r = o.plan_cost(j, t, G, S, p)
                B = 4 * S if pr.b_mode == 0 else int(pr.b_values[p % nB])
                k = p // nB
                g = G // S
                if B * (g >> k) > pr.gb[j]:
                    assert not r["feasible"]
                    continue
                if not r["feasible"]:
                    continue
                assert r["t_iter"] == flow_shop_makespan(list(r["T"]), B) + max(r["sync"])
                checked += 1
    assert checked > 200


# ---------------------------------------------------------------- Π9(i) pure DP
def test_pure_data_parallel_reduces_to_dp_step(oracle_mod):
    rng = np.random.default_rng(5)
    for _ in range(100):
        L = int(rng.integers(1, 12))
        c = rng.integers(1, 1000, size=L).tolist()
        w = rng.integers(0, 10 ** 6, size=L).tolist()
        gpn = int(rng.choice([1, 2, 4, 8]))
        ai, ax = int(rng.integers(1, 100)), int(rng.integers(1, 1000))
        bi, bx = int(rng.integers(1, MiB)), int(rng.integers(1, 8 * MiB))
        GB = int(rng.choice([8, 16, 64]))
        pr = problem_from([dict(cap=8, gpn=gpn, alpha_in=ai, beta_in=bi, alpha_x=ax, beta_x=bx)],
                          [dict(c=c, ng=4, gb=GB, w=w, kst=1)], k_max=3, g_max=8, gpu_set=1)
        o = oracle_mod.Oracle(pr)
        for G in (1, 2, 4, 8):
            r = o.plan_cost(0, 0, G, 1, 0)          # S = 1, k = 0 -> tp 1, dp = G, B = 4
            if 4 * G > GB:
                assert not r["feasible"]
                continue
            dp = G
            a, b = (ai, bi) if G <= gpn else (ax, bx)
            ar = 0 if dp == 1 else 2 * (dp - 1) * a + -(-(2 * (dp - 1) * sum(w) * b) // (dp * MiB))
            # B cancels: B * (GB / (B dp)) * sum(c) = (GB/dp) sum(c) -- the plain DP step
            assert r["t_iter"] == (GB // dp) * sum(c) + ar


# ---------------------------------------------------------------- O1 enumeration
def test_enumeration_counts(oracle_mod):
    # SPEC.md:198 example: N_G = 8, 2 types with capacity >= 16, 16 operators ->
    # G in {4, 8, 16}; S in {1..G} powers of two -> 3 + 4 + 5 = 12 per type.
    jobs = [dict(c=[1] * 16, ng=8, gb=64)]
    pr = problem_from([dict(cap=16), dict(cap=32)], jobs, k_max=6, g_max=64, gpu_set=0, s_max=16)
    assert oracle_mod.Oracle(pr).count()[0] == 24
    # N_G = 1 -> G in {1, 2}: S {1} and {1, 2}
    pr = problem_from([dict(cap=16)], [dict(c=[1] * 16, ng=1)], k_max=6, g_max=64, gpu_set=0)
    cells = oracle_mod.Oracle(pr).enumerate()
    assert list(zip(cells["G"], cells["S"])) == [(1, 1), (2, 1), (2, 2)]
    # capacity 8, N_G = 8 -> 2 N_G skipped
    pr = problem_from([dict(cap=8)], [dict(c=[1] * 16, ng=8)], k_max=6, g_max=64, gpu_set=0)
    assert set(oracle_mod.Oracle(pr).enumerate()["G"]) == {4, 8}
    # BASELINE configs 1-2 (12 Cells / 20 plans; ~200 / ~470)
    assert oracle_mod.Oracle(W.make_config(1)).count() == (12, 20)
    n, p = oracle_mod.Oracle(W.make_config(2)).count()
    assert 150 < n < 260 and 350 < p < 600


def test_enumeration_matches_definition(oracle_mod):
    for seed in range(300):
        pr = W.random_tiny(seed, max_layers=12, n_types=3, n_jobs=4)
        cells = oracle_mod.Oracle(pr).enumerate()
        got = list(zip(*(cells[k].tolist() for k in ("job", "type", "G", "S", "nplans"))))
        assert got == enumerate_cells_ref(pr)


# ---------------------------------------------------------------- O4 argmin
def test_estimate_is_first_minimum_over_all_plans(oracle_mod):
    for seed in range(120):
        pr = W.random_tiny(seed, max_layers=8)
        o = oracle_mod.Oracle(pr)
        cells = o.enumerate()
        t_ns, plan = o.estimate(cells)
        for i in range(len(cells["G"])):
            j, t, G, S = (int(cells[k][i]) for k in ("job", "type", "G", "S"))
            costs = []
            for p in range(int(cells["nplans"][i])):
                r = o.plan_cost(j, t, G, S, p)
                costs.append(r["t_iter"] if r["feasible"] else INF)
            best = min(costs)
            want_p = costs.index(best) if best < INF else -1
            assert (int(plan[i]), int(t_ns[i])) == (want_p, best)


def test_estimate_split_is_bruteforce_optimal_over_all_plans(oracle_mod):
    """Brute force over every split AND every plan of tiny Cells: the best plan
    under the R0 split is the best plan under the brute-force R0 split."""
    for seed in range(40):
        pr = W.random_tiny(1000 + seed, max_layers=7, n_types=1, n_jobs=2)
        o = oracle_mod.Oracle(pr)
        for j in range(pr.n_jobs):
            L = int(pr.n_layers[j])
            c0 = pr.c[0, 0, pr.layer_off[j]:pr.layer_off[j + 1]].tolist()
            F = brute_prefix_opt(c0)
            for S in (1, 2, 4):
                if S <= L:
                    assert tuple(int(x) for x in o.split(j, 0, S)) == brute_r0_split(c0, S, F)[0]


# ---------------------------------------------------------------- Π7 round
def _round_problem(fx, d):
    jobs = [dict(c=[1], ng=jb["ng"], submit=jb["submit"], id=jb["id"]) for jb in fx["jobs"]]
    pr = problem_from([dict(cap=c) for c in fx["cap"]], jobs, k_max=2, g_max=4, depth=d)
    cells = {k: [] for k in ("job", "type", "G", "S", "nplans")}
    t_ns = []
    for j, jb in enumerate(fx["jobs"]):
        for (t, G, T) in sorted(jb["options"]):
            for k, v in (("job", j), ("type", t), ("G", G), ("S", 1), ("nplans", 1)):
                cells[k].append(v)
            t_ns.append(T)
    cells = {k: np.array(v, np.int32) for k, v in cells.items()}
    return pr, cells, np.array(t_ns, np.int64)


def test_round_hand_vector(oracle_mod):
    fx = golden("round_pi7.json")
    for d, key in ((0, "d0"), (1, "d1"), (3, "d1")):
        pr, cells, t_ns = _round_problem(fx, d)
        dec, fa, tot = oracle_mod.Oracle(pr).round(cells, t_ns)
        e = fx["expect"][key]
        for j, ch in enumerate(e["choice"]):
            if ch is None:
                assert dec[j] == -1
            else:
                assert (int(cells["type"][dec[j]]), int(cells["G"][dec[j]])) == tuple(ch)
        assert list(fa) == e["free_after"]
        assert math.isclose(tot, e["total"], rel_tol=1e-12)


def test_round_edge_vectors(oracle_mod):
    fx = golden("round_edges.json")
    for key in ("equal", "tie", "vtie", "ref", "prio"):
        case = fx[key]
        pr, cells, t_ns = _round_problem(case, case["depth"])
        dec, fa, tot = oracle_mod.Oracle(pr).round(cells, t_ns)
        for j, ch in enumerate(case["choice"]):
            if ch is None:
                assert dec[j] == -1, key
            else:
                assert (int(cells["type"][dec[j]]), int(cells["G"][dec[j]])) == tuple(ch), key
        assert list(fa) == case["free_after"] and tot == case["total"], key


def test_round_option_prefers_fewer_stages_on_equal_time(oracle_mod):
    """O_j keeps, per (t, G), the Cell with min (T_c, S_c) (§N6): two Cells of
    the same (t, G) with equal T -> the one with fewer stages is decided."""
    pr = problem_from([dict(cap=4)], [dict(c=[1, 1], ng=2)], k_max=2, g_max=4, depth=0)
    cells = {k: np.array(v, np.int32) for k, v in
             dict(job=[0, 0, 0], type=[0, 0, 0], G=[1, 2, 2], S=[1, 1, 2], nplans=[1, 1, 1]).items()}
    for t_ns, want in (([90, 70, 70], 1), ([90, 70, 60], 2), ([90, 60, 70], 1)):
        dec, _, _ = oracle_mod.Oracle(pr).round(cells, np.array(t_ns, np.int64))
        assert dec[0] == want


def test_round_d0_abundant_capacity_is_per_job_argmin(oracle_mod):
    """Π9(ii): with d = 0 and free >= sum N_G, every job independently takes
    min kappa = (T, G, t) over its options with G <= N_G; nothing else moves."""
    for cfg in (2, 3):
        pr = W.make_config(cfg)
        pr.depth = 0
        big = np.full(pr.n_types, 1 << 20, np.int32)
        pr.cap = big
        o = oracle_mod.Oracle(pr)
        cells = o.enumerate()
        t_ns, _ = o.estimate(cells)
        dec, fa, _ = o.round(cells, t_ns, free_in=big)
        best = {}
        for i in range(len(t_ns)):
            j = int(cells["job"][i])
            if t_ns[i] == INF or cells["G"][i] > pr.ng[j]:
                continue
            key = (int(t_ns[i]), int(cells["G"][i]), int(cells["type"][i]), int(cells["S"][i]))
            if j not in best or key < best[j][0]:
                best[j] = (key, i)
        for j in range(pr.n_jobs):
            if dec[j] == -2:
                assert (t_ns[cells["job"] == j] == INF).all()
            elif j in best:
                assert dec[j] == best[j][1]
            else:
                assert dec[j] == -1


# ---------------------------------------------------------------- Π8 invariants
@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_invariants_on_configs(oracle_mod, cfg):
    pr = W.make_config(cfg)
    o = oracle_mod.Oracle(pr)
    cells = o.enumerate()
    t_ns, plan = o.estimate(cells)
    dec, fa, tot = o.round(cells, t_ns)
    # splits cover every layer exactly once, S stages of g = G/S GPUs (sum g = G)
    rng = np.random.default_rng(cfg)
    for i in rng.choice(len(t_ns), size=min(60, len(t_ns)), replace=False):
        j, t, G, S = (int(cells[k][i]) for k in ("job", "type", "G", "S"))
        b = o.split(j, t, S)
        assert b[0] == 0 and b[-1] == pr.n_layers[j] and np.all(np.diff(b) >= 1)
        assert (G // S) * S == G
        # best <= every feasible plan
        for p in range(int(cells["nplans"][i])):
            r = o.plan_cost(j, t, G, S, p)
            if r["feasible"]:
                assert t_ns[i] <= r["t_iter"]
    # allocations within capacity, admitted jobs on feasible Cells
    used = np.zeros(pr.n_types, np.int64)
    for j in range(pr.n_jobs):
        if dec[j] >= 0:
            assert cells["job"][dec[j]] == j and t_ns[dec[j]] < INF
            used[cells["type"][dec[j]]] += cells["G"][dec[j]]
    assert np.all(used <= pr.cap) and np.all(fa == pr.cap - used)
    # determinism
    dec2, fa2, tot2 = o.round(cells, t_ns)
    assert np.array_equal(dec, dec2) and np.array_equal(fa, fa2) and tot == tot2


def test_sweep_best_never_worse_than_gpipe_rule(oracle_mod):
    """cfg1: B = 4S is in the sweep set {1..16} for S <= 4, so the sweep's best
    can only be better or equal (Π8)."""
    a = oracle_mod.Oracle(W.make_config(1))
    b = oracle_mod.Oracle(W.make_config(1, variant="sweep"))
    ca, cb = a.enumerate(), b.enumerate()
    ta, _ = a.estimate(ca)
    tb, _ = b.estimate(cb)
    assert np.array_equal(ca["G"], cb["G"]) and np.all(tb <= ta)


# ---------------------------------------------------------------- NEXT-4 round state
def test_round_state_hand_vector(oracle_mod):
    fx = golden("round_state.json")
    for d, key in ((1, "d1"), (3, "d1"), (0, "d0")):
        pr, cells, t_ns = _round_problem(fx, d)
        run = np.full(pr.n_jobs, -1, np.int64)
        for j, rc in enumerate(fx["running"]):
            if rc is not None:
                run[j] = [i for i in range(len(t_ns)) if cells["job"][i] == j and
                          (cells["type"][i], cells["G"][i]) == tuple(rc)][0]
        dec, fa, tot = oracle_mod.Oracle(pr).round_state(cells, t_ns, fx["free"], run_cell=run)
        e = fx["expect"][key]
        for j, ch in enumerate(e["choice"]):
            if ch is None:
                assert dec[j] == -1
            else:
                assert (int(cells["type"][dec[j]]), int(cells["G"][dec[j]])) == tuple(ch)
        assert list(fa) == e["free_after"] and tot == e["total"]


def test_round_state_reduces_to_round(oracle_mod):
    """No running job and every job active: the state round is the round;
    inactive jobs get -3 and are invisible to the others."""
    pr = W.make_config(3)
    o = oracle_mod.Oracle(pr)
    cells = o.enumerate()
    t_ns, _ = o.estimate(cells)
    d1, f1, t1 = o.round(cells, t_ns)
    d2, f2, t2 = o.round_state(cells, t_ns, pr.cap)
    assert np.array_equal(d1, d2) and np.array_equal(f1, f2) and t1 == t2
    act = np.zeros(pr.n_jobs, np.uint8)
    act[::2] = 1
    d3, _, _ = o.round_state(cells, t_ns, pr.cap, active=act)
    assert np.all(d3[1::2] == -3) and np.all(d3[::2] != -3)
