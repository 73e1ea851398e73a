"""NEXT-2: pins of the oracle's paper stage determination.

PAPER.md:266-283 maps each operator to G * FLOPs_l / FLOPs GPUs, cuts the model
at the S-1 smallest inter-operator communications, and gives each stage the
sum of its operators' GPUs, "approximating a power of 2".  Readings R-8..R-10
 fix what the paper leaves open.  Pins: the paper's worked
numbers (0.5 / 1.5 GPU), SPEC's uniform example, rounding cases, a hand
vector for the node-packing link rules, brute force over every cut set, and
reduction to the pinned uniform path (§N3 split, §N5 cost) where the paper's
stages coincide with it.
"""
import itertools

import numpy as np
import pytest

from helpers import golden, problem_from
from paper_2403_16125_b200 import workload as W

G = golden("paper_stages.json")


def one_job(c, bnd, *, w=None, gb=1, gpn=64, cap=64, g_max=64, alpha_in=1, alpha_x=1):
    L = len(c)
    return problem_from([dict(cap=cap, gpn=gpn, alpha_in=alpha_in, alpha_x=alpha_x)],
                        [dict(c=list(c), bnd=list(bnd), w=list(w or [0] * L), ng=1, gb=gb)],
                        k_max=6, g_max=g_max)


def test_paper_fractional_mapping(oracle_mod):
    ex = G["paper_fig_stage_partition"]
    n = len(ex["flops"])
    pr = one_job(ex["flops"], [1] * n)
    o = oracle_mod.Oracle(pr)
    num, den = o.paper_fractional(0, 0, ex["G"], n, np.arange(n + 1))
    assert np.allclose(num / den, ex["fractional_gpus"])
    assert num[0] * 2 == den and num[1] * 2 == 3 * den  # exactly 0.5 and 1.5


def test_round_pow2_cases(oracle_mod):
    for num, den, want in G["round_pow2"]["cases"]:
        assert oracle_mod.paper_round_pow2(num, den) == want, (num, den)


def test_spec_uniform_example(oracle_mod):
    ex = G["spec_uniform"]
    pr = one_job([5] * ex["L"], [7] * ex["L"])
    o = oracle_mod.Oracle(pr)
    b, g = o.paper_stages(0, 0, ex["G"], ex["S"])
    assert list(b) == ex["cuts"] and list(g) == ex["gpus"]


def test_single_stage_takes_everything(oracle_mod):
    rng = np.random.default_rng(3)
    c = rng.integers(1, 50, 9)
    pr = one_job(c, rng.integers(1, 9, 9))
    o = oracle_mod.Oracle(pr)
    for Gc in (1, 2, 8, 32):
        b, g = o.paper_stages(0, 0, Gc, 1)
        assert list(b) == [0, 9] and list(g) == [Gc]


def test_link_rules_hand_vector(oracle_mod):
    ex = G["links_hand"]
    pr = one_job(ex["c"], ex["bnd"], w=ex["w"], gb=ex["gb"], gpn=ex["gpn"], cap=8,
                 alpha_in=ex["alpha_in"], alpha_x=ex["alpha_x"])
    o = oracle_mod.Oracle(pr)
    b, g = o.paper_stages(0, 0, ex["G"], ex["S"])
    assert list(b) == ex["cuts"] and list(g) == ex["gpus"]
    t, feas = o.paper_plan_cost(0, 0, ex["S"], b, g, 0)
    assert feas and t == ex["t_iter_p0"]


def brute_cuts(c, bnd, S):
    """Every cut set: keep those whose sorted gap bytes are lexicographically
    smallest (the S-1 smallest communications), then the min-max compute."""
    L = len(c)
    P = np.concatenate([[0], np.cumsum(c)])
    best = None
    for cs in itertools.combinations(range(1, L), S - 1):
        key_bytes = sorted(bnd[q - 1] for q in cs)
        b = (0,) + cs + (L,)
        mx = max(P[b[i + 1]] - P[b[i]] for i in range(S))
        key = (key_bytes, mx)
        if best is None or key < best[0]:
            best = (key, [b])
        elif key == best[0]:
            best[1].append(b)
    return best[0], best[1]


@pytest.mark.parametrize("seed", range(60))
def test_cuts_bruteforce(oracle_mod, seed):
    rng = np.random.default_rng(1000 + seed)
    L = int(rng.integers(2, 10))
    c = rng.integers(1, 6 if seed % 2 else 40, L)
    bnd = rng.integers(1, 3 if seed % 3 == 0 else 50, L)  # many ties on some seeds
    pr = one_job(c, bnd)
    o = oracle_mod.Oracle(pr)
    P = np.concatenate([[0], np.cumsum(c)])
    for S in range(1, L + 1):
        b, _ = o.paper_stages(0, 0, 64, S)
        (kb, mx), sets = brute_cuts(c, bnd, S)
        assert sorted(bnd[q - 1] for q in b[1:-1]) == kb          # S-1 smallest bytes
        assert max(P[b[i + 1]] - P[b[i]] for i in range(S)) == mx  # min-max among them
        assert tuple(int(x) for x in b) in sets
        if len(sets) == 1:
            assert tuple(int(x) for x in b) == sets[0]


@pytest.mark.parametrize("seed", range(40))
def test_gpus_conservation_and_rule(oracle_mod, seed):
    rng = np.random.default_rng(2000 + seed)
    L = int(rng.integers(1, 12))
    c = rng.integers(1, 100, L)
    pr = one_job(c, rng.integers(1, 5, L))
    o = oracle_mod.Oracle(pr)
    P = np.concatenate([[0], np.cumsum(c)])
    for S in range(1, L + 1):
        for Gc in (1 << e for e in range(0, 8)):
            if Gc < S:
                continue
            b, g = o.paper_stages(0, 0, Gc, S)
            assert g.sum() == Gc and np.all(g >= 1)
            assert np.all((g & (g - 1)) == 0)
            F = np.array([P[b[i + 1]] - P[b[i]] for i in range(S)])
            init = [oracle_mod.paper_round_pow2(int(Gc * f), int(P[-1])) for f in F]
            # the repair only moves the sum toward G: stages change only if it was off
            if sum(init) == Gc:
                assert list(g) == init


def test_equal_bytes_reduce_to_d1_split(oracle_mod):
    """With every boundary equal, the cut rule is the §N3 min-max split (R0)."""
    rng = np.random.default_rng(7)
    for _ in range(30):
        L = int(rng.integers(2, 14))
        c = rng.integers(1, 30, L)
        pr = one_job(c, [9] * L)
        o = oracle_mod.Oracle(pr)
        for S in range(1, L + 1):
            b, _ = o.paper_stages(0, 0, 64, S)
            assert np.array_equal(b, o.split(0, 0, S))


def test_uniform_stages_reduce_to_uniform_estimate(oracle_mod):
    """Cells whose paper stages equal the §N3 split with g_s = G/S for every s
    must cost exactly as the pinned uniform path (same plans, same links)."""
    hit = 0
    for cfg in (1, 2):
        pr = W.make_config(cfg)
        o = oracle_mod.Oracle(pr)
        cells = o.enumerate()
        t_u, p_u = o.estimate(cells)
        t_p, p_p, lg = o.estimate_paper(cells)
        for i in range(len(t_u)):
            j, t, Gc, S = (int(cells[k][i]) for k in ("job", "type", "G", "S"))
            b, g = o.paper_stages(j, t, Gc, S)
            if np.array_equal(b, o.split(j, t, S)) and np.all(g == Gc // S):
                hit += 1
                assert t_p[i] == t_u[i] and p_p[i] == p_u[i], (cfg, i)
                for p in range(int(cells["nplans"][i])):
                    tp_, fe = o.paper_plan_cost(j, t, S, b, g, p)
                    ref = o.plan_cost(j, t, Gc, S, p)
                    assert fe == ref["feasible"]
                    if fe:
                        assert tp_ == ref["t_iter"]
            assert np.all(lg[i, :S] == np.log2(g).astype(int)) and np.all(lg[i, S:] == -1)
    assert hit > 20


def test_estimate_is_first_minimum_over_plans(oracle_mod):
    pr = W.make_config(2)
    o = oracle_mod.Oracle(pr)
    cells = o.enumerate()
    t_p, p_p, _ = o.estimate_paper(cells)
    nB = 1 if pr.b_mode == 0 else len(pr.b_values)
    for i in range(0, len(t_p), 3):
        j, t, Gc, S = (int(cells[k][i]) for k in ("job", "type", "G", "S"))
        b, g = o.paper_stages(j, t, Gc, S)
        np_ = (int(np.log2(g.min())) + 1) * nB
        costs = [o.paper_plan_cost(j, t, S, b, g, p) for p in range(np_)]
        feas = [(tt, p) for p, (tt, fe) in enumerate(costs) if fe]
        if not feas:
            assert p_p[i] == -1 and t_p[i] == np.iinfo(np.int64).max
        else:
            assert (t_p[i], p_p[i]) == min(feas)


def test_repair_hand_vector(oracle_mod):
    ex = G["repair_hand"]
    n = len(ex["flops"])
    pr = one_job(ex["flops"], [1] * n)
    o = oracle_mod.Oracle(pr)
    num, den = o.paper_fractional(0, 0, ex["G"], n, np.arange(n + 1))
    assert [oracle_mod.paper_round_pow2(int(x), int(den)) for x in num] == ex["rounded"]
    b, g = o.paper_stages(0, 0, ex["G"], ex["S"])
    assert list(b) == list(range(n + 1)) and list(g) == ex["gpus"]
