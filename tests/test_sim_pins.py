"""Pins of the oracle trace simulator (NEXT-4): a hand-computed two-job
trace with and without resource scaling, and invariants on generated traces."""
import math

import numpy as np
import pytest

from helpers import golden
from paper_2403_16125_b200 import workload as W
from test_oracle_pins import _round_problem

NS = 10 ** 9


def test_hand_trace(oracle_mod):
    from oracle import sim
    fx = golden("sim_trace.json")
    for d, key in ((0, "d0"), (3, "d3")):
        pr, cells, t_ns = _round_problem(fx, d)
        out = sim.simulate(oracle_mod.Oracle(pr), cells, t_ns, [j["iters"] for j in fx["jobs"]],
                           fx["penalty_s"])
        e = fx["expect"][key]
        assert list(out["first_start"] // NS) == e["first_start_s"], key
        assert list(out["finish"] // NS) == e["finish_s"], key
        assert list(out["restarts"]) == e["restarts"], key
        assert np.all(out["state"] == 3)


def test_trace_invariants(oracle_mod):
    from oracle import sim
    pr = W.subset(W.make_config(3), 120)
    o = oracle_mod.Oracle(pr)
    cells = o.enumerate()
    t_ns, _ = o.estimate(cells)
    it = W.iterations_for(pr)
    out = sim.simulate(o, cells, t_ns, it, 30)
    done = out["state"] == 3
    sub = pr.submit.astype(np.int64) * NS
    assert done.sum() + (out["state"] == 4).sum() + (out["state"] == 5).sum() == pr.n_jobs
    assert np.all(out["first_start"][done] >= sub[done])
    assert np.all(out["finish"][done] > out["first_start"][done])
    # a job never finishes faster than its iterations on its fastest feasible Cell
    for j in np.where(done)[0]:
        best = t_ns[(cells["job"] == j) & (t_ns < np.iinfo(np.int64).max)].min()
        assert out["finish"][j] - out["first_start"][j] >= it[j] * best
    assert out["rounds"] > 0


# ---------------------------------------------------------------- NEXT-4 ablations (NA / NH)
def _state_case(oracle_mod, case, policy):
    pr, cells, t_ns = _round_problem(case, case["depth"])
    run = np.full(pr.n_jobs, -1, np.int64)
    for j, rc in enumerate(case["running"]):
        if rc is not None:
            run[j] = [i for i in range(len(t_ns)) if cells["job"][i] == j and
                      (cells["type"][i], cells["G"][i]) == tuple(rc)][0]
    dec, fa, tot = oracle_mod.Oracle(pr).round_state(cells, t_ns, case["free"], run_cell=run,
                                                     policy=policy)
    return [None if d < 0 else (int(cells["type"][d]), int(cells["G"][d])) for d in dec], list(fa), tot


@pytest.mark.parametrize("key,bit", [("na", 1), ("nh", 2)])
def test_round_policy_hand_vectors(oracle_mod, key, bit):
    """PAPER.md:783-792 ablations on hand-computed states (tests/golden/round_policy.json)."""
    case = golden("round_policy.json")[key]
    for policy, want in ((0, case["expect"]["full"]), (bit, case["expect"][key])):
        ch, fa, tot = _state_case(oracle_mod, case, policy)
        assert ch == [None if c is None else tuple(c) for c in want["choice"]], policy
        assert fa == want["free_after"] and math.isclose(tot, want["total"], rel_tol=1e-15)


@pytest.mark.parametrize("cfg", [2, 3])
def test_round_policy_invariants(oracle_mod, cfg):
    """NA: every admitted job runs on exactly N_G GPUs.  NH: a running job that
    stays admitted keeps its GPU type.  NH with one GPU type, and policy 0, are
    the full round."""
    pr = W.make_config(cfg)
    o = oracle_mod.Oracle(pr)
    cells = o.enumerate()
    t_ns, _ = o.estimate(cells)
    d0, f0, t0 = o.round_state(cells, t_ns, pr.cap)
    dn, _, _ = o.round_state(cells, t_ns, pr.cap, policy=1)
    adm = dn >= 0
    assert adm.any()
    assert np.all(cells["G"][dn[adm]] == pr.ng[adm])
    assert (d0 >= 0).sum() >= 1
    # a state with running jobs: every running job keeps its type under NH
    run = np.where(d0 >= 0, d0, -1).astype(np.int64)
    rng = np.random.default_rng(cfg)
    run[rng.random(pr.n_jobs) < 0.3] = -1
    used = np.zeros(pr.n_types, np.int64)
    for j in np.where(run >= 0)[0]:
        used[cells["type"][run[j]]] += cells["G"][run[j]]
    free = (pr.cap - used).astype(np.int32)
    dh, _, _ = o.round_state(cells, t_ns, free, run_cell=run, policy=2)
    kept = (run >= 0) & (dh >= 0)
    assert kept.any()
    assert np.all(cells["type"][dh[kept]] == cells["type"][run[kept]])


def test_round_policy_nh_single_type_is_full_round(oracle_mod):
    """With one GPU type there is no type to change: NH == the full round."""
    for seed in range(12):
        pr = W.random_tiny(500 + seed, n_types=1, n_jobs=5)
        o = oracle_mod.Oracle(pr)
        cells = o.enumerate()
        t_ns, _ = o.estimate(cells)
        a = o.round_state(cells, t_ns, pr.cap)
        b = o.round_state(cells, t_ns, pr.cap, policy=2)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and a[2] == b[2]


# ---------------------------------------------------------------- deadline-aware variant (R-12)
def test_round_deadline_bound_hand(oracle_mod):
    """t_max filters options: round_state.json's state with
    J0's bound 90 leaves J0 only (0,4,80) -- G 4 > N_G 2, so no admissible
    option: J0 pending, J1 untouched; a running job keeps its (type, G) even
    when its own T exceeds its bound."""
    case = golden("round_state.json")
    pr, cells, t_ns = _round_problem(case, 1)
    run = np.full(pr.n_jobs, -1, np.int64)
    run[1] = [i for i in range(len(t_ns)) if cells["job"][i] == 1 and cells["G"][i] == 4][0]
    o = oracle_mod.Oracle(pr)
    dec, fa, tot = o.round_state(cells, t_ns, case["free"], run_cell=run,
                                 t_max=np.array([90, 50], np.int64))
    assert dec[0] == -1 and dec[1] == run[1] and list(fa) == [0] and tot == 1.0
    # without the bound the hand vector's scale-down happens (d1 expectation)
    dec, _, tot = o.round_state(cells, t_ns, case["free"], run_cell=run,
                                t_max=np.array([10 ** 12, 10 ** 12], np.int64))
    assert dec[0] >= 0 and tot == 1.5


def test_sim_deadlines_every_finished_job_meets_it(oracle_mod):
    """Deadline-aware simulation: every job that finishes does so by its
    deadline, and infinite deadlines reproduce the plain simulation."""
    from oracle import sim
    pr = W.subset(W.make_config(2), 8)
    pr.depth = 3
    o = oracle_mod.Oracle(pr)
    cells = o.enumerate()
    t_ns, _ = o.estimate(cells)
    it = W.iterations_for(pr, seed=2)
    plain = sim.simulate(o, cells, t_ns, it, 30)
    inf = sim.simulate(o, cells, t_ns, it, 30, deadlines=np.full(pr.n_jobs, 2 ** 62, np.int64))
    for k in ("first_start", "finish", "restarts", "state"):
        assert np.array_equal(plain[k], inf[k]), k
    dl = deadlines_for(pr, cells, t_ns, it, seed=7)
    r = sim.simulate(o, cells, t_ns, it, 30, deadlines=dl)
    done = r["state"] == 3
    assert np.all(r["finish"][done] <= dl[done])
    assert (r["state"] == 4).any() or done.all()


def deadlines_for(pr, cells, t_ns, it, seed):
    """Synthetic deadlines: submit + lambda * N * (fastest Cell's T), lambda ~ U[0.8, 2.5]."""
    rng = np.random.default_rng(seed)
    INF = np.iinfo(np.int64).max
    best = np.full(pr.n_jobs, INF, np.int64)
    np.minimum.at(best, cells["job"], t_ns)
    lam = rng.uniform(0.8, 2.5, pr.n_jobs)
    base = np.where(best == INF, 0, best).astype(np.float64) * np.asarray(it, np.float64)
    return (np.asarray(pr.submit, np.int64) * NS + (lam * base).astype(np.int64)).astype(np.int64)


# ---------------------------------------------------------------- opportunistic execution (R-14)
def test_opportunistic_hand_trace(oracle_mod):
    """PAPER.md:504-507 on a hand trace (tests/golden/sim_opportunistic.json)."""
    from oracle import sim
    fx = golden("sim_opportunistic.json")
    pr, cells, t_ns = _round_problem(fx, 0)
    it = [j["iters"] for j in fx["jobs"]]
    for key, opp in (("plain", False), ("opportunistic", True)):
        out = sim.simulate(oracle_mod.Oracle(pr), cells, t_ns, it, fx["penalty_s"], opportunistic=opp)
        e = fx["expect"][key]
        assert list(out["first_start"] // NS) == e["first_start_s"], key
        assert list(out["finish"] // NS) == e["finish_s"], key
        assert list(out["restarts"]) == e["restarts"], key
        assert np.all(out["state"] == 3), key


def test_opportunistic_invariants(oracle_mod):
    """With opportunistic execution every job still finishes at most once and
    never faster than its iterations on its fastest Cell; suspended jobs are
    counted as restarts."""
    from oracle import sim
    pr = W.subset(W.make_config(3), 120)
    o = oracle_mod.Oracle(pr)
    cells = o.enumerate()
    t_ns, _ = o.estimate(cells)
    it = W.iterations_for(pr)
    out = sim.simulate(o, cells, t_ns, it, 30, opportunistic=True)
    done = out["state"] == 3
    assert done.sum() + (out["state"] == 4).sum() + (out["state"] == 5).sum() == pr.n_jobs
    for j in np.where(done)[0]:
        best = t_ns[(cells["job"] == j) & (t_ns < np.iinfo(np.int64).max)].min()
        assert out["finish"][j] - out["first_start"][j] >= it[j] * best
