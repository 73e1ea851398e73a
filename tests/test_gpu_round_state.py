"""GPU NEXT-4 round from a cluster state vs the oracle (bit-exact decisions,
free counts and fp64 total) on random states: a random active subset, some
active jobs running on Cells chosen by an earlier round."""
import numpy as np
import pytest

from paper_2403_16125_b200 import workload as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA GPU")
    from paper_2403_16125_b200 import build
    build.build()
    import paper_2403_16125_b200 as p
    return p


@pytest.mark.parametrize("cfg,seed", [(2, 1), (3, 2), (3, 3), (4, 4)])
def test_random_states(pkg, oracle_mod, cfg, seed):
    pr = W.make_config(cfg)
    o = oracle_mod.Oracle(pr)
    cells = o.enumerate()
    t_ns, _ = o.estimate(cells)
    rng = np.random.default_rng(seed)
    with pkg.Crius(pr) as cr:
        cr.enumerate()
        res = cr.estimate()
        # state 1: half the jobs active, run a round, keep its admissions running
        act = (rng.random(pr.n_jobs) < 0.5).astype(np.uint8)
        dg, fg, tg = cr.schedule_round_state(res, pr.cap, active=act)
        do, fo, to = o.round_state(cells, t_ns, pr.cap, active=act)
        assert np.array_equal(dg, do) and np.array_equal(fg, fo) and tg == to
        run = np.where(dg >= 0, dg, -1).astype(np.int64)
        # state 2: a quarter of the running jobs finished, new jobs arrive
        done = (run >= 0) & (rng.random(pr.n_jobs) < 0.25)
        run[done] = -1
        act2 = act.copy()
        act2[done] = 0
        act2[(act == 0) & (rng.random(pr.n_jobs) < 0.5)] = 1
        used = np.zeros(pr.n_types, np.int64)
        for j in np.where(run >= 0)[0]:
            used[cells["type"][run[j]]] += cells["G"][run[j]]
        free = (pr.cap - used).astype(np.int32)
        for d in (pr.depth, 0, 1):
            pr.depth = d
            o2 = oracle_mod.Oracle(pr)
            with pkg.Crius(pr) as cr2:
                cr2.enumerate()
                r2 = cr2.estimate()
                dg, fg, tg = cr2.schedule_round_state(r2, free, run_cell=run, active=act2)
            do, fo, to = o2.round_state(cells, t_ns, free, run_cell=run, active=act2)
            assert np.array_equal(dg, do), d
            assert np.array_equal(fg, fo) and tg == to, d


@pytest.mark.parametrize("cfg,seed,policy", [(2, 5, 1), (3, 6, 1), (3, 7, 2), (4, 8, 2), (3, 9, 3),
                                             (4, 10, 3)])
def test_policy_states(pkg, oracle_mod, cfg, seed, policy):
    """NEXT-4 ablations (NA = 1, NH = 2, both = 3) on random cluster states:
    decisions, free counts and fp64 total bit-exact to the oracle."""
    pr = W.make_config(cfg)
    o = oracle_mod.Oracle(pr)
    cells = o.enumerate()
    t_ns, _ = o.estimate(cells)
    rng = np.random.default_rng(seed)
    with pkg.Crius(pr) as cr:
        cr.enumerate()
        res = cr.estimate()
        cr.set_round_policy(policy)
        act = (rng.random(pr.n_jobs) < 0.6).astype(np.uint8)
        dg, fg, tg = cr.schedule_round_state(res, pr.cap, active=act)
        do, fo, to = o.round_state(cells, t_ns, pr.cap, active=act, policy=policy)
        assert np.array_equal(dg, do) and np.array_equal(fg, fo) and tg == to
        # second state: the admitted jobs run, some finish, new ones arrive
        run = np.where(dg >= 0, dg, -1).astype(np.int64)
        run[rng.random(pr.n_jobs) < 0.25] = -1
        act2 = act.copy()
        act2[(act == 0) & (rng.random(pr.n_jobs) < 0.5)] = 1
        act2[(run < 0) & (dg >= 0)] = 0
        used = np.zeros(pr.n_types, np.int64)
        for j in np.where(run >= 0)[0]:
            used[cells["type"][run[j]]] += cells["G"][run[j]]
        free = (pr.cap - used).astype(np.int32)
        dg, fg, tg = cr.schedule_round_state(res, free, run_cell=run, active=act2)
        do, fo, to = o.round_state(cells, t_ns, free, run_cell=run, active=act2, policy=policy)
        assert np.array_equal(dg, do) and np.array_equal(fg, fo) and tg == to


@pytest.mark.parametrize("cfg,seed,policy", [(2, 11, 0), (3, 12, 0), (4, 13, 0), (3, 14, 3)])
def test_deadline_bound_states(pkg, oracle_mod, cfg, seed, policy):
    """Deadline bounds (R-12) on random states: per-job t_max around the jobs'
    own option times (some bind, some not), running jobs exempt on their
    (type, G); bit-exact to the oracle."""
    pr = W.make_config(cfg)
    o = oracle_mod.Oracle(pr)
    cells = o.enumerate()
    t_ns, _ = o.estimate(cells)
    INF = np.iinfo(np.int64).max
    rng = np.random.default_rng(seed)
    best = np.full(pr.n_jobs, INF, np.int64)
    np.minimum.at(best, cells["job"], t_ns)
    scale = rng.uniform(0.9, 1.6, pr.n_jobs)
    tmax = np.where(best == INF, -1, (np.where(best == INF, 0, best) * scale).astype(np.int64))
    with pkg.Crius(pr) as cr:
        cr.enumerate()
        res = cr.estimate()
        cr.set_round_policy(policy)
        dg0, _, _ = cr.schedule_round_state(res, pr.cap)
        run = np.where(dg0 >= 0, dg0, -1).astype(np.int64)
        run[rng.random(pr.n_jobs) < 0.4] = -1
        used = np.zeros(pr.n_types, np.int64)
        for j in np.where(run >= 0)[0]:
            used[cells["type"][run[j]]] += cells["G"][run[j]]
        free = (pr.cap - used).astype(np.int32)
        cr.set_deadline_bounds(tmax)
        dg, fg, tg = cr.schedule_round_state(res, free, run_cell=run)
        cr.set_deadline_bounds(None)
        do0, _, _ = o.round_state(cells, t_ns, pr.cap, policy=policy)
        assert np.array_equal(dg0, do0)
        do, fo, to = o.round_state(cells, t_ns, free, run_cell=run, policy=policy, t_max=tmax)
        assert np.array_equal(dg, do) and np.array_equal(fg, fo) and tg == to
