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
