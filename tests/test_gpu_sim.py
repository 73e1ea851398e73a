"""NEXT-4: the product trace simulator (GPU rounds, paper_2403_16125_b200.sim)
vs the oracle simulator: identical start/finish times, restarts and final
states on generated traces."""
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


@pytest.mark.parametrize("cfg,n,depth,pen", [(2, 8, 3, 30), (3, 150, 3, 30), (3, 150, 0, 30),
                                             (3, 300, 1, 120)])
def test_sim_matches_oracle(pkg, oracle_mod, cfg, n, depth, pen):
    from oracle import sim as osim
    from paper_2403_16125_b200 import sim
    pr = W.subset(W.make_config(cfg), n)
    pr.depth = depth
    it = W.iterations_for(pr, seed=cfg)
    with pkg.Crius(pr) as cr:
        got = sim.simulate(cr, pr, it, penalty_s=pen)
    o = oracle_mod.Oracle(pr)
    cells = o.enumerate()
    t_ns, _ = o.estimate(cells)
    want = osim.simulate(o, cells, t_ns, it, pen)
    assert got.rounds == want["rounds"]
    assert np.array_equal(got.first_start, want["first_start"])
    assert np.array_equal(got.finish, want["finish"])
    assert np.array_equal(got.restarts, want["restarts"])
    assert np.array_equal(got.state, want["state"])


@pytest.mark.parametrize("policy", [1, 2, 3])
def test_sim_policy_matches_oracle(pkg, oracle_mod, policy):
    """The ablation runs (NA / NH / both) of the simulator match the oracle's."""
    from oracle import sim as osim
    from paper_2403_16125_b200 import sim
    pr = W.subset(W.make_config(3), 150)
    it = W.iterations_for(pr, seed=3)
    with pkg.Crius(pr) as cr:
        got = sim.simulate(cr, pr, it, penalty_s=30, policy=policy)
    o = oracle_mod.Oracle(pr)
    cells = o.enumerate()
    t_ns, _ = o.estimate(cells)
    want = osim.simulate(o, cells, t_ns, it, 30, policy=policy)
    assert got.rounds == want["rounds"]
    assert np.array_equal(got.first_start, want["first_start"])
    assert np.array_equal(got.finish, want["finish"])
    assert np.array_equal(got.restarts, want["restarts"])
    assert np.array_equal(got.state, want["state"])


@pytest.mark.parametrize("cfg,n,policy", [(2, 8, 0), (3, 150, 0), (3, 150, 2)])
def test_sim_deadlines_match_oracle(pkg, oracle_mod, cfg, n, policy):
    """The deadline-aware simulation (early drops + t_max-bounded options)
    matches the oracle's; finished jobs meet their deadlines."""
    from oracle import sim as osim
    from paper_2403_16125_b200 import sim
    from test_sim_pins import deadlines_for
    pr = W.subset(W.make_config(cfg), n)
    pr.depth = 3
    it = W.iterations_for(pr, seed=cfg)
    o = oracle_mod.Oracle(pr)
    cells = o.enumerate()
    t_ns, _ = o.estimate(cells)
    dl = deadlines_for(pr, cells, t_ns, it, seed=cfg + 40)
    with pkg.Crius(pr) as cr:
        got = sim.simulate(cr, pr, it, penalty_s=30, policy=policy, deadlines=dl)
    want = osim.simulate(o, cells, t_ns, it, 30, policy=policy, deadlines=dl)
    assert got.rounds == want["rounds"]
    for k in ("first_start", "finish", "restarts", "state"):
        assert np.array_equal(getattr(got, k), want[k]), k
    done = got.state == sim.DONE
    assert np.all(got.finish[done] <= dl[done])


@pytest.mark.parametrize("cfg,n,depth,policy,ddl", [(2, 8, 0, 0, False), (3, 150, 3, 0, False),
                                                   (3, 150, 0, 0, False), (3, 150, 3, 2, True)])
def test_sim_opportunistic_matches_oracle(pkg, oracle_mod, cfg, n, depth, policy, ddl):
    """Opportunistic execution (R-14; with NH and deadlines in the last case):
    suspensions, resumptions and every event time identical to the oracle's."""
    from oracle import sim as osim
    from paper_2403_16125_b200 import sim
    from test_sim_pins import deadlines_for
    pr = W.subset(W.make_config(cfg), n)
    pr.depth = depth
    it = W.iterations_for(pr, seed=cfg)
    o = oracle_mod.Oracle(pr)
    cells = o.enumerate()
    t_ns, _ = o.estimate(cells)
    dl = deadlines_for(pr, cells, t_ns, it, seed=cfg + 50) if ddl else None
    with pkg.Crius(pr) as cr:
        got = sim.simulate(cr, pr, it, penalty_s=30, policy=policy, deadlines=dl, opportunistic=True)
    want = osim.simulate(o, cells, t_ns, it, 30, policy=policy, deadlines=dl, opportunistic=True)
    assert got.rounds == want["rounds"]
    for k in ("first_start", "finish", "restarts", "state"):
        assert np.array_equal(getattr(got, k), want[k]), k
