"""Pins of the oracle trace simulator (NEXT-4): a hand-computed two-job
trace with and without resource scaling, and invariants on generated traces."""
import numpy as np

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
