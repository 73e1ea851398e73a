"""Pins of the NEXT-3 tuner oracle (Cell-guided parallelism tuning,
PAPER.md:392-412): SPEC's pruning examples, the work bound, containment
(tuned <= estimate, the estimated plan is in the pruned space), the full
assembled optimum as a lower bound, and brute force over the pruned product."""
import itertools

import numpy as np

from helpers import golden
from paper_2403_16125_b200 import workload as W

INF = np.iinfo(np.int64).max


def test_pruning_examples(oracle_mod):
    for c in golden("tuner_spec.json")["cases"]:
        ks = oracle_mod.tune_choices(c["g"], c["favour"] == "tp")
        assert ks == c["k"], c
        if "pairs" in c:
            assert [[c["g"] >> k, 1 << k] for k in ks] == c["pairs"]


def test_pruning_properties(oracle_mod):
    for e in range(0, 9):
        g = 1 << e
        dp, tp = oracle_mod.tune_choices(g, 0), oracle_mod.tune_choices(g, 1)
        assert dp[0] == 0 and tp[-1] == e              # dp-only / tp-only endpoints survive
        assert set(dp) | set(tp) == set(range(e + 1))  # the halves cover the axis
        assert set(dp) & set(tp)                       # half-hybrid in both
        assert len(dp) <= e // 2 + 2 and len(tp) <= e // 2 + 2   # SPEC.md:414 work bound
        if e % 2 == 0:
            assert set(dp) & set(tp) == {e // 2}       # sqrt(g) x sqrt(g) exactly


def test_tuned_between_full_optimum_and_estimate(oracle_mod):
    checked = 0
    for seed in range(25):
        pr = W.random_tiny(700 + seed, max_layers=6, n_types=1, n_jobs=2)
        o = oracle_mod.Oracle(pr)
        cells = o.enumerate()
        nB = 1 if pr.b_mode == 0 else len(pr.b_values)
        for form in (0, 1):
            t_est, b_est, k_est = o.estimate_assembled(cells, 1, form)
            t_full, _, _ = o.estimate_assembled(cells, 2, form)
            t_tun, b_tun, k_tun = o.tune_assembled(cells, form, k_est)
            for i in range(len(cells["G"])):
                assert t_full[i] <= t_tun[i] <= t_est[i]
                j, t, G, S = (int(cells[k][i]) for k in ("job", "type", "G", "S"))
                g = G // S
                ch = [oracle_mod.tune_choices(g, k_est[i][s] > 0) for s in range(S)]
                best = INF
                for bi in range(nB):
                    for ks in itertools.product(*ch):
                        lat, ok = o.assembled_cost(form, j, t, G, S, bi, np.array(ks, np.int8))
                        if ok:
                            best = min(best, lat)
                assert t_tun[i] == best
                if best < INF:
                    assert all(k_tun[i][s] in ch[s] for s in range(S))
                    lat, ok = o.assembled_cost(form, j, t, G, S, int(b_tun[i]), k_tun[i])
                    assert ok and lat == best
                checked += 1
    assert checked > 100
