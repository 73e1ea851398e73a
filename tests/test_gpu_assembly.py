"""GPU NEXT-1 (per-stage parallelism assembly) vs the brute-force oracle.

The best latency per Cell is unique and must be bit-exact; several assembled
plans can attain it, so the GPU's plan (microbatch index + per-stage tp) is
checked for validity: the oracle recomputes its latency, which must equal the
optimum."""
import numpy as np
import pytest

from paper_2403_16125_b200 import workload as W

pytestmark = pytest.mark.gpu
INF = np.iinfo(np.int64).max


@pytest.fixture(scope="module")
def pkg():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA GPU")
    from paper_2403_16125_b200 import build
    build.build()
    import paper_2403_16125_b200 as p
    return p


def run(pkg, pr, mode, form):
    import torch
    with pkg.Crius(pr) as cr:
        n, _, _ = cr.enumerate()
        ms = cr.max_stages()
        sk = torch.full((max(n, 1), ms), -9, dtype=torch.int8, device="cuda")
        res = cr.estimate_assembled(mode, form, stage_tp=sk)
        t_ns, b, fl = pkg.decode(res)
        return t_ns[:n], b[:n], fl[:n], sk.cpu().numpy()[:n]


def check(oracle_mod, pr, got, mode, form, sample=None):
    o = oracle_mod.Oracle(pr)
    cells = o.enumerate()
    idx = range(len(cells["G"])) if sample is None else sample
    t_g, b_g, f_g, sk_g = got
    for i in idx:
        t_o, _, _ = o.estimate_assembled(cells, mode, form, i, i + 1)
        assert t_g[i] == t_o[0], (i, t_g[i], t_o[0])
        assert f_g[i] == (t_o[0] < INF)
        if t_o[0] < INF:
            j, t, G, S = (int(cells[k][i]) for k in ("job", "type", "G", "S"))
            assert np.all(sk_g[i][S:] == -1)
            lat, ok = o.assembled_cost(form, j, t, G, S, int(b_g[i]), sk_g[i])
            assert ok and lat == t_g[i], (i, lat, t_g[i])
        else:
            assert b_g[i] == -1


@pytest.mark.parametrize("seed", range(25))
@pytest.mark.parametrize("mode,form", [(1, 0), (1, 1), (2, 0), (2, 1)])
def test_tiny_bruteforce(pkg, oracle_mod, seed, mode, form):
    pr = W.random_tiny(seed, max_layers=8, n_types=2, n_jobs=3)
    check(oracle_mod, pr, run(pkg, pr, mode, form), mode, form)


@pytest.mark.parametrize("form", [0, 1])
def test_cfg2_paper_assembly(pkg, oracle_mod, form):
    pr = W.make_config(2)
    check(oracle_mod, pr, run(pkg, pr, 1, form), 1, form)


def test_cfg1_all_factorisations(pkg, oracle_mod):
    for var in (None, "sweep"):
        pr = W.make_config(1, variant=var)
        for form in (0, 1):
            check(oracle_mod, pr, run(pkg, pr, 2, form), 2, form)


def test_cfg4_sampled_paper_assembly(pkg, oracle_mod):
    pr = W.make_config(4)
    got = run(pkg, pr, 1, 1)
    o = oracle_mod.Oracle(pr)
    cells = o.enumerate()
    rng = np.random.default_rng(4)
    small = np.where(cells["S"] <= 8)[0]
    check(oracle_mod, pr, got, 1, 1, sample=rng.choice(small, 300, replace=False))


# ---------------------------------------------------------------- NEXT-3 tuner
def run_tune(pkg, pr, favor_np, form):
    import torch
    with pkg.Crius(pr) as cr:
        n, _, _ = cr.enumerate()
        ms = cr.max_stages()
        fav = torch.from_numpy(np.ascontiguousarray(favor_np[:, :ms], np.int8)).cuda()
        sk = torch.full((max(n, 1), ms), -9, dtype=torch.int8, device="cuda")
        res = cr.tune_assembled(fav, form, stage_tp=sk)
        t_ns, b, fl = pkg.decode(res)
        return t_ns[:n], b[:n], fl[:n], sk.cpu().numpy()[:n]


@pytest.mark.parametrize("seed", range(20))
@pytest.mark.parametrize("form", [0, 1])
def test_tuner_seeded_favours(pkg, oracle_mod, seed, form):
    """Favours are a seeded input: the tuned optimum is unique -> bit-exact."""
    pr = W.random_tiny(900 + seed, max_layers=8, n_types=2, n_jobs=3)
    o = oracle_mod.Oracle(pr)
    cells = o.enumerate()
    ms = int(cells["S"].max())
    rng = np.random.default_rng(seed)
    favor = rng.integers(0, 2, size=(len(cells["G"]), ms)).astype(np.int8) * 3
    t_g, b_g, f_g, k_g = run_tune(pkg, pr, favor, form)
    t_o, _, _ = o.tune_assembled(cells, form, favor)
    assert np.array_equal(t_g, t_o)
    for i in range(len(t_o)):
        if t_o[i] == INF:
            assert b_g[i] == -1 and f_g[i] == 0
            continue
        j, t, G, S = (int(cells[k][i]) for k in ("job", "type", "G", "S"))
        ch = [oracle_mod.tune_choices(G // S, favor[i][s] > 0) for s in range(S)]
        assert all(k_g[i][s] in ch[s] for s in range(S))
        lat, ok = o.assembled_cost(form, j, t, G, S, int(b_g[i]), k_g[i])
        assert ok and lat == t_g[i]


def test_tuner_after_estimate_cfg2(pkg, oracle_mod):
    """Estimate (paper assembly) -> favours -> tune, all on the GPU: the tuned
    plan lies in the pruned space of the estimate's plan, attains the oracle's
    brute-force optimum of that space and never loses to the estimate."""
    pr = W.make_config(2)
    for form in (0, 1):
        t_e, b_e, f_e, k_e = run(pkg, pr, 1, form)
        t_t, b_t, f_t, k_t = run_tune(pkg, pr, k_e, form)
        o = oracle_mod.Oracle(pr)
        cells = o.enumerate()
        t_o, _, _ = o.tune_assembled(cells, form, k_e)
        assert np.array_equal(t_t, t_o)
        assert np.all(t_t <= t_e)
