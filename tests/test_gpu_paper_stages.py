"""GPU NEXT-2 (the paper's stage determination) vs the oracle, bit for bit.

crius_estimate_paper_stages must reproduce the oracle's cuts (the S-1
smallest boundary bytes, ties by the min-max R0 rule), the power-of-two GPUs
per stage and the best plan (t_ns, plan index) of every Cell; see
tests/test_paper_stages_pins.py for what pins the oracle to the paper."""
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


def run(pkg, pr):
    import torch
    with pkg.Crius(pr) as cr:
        n, _, u = cr.enumerate()
        ms = cr.max_stages()
        lg = torch.full((max(n, 1), ms), -9, dtype=torch.int8, device="cuda")
        sp = torch.full((max(u, 1) * cr.split_stride(),), -7, dtype=torch.int16, device="cuda")
        res = cr.estimate_paper_stages(splits=sp, stage_lg=lg)
        t_ns, plan, fl = pkg.decode(res)
        cells = {k: v.cpu().numpy() for k, v in cr.cells().items()}
        return dict(n=n, t=t_ns[:n], plan=plan[:n], flags=fl[:n], lg=lg.cpu().numpy()[:n],
                    splits=sp.cpu().numpy().reshape(max(u, 1), -1), cells=cells, ms=ms)


def check(oracle_mod, pr, g, sample=None):
    o = oracle_mod.Oracle(pr)
    cells = o.enumerate()
    idx = np.arange(g["n"]) if sample is None else np.asarray(sample)
    ucb = g["cells"]["unit_cell_begin"]
    for i in idx:
        i = int(i)
        t_o, p_o, lg_o = o.estimate_paper(cells, i, i + 1, kstride=g["ms"])
        assert g["t"][i] == t_o[0] and g["plan"][i] == p_o[0], (i, g["t"][i], t_o[0], g["plan"][i], p_o[0])
        assert g["flags"][i] == (p_o[0] >= 0)
        assert np.array_equal(g["lg"][i], lg_o[0]), i
        j, t, G, S = (int(cells[k][i]) for k in ("job", "type", "G", "S"))
        b, _ = o.paper_stages(j, t, G, S)
        u = j * pr.n_types + t
        assert ucb[u] <= i < ucb[u + 1]
        si = int(np.log2(S))
        at = (S - 1) + si
        assert np.array_equal(g["splits"][u][at:at + S + 1], b), (i, S)


@pytest.mark.parametrize("seed", range(30))
def test_tiny_random(pkg, oracle_mod, seed):
    pr = W.random_tiny(seed, max_layers=9, n_types=2, n_jobs=3)
    check(oracle_mod, pr, run(pkg, pr))


@pytest.mark.parametrize("cfg,variant", [(1, None), (1, "sweep"), (2, None), (3, None)])
def test_configs(pkg, oracle_mod, cfg, variant):
    pr = W.make_config(cfg, variant=variant)
    check(oracle_mod, pr, run(pkg, pr))


@pytest.mark.parametrize("cfg,variant", [(4, None), (4, "pow2")])
def test_cfg4_sampled(pkg, oracle_mod, cfg, variant):
    pr = W.make_config(cfg, variant=variant)
    g = run(pkg, pr)
    rng = np.random.default_rng(11)
    check(oracle_mod, pr, g, sample=rng.choice(g["n"], 300, replace=False))
