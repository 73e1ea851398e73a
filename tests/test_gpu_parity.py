"""GPU path (libcrius through the C-ABI) vs the CPU oracle, element by element.

Contract (BASELINE.json north_star): Cells, stage splits, plan indices and
schedule decisions bit-exact; fp64 times (t_ns / 1e9) within 1e-9 relative
(they are in fact bit-identical: both sides produce the same int64 ns).
Every input is seeded and synthetic (paper_2403_16125_b200.workload).
"""
import os

import numpy as np
import pytest

from paper_2403_16125_b200 import workload as W

pytestmark = pytest.mark.gpu
INF = np.iinfo(np.int64).max


@pytest.fixture(scope="module")
def crius():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA GPU")
    from paper_2403_16125_b200 import build
    build.build()
    import paper_2403_16125_b200 as pkg
    return pkg


def gpu_run(pkg, pr, splits=False, free=None, round_=True):
    import torch
    with pkg.Crius(pr) as cr:
        n, p, u = cr.enumerate()
        cells = {k: v.cpu().numpy() for k, v in cr.cells().items()}
        sp = None
        if splits:
            sp = torch.full((max(u, 1) * cr.split_stride(),), -7, dtype=torch.int16, device="cuda")
        res = cr.estimate(splits=sp)
        t_ns, plan, flags = pkg.decode(res)
        out = dict(cells=cells, t_ns=t_ns[:n], plan=plan[:n], flags=flags[:n], n=n, p=p, u=u,
                   stride=cr.split_stride(), launches=cr.launches())
        if splits:
            out["splits"] = sp.cpu().numpy().reshape(u, -1)
        if round_:
            out["round"] = cr.schedule_round(res, free=free)
        return out


def oracle_run(oracle_mod, pr, free=None, c_range=None):
    o = oracle_mod.Oracle(pr)
    cells = o.enumerate()
    if c_range is None:
        t_ns, plan = o.estimate(cells)
    else:
        t_ns, plan = o.estimate(cells, *c_range)
    rnd = o.round(cells, t_ns, free_in=free) if c_range is None else None
    return o, cells, t_ns, plan, rnd


def assert_same(g, o_cells, o_t, o_plan, o_round=None):
    for k in ("job", "type", "G", "S", "nplans"):
        assert np.array_equal(g["cells"][k], o_cells[k]), k
    assert np.array_equal(g["t_ns"], o_t)
    assert np.array_equal(g["plan"], o_plan)
    assert np.array_equal(g["flags"], (o_plan >= 0).astype(np.int32))
    # fp64 contract: (double)t_ns / 1e9, relative error <= 1e-9
    fin = o_t < INF
    ts_g = g["t_ns"][fin].astype(np.float64) / 1e9
    ts_o = o_t[fin].astype(np.float64) / 1e9
    assert np.all(np.abs(ts_g - ts_o) <= 1e-9 * np.abs(ts_o))
    if o_round is not None:
        dg, fg, tg = g["round"]
        do, fo, to = o_round
        assert np.array_equal(dg, do)
        assert np.array_equal(fg, fo)
        assert tg == to and abs(tg - to) <= 1e-9 * abs(to)


def check_splits(g, o, pr, sample=None, seed=0):
    u = g["u"]
    units = range(u) if sample is None else np.random.default_rng(seed).choice(u, sample, replace=False)
    ucb = g["cells"]["unit_cell_begin"]
    for uu in units:
        row = g["splits"][uu]
        if ucb[uu + 1] == ucb[uu]:
            assert np.all(row == -1)
            continue
        j, t = divmod(int(uu), pr.n_types)
        smax = int(g["cells"]["S"][ucb[uu]:ucb[uu + 1]].max())
        si = 0
        while (1 << si) <= smax:
            S = 1 << si
            at = (S - 1) + si
            assert np.array_equal(row[at:at + S + 1], o.split(j, t, S)), (uu, S)
            si += 1
        assert np.all(row[(1 << si) - 1 + si:] == -1)


CONFIGS = [(1, None, True), (1, "sweep", True), (1, None, False), (2, None, True),
           (3, None, True), (4, None, True)]


@pytest.mark.parametrize("cfg,variant,jitter", CONFIGS)
def test_configs_bit_exact(crius, oracle_mod, cfg, variant, jitter):
    pr = W.make_config(cfg, variant=variant, jitter=jitter)
    g = gpu_run(crius, pr, splits=True)
    o, cells, t_ns, plan, rnd = oracle_run(oracle_mod, pr)
    assert (g["n"], g["p"]) == o.count()
    assert_same(g, cells, t_ns, plan, rnd)
    check_splits(g, o, pr, sample=None if g["u"] <= 400 else 300, seed=cfg)
    assert g["launches"] > 0


@pytest.mark.parametrize("seed", [101, 102, 103])
def test_other_seeds(crius, oracle_mod, seed):
    for cfg in (2, 3):
        pr = W.make_config(cfg, seed=seed)
        g = gpu_run(crius, pr)
        _, cells, t_ns, plan, rnd = oracle_run(oracle_mod, pr)
        assert_same(g, cells, t_ns, plan, rnd)


def test_cfg4_all_pow2(crius, oracle_mod):
    pr = W.make_config(4, variant="pow2")
    g = gpu_run(crius, pr, splits=True)
    _, cells, t_ns, plan, rnd = oracle_run(oracle_mod, pr)
    assert_same(g, cells, t_ns, plan, rnd)


@pytest.mark.parametrize("form", ["0", "1"])
def test_plan_forms(crius, oracle_mod, monkeypatch, form):
    """b_mode 0 evaluates plans either one per lane or one (plan, stage) per lane
    with butterflies over aligned lane groups; the library picks per launch by
    plans per unit (cfg4: per stage, the all-pow2 variant: per plan).
    CRIUS_EST_PER_STAGE forces each form on the configs that default to the
    other, and on small and tiny cases (ragged chunks, S up to 16)."""
    monkeypatch.setenv("CRIUS_EST_PER_STAGE", form)
    cases = [W.make_config(4, variant="pow2" if form == "1" else None), W.make_config(2)]
    cases += [W.random_tiny(s, max_layers=12, n_types=3, n_jobs=6) for s in range(10)]
    for pr in cases:
        g = gpu_run(crius, pr, splits=True)
        o, cells, t_ns, plan, rnd = oracle_run(oracle_mod, pr)
        assert_same(g, cells, t_ns, plan, rnd)


def test_cfg5_sampled_units(crius, oracle_mod):
    """Full-size cfg5 (96 layers, S <= 32, 7 B values): the GPU estimates every
    Cell; the oracle recomputes the Cells of 200 sampled units one by one."""
    pr = W.make_config(5)
    g = gpu_run(crius, pr, splits=True, round_=False)
    o = oracle_mod.Oracle(pr)
    cells = o.enumerate()  # the oracle's own Cell list, compared with the GPU's
    for k in ("job", "type", "G", "S", "nplans"):
        assert np.array_equal(g["cells"][k], cells[k]), k
    unit = cells["job"].astype(np.int64) * pr.n_types + cells["type"]
    ucb = np.searchsorted(unit, np.arange(g["u"] + 1), side="left")
    rng = np.random.default_rng(5)
    for uu in rng.choice(g["u"], 200, replace=False):
        c0, c1 = int(ucb[uu]), int(ucb[uu + 1])
        if c0 == c1:
            continue
        t_ns, plan = o.estimate(cells, c0, c1)
        assert np.array_equal(g["t_ns"][c0:c1], t_ns), uu
        assert np.array_equal(g["plan"][c0:c1], plan), uu
    check_splits(g, o, pr, sample=100, seed=55)


_PAR = {}


def _par_estimate(args):
    """Worker (a fresh forkserver process): rebuild the seeded problem and run
    the plain single-threaded oracle on Cells [c0, c1)."""
    import oracle
    cfg, jitter, scale, c0, c1 = args
    key = (cfg, jitter, scale)
    if _PAR.get("key") != key:
        pr = W.make_config(cfg, jitter=jitter, scale=scale)
        o = oracle.Oracle(pr)
        _PAR.update(key=key, o=o, cells=o.enumerate())
    return _PAR["o"].estimate(_PAR["cells"], c0, c1)


def oracle_estimate_parallel(cfg, jitter, cells, scale=1):
    """The oracle's estimate of every Cell, sharded over the host's cores by
    contiguous work-balanced Cell ranges (each worker runs the plain
    single-threaded oracle on its range)."""
    import multiprocessing as mp
    n = len(cells["job"])
    P = max(1, len(os.sched_getaffinity(0)))
    w = (cells["nplans"].astype(np.int64) * cells["S"]).cumsum()
    # 4 ranges per worker: the per-Cell cost varies, so finer pieces balance better
    Q = 4 * P
    cuts = [0] + [int(np.searchsorted(w, w[-1] * r / Q)) for r in range(1, Q)] + [n]
    ranges = [(cfg, jitter, scale, cuts[r], cuts[r + 1]) for r in range(Q) if cuts[r + 1] > cuts[r]]
    with mp.get_context("forkserver").Pool(P) as pool:
        parts = pool.map(_par_estimate, ranges, chunksize=1)
    return np.concatenate([p[0] for p in parts]), np.concatenate([p[1] for p in parts])


@pytest.mark.parametrize("jitter", [True, False])
def test_cfg5_full_space(crius, oracle_mod, jitter):
    """BASELINE config 5 (stress: 96-layer GPT jobs, S <= 32, all-pow2, the
    7-value B sweep; 1.56 M Cells, 41 M plans) over the WHOLE Cell space: every
    Cell's t_ns, plan and flags equal the oracle's (the oracle sharded over the
    host cores), and the round equals the oracle's round on its own estimates
    (decisions, free counts, fp64 total) -- PAPER.md:386-390 (every plan
    estimated), :432-464 (Alg. 1).  jitter False: u == 1, identical layers (ties)."""
    pr = W.make_config(5, jitter=jitter)
    g = gpu_run(crius, pr, splits=False, round_=True)
    o = oracle_mod.Oracle(pr)
    cells = o.enumerate()
    o_t, o_plan = oracle_estimate_parallel(5, jitter, cells)
    o_round = o.round(cells, o_t)
    assert_same(g, cells, o_t, o_plan, o_round)


@pytest.mark.parametrize("seed", range(40))
def test_random_tiny(crius, oracle_mod, seed):
    pr = W.random_tiny(seed, max_layers=12, n_types=3, n_jobs=6)
    g = gpu_run(crius, pr, splits=True)
    o, cells, t_ns, plan, rnd = oracle_run(oracle_mod, pr)
    assert_same(g, cells, t_ns, plan, rnd)
    check_splits(g, o, pr)


def test_edge_uniform_layers_max_ties(crius, oracle_mod):
    pr = W.make_config(5, jitter=False)
    pr_small = W.assemble("u", W.CFG4_CLUSTER, ["GPT96"] * 50, pr.ng[:50], pr.gb[:50],
                          np.random.default_rng(0), jitter=False, gpu_set=1, s_max=32, g_max=64,
                          b_mode=1, b_values=W.B_SWEEP.copy(), depth=3)
    g = gpu_run(crius, pr_small, splits=True)
    o, cells, t_ns, plan, rnd = oracle_run(oracle_mod, pr_small)
    assert_same(g, cells, t_ns, plan, rnd)
    check_splits(g, o, pr_small)


def test_edge_single_layer_and_S_equals_L(crius, oracle_mod):
    from helpers import problem_from
    jobs = [dict(c=[5], ng=4, gb=16, w=[10], act=[1], bnd=[3], tpv=[2], tpn=[1]),
            dict(c=[3, 1, 4, 1, 5, 9, 2, 6], ng=8, gb=64, w=[1] * 8, act=[2] * 8, bnd=[4] * 8,
                 tpv=[8] * 8, tpn=[2] * 8, submit=1, id=1)]
    pr = problem_from([dict(cap=16, gpn=4), dict(cap=8, gpn=2)], jobs, k_max=3, g_max=8,
                      gpu_set=1, s_max=64)
    g = gpu_run(crius, pr, splits=True)
    o, cells, t_ns, plan, rnd = oracle_run(oracle_mod, pr)
    assert_same(g, cells, t_ns, plan, rnd)
    check_splits(g, o, pr)
    assert (g["cells"]["S"] == 8).any()


def test_edge_memory_infeasible_everywhere(crius, oracle_mod):
    pr = W.make_config(2)
    pr.mem = np.ones_like(pr.mem)
    g = gpu_run(crius, pr)
    _, cells, t_ns, plan, rnd = oracle_run(oracle_mod, pr)
    assert_same(g, cells, t_ns, plan, rnd)
    assert np.all(g["plan"] == -1) and np.all(g["round"][0] == -2)


def test_edge_no_free_gpus(crius, oracle_mod):
    pr = W.make_config(3)
    free = np.zeros(pr.n_types, np.int32)
    g = gpu_run(crius, pr, free=free)
    _, cells, t_ns, plan, rnd = oracle_run(oracle_mod, pr, free=free)
    assert_same(g, cells, t_ns, plan, rnd)
    assert np.all(g["round"][0] < 0)


@pytest.mark.parametrize("depth", [0, 1, 2, 5])
def test_round_depths(crius, oracle_mod, depth):
    pr = W.make_config(3)
    pr.depth = depth
    g = gpu_run(crius, pr)
    _, cells, t_ns, plan, rnd = oracle_run(oracle_mod, pr)
    assert_same(g, cells, t_ns, plan, rnd)


@pytest.mark.parametrize("cfg,variant", [(4, None), (3, None)])
def test_rank_invariance_emulated(crius, oracle_mod, cfg, variant):
    """A7 on one GPU: the R = 2/4/8 ranks' contiguous unit ranges estimated one
    after another into padded chunks and compacted (the all-gather's layout)
    equal the ORACLE's records (t_ns, plan, flags) for every Cell, and the round
    on them equals the oracle's round (decisions, free counts, fp64 total) --
    north_star: every rank gets every Cell's best plan, decisions bit-exact."""
    import torch
    pkg = crius
    pr = W.make_config(cfg, variant=variant)
    _, o_cells, o_t, o_plan, (do, fo, to) = oracle_run(oracle_mod, pr)
    with pkg.Crius(pr) as cr:
        n, _, u = cr.enumerate()
        cells = {k: v.cpu().numpy() for k, v in cr.cells().items()}
        for world in (2, 4, 8):
            ub, cb = cr.partition(world)
            assert ub[0] == 0 and ub[-1] == u and cb[-1] == n and np.all(np.diff(ub) >= 0)
            chunk = int(max(cb[r + 1] - cb[r] for r in range(world)))
            gathered = torch.full((world * chunk, 2), -1, dtype=torch.int64, device="cuda")
            for r in range(world):
                cr.estimate(ub[r], ub[r + 1], out=gathered[r * chunk:(r + 1) * chunk])
            full = cr.compact(gathered, chunk, world, cb)
            t_ns, plan, flags = pkg.decode(full)
            dg, fg, tg = cr.schedule_round(full)
            assert_same({"cells": cells, "t_ns": t_ns[:n], "plan": plan[:n], "flags": flags[:n],
                         "round": (dg, fg, tg)}, o_cells, o_t, o_plan, (do, fo, to))


def test_update_profiles_and_repeat(crius, oracle_mod):
    pkg = crius
    a, b = W.make_config(3, seed=3), W.make_config(3, seed=3)
    b.c = (b.c * 2).astype(np.int32)
    with pkg.Crius(a) as cr:
        cr.enumerate()
        r1 = pkg.decode(cr.estimate())[0]
        r1b = pkg.decode(cr.estimate())[0]
        assert np.array_equal(r1, r1b)
        cr.update(b)
        cr.enumerate()
        r2 = pkg.decode(cr.estimate())[0][:cr.n_cells]
    _, _, t_ns, _, _ = oracle_run(oracle_mod, b)
    assert np.array_equal(r2, t_ns)


@pytest.mark.parametrize("cfg,chunks", [(2, 1), (2, 5), (3, 64), (4, 4)])
def test_update_estimate_pipelined(crius, oracle_mod, cfg, chunks):
    """crius_update_estimate (row upload pipelined against the per-range checks
    and estimates, records at global Cell index) from pinned host arrays: same
    records and splits as update + enumerate + estimate, and the oracle's."""
    import torch
    pkg = crius
    a, b = W.make_config(cfg, seed=5), W.make_config(cfg, seed=5)
    b.c = (b.c * 3).astype(np.int32)
    b.tpv = b.tpv + 11
    for k in ("c", "w", "act", "bnd", "tpv", "tpn"):
        setattr(b, k, torch.from_numpy(np.ascontiguousarray(getattr(b, k))).pin_memory().numpy())
    with pkg.Crius(a) as cr:
        cr.enumerate()
        cr.estimate()
        u = cr.n_units
        sp = torch.full((u * cr.split_stride(),), -7, dtype=torch.int16, device="cuda")
        got = cr.update_estimate(b, chunks=chunks, splits=sp)
        t_got, plan_got, _ = pkg.decode(got)
        n = cr.n_cells
        sp2 = torch.full_like(sp, -7)
        cr.update(b)
        cr.enumerate()
        ref = cr.estimate(splits=sp2)
        t_ref, plan_ref, _ = pkg.decode(ref)
    assert np.array_equal(t_got[:n], t_ref[:n]) and np.array_equal(plan_got[:n], plan_ref[:n])
    assert torch.equal(sp, sp2)
    _, _, o_t, o_plan, _ = oracle_run(oracle_mod, b)
    assert np.array_equal(t_got[:n], o_t) and np.array_equal(plan_got[:n], o_plan)


def test_update_estimate_rejects_bad_rows(crius, oracle_mod):
    """A row failing the bound checks: EINVAL naming the job, the records are
    not usable (estimate before a new enumeration is refused), and a valid batch
    afterwards works again."""
    pkg = crius
    a, b = W.make_config(2), W.make_config(2)
    b.c = b.c.copy()
    b.c.reshape(-1)[int(b.layer_off[7]) + 1] = 0
    with pkg.Crius(a) as cr:
        cr.enumerate()
        with pytest.raises(pkg.CriusError) as e:
            cr.update_estimate(b, chunks=3)
        assert e.value.code == 2
        with pytest.raises(pkg.CriusError):
            cr.estimate()
        got = pkg.decode(cr.update_estimate(a, chunks=3))[0][:cr.n_cells]
    _, _, o_t, _, _ = oracle_run(oracle_mod, a)
    assert np.array_equal(got, o_t)


def test_update_profiles_range(crius, oracle_mod):
    """crius_update_profiles_range: only the rows of jobs [j0, j1) are re-copied,
    so the library estimates only units of those jobs (a range reaching other
    jobs is rejected: their rows may be stale) and those Cells match the oracle
    on the new values."""
    pkg = crius
    a, b = W.make_config(3, seed=3), W.make_config(3, seed=3)
    b.c = (b.c * 2).astype(np.int32)
    b.bnd = b.bnd + 7
    j0, j1 = 300, 650
    T = a.n_types
    with pkg.Crius(a) as cr:
        cr.enumerate()
        cr.update(b, j0, j1)
        n, _, _ = cr.enumerate()
        cells = {k: v.cpu().numpy() for k, v in cr.cells().items()}
        with pytest.raises(pkg.CriusError) as e:
            cr.estimate()
        assert e.value.code == 2 and "did not upload" in str(e.value)
        with pytest.raises(pkg.CriusError):
            cr.estimate(j0 * T - 1, j1 * T)
        inr = (cells["job"] >= j0) & (cells["job"] < j1)
        got = pkg.decode(cr.estimate(j0 * T, j1 * T))[0][:int(inr.sum())]
    _, _, t_b, _, _ = oracle_run(oracle_mod, b)
    assert inr.any() and (~inr).any()
    assert np.array_equal(got, t_b[inr])
    with pkg.Crius(a) as cr:
        with pytest.raises(pkg.CriusError):
            cr.update(b, 5, a.n_jobs + 1)


def test_loader_rejects_overflow(crius):
    pkg = crius
    pr = W.make_config(2)
    pr.c = np.full_like(pr.c, 2 ** 31 - 1)
    pr.gb = np.full_like(pr.gb, 2 ** 20)   # 34 layers * 2^31 ns * 2^20 samples > 2^52
    with pytest.raises(pkg.CriusError) as e:
        pkg.Crius(pr)
    assert e.value.code == 2 and "2^52" in str(e.value)


@pytest.mark.parametrize("field,value,msg", [("c", 0, "compute_ns must be >= 1"),
                                             ("w", -1, "negative per-layer value"),
                                             ("act", 2 ** 58, "kst*sum(w) + GB*sum(act) >= 2^62"),
                                             ("tpv", 2 ** 58, "alpha-beta numerator >= 2^63")])
def test_loader_rejects_per_layer(crius, field, value, msg):
    """The §N0 checks run on the device per job (k_profile_check); a violation
    names the job and the bound, and the range update checks only its rows."""
    pkg = crius
    pr = W.make_config(2)
    bad = getattr(pr, field).copy()
    if field == "c":
        bad[0, 0, pr.layer_off[3]] = value
    else:
        bad[pr.layer_off[3]] = value
    setattr(pr, field, bad)
    with pytest.raises(pkg.CriusError) as e:
        pkg.Crius(pr)
    assert e.value.code == 2 and msg in str(e.value)
    if field != "c":
        assert "job 3" in str(e.value)
    good = W.make_config(2)
    with pkg.Crius(good) as cr:
        cr.update(pr, 4, pr.n_jobs)       # rows of job 3 are not re-checked
        with pytest.raises(pkg.CriusError):
            cr.update(pr, 0, pr.n_jobs)


def test_cfg5_x10_full_space(crius, oracle_mod):
    """100k-job stress (15.6 M Cells, 414 M plans): every Cell and the round
    against the oracle (its estimate sharded over the host cores), and the
    round's invariants (every admitted job on one of its own feasible Cells,
    capacity conserved)."""
    pkg = crius
    pr = W.make_config(5, scale=10)
    with pkg.Crius(pr) as cr:
        n, p, u = cr.enumerate()
        res = cr.estimate()
        t_g, p_g, f_g = pkg.decode(res)
        cg = {k: v.cpu().numpy() for k, v in cr.cells().items()}
        dec, fa, tot = cr.schedule_round(res)
    o = oracle_mod.Oracle(pr)
    cells = o.enumerate()
    o_t, o_plan = oracle_estimate_parallel(5, True, cells, scale=10)
    assert_same({"cells": cg, "t_ns": t_g[:n], "plan": p_g[:n], "flags": f_g[:n],
                 "round": (dec, fa, tot)}, cells, o_t, o_plan, o.round(cells, o_t))
    used = np.zeros(pr.n_types, np.int64)
    for j in np.where(dec >= 0)[0]:
        assert cells["job"][dec[j]] == j and t_g[dec[j]] < INF
        used[cells["type"][dec[j]]] += cells["G"][dec[j]]
    assert np.all(used + fa == pr.cap)


@pytest.mark.parametrize("cfg", [2, 4])
def test_exchange_world1_equals_oracle(crius, oracle_mod, cfg):
    """The fused exchange path on one GPU (world 1: the window is the rank's own):
    estimate kernel -> window stores + release flag -> device-side acquire wait ->
    round.  5 steps (both window halves, epochs 1..5), each bit-exact to the oracle;
    a sub-range per step exercises the empty-range signal too."""
    pr = W.make_config(cfg)
    o = oracle_mod.Oracle(pr)
    cells = o.enumerate()
    t_ref, p_ref = o.estimate(cells)
    d_ref, f_ref, tot_ref = o.round(cells, t_ref)
    with crius.Crius(pr) as cr:
        n, _, u = cr.enumerate()
        h = cr.exchange_init(0, 1)
        assert len(h) == 64
        cr.exchange_open(h)
        for step in range(5):
            cr.estimate_exchange(0, u)
            full = cr.exchange_wait()
            t_ns, plan, _ = crius.decode(full[:n])
            assert np.array_equal(t_ns, t_ref) and np.array_equal(plan, p_ref), step
            dec, fa, tot = cr.schedule_round(full)
            assert np.array_equal(dec, d_ref) and np.array_equal(fa, f_ref) and tot == tot_ref
        # an empty range still signals (the wait completes); the window keeps old values
        cr.estimate_exchange(0, 0)
        cr.exchange_wait()
        import torch
        torch.cuda.synchronize()
        cr.exchange_close()


def test_exchange_rejects_misuse(crius):
    pr = W.make_config(1)
    with crius.Crius(pr) as cr:
        cr.enumerate()
        with pytest.raises(Exception, match="not open"):
            cr.estimate_exchange(0, 1)
        with pytest.raises(Exception, match="world"):
            cr.exchange_init(0, 9)
        h = cr.exchange_init(0, 1, capacity=1)
        cr.exchange_open(h)
        with pytest.raises(Exception, match="exchange window"):
            cr.estimate_exchange(0, 1)
