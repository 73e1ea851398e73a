"""The round kernel's configuration paths vs the oracle.

k_round keeps the admitted-job records and per-type lists in shared memory
when its bound on their number fits (global memory beyond; CRIUS_ROUND_SMEM
caps the shared memory it may use, so 0 forces the global path), and its
batch width is the CTA size (CRIUS_ROUND_THREADS at build time).  The default
build takes the shared-memory path at every shipped config, so this test runs
full rounds in child processes with the global path forced and with other CTA
sizes, and compares decisions, free counts and the total with the oracle's,
bit for bit.  The round-state case (running multi-GPU jobs that ScaleResource
may shrink, so more jobs than free GPUs can be admitted) runs on the global
path too.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_2403_16125_b200 import workload as W

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

VARIANTS = {
    "rt512.so": ["CRIUS_ROUND_THREADS=512"],
    "rt1024.so": ["CRIUS_ROUND_THREADS=1024"],
}

CHILD = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2403_16125_b200 as pkg
from paper_2403_16125_b200 import workload as W
cfg, variant, out, state = int(sys.argv[2]), (sys.argv[3] or None), sys.argv[4], sys.argv[5]
pr = W.make_config(cfg, variant=variant)
with pkg.Crius(pr) as cr:
    cr.enumerate()
    res = cr.estimate()
    if state:
        z = np.load(state)
        dec, fa, tot = cr.schedule_round_state(res, z["free"], z["run_cell"])
    else:
        dec, fa, tot = cr.schedule_round(res)
    st = cr.round_stats()
np.savez(out, dec=dec, fa=fa, tot=np.float64(tot), smem=np.int64(st["records_in_smem"]))
"""


@pytest.fixture(scope="module")
def variants():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA GPU")
    from paper_2403_16125_b200 import build
    v = {name: build.build_variant(name, defs) for name, defs in VARIANTS.items()}
    v["global.so"] = build.build()  # the default library with shared memory capped at 0
    return v


def _run(path, cfg, variant, out, state="", smem_cap=None):
    env = dict(os.environ, CRIUS_LIB=path)
    if smem_cap is not None:
        env["CRIUS_ROUND_SMEM"] = str(smem_cap)
    subprocess.run([sys.executable, "-c", CHILD, ROOT, str(cfg), variant or "", out, state],
                   env=env, check=True, timeout=300)
    return np.load(out)


@pytest.mark.parametrize("cfg,variant", [(3, None), (4, None), (4, "pow2")])
def test_round_paths(variants, oracle_mod, tmp_path, cfg, variant):
    pr = W.make_config(cfg, variant=variant)
    o = oracle_mod.Oracle(pr)
    cells = o.enumerate()
    t_ns, _ = o.estimate(cells)
    do, fo, to = o.round(cells, t_ns)
    for name, path in variants.items():
        r = _run(path, cfg, variant, str(tmp_path / f"{name}.npz"),
                 smem_cap=0 if name == "global.so" else None)
        if name == "global.so":
            assert int(r["smem"]) == 0
        assert np.array_equal(r["dec"], do), name
        assert np.array_equal(r["fa"], fo), name
        assert float(r["tot"]) == to, name


@pytest.mark.parametrize("cfg", [3, 4])
def test_round_state_global_records(variants, oracle_mod, tmp_path, cfg):
    """Running jobs on large Cells, few free GPUs: ScaleResource shrinks them, so
    the admitted count exceeds the free GPUs (the records bound must count the
    running jobs' GPUs).  Global-record path vs the oracle."""
    pr = W.make_config(cfg)
    o = oracle_mod.Oracle(pr)
    cells = o.enumerate()
    t_ns, _ = o.estimate(cells)
    rng = np.random.default_rng(7)
    J, T = pr.n_jobs, pr.n_types
    job, typ, G = cells["job"], cells["type"], cells["G"]
    # every 7th job runs on its largest feasible Cell (while capacity lasts)
    run_cell = np.full(J, -1, np.int64)
    used = np.zeros(T, np.int64)
    cap = np.asarray(pr.cap, np.int64)
    for j in range(0, J, 7):
        ids = np.nonzero((job == j) & (t_ns < np.iinfo(np.int64).max))[0]
        if len(ids) == 0:
            continue
        c = ids[np.argmax(G[ids])]
        if used[typ[c]] + G[c] <= cap[typ[c]]:
            run_cell[j] = c
            used[typ[c]] += G[c]
    free = np.maximum(0, cap - used - rng.integers(0, 4, T)).astype(np.int32)
    do, fo, to = o.round_state(cells, t_ns, free, run_cell)
    st = str(tmp_path / "state.npz")
    np.savez(st, free=free, run_cell=run_cell)
    for name, path in variants.items():
        r = _run(path, cfg, None, str(tmp_path / f"s_{name}.npz"), state=st,
                 smem_cap=0 if name == "global.so" else None)
        assert np.array_equal(r["dec"], do), name
        assert np.array_equal(r["fa"], fo), name
        assert float(r["tot"]) == to, name
