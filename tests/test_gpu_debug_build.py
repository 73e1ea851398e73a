"""The kernels' device-side invariant checks (CRIUS_CHECK, -DCRIUS_DEBUG).

compute-sanitizer is refused on this GPU pool (profiles/r2/), so the library is
rebuilt with its bound checks compiled in (window, admitted-record, type-list
and option-pool bounds, option indices, DP argmin ranges): a violated bound
traps the kernel.  Round, estimate and round-state cases run in a child process
against that build and must still equal the oracle bit for bit.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_2403_16125_b200 import workload as W

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2403_16125_b200 as pkg
from paper_2403_16125_b200 import workload as W
cfg, variant, out, state = int(sys.argv[2]), (sys.argv[3] or None), sys.argv[4], sys.argv[5]
pr = W.make_config(cfg, variant=variant)
with pkg.Crius(pr) as cr:
    n, _, _ = cr.enumerate()
    res = cr.estimate()
    t_ns, plan, _ = pkg.decode(res)
    if state:
        z = np.load(state)
        dec, fa, tot = cr.schedule_round_state(res, z["free"], z["run_cell"])
    else:
        dec, fa, tot = cr.schedule_round(res)
np.savez(out, t=t_ns[:n], p=plan[:n], dec=dec, fa=fa, tot=np.float64(tot))
"""


@pytest.fixture(scope="module")
def debug_lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA GPU")
    from paper_2403_16125_b200 import build
    return build.build_debug()


def _child(lib, cfg, variant, out, state=""):
    env = dict(os.environ, CRIUS_LIB=lib)
    subprocess.run([sys.executable, "-c", CHILD, ROOT, str(cfg), variant or "", out, state],
                   env=env, check=True, timeout=600)
    return np.load(out)


@pytest.mark.parametrize("cfg,variant", [(2, None), (3, None), (4, None), (4, "pow2")])
def test_debug_build_parity(debug_lib, oracle_mod, tmp_path, cfg, variant):
    pr = W.make_config(cfg, variant=variant)
    o = oracle_mod.Oracle(pr)
    cells = o.enumerate()
    t_ns, plan = o.estimate(cells)
    do, fo, to = o.round(cells, t_ns)
    r = _child(debug_lib, cfg, variant, str(tmp_path / "d.npz"))
    assert np.array_equal(r["t"], t_ns) and np.array_equal(r["p"], plan)
    assert np.array_equal(r["dec"], do) and np.array_equal(r["fa"], fo) and float(r["tot"]) == to


def test_debug_build_round_state(debug_lib, oracle_mod, tmp_path):
    pr = W.make_config(3)
    o = oracle_mod.Oracle(pr)
    cells = o.enumerate()
    t_ns, _ = o.estimate(cells)
    run_cell = np.full(pr.n_jobs, -1, np.int64)
    used = np.zeros(pr.n_types, np.int64)
    for j in range(0, pr.n_jobs, 5):
        ids = np.nonzero((cells["job"] == j) & (t_ns < np.iinfo(np.int64).max))[0]
        if len(ids):
            c = ids[np.argmax(cells["G"][ids])]
            if used[cells["type"][c]] + cells["G"][c] <= pr.cap[cells["type"][c]]:
                run_cell[j] = c
                used[cells["type"][c]] += cells["G"][c]
    free = (pr.cap - used).astype(np.int32)
    do, fo, to = o.round_state(cells, t_ns, free, run_cell)
    st = str(tmp_path / "s.npz")
    np.savez(st, free=free, run_cell=run_cell)
    r = _child(debug_lib, 3, None, str(tmp_path / "d.npz"), st)
    assert np.array_equal(r["dec"], do) and np.array_equal(r["fa"], fo) and float(r["tot"]) == to
