"""The round kernel's capacity fallbacks vs the oracle.

k_round_greedy keeps the other-type move caches of the listed jobs in shared
memory up to kECap entries (global memory beyond) and stages their options in
a pool of kPool records (refills re-read global memory when a job got no
room); the per-type move loops run on CRIUS_SEQ_WARPS warps; the admitted-job
records live in shared memory up to kAdmSmem jobs (global memory beyond).  The default
build hits the fast paths on most recomputations, so this test rebuilds the
library with tiny capacities (every fallback taken) and with one warp per type,
runs full rounds in a child process (CRIUS_LIB selects the variant) and
compares the decisions with the oracle's, bit for bit.
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
    "caps_tiny.so": ["CRIUS_ECAP=4", "CRIUS_POOL=16", "CRIUS_SEQ_WARPS=1"],
    "caps_nopool.so": ["CRIUS_POOL=1", "CRIUS_SEQ_WARPS=2"],
    "adm_global.so": ["CRIUS_ADM_SMEM=16", "CRIUS_SEQ_WARPS=8"],
}

CHILD = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2403_16125_b200 as pkg
from paper_2403_16125_b200 import workload as W
cfg, variant, out = int(sys.argv[2]), (sys.argv[3] or None), sys.argv[4]
pr = W.make_config(cfg, variant=variant)
with pkg.Crius(pr) as cr:
    cr.enumerate()
    dec, fa, tot = cr.schedule_round(cr.estimate())
np.savez(out, dec=dec, fa=fa, tot=np.float64(tot))
"""


@pytest.fixture(scope="module")
def variants():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA GPU")
    from paper_2403_16125_b200 import build
    return {name: build.build_variant(name, defs) for name, defs in VARIANTS.items()}


@pytest.mark.parametrize("cfg,variant", [(3, None), (4, None), (4, "pow2")])
def test_round_fallback_paths(variants, oracle_mod, tmp_path, cfg, variant):
    pr = W.make_config(cfg, variant=variant)
    o = oracle_mod.Oracle(pr)
    cells = o.enumerate()
    t_ns, _ = o.estimate(cells)
    do, fo, to = o.round(cells, t_ns)
    for name, path in variants.items():
        out = str(tmp_path / f"{name}.npz")
        env = dict(os.environ, CRIUS_LIB=path)
        subprocess.run([sys.executable, "-c", CHILD, ROOT, str(cfg), variant or "", out],
                       env=env, check=True, timeout=300)
        r = np.load(out)
        assert np.array_equal(r["dec"], do), name
        assert np.array_equal(r["fa"], fo), name
        assert float(r["tot"]) == to, name
