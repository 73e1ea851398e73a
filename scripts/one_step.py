"""One hot-path step (enumerate, estimate, round) on cuda:0 -- for ncu captures."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_16125_b200 as pkg  # noqa: E402
from paper_2403_16125_b200 import workload as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--variant", default=None)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
pr = W.make_config(a.config, variant=a.variant)
with pkg.Crius(pr, device=0) as cr:
    for _ in range(a.reps):
        cr.enumerate()
        res = cr.estimate()
        dec, fa, tot = cr.schedule_round(res)
    print("ok", cr.n_cells, cr.n_plans, int((dec >= 0).sum()), tot, cr.round_stats())
