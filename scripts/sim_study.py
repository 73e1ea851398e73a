"""Trace simulation study (NEXT-4): JCT / queueing / makespan / restarts of
the synthetic traces under search depth d and the
ablations NA / NH (--policies 0,1,2), GPU rounds."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2403_16125_b200 as pkg  # noqa: E402
from paper_2403_16125_b200 import sim  # noqa: E402
from paper_2403_16125_b200 import workload as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--jobs", type=int, default=0)
ap.add_argument("--depths", default="0,1,3")
ap.add_argument("--penalty", type=int, default=30)
ap.add_argument("--policies", default="0", help="0 full, 1 NA, 2 NH, 3 both")
ap.add_argument("--opportunistic", action="store_true",
                help="opportunistic execution (suspend later jobs for a waiting one, PAPER.md:504-507)")
ap.add_argument("--deadlines", type=float, default=0.0,
                help="> 0: deadline-aware runs, deadline = submit + U[lo, hi] x N x fastest T, "
                     "lo = this value, hi = 2.5 (ElasticFlow-style, PAPER.md:753-780)")
a = ap.parse_args()
base = W.make_config(a.config)
if a.jobs:
    base = W.subset(base, a.jobs)
it = W.iterations_for(base, seed=a.config)
for pol in [int(x) for x in a.policies.split(",")]:
    for d in [int(x) for x in a.depths.split(",")]:
        base.depth = d
        with pkg.Crius(base) as cr:
            dl = None
            if a.deadlines > 0:
                cr.enumerate()
                res = cr.estimate()
                tc = res[:cr.n_cells, 0].cpu().numpy()
                job = cr.cells()["job"].cpu().numpy()
                best = np.full(base.n_jobs, np.iinfo(np.int64).max, np.int64)
                np.minimum.at(best, job, tc)
                best = np.where(best == np.iinfo(np.int64).max, 0, best)
                lam = np.random.default_rng(a.config).uniform(a.deadlines, 2.5, base.n_jobs)
                dl = base.submit.astype(np.int64) * sim.NS + (lam * best * it).astype(np.int64)
            t0 = time.perf_counter()
            r = sim.simulate(cr, base, it, penalty_s=a.penalty, policy=pol, deadlines=dl,
                             opportunistic=a.opportunistic)
            dt = time.perf_counter() - t0
        s = r.summary(base.submit.astype(np.int64) * sim.NS)
        done = r.state == sim.DONE
        span = s["makespan_s"] or 0.0
        # cluster throughput: samples of the finished jobs per second of makespan
        s["samples_per_s"] = (float((it[done] * base.gb[done]).sum()) / span) if span else None
        if dl is not None:
            s["deadline_ratio"] = float((done & (r.finish <= dl)).sum() / base.n_jobs)
        s.update(config=base.name, depth=d, policy=["full", "NA", "NH", "NA+NH"][pol],
                 deadlines=a.deadlines or None, opportunistic=a.opportunistic,
                 wall_s=round(dt, 2), rounds_per_s=round(r.rounds / dt, 1))
        print(json.dumps(s), flush=True)
