"""Trace simulation study (NEXT-4): JCT / queueing / makespan / restarts of
the synthetic traces under search depth d, GPU rounds."""
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
a = ap.parse_args()
base = W.make_config(a.config)
if a.jobs:
    base = W.subset(base, a.jobs)
it = W.iterations_for(base, seed=a.config)
for d in [int(x) for x in a.depths.split(",")]:
    base.depth = d
    with pkg.Crius(base) as cr:
        t0 = time.perf_counter()
        r = sim.simulate(cr, base, it, penalty_s=a.penalty)
        dt = time.perf_counter() - t0
    s = r.summary(base.submit.astype(np.int64) * sim.NS)
    s.update(config=base.name, depth=d, wall_s=round(dt, 2), rounds_per_s=round(r.rounds / dt, 1))
    print(json.dumps(s), flush=True)
