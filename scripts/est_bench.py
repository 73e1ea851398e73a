"""Time crius_estimate_cells alone (CUDA events, median of N) for a config."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2403_16125_b200 as pkg  # noqa: E402
from paper_2403_16125_b200 import workload as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="4,5")
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
tag = os.path.basename(os.environ.get("CRIUS_LIB", "default"))
for cfg in a.configs.split(","):
    var = None
    if "-" in cfg:
        cfg, var = cfg.split("-")
    pr = W.make_config(int(cfg), variant=var)
    with pkg.Crius(pr) as cr:
        n, p, _ = cr.enumerate()
        out = cr.new_results(n)
        for _ in range(3):
            cr.estimate(out=out)
        ts = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            cr.estimate(out=out)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        ms = ts[len(ts) // 2]
        print(f"{tag:24s} cfg{cfg}{'-'+var if var else ''}: estimate {ms:.4f} ms  {p / ms / 1e6:.3f} G plans/s", flush=True)
