"""Time crius_schedule_round alone (CUDA events, median of N) for configs; print round stats."""
import argparse
import os
import sys
import zlib

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2403_16125_b200 as pkg  # noqa: E402
from paper_2403_16125_b200 import workload as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="4,5,3")
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--stats", action="store_true")
a = ap.parse_args()
tag = os.path.basename(os.environ.get("CRIUS_LIB", "default"))
for cfg in a.configs.split(","):
    var = None
    if "-" in cfg:
        cfg, var = cfg.split("-")
    pr = W.make_config(int(cfg), variant=var)
    with pkg.Crius(pr) as cr:
        n, p, _ = cr.enumerate()
        res = cr.estimate()
        for _ in range(3):
            dec0 = cr.schedule_round(res)[0]
        ts = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            dec = cr.schedule_round(res)[0]
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
            assert (dec == dec0).all()
        ts.sort()
        st = cr.round_stats()
        print(f"{tag:16s} cfg{cfg}{'-'+var if var else ''}: round {ts[len(ts) // 2]:.4f} ms "
              f"admitted {st['admitted']} decisions-crc {zlib.crc32(dec0.tobytes()):08x}",
              flush=True)
        if a.stats:
            print("   ", st, flush=True)
