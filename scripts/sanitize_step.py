"""Small hot-path runs for compute-sanitizer: cfg1/cfg2 estimate + round,
NEXT-1 assembly and NEXT-3 tuning, and a tiny random problem."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2403_16125_b200 as pkg  # noqa: E402
from paper_2403_16125_b200 import workload as W  # noqa: E402

for pr in (W.make_config(1), W.make_config(1, variant="sweep"), W.make_config(2),
           W.random_tiny(3, max_layers=8, n_types=3, n_jobs=5)):
    with pkg.Crius(pr) as cr:
        n, _, u = cr.enumerate()
        sp = torch.empty((u * cr.split_stride(),), dtype=torch.int16, device="cuda")
        res = cr.estimate(splits=sp)
        dec, fa, tot = cr.schedule_round(res)
        sk = torch.empty((n, cr.max_stages()), dtype=torch.int8, device="cuda")
        cr.estimate_assembled(1, 1, stage_tp=sk)
        cr.tune_assembled(sk, 1)
        ub, cb = cr.partition(2)
        ch = int(max(cb[1] - cb[0], cb[2] - cb[1]))
        g = cr.new_results(2 * ch)
        cr.estimate(ub[0], ub[1], out=g[:ch])
        cr.estimate(ub[1], ub[2], out=g[ch:])
        cr.compact(g, ch, 2, cb)
        torch.cuda.synchronize()
        print(pr.name, n, int((dec >= 0).sum()), tot)
print("sanitize ok")
