"""World-size-2 (and 3) CPU test of the multi-GPU orchestration (sharded.py)
over the gloo backend: contiguous unit ranges per rank, one all-gather of the
16-byte Cell records, removal of the per-rank padding, replicated round.

The per-rank estimate is done by a test-only stand-in context backed by the
CPU oracle (the CUDA path is covered by tests/test_gpu_parity.py, including
the same flow emulated on one GPU); what is under test here is the exchange.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2403_16125_b200 import sharded
from paper_2403_16125_b200 import workload as W

INF = np.iinfo(np.int64).max


class OracleCtx:
    """Same methods as Crius, on CPU tensors, estimates from the oracle."""

    def __init__(self, pr):
        import oracle
        self.pr = pr
        self.o = oracle.Oracle(pr)
        self.cells = self.o.enumerate()
        unit = self.cells["job"].astype(np.int64) * pr.n_types + self.cells["type"]
        self.n_units = pr.n_jobs * pr.n_types
        self.ucb = np.searchsorted(unit, np.arange(self.n_units + 1), side="left")
        self.n_cells = len(unit)

    def partition(self, world):
        ub = np.array([self.n_units * r // world for r in range(world + 1)], np.int64)
        return ub, self.ucb[ub].astype(np.int64)

    def new_results(self, n):
        return torch.full((max(n, 1), 2), -1, dtype=torch.int64)

    def estimate(self, u0, u1, out):
        c0, c1 = int(self.ucb[u0]), int(self.ucb[u1])
        t_ns, plan = self.o.estimate(self.cells, c0, c1)
        out[:c1 - c0, 0] = torch.from_numpy(t_ns)
        pf = np.stack([plan, (plan >= 0).astype(np.int32)], 1).astype(np.int32)
        out[:c1 - c0, 1] = torch.from_numpy(pf.view(np.int64).reshape(-1))
        return out

    def compact(self, gathered, chunk, world, cb, out=None):
        out = self.new_results(self.n_cells) if out is None else out
        for r in range(world):
            n = int(cb[r + 1] - cb[r])
            out[int(cb[r]):int(cb[r]) + n] = gathered[r * chunk:r * chunk + n]
        return out


def _worker(rank, world, port, cfg, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    pr = W.make_config(cfg)
    ctx = OracleCtx(pr)
    plan = sharded.ShardPlan(ctx, world)
    full = sharded.estimate_all(ctx, plan, rank)
    t_ns = full[:plan.n_cells, 0].numpy().copy()
    dec, fa, tot = ctx.o.round(ctx.cells, t_ns)
    q.put((rank, t_ns, dec, fa, tot))
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,cfg", [(2, 2), (2, 3), (3, 2)])
def test_sharded_flow_gloo(world, cfg, oracle_mod):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, cfg, q)) for r in range(world)]
    for p in ps:
        p.start()
    outs = [q.get(timeout=300) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    o = oracle_mod.Oracle(W.make_config(cfg))
    cells = o.enumerate()
    t_ref, _ = o.estimate(cells)
    d_ref, f_ref, tot_ref = o.round(cells, t_ref)
    for rank, t_ns, dec, fa, tot in outs:
        assert np.array_equal(t_ns, t_ref), rank
        assert np.array_equal(dec, d_ref) and np.array_equal(fa, f_ref) and tot == tot_ref
