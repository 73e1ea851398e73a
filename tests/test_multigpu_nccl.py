"""N-GPU (NCCL over NVLink) run of the sharded hot path, one process per GPU:
contiguous unit ranges, one all_gather_into_tensor of the 16-byte Cell
records, device-side compaction, replicated round.  Every rank's records and
decisions must be byte-identical to the oracle's.  Skips with < 2 GPUs."""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _make(cfg):
    from paper_2403_16125_b200 import workload as W
    if isinstance(cfg, str):  # "tiny<seed>": one job, one GPU type -> one unit
        return W.random_tiny(int(cfg[4:]), n_types=1, n_jobs=1)
    return W.make_config(cfg)


def _worker_p2p(rank, world, port, cfg, steps, q):
    """The fused exchange: estimate kernel -> P2P stores into every rank's window
    + arrival flags; several steps (double-buffered windows, epochs)."""
    import torch.distributed as dist
    import paper_2403_16125_b200 as pkg
    from paper_2403_16125_b200 import sharded
    from paper_2403_16125_b200 import workload as W
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    pr = _make(cfg)
    outs = []
    with pkg.Crius(pr, device=rank) as cr:
        cr.enumerate()
        plan = sharded.ShardPlan(cr, world)
        xch = sharded.PeerExchange(cr, rank, world)
        for _ in range(steps):
            full = xch.estimate_all(plan)
            dec, fa, tot = cr.schedule_round(full)
            t_ns, plan_idx, _ = pkg.decode(full[:plan.n_cells])
            outs.append((t_ns, plan_idx, dec, fa, tot))
        xch.close()
    q.put((rank, outs))
    dist.destroy_process_group()


def _worker(rank, world, port, cfg, q):
    import torch.distributed as dist
    import paper_2403_16125_b200 as pkg
    from paper_2403_16125_b200 import sharded
    from paper_2403_16125_b200 import workload as W
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    pr = W.make_config(cfg)
    with pkg.Crius(pr, device=rank) as cr:
        cr.enumerate()
        plan = sharded.ShardPlan(cr, world)
        full = sharded.estimate_all(cr, plan, rank)
        t_ns, plan_idx, _ = pkg.decode(full[:plan.n_cells])
        dec, fa, tot = cr.schedule_round(full)
    q.put((rank, t_ns, plan_idx, dec, fa, tot))
    dist.destroy_process_group()


@pytest.mark.parametrize("cfg", [3, 4])
def test_nccl_sharded_equals_oracle(oracle_mod, cfg):
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    world = min(torch.cuda.device_count(), 4)
    import torch.multiprocessing as mp
    from paper_2403_16125_b200 import workload as W
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, cfg, q)) for r in range(world)]
    for p in ps:
        p.start()
    outs = [q.get(timeout=600) for _ in range(world)]
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    o = oracle_mod.Oracle(W.make_config(cfg))
    cells = o.enumerate()
    t_ref, p_ref = o.estimate(cells)
    d_ref, f_ref, tot_ref = o.round(cells, t_ref)
    for rank, t_ns, plan_idx, dec, fa, tot in outs:
        assert np.array_equal(t_ns, t_ref) and np.array_equal(plan_idx, p_ref), rank
        assert np.array_equal(dec, d_ref) and np.array_equal(fa, f_ref) and tot == tot_ref, rank


@pytest.mark.parametrize("cfg", [3, 4, "tiny7"])
def test_p2p_exchange_equals_oracle(oracle_mod, cfg):
    """("tiny7": a single unit, so every rank but one has an empty range and
    only signals.)"""
    """Fused estimate + NVLink P2P exchange on every GPU of the box (<= 8): every
    rank's records and decisions byte-identical to the oracle, 3 steps each."""
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    world = min(torch.cuda.device_count(), 8)
    import torch.multiprocessing as mp
    from paper_2403_16125_b200 import workload as W
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker_p2p, args=(r, world, port, cfg, 3, q)) for r in range(world)]
    for p in ps:
        p.start()
    outs = [q.get(timeout=600) for _ in range(world)]
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    o = oracle_mod.Oracle(_make(cfg))
    cells = o.enumerate()
    t_ref, p_ref = o.estimate(cells)
    d_ref, f_ref, tot_ref = o.round(cells, t_ref)
    for rank, steps in outs:
        assert len(steps) == 3
        for t_ns, plan_idx, dec, fa, tot in steps:
            assert np.array_equal(t_ns, t_ref) and np.array_equal(plan_idx, p_ref), rank
            assert np.array_equal(dec, d_ref) and np.array_equal(fa, f_ref) and tot == tot_ref, rank
