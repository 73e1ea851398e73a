"""Multi-GPU sharding of the Cell space.

The unit (job, GPU type) is the independent piece of work: its stage DP, every
Cell (G, S) and every plan depend only on that job's profile rows and that
type's parameters.  Each rank estimates one contiguous, work-balanced range of
units (crius_partition_units), so its Cells are one contiguous range; ONE
all-gather (NCCL over NVLink 5 / NVSwitch through torch.distributed) gives
every rank every Cell's 16-byte record, the per-rank padding is removed on the
device (crius_compact_gathered), and every rank runs the same deterministic
round -- no further exchange is needed.

`ctx` is a `Crius` context (or anything with the same partition / new_results /
estimate / compact methods).
"""
from __future__ import annotations


class ShardPlan:
    """Unit/Cell ranges of every rank and the padded chunk size."""

    def __init__(self, ctx, world):
        self.world = world
        self.unit_begin, self.cell_begin = ctx.partition(world)
        self.chunk = int(max(self.cell_begin[r + 1] - self.cell_begin[r] for r in range(world)))
        self.n_cells = int(self.cell_begin[world])

    def job_range(self, rank, n_types):
        """Jobs whose units (job * n_types + type) fall in rank's unit range: the
        per-layer profile rows that rank needs (crius_update_profiles_range)."""
        u0, u1 = int(self.unit_begin[rank]), int(self.unit_begin[rank + 1])
        if u1 <= u0:
            return 0, 0
        return u0 // n_types, (u1 + n_types - 1) // n_types


def estimate_all(ctx, plan: ShardPlan, rank, mine=None, gathered=None, full=None, group=None):
    """Estimate this rank's range, all-gather all ranks' records, compact.
    Returns the full [n_cells, 2] record tensor (identical on every rank)."""
    import torch.distributed as dist
    w = plan.world
    if mine is None:
        mine = ctx.new_results(plan.chunk)
    ctx.estimate(int(plan.unit_begin[rank]), int(plan.unit_begin[rank + 1]), out=mine)
    if w == 1:
        return mine
    if gathered is None:
        gathered = ctx.new_results(w * plan.chunk)
    dist.all_gather_into_tensor(gathered, mine[:plan.chunk], group=group)
    return ctx.compact(gathered, plan.chunk, w, plan.cell_begin, out=full)


class PeerExchange:
    """The fused exchange (crius_exchange_*): the estimate kernel stores every
    Cell record into every rank's window over NVLink peer memory and signals
    per-rank arrival flags -- no NCCL all-gather, no compaction.  Setup exchanges
    the 64-byte CUDA IPC handles once over the process group (plumbing only)."""

    def __init__(self, ctx, rank, world, capacity=None, group=None):
        import torch
        import torch.distributed as dist
        self.ctx, self.rank, self.world = ctx, rank, world
        h = ctx.exchange_init(rank, world, capacity)
        mine = torch.frombuffer(bytearray(h), dtype=torch.uint8).to(f"cuda:{ctx.device}")
        allh = torch.empty(world * 64, dtype=torch.uint8, device=f"cuda:{ctx.device}")
        dist.all_gather_into_tensor(allh, mine, group=group)
        ctx.exchange_open(allh.cpu().numpy().tobytes())
        dist.barrier(group=group)  # every window is mapped before anyone stores into it

    def estimate_all(self, plan: ShardPlan, stream=None):
        """This rank's unit range -> every rank's window; returns all n_cells
        records (a view of this rank's window, valid until the step after next)."""
        self.ctx.estimate_exchange(int(plan.unit_begin[self.rank]),
                                   int(plan.unit_begin[self.rank + 1]), stream=stream)
        return self.ctx.exchange_wait(stream=stream)

    def close(self):
        self.ctx.exchange_close()
