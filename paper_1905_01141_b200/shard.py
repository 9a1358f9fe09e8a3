"""Multi-GPU plumbing for the decode path: cells are sharded
over ranks in contiguous ranges; CBs never cross ranks, so the only
collectives are one SUM reduction of the counters and one MAX of the time."""
from __future__ import annotations

import torch

COUNTERS = ("n_cb", "n_crc_ok", "info_bits", "sum_k", "counted_ops")


def cells_for_rank(rank: int, world: int, n_cells: int) -> list[int]:
    """Contiguous, balanced cell range of ``rank`` (sizes differ by at most 1)."""
    per, extra = divmod(n_cells, world)
    lo = rank * per + min(rank, extra)
    return list(range(lo, lo + per + (1 if rank < extra else 0)))


def reduce_counters(values, elapsed_ms: float, dist=None, device="cpu"):
    """-> (dict of summed counters, max elapsed ms over ranks)."""
    c = torch.tensor([float(v) for v in values], dtype=torch.float64, device=device)
    t = torch.tensor([float(elapsed_ms)], dtype=torch.float64, device=device)
    if dist is not None and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(c, op=dist.ReduceOp.SUM)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return dict(zip(COUNTERS, (int(x) for x in c.tolist()))), t.item()
