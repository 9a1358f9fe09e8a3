"""Multi-GPU plumbing for the decode path: cells are sharded
over ranks in contiguous ranges; CBs never cross ranks, so the only
collectives are one SUM reduction of the counters and one MAX of the time
(after the timed region), plus -- for evidence, not for the path -- a gather
of per-cell output digests so that runs at different rank counts can be
compared CB for CB (the determinism contract)."""
from __future__ import annotations

import hashlib

import numpy as np
import torch

COUNTERS = ("n_cb", "n_crc_ok", "info_bits", "sum_k", "counted_ops")


def cells_for_rank(rank: int, world: int, n_cells: int) -> list[int]:
    """Contiguous, balanced cell range of ``rank`` (sizes differ by at most 1)."""
    per, extra = divmod(n_cells, world)
    lo = rank * per + min(rank, extra)
    return list(range(lo, lo + per + (1 if rank < extra else 0)))


def reduce_counters(values, elapsed_ms: float, dist=None, device="cpu"):
    """-> (dict of summed counters, max elapsed ms over ranks).  Counters travel
    as int64 (exact at any size); the time as float64."""
    c = torch.tensor([int(v) for v in values], dtype=torch.int64, device=device)
    t = torch.tensor([float(elapsed_ms)], dtype=torch.float64, device=device)
    if dist is not None and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(c, op=dist.ReduceOp.SUM)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return dict(zip(COUNTERS, (int(x) for x in c.tolist()))), t.item()


def cell_digests(desc: np.ndarray, cb_cell: np.ndarray, words: np.ndarray, crc_ok: np.ndarray) -> dict[int, str]:
    """Per cell: SHA-256 over its CBs in batch order of (the CB's ceil(K/32)
    packed output words, little-endian) || (its crc_ok byte).  A CB's outputs
    depend only on its own inputs, so a cell's digest is the same whatever
    the rank count or batch composition that decoded it."""
    words = np.ascontiguousarray(words).view(np.uint32)
    ok = np.ascontiguousarray(crc_ok, np.uint8)
    out: dict[int, hashlib._Hash] = {}
    for i in range(desc.size):
        c = int(cb_cell[i])
        h = out.get(c)
        if h is None:
            h = out[c] = hashlib.sha256()
        o, n = int(desc["bit_off"][i]), (int(desc["K"][i]) + 31) // 32
        h.update(words[o:o + n].tobytes())
        h.update(ok[i:i + 1].tobytes())
    return {c: h.hexdigest() for c, h in out.items()}


def gather_digests(local: dict, dist=None) -> dict:
    """Union of every rank's per-cell digests (gathered to all ranks)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return dict(local)
    parts = [None] * dist.get_world_size()
    dist.all_gather_object(parts, dict(local))
    merged: dict = {}
    for p in parts:
        for k, v in p.items():
            if k in merged and merged[k] != v:
                raise RuntimeError(f"cell {k} decoded differently by two ranks")
            merged[k] = v
    return merged


def combined_digest(cells: dict) -> str:
    """One SHA-256 over the sorted (cell, digest) pairs: equal for two runs iff
    they decoded the same cells to the same outputs."""
    h = hashlib.sha256()
    for k in sorted(cells):
        h.update(f"{k}:{cells[k]};".encode())
    return h.hexdigest()


def sha256_tensors(ts, chunk_bytes: int = 1 << 28) -> str:
    """SHA-256 of the concatenated bytes of tensors (device or host), copied to
    the host in bounded chunks."""
    h = hashlib.sha256()
    for t in ts:
        flat = t.reshape(-1)
        step = max(1, chunk_bytes // max(1, flat.element_size()))
        for i in range(0, flat.numel(), step):
            h.update(flat[i:i + step].cpu().numpy().tobytes())
    return h.hexdigest()
