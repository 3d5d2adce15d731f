"""Independent instances across ranks: contiguous shards and
the one end-of-solve gather.

The reference solves every instance on its own (``SPEC.md:384``: instances
are independent; ``builders.py:355-372`` builds one per weight row,
``builders.py:302-318`` one per tomography slice).  Here each rank runs its
own persistent kernel over a contiguous block of instances with no
inter-GPU traffic, and a single collective at the end assembles the
per-instance results on every rank.  The same code runs on NCCL (GPU
tensors) and gloo (CPU tensors, the CPU tests).
"""

from __future__ import annotations

import numpy as np


def shard_rows(total: int, rank: int, world: int) -> np.ndarray:
    """Contiguous shard of ``rank``: ids [r*T/W, (r+1)*T/W) (sizes differ by <= 1)."""
    lo = (total * rank) // world
    hi = (total * (rank + 1)) // world
    return np.arange(lo, hi)


def gather_rows(ids: np.ndarray, fields: dict, total: int, group=None) -> tuple[np.ndarray, dict]:
    """All-gather per-instance arrays from every rank and return them sorted
    by instance id.  ``fields`` maps a name to an array whose first axis is
    aligned with ``ids`` (any trailing shape, int or float dtype; values of
    integer fields must fit in int64).  One all_gather of the counts, then
    one per field (padded to the largest shard).  Without an initialized
    process group this is the identity."""
    import torch
    import torch.distributed as dist

    ids = np.asarray(ids, dtype=np.int64)
    if not dist.is_initialized():
        order = np.argsort(ids, kind="stable")
        return ids[order], {k: np.asarray(v)[order] for k, v in fields.items()}
    world = dist.get_world_size(group)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    k = ids.size
    counts = torch.tensor([k], dtype=torch.int64, device=dev)
    all_counts = [torch.zeros_like(counts) for _ in range(world)]
    dist.all_gather(all_counts, counts, group=group)
    cnts = [int(c.item()) for c in all_counts]
    maxr = max(max(cnts), 1)

    def exchange(a: np.ndarray) -> np.ndarray:
        # each field travels in its own dtype (int8 codes: 1 byte per variable)
        a = np.asarray(a)
        tail = a.shape[1:]
        width = int(np.prod(tail)) if tail else 1
        npdt = a.dtype if a.dtype in (np.int8, np.uint8, np.int16, np.int32, np.int64, np.float32,
                                      np.float64) else (np.float64 if a.dtype.kind == "f" else np.int64)
        dt = torch.from_numpy(np.zeros(1, dtype=npdt)).dtype
        buf = torch.zeros((maxr, width), dtype=dt, device=dev)
        if k:
            buf[:k] = torch.from_numpy(np.ascontiguousarray(a.reshape(k, width), dtype=npdt)).to(dev)
        parts = [torch.empty_like(buf) for _ in range(world)]
        dist.all_gather(parts, buf, group=group)
        out = np.concatenate([parts[w][:cnts[w]].cpu().numpy() for w in range(world)])
        return out.reshape((out.shape[0],) + tail).astype(a.dtype, copy=False)

    all_ids = exchange(ids)
    order = np.argsort(all_ids, kind="stable")
    return all_ids[order], {name: exchange(v)[order] for name, v in fields.items()}
