"""Multi-GPU plumbing: one process per GPU, torch.distributed over NCCL.

The data path needs only three collectives, all here:
  * broadcast_graph  — rank 0's PCSR/signature buffers to every rank, once per graph
                       (PCSR is replicated, PAPER.md keeps one GPU; §8(e) 'Replication');
  * allreduce_counts — the per-query match counts after each rank ran its shard of M rows;
  * gather_tables    — optional: the rank-local match tables to rank 0 in rank order, which
                       reproduces the 1-GPU row order because shards are contiguous.
Every rank runs filter, plan and the levels before the shard level redundantly (identical,
cheap) and then keeps its F-weighted contiguous slice of rows (gsi_query_opts.shard_*).

Buffers are passed as torch tensors; on GPU they are zero-copy views of library memory
(gsi.torch_view), in the CPU tests (gloo) plain CPU tensors.
"""
from __future__ import annotations

from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np
import torch
import torch.distributed as dist


def broadcast_graph(meta: Optional[bytes], views: Optional[Sequence[torch.Tensor]],
                    alloc_like: Callable[[bytes], Tuple[object, Sequence[torch.Tensor]]], src: int = 0):
    """Replicate a graph.  On `src`, `meta`/`views` describe the built graph; on the other
    ranks `alloc_like(meta)` must return (graph, views) with the same buffer sizes, which this
    function then fills.  Returns (graph-or-None, views, meta)."""
    rank = dist.get_rank()
    obj = [meta if rank == src else None]
    dist.broadcast_object_list(obj, src=src)
    meta = obj[0]
    graph = None
    if rank != src:
        graph, views = alloc_like(meta)
    for v in views:
        if v.numel():
            dist.broadcast(v, src=src)
    return graph, views, meta


def broadcast_queries(queries: Optional[list], src: int = 0) -> list:
    obj = [queries]
    dist.broadcast_object_list(obj, src=src)
    return obj[0]


def allreduce_counts(counts: torch.Tensor) -> torch.Tensor:
    """Sum of the per-rank shard counts (uint64 semantics in int64 storage)."""
    dist.all_reduce(counts, op=dist.ReduceOp.SUM)
    return counts


def gather_tables(local, k: int, dst: int = 0, device: Optional[str] = None) -> Optional[np.ndarray]:
    """Concatenate the rank-local tables on `dst` in rank order (None elsewhere).  `local` is a
    numpy array or a torch tensor (a device-resident result table stays on the device: the
    gather then runs over NCCL with no host staging).  device=None: CUDA under NCCL, else CPU."""
    if device is None:
        device = f"cuda:{torch.cuda.current_device()}" if dist.get_backend() == "nccl" else "cpu"
    ws, rank = dist.get_world_size(), dist.get_rank()
    if isinstance(local, torch.Tensor):
        loc_t = local.to(device=device, dtype=torch.int32).reshape(-1, k)
    else:
        loc_t = torch.as_tensor(np.ascontiguousarray(local, dtype=np.int32).reshape(-1, k)).to(device)
    n = torch.tensor([loc_t.shape[0]], dtype=torch.int64, device=device)
    sizes = [torch.zeros(1, dtype=torch.int64, device=device) for _ in range(ws)]
    dist.all_gather(sizes, n)
    sizes = [int(s.item()) for s in sizes]
    mx = max(sizes) if sizes else 0
    buf = torch.zeros((max(mx, 1), k), dtype=torch.int32, device=device)
    if loc_t.shape[0]:
        buf[: loc_t.shape[0]] = loc_t
    outs = [torch.zeros_like(buf) for _ in range(ws)] if rank == dst else None
    if ws == 1:
        outs = [buf]
    else:
        dist.gather(buf, gather_list=outs, dst=dst)
    if rank != dst:
        return None
    return np.concatenate([o[:s].cpu().numpy() for o, s in zip(outs, sizes)]) if sum(sizes) else \
        np.zeros((0, k), np.int32)


def shard_bounds(F: np.ndarray, rank: int, world: int) -> Tuple[int, int]:
    """Host mirror of the device shard split (k_shard_bounds): with
    T = F[|M|], rank r keeps rows i with ceil(r T / W) <= F[i] < ceil((r+1) T / W), i.e. the
    contiguous row range [a_r, a_{r+1}) with a_r = lower_bound(F[0..|M|), ceil(r T / W)),
    a_0 = 0, a_W = |M|.  Ranges partition the rows and each rank's slot share is within one
    row's buffer of T / W."""
    nM = len(F) - 1
    T = int(F[nM])

    def a(r):
        if r <= 0:
            return 0
        if r >= world:
            return nM
        target = (r * T + world - 1) // world
        return int(np.searchsorted(F[:nM], target, side="left"))
    return a(rank), a(rank + 1)
