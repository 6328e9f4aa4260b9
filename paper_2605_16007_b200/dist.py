"""Multi-GPU plumbing for the sharded search (P:L397-407 [sec 3.4]).

One process per GPU.  The index is sharded by contiguous id slices (every
inverted list is split across all ranks, R#21); rank 0 trains the
rotation P and the centroids and broadcasts them; the NCCL communicator of the
C library is bootstrapped by broadcasting its unique id through the torch
process group.  The exchange step itself (all-gather of the per-rank top-k +
merge by (dist, id)) runs inside ``rabitq_search_sharded``; ``allgather_topk``
is the same exchange through torch.distributed (used by the gloo tests and as
a fallback-free alternative when the caller already holds per-rank results).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(N: int, rank: int, world: int):
    """Contiguous id slice [lo, hi) of `rank` (sizes differ by at most 1)."""
    return (N * rank) // world, (N * (rank + 1)) // world


def broadcast_params(P: torch.Tensor, C: torch.Tensor, src: int = 0):
    """Rank `src`'s rotation P [D x D] and rotated centroids C [nlist x D] to all ranks (in place)."""
    dist.broadcast(P, src)
    dist.broadcast(C, src)
    return P, C


def share_unique_id(uid):
    """Broadcast rank 0's 128-byte NCCL unique id (bytes) through the process group."""
    obj = [uid if dist.get_rank() == 0 else None]
    dist.broadcast_object_list(obj, 0)
    return obj[0]


def allgather_topk(ids: torch.Tensor, dists: torch.Tensor):
    """Per-rank [nq x k] top-k -> [G x nq x k] on every rank (the exchange step)."""
    G = dist.get_world_size()
    gi = torch.empty((G,) + tuple(ids.shape), dtype=ids.dtype, device=ids.device)
    gd = torch.empty((G,) + tuple(dists.shape), dtype=dists.dtype, device=dists.device)
    if dist.get_backend() == "nccl":
        dist.all_gather_into_tensor(gi, ids.contiguous())
        dist.all_gather_into_tensor(gd, dists.contiguous())
    else:
        dist.all_gather(list(gi.unbind(0)), ids.contiguous())
        dist.all_gather(list(gd.unbind(0)), dists.contiguous())
    return gi, gd
