"""Repetition sharding across GPUs (one process per GPU, torch.distributed).

Repetition trees are independent (cpsjoin.py:346-349) and
their seeds are host-derived and prefix-stable, so rank r runs trees
r, r + W, r + 2W, ...  The join then needs one real exchange step: the
verified pairs of every rank are gathered (sizes first, then padded
keys/similarities) and merged by sort + unique, and the counters are
all-reduced (sum for pre/candidates/results, max for max_depth and
peak_live_members).  The result is identical to the single-GPU join for any
world size because union, dedup, sums and maxima are order-independent.
"""
from __future__ import annotations

import numpy as np

from .core import Counters
from .cpsjoin import CPSJoinParams, JoinArrays, cpsjoin_self_arrays


def _gpu_local(emb, params: CPSJoinParams, rep_indices):
    return cpsjoin_self_arrays(emb, params, rep_indices=rep_indices)


def _all_gather_var(x: np.ndarray, device, group=None) -> np.ndarray:
    """Concatenate a 1-D int64/float64 array across ranks (rank order)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    n = torch.tensor([len(x)], dtype=torch.int64, device=device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    m = max(sizes) if sizes else 0
    buf = torch.zeros(max(m, 1), dtype=torch.from_numpy(x[:0]).dtype, device=device)
    if len(x):
        buf[:len(x)] = torch.from_numpy(np.ascontiguousarray(x)).to(device)
    outs = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(outs, buf, group=group)
    return np.concatenate([o[:s].cpu().numpy() for o, s in zip(outs, sizes)]) if world else x


def merge_results(parts_keys: np.ndarray, parts_sims: np.ndarray):
    """Sort + unique by pair key (first occurrence kept; duplicates carry
    identical similarities)."""
    keys, first = np.unique(parts_keys.astype(np.uint64), return_index=True)
    return keys, parts_sims[first]


def shard_reps(emb, params: CPSJoinParams, rank: int, world: int, group=None, device=None,
               local_join=None) -> JoinArrays:
    """cpsjoin_self over `world` ranks; every rank returns the full result."""
    if world <= 1:
        return (local_join or _gpu_local)(emb, params, None)
    import torch
    import torch.distributed as dist
    idx = np.arange(rank, params.repetitions, world, dtype=np.int64)
    local = (local_join or _gpu_local)(emb, params, idx)
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" \
            else torch.device("cpu")
    keys = (local.a.astype(np.uint64) << np.uint64(32)) | local.b.astype(np.uint64)
    all_keys = _all_gather_var(keys.view(np.int64), device, group).view(np.uint64)
    all_sims = _all_gather_var(local.similarity.astype(np.float64), device, group)
    all_caps = _all_gather_var(local.depth_cap_sizes.astype(np.int64), device, group)
    keys, sims = merge_results(all_keys, all_sims)
    c = local.counters
    s = torch.tensor([c.pre_candidates, c.candidates, c.results], dtype=torch.int64, device=device)
    mx = torch.tensor([c.max_depth, c.peak_live_members], dtype=torch.int64, device=device)
    dist.all_reduce(s, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=group)
    s, mx = s.cpu().tolist(), mx.cpu().tolist()
    counters = Counters(s[0], s[1], s[2], mx[0], mx[1])
    a = (keys >> np.uint64(32)).astype(np.int64)
    b = (keys & np.uint64(0xFFFFFFFF)).astype(np.int64)
    return JoinArrays(a, b, sims, counters, all_caps, dict(local.stats, world=world))
