"""Multi-GPU CPSJoin: set-sharded embedding + repetition sharding (one
process per GPU, torch.distributed over NCCL).

Embedding is per set: `embed_sharded` runs K1 on each rank's n/W slice of
the sets and all-gathers the value and sketch rows (NVLink), so the
dominant preprocessing cost divides by W.

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


def shard_range(n: int, rank: int, world: int) -> tuple[int, int, int]:
    """Set shard of `rank`: [lo, hi) with a common padded size S."""
    S = -(-n // world) if n else 0
    lo = min(n, rank * S)
    return lo, min(n, lo + S), S


def _gpu_k1(eparams, sketch, d_tok, d_off, d, lo, hi, vals_out, sk_out):
    """K1 over sets [lo, hi) of a device CSR into shard buffers (values
    skipped when eparams is None, sketches when sketch is None)."""
    import torch

    from ._native import Context
    from .hashing import sketch_family
    ctx = Context.get()
    n_loc = hi - lo
    if n_loc <= 0:
        return
    max_token = min(int(d) - 1, 0xFFFFFFFF) if d else 0xFFFFFFFF
    stream = torch.cuda.current_stream().cuda_stream
    offp = d_off.data_ptr() + 8 * lo
    if eparams is not None:
        ctx.check(ctx.lib.cpsj_minhash_sketch(ctx.handle, eparams.device(ctx).handle, d_tok.data_ptr(), offp,
                                              n_loc, max_token, vals_out.data_ptr(), None, stream))
    if sketch is not None:
        ctx.check(ctx.lib.cpsj_minhash_sketch(ctx.handle, sketch_family(*sketch).device(ctx).handle,
                                              d_tok.data_ptr(), offp, n_loc, max_token, None, sk_out.data_ptr(),
                                              stream))


def _gather_rows(shard, world: int, group=None):
    """All-gather equal-size row shards into one (world * S, ...) tensor."""
    import torch
    import torch.distributed as dist
    if dist.get_backend(group) == "nccl":
        out = torch.empty((world * shard.shape[0],) + tuple(shard.shape[1:]), dtype=shard.dtype, device=shard.device)
        dist.all_gather_into_tensor(out, shard.contiguous(), group=group)
        return out
    # gloo (CPU tests, functional runs): stage through host memory
    host = shard.detach().cpu().contiguous()
    parts = [torch.empty_like(host) for _ in range(world)]
    dist.all_gather(parts, host, group=group)
    return torch.cat(parts).to(shard.device)


def embed_sharded(eparams, d_tok, d_off, d: int, sketch, rank: int, world: int, group=None, local_k1=None):
    """Set-sharded embedding: rank r runs K1 (values and, with ``sketch =
    (ell, seed)``, the sketches) on its n/W slice of the sets, and one
    all-gather per array replicates the (n, t) values and (n, ell) sketches
    on every rank (the join's node sketches, splits and BruteForce read any
    row).  Every rank holds the full CSR: verification reads any row too.
    Returns (values, sketches) as device tensors of n rows."""
    import torch
    n = int(d_off.shape[0]) - 1
    lo, hi, S = shard_range(n, rank, world)
    vals = torch.zeros((max(S, 1), eparams.t if eparams else 1), dtype=torch.int32, device=d_tok.device)
    sk = torch.zeros((max(S, 1), sketch[0] if sketch else 1), dtype=torch.int64, device=d_tok.device)
    (local_k1 or _gpu_k1)(eparams, sketch, d_tok, d_off, d, lo, hi, vals, sk)
    if world <= 1:
        return (vals[:n] if eparams else None), (sk[:n] if sketch else None)
    all_vals = _gather_rows(vals, world, group)[:n] if eparams else None
    all_sk = _gather_rows(sk, world, group)[:n] if sketch else None
    return all_vals, all_sk


class _DeviceArray:
    """CUDA Array Interface view of library-owned device memory (lets
    torch.as_tensor wrap it without a copy)."""

    def __init__(self, ptr: int, shape: tuple, typestr: str, owner):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None}
        self._owner = owner


class PeerArrays:
    """The (n, t) values and (n, ell) sketch arrays of a node-wide K1 as
    CUDA IPC exchange buffers: every rank allocates its own pair
    (cpsj_xbuf_create), the 64-byte handles are all-gathered once, and every
    rank maps every peer's pair (cpsj_xbuf_open, NVLink peer access).  K1 then
    writes each row it computes to all ranks' buffers
    (cpsj_minhash_sketch_multi), so the all-gather of the set-sharded
    embedding happens inside the kernel's epilogue."""

    def __init__(self, ctx, n: int, t: int, ell: int, rank: int, world: int, group=None, nnz: int | None = None):
        import ctypes

        import torch
        import torch.distributed as dist

        from ._native import IPC_HANDLE_BYTES, P
        if world > 8:
            raise ValueError("peer exchange supports up to 8 ranks per node")
        self.ctx, self.n, self.t, self.ell, self.rank, self.world = ctx, n, t, ell, rank, world
        self.nnz = nnz
        self._own, self._opened = [], []
        handles = []
        sizes = [max(1, n * t * 4), max(1, n * ell * 8)]
        if nnz is not None:
            # the CSR too (tokens, offsets): each rank uploads only its slice
            # and pushes it to the peers (csr_from_host_sharded)
            sizes += [max(1, nnz * 4), (n + 1) * 8]
        for nbytes in sizes:
            p = P()
            h = (ctypes.c_uint8 * IPC_HANDLE_BYTES)()
            ctx.check(ctx.lib.cpsj_xbuf_create(ctx.handle, nbytes, ctypes.byref(p), h))
            self._own.append(int(p.value))
            handles.append(bytes(h))
        gathered = [None] * world
        dist.all_gather_object(gathered, handles, group=group)
        self.values_ptrs, self.sketch_ptrs, self.tokens_ptrs, self.offsets_ptrs = [], [], [], []
        for r in range(world):
            if r == rank:
                ptrs = list(self._own)
            else:
                ptrs = []
                for hb in gathered[r]:
                    p = P()
                    buf = (ctypes.c_uint8 * IPC_HANDLE_BYTES).from_buffer_copy(hb)
                    ctx.check(ctx.lib.cpsj_xbuf_open(ctx.handle, buf, ctypes.byref(p)))
                    self._opened.append(int(p.value))
                    ptrs.append(int(p.value))
            self.values_ptrs.append(ptrs[0])
            self.sketch_ptrs.append(ptrs[1])
            if nnz is not None:
                self.tokens_ptrs.append(ptrs[2])
                self.offsets_ptrs.append(ptrs[3])
        dev = torch.device("cuda", ctx.device)
        self.values = torch.as_tensor(_DeviceArray(self._own[0], (n, t), "<i4", self), device=dev)
        self.sketch = torch.as_tensor(_DeviceArray(self._own[1], (n, ell), "<i8", self), device=dev)
        if nnz is not None:
            self.tokens = torch.as_tensor(_DeviceArray(self._own[2], (nnz,), "<i4", self), device=dev)
            self.offsets = torch.as_tensor(_DeviceArray(self._own[3], (n + 1,), "<i8", self), device=dev)

    def close(self):
        for p in self._opened:
            self.ctx.lib.cpsj_xbuf_close(self.ctx.handle, p, 1)
        for p in self._own:
            self.ctx.lib.cpsj_xbuf_close(self.ctx.handle, p, 0)
        self._opened, self._own = [], []


def _k1_to_peers(ctx, fam, d_tok, d_off, d: int, lo: int, hi: int, ptrs: list, is_sketch: bool):
    import ctypes

    import torch

    from ._native import K1Dsts
    n_loc = hi - lo
    if n_loc <= 0:
        return
    dst = K1Dsts()
    for i, p in enumerate(ptrs):
        if is_sketch:
            dst.d_sketch[i] = p
        else:
            dst.d_values[i] = p
    dst.n_dsts = len(ptrs)
    dst.row0 = lo
    max_token = min(int(d) - 1, 0xFFFFFFFF) if d else 0xFFFFFFFF
    stream = torch.cuda.current_stream().cuda_stream
    ctx.check(ctx.lib.cpsj_minhash_sketch_multi(ctx.handle, fam.handle, d_tok.data_ptr(), d_off.data_ptr() + 8 * lo,
                                                n_loc, max_token, ctypes.byref(dst), stream))


def embed_sharded_p2p(eparams, d_tok, d_off, d: int, sketch, rank: int, world: int, peers: PeerArrays,
                      group=None):
    """Set-sharded embedding with the all-gather fused into K1: rank r
    hashes sets [r n/W, (r+1) n/W) and stores each row into every rank's
    PeerArrays over NVLink; one barrier (a 1-element all-reduce, stream
    ordered under NCCL) publishes the rows.  Returns (values, sketches) =
    this rank's full (n, t) / (n, ell) arrays."""
    import torch
    import torch.distributed as dist

    from ._native import Context
    from .hashing import sketch_family
    ctx = Context.get()
    n = int(d_off.shape[0]) - 1
    lo, hi, _ = shard_range(n, rank, world)
    nccl = world > 1 and dist.get_backend(group) == "nccl"
    if nccl:
        # write-after-read guard: no peer may still be reading the previous
        # contents (stream ordered, no host synchronisation)
        flag = torch.zeros(1, dtype=torch.int32, device=d_tok.device)
        dist.all_reduce(flag, group=group)
    elif world > 1:
        torch.cuda.synchronize()
        dist.barrier(group=group)
    if eparams is not None:
        _k1_to_peers(ctx, eparams.device(ctx), d_tok, d_off, d, lo, hi, peers.values_ptrs, False)
    if sketch is not None:
        _k1_to_peers(ctx, sketch_family(*sketch).device(ctx), d_tok, d_off, d, lo, hi, peers.sketch_ptrs, True)
    if nccl:
        flag = torch.zeros(1, dtype=torch.int32, device=d_tok.device)
        dist.all_reduce(flag, group=group)        # every rank's K1 stores precede the readers
    elif world > 1:
        torch.cuda.synchronize()
        dist.barrier(group=group)
    return (peers.values if eparams is not None else None), (peers.sketch if sketch is not None else None)


def _stream_barrier(device, group=None):
    """All ranks reach this point in stream order (a 1-element NCCL
    all-reduce: no host synchronisation); gloo falls back to a host barrier
    after draining the device (functional runs)."""
    import torch
    import torch.distributed as dist
    if dist.get_backend(group) == "nccl":
        flag = torch.zeros(1, dtype=torch.int32, device=device)
        dist.all_reduce(flag, group=group)
    else:
        torch.cuda.synchronize()
        dist.barrier(group=group)


def csr_from_host_sharded(tok_host, off_host, rank: int, world: int, peers: PeerArrays, group=None,
                          side_stream=None):
    """End-to-end input staging for the set-sharded path: rank r copies only
    ITS slice of the CSR (sets shard_range(n, r, W): tokens
    off[lo]..off[hi] and offsets lo..hi) from pinned host memory into its own
    full-size CSR buffer, then pushes that slice to every peer's buffer
    (cpsj_copy_async over NVLink) on `side_stream`, so the push overlaps the
    K1 launches that only need the local slice.  The caller joins the side
    stream and runs a barrier (embed_sharded_p2p's closing all-reduce) before
    any rank reads the full CSR.  Host->device bytes per rank = the slice
    (about 1/W of the CSR) instead of the whole CSR.
    Returns (tokens, offsets) = this rank's full-size device buffers and the
    host->device byte count."""
    import torch
    ctx = peers.ctx
    n = peers.n
    lo, hi, _ = shard_range(n, rank, world)
    main = torch.cuda.current_stream()
    t0, t1 = int(off_host[lo]), int(off_host[hi])
    h2d = 0
    # own slice first (the K1 launches read it), on the main stream
    if t1 > t0:
        ctx.check(ctx.lib.cpsj_copy_async(ctx.handle, peers.tokens_ptrs[rank] + 4 * t0,
                                          tok_host.data_ptr() + 4 * t0, 4 * (t1 - t0), main.cuda_stream))
        h2d += 4 * (t1 - t0)
    if hi >= lo:
        ctx.check(ctx.lib.cpsj_copy_async(ctx.handle, peers.offsets_ptrs[rank] + 8 * lo,
                                          off_host.data_ptr() + 8 * lo, 8 * (hi - lo + 1), main.cuda_stream))
        h2d += 8 * (hi - lo + 1)
    if world > 1:
        ss = side_stream if side_stream is not None else main
        if ss is not main:
            ss.wait_stream(main)
        for r in range(world):
            if r == rank:
                continue
            if t1 > t0:
                ctx.check(ctx.lib.cpsj_copy_async(ctx.handle, peers.tokens_ptrs[r] + 4 * t0,
                                                  peers.tokens_ptrs[rank] + 4 * t0, 4 * (t1 - t0), ss.cuda_stream))
            ctx.check(ctx.lib.cpsj_copy_async(ctx.handle, peers.offsets_ptrs[r] + 8 * lo,
                                              peers.offsets_ptrs[rank] + 8 * lo, 8 * (hi - lo + 1), ss.cuda_stream))
    return peers.tokens, peers.offsets, h2d


def embed_sharded_p2p_from_host(eparams, tok_host, off_host, d: int, sketch, rank: int, world: int,
                                peers: PeerArrays, group=None, side_stream=None):
    """The whole set-sharded embedding from pinned host buffers: one barrier
    (write-after-read guard), this rank's CSR slice host->device and pushed
    to the peers (csr_from_host_sharded, overlapping K1), K1 values and
    sketches of the slice stored to every rank (cpsj_minhash_sketch_multi),
    and one closing barrier.  Returns (tokens, offsets, values, sketches,
    h2d_bytes); every rank then holds the full CSR and full arrays."""
    import torch

    from ._native import Context
    from .hashing import sketch_family
    ctx = Context.get()
    dev = torch.device("cuda", ctx.device)
    n = peers.n
    lo, hi, _ = shard_range(n, rank, world)
    if world > 1:
        _stream_barrier(dev, group)
    d_tok, d_off, h2d = csr_from_host_sharded(tok_host, off_host, rank, world, peers, group, side_stream)
    if eparams is not None:
        _k1_to_peers(ctx, eparams.device(ctx), d_tok, d_off, d, lo, hi, peers.values_ptrs, False)
    if sketch is not None:
        _k1_to_peers(ctx, sketch_family(*sketch).device(ctx), d_tok, d_off, d, lo, hi, peers.sketch_ptrs, True)
    if side_stream is not None:
        torch.cuda.current_stream().wait_stream(side_stream)
    if world > 1:
        _stream_barrier(dev, group)      # every rank's slices and K1 rows precede the readers
    return d_tok, d_off, (peers.values if eparams is not None else None), \
        (peers.sketch if sketch is not None else None), h2d


def embedded_from_parts(eparams, d_tok, d_off, d: int, values, sketches, sketch_key=None, host_csr=None):
    """EmbeddedDataset over device tensors produced by embed_sharded."""
    import torch

    from .embed import EmbeddedDataset
    n = int(d_off.shape[0]) - 1
    emb = EmbeddedDataset(None, None, None, eparams.t, eparams.seed, None, None, np.arange(n, dtype=np.int64))
    emb._dev.update(values=values, tokens=d_tok, offsets=d_off)
    emb._dev["sizes"] = (d_off[1:] - d_off[:-1]).to(torch.int32)
    emb._n = n
    emb._width = int(d)
    emb._ids_checked, emb._ids_ok = (id(emb.source_ids), n), True
    emb._sizes_fn = lambda: emb._dev["sizes"].cpu().numpy().astype(np.int64)
    if host_csr is not None:
        emb._csr_arrays = (host_csr[0], host_csr[1], int(d))
    if sketches is not None and sketch_key is not None:
        emb._dev_sketch[tuple(sketch_key)] = sketches
    return emb


def merge_results(parts_keys: np.ndarray, parts_sims: np.ndarray):
    """Sort + unique by pair key (first occurrence kept; duplicates carry
    identical similarities)."""
    keys, first = np.unique(parts_keys.astype(np.uint64), return_index=True)
    return keys, parts_sims[first]


def shard_reps(emb, params: CPSJoinParams, rank: int, world: int, group=None, device=None,
               local_join=None) -> JoinArrays:
    """cpsjoin_self over `world` ranks, repetition trees round-robin; every
    rank returns the full result."""
    if world <= 1:
        return (local_join or _gpu_local)(emb, params, None)
    idx = np.arange(rank, params.repetitions, world, dtype=np.int64)
    local = (local_join or _gpu_local)(emb, params, idx)
    return merge_ranks(local, world, group, device)


def shard_frontier(emb, params: CPSJoinParams, rank: int, world: int, depth: int = 1, group=None, device=None,
                   local_join=None) -> JoinArrays:
    """cpsjoin_self over `world` ranks, sharding the tree frontier: every
    rank builds every repetition's levels above `depth` (the root split is
    cheap and identical everywhere), then keeps its size-balanced contiguous
    share of the nodes of level `depth` (cost-weighted cut, see cpsj_plan in
    include/cpsjoin_b200.h) and everything below them (SURVEY.md 8(e):
    scales past R GPUs, where repetition sharding stops).  Ranks != 0 count
    only what they found below the cut, so the counter sums and the pair
    union equal the unsharded join."""
    if world <= 1:
        return (local_join or _gpu_local)(emb, params, None)
    local = (local_join or _gpu_frontier)(emb, params, (rank, world, depth))
    return merge_ranks(local, world, group, device)


def _gpu_frontier(emb, params: CPSJoinParams, frontier):
    return cpsjoin_self_arrays(emb, params, frontier=frontier)


def merge_ranks(local: JoinArrays, world: int, group=None, device=None) -> JoinArrays:
    """Union of the ranks' pairs (gather + sort/unique) and their counters
    (sum of pre/candidates/results, max of depth and peak)."""
    import torch
    import torch.distributed as dist
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
