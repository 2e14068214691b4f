"""MinHash embedding of records (drop-in for the reference's simjoin.embed).

``embed_dataset`` runs K1 (csrc/minhash.cu) over the CSR of the dataset and
keeps the (n, t) value matrix resident on the GPU; ``EmbeddedDataset``
exposes the reference's attributes (values, dense, d, t, seed, verify_csr,
sizes, source_ids, side, origin) and the cached ``sketches(ell, seed)``,
materialising host copies only when they are read.
"""
from __future__ import annotations

import numpy as np

from .core import Dataset, Record
from .hashing import KIND_EMBED, derive_rng, minhash_segments_many, sketch_family

DEFAULT_T = 128


class EmbeddingParams:
    """t independent MinHash functions drawn from a master seed
    (reference embed.py:36-48)."""

    def __init__(self, t: int = DEFAULT_T, seed: int = 0):
        if t < 1:
            raise ValueError("embedding size t must be at least 1")
        self.t = t
        self.seed = seed
        self.tables = derive_rng(seed, KIND_EMBED).integers(0, 2 ** 64, size=(t, 4, 256), dtype=np.uint64)
        self._device = {}

    def device(self, ctx):
        fam = self._device.get(ctx.device)
        if fam is None:
            from ._native import Family
            fam = self._device[ctx.device] = Family(ctx, self.tables)
        return fam


def dense_remap_device(d_values, t: int):
    """The reference's first-seen dense remap of an embedding
    (_first_seen_dense over keys (i << 32) | values[r, i], embed.py:108-114,
    129-132) on the GPU (cpsj_dense_remap, csrc/dense.cu).  d_values: (n, t)
    int32 device tensor (u32 bits).  Returns ((n, t) int32 device tensor of
    dense ids, d)."""
    import ctypes
    torch = _torch()
    from ._native import Context, i64
    ctx = Context.get()
    n = int(d_values.shape[0])
    out = torch.empty((n, t), dtype=torch.int32, device=d_values.device)
    d = i64()
    stream = torch.cuda.current_stream(d_values.device).cuda_stream
    ctx.check(ctx.lib.cpsj_dense_remap(ctx.handle, d_values.data_ptr(), n, int(t), out.data_ptr(), ctypes.byref(d),
                                       stream))
    return out, int(d.value)


def _torch():
    import torch
    return torch


class EmbeddedDataset:
    """Records embedded to t MinHash values each, plus verification data
    (reference embed.py:51-98).  Device copies are made lazily and dropped
    whenever a host attribute is reassigned."""

    def __init__(self, values, dense, d, t: int, seed: int, verify_csr, sizes, source_ids,
                 side=None, origin: Dataset | None = None):
        self._values = None if values is None else np.asarray(values, dtype=np.uint32)
        self._dense = None if dense is None else np.asarray(dense)
        self._d = d
        self.t = t
        self.seed = seed
        self._csr = verify_csr
        self._csr_arrays = None
        self._sizes = None if sizes is None else np.asarray(sizes, dtype=np.int64)
        self.source_ids = source_ids
        self.side = side
        self.origin = origin
        self._n = None
        self._sketch_cache: dict = {}
        self._dev_sketch: dict = {}
        self._dev: dict = {}
        self._width = None      # token universe bound of the CSR, if known
        self._sizes_fn = None   # lazy host sizes for device-only datasets

    # ------------------------------------------------------------- internal
    @classmethod
    def _device_backed(cls, dev_values, t, seed, tokens, offsets, d_universe, origin, dev_csr):
        obj = cls(None, None, None, t, seed, None, np.diff(offsets), np.arange(len(offsets) - 1, dtype=np.int64),
                  origin=origin)
        obj._csr_arrays = (tokens, offsets, d_universe)
        obj._width = d_universe
        obj._dev["values"] = dev_values
        obj._dev["tokens"], obj._dev["offsets"] = dev_csr
        obj._n = len(offsets) - 1
        obj._ids_checked, obj._ids_ok = (id(obj.source_ids), obj._n), True
        return obj

    def _csr_host(self):
        if self._csr_arrays is None:
            m = self._csr
            self._csr_arrays = (np.asarray(m.indices).astype(np.uint32, copy=False),
                                np.asarray(m.indptr).astype(np.int64, copy=False), int(m.shape[1]))
        return self._csr_arrays

    def device_inputs(self, ctx):
        """Device tensors the join reads: tokens, offsets, sizes (i32), values."""
        torch = _torch()
        dev = torch.device("cuda", ctx.device)
        if "tokens" not in self._dev:
            tok, off, _ = self._csr_host()
            self._dev["tokens"] = torch.from_numpy(np.ascontiguousarray(tok).view(np.int32)).to(dev, non_blocking=True)
            self._dev["offsets"] = torch.from_numpy(np.ascontiguousarray(off)).to(dev, non_blocking=True)
        if "sizes" not in self._dev:
            self._dev["sizes"] = torch.from_numpy(self.sizes.astype(np.int32)).to(dev, non_blocking=True)
        if "values" not in self._dev:
            v = np.ascontiguousarray(self.values, dtype=np.uint32)
            self._dev["values"] = torch.from_numpy(v.view(np.int32)).to(dev, non_blocking=True)
        return self._dev["tokens"], self._dev["offsets"], self._dev["sizes"], self._dev["values"]

    def device_side(self, ctx):
        """emb.side as a device int8 tensor (None for a self-join dataset)."""
        if self.side is None:
            return None
        key = id(self.side)
        if self._dev.get("side_key") != key:
            torch = _torch()
            self._dev["side"] = torch.from_numpy(np.ascontiguousarray(self.side, dtype=np.int8)).to(
                torch.device("cuda", ctx.device))
            self._dev["side_key"] = key
        return self._dev["side"]

    def ids_are_rows(self) -> bool:
        """True when source_ids == arange(n) (checked once per array)."""
        src = self.source_ids
        key = (id(src), len(self))
        if getattr(self, "_ids_checked", None) != key:
            ok = src is None or (len(src) == len(self) and np.array_equal(src, np.arange(len(self))))
            self._ids_checked = key
            self._ids_ok = ok
        return self._ids_ok

    # ------------------------------------------------------------ reference
    def __len__(self) -> int:
        if self._n is None:
            self._n = len(self._values) if self._values is not None else len(self._csr_host()[1]) - 1
        return self._n

    @property
    def values(self) -> np.ndarray:
        if self._values is None:
            self._values = self._dev["values"].cpu().numpy().view(np.uint32)
        return self._values

    @values.setter
    def values(self, v):
        self._values = np.asarray(v, dtype=np.uint32)
        self._values_host_set = True
        self._dev.pop("values", None)
        self._dense = None
        self._d = None
        self._n = len(self._values)

    @property
    def dense(self) -> np.ndarray:
        if self._dense is None:
            self._compute_dense()
        return self._dense

    @dense.setter
    def dense(self, v):
        self._dense = v

    @property
    def d(self) -> int:
        if self._d is None:
            self._compute_dense()
        return self._d

    @d.setter
    def d(self, v):
        self._d = v

    def _compute_dense(self):
        # GPU remap (csrc/dense.cu); read lazily -- only embedded_record and
        # the reference-facing attributes use it, the join never does
        n, t = len(self), self.t
        if n == 0:
            self._dense, self._d = np.zeros((0, t), dtype=np.uint32), 0
            return
        if "values" in self._dev:
            dv = self._dev["values"]
        else:
            from ._native import Context
            ctx = Context.get()
            dv = _torch().from_numpy(np.ascontiguousarray(self.values, dtype=np.uint32).view(np.int32)).to(
                _torch().device("cuda", ctx.device))
        dense, d = dense_remap_device(dv, t)
        self._dense, self._d = dense.cpu().numpy().view(np.uint32), d

    @property
    def verify_csr(self):
        if self._csr is None:
            from scipy.sparse import csr_matrix
            tok, off, width = self._csr_arrays
            self._csr = csr_matrix((np.ones(len(tok), dtype=np.int32), tok.astype(np.int32), off),
                                   shape=(len(off) - 1, width))
        return self._csr

    @verify_csr.setter
    def verify_csr(self, m):
        self._csr = m
        self._csr_arrays = None
        self._dev.pop("tokens", None)
        self._dev.pop("offsets", None)

    @property
    def sizes(self) -> np.ndarray:
        if self._sizes is None and self._sizes_fn is not None:
            self._sizes = self._sizes_fn()
        return self._sizes

    @sizes.setter
    def sizes(self, v):
        self._sizes = np.asarray(v, dtype=np.int64)
        self._dev.pop("sizes", None)

    def embedded_record(self, row: int) -> np.ndarray:
        return np.sort(self.dense[row])

    def original_record(self, row: int) -> Record:
        tok, off, _ = self._csr_host()
        return Record(int(self.source_ids[row]), tok[off[row]:off[row + 1]].astype(np.uint32))

    def sketches_device(self, ell: int, seed: int):
        """(n, ell) sketch matrix as a device tensor (int64 view of u64),
        computed once per (ell, seed) by K1 (hashing.py:197-211)."""
        key = (ell, seed)
        if key not in self._dev_sketch:
            torch = _torch()
            from ._native import Context
            ctx = Context.get()
            n = len(self)
            dev = torch.device("cuda", ctx.device)
            out = torch.zeros((n, ell), dtype=torch.int64, device=dev)
            if n > 0:
                tok, off, sizes, _ = self.device_inputs(ctx)
                fam = sketch_family(ell, seed).device(ctx)
                width = self._width if self._width is not None else self._csr_host()[2]
                stream = torch.cuda.current_stream(dev).cuda_stream
                ctx.check(ctx.lib.cpsj_minhash_sketch(ctx.handle, fam.handle, tok.data_ptr(), off.data_ptr(), n,
                                                      max(0, min(int(width) - 1, 0xFFFFFFFF)) if width else
                                                      0xFFFFFFFF, None, out.data_ptr(), stream))
            self._dev_sketch[key] = out
        return self._dev_sketch[key]

    def sketches(self, ell: int, seed: int) -> np.ndarray:
        """(n, ell) sketch matrix of the original records, cached per family."""
        key = (ell, seed)
        if key not in self._sketch_cache:
            self._sketch_cache[key] = self.sketches_device(ell, seed).cpu().numpy().view(np.uint64)
        return self._sketch_cache[key]


def embed_record(params: EmbeddingParams, x: Record) -> list[tuple[int, int]]:
    if len(x) == 0:
        raise ValueError("cannot embed an empty record")
    tok = np.asarray(x.tokens, dtype=np.uint32)
    vals = minhash_segments_many(params.tables, tok, np.array([0, len(tok)], dtype=np.int64))[0]
    return [(i, int(v)) for i, v in enumerate(vals)]


def embed_device_csr(params: EmbeddingParams, d_tokens, d_offsets, d: int, host_csr=None,
                     origin: Dataset | None = None) -> EmbeddedDataset:
    """embed_dataset for a CSR that is already resident on the GPU (torch
    int32 token / int64 offset tensors).  ``host_csr`` = (tokens, offsets)
    numpy arrays, if the caller has them, back the lazy host attributes."""
    torch = _torch()
    from ._native import Context
    ctx = Context.get()
    n = int(d_offsets.shape[0]) - 1
    t = params.t
    fam = params.device(ctx)
    dev = torch.device("cuda", ctx.device)
    d_vals = torch.empty((max(n, 0), t), dtype=torch.int32, device=dev)
    max_token = min(int(d) - 1, 0xFFFFFFFF) if d and d > 0 else 0xFFFFFFFF
    stream = torch.cuda.current_stream(dev).cuda_stream
    if n > 0:
        ctx.check(ctx.lib.cpsj_minhash_sketch(ctx.handle, fam.handle, d_tokens.data_ptr(), d_offsets.data_ptr(), n,
                                              max_token, d_vals.data_ptr(), None, stream))
    if host_csr is None:
        host_csr = (None, None)
    tok, off = host_csr
    obj = EmbeddedDataset(None, None, None, t, params.seed, None, None, np.arange(n, dtype=np.int64), origin=origin)
    obj._csr_arrays = (tok, off, int(d)) if tok is not None else None
    obj._width = int(d)
    obj._dev.update(values=d_vals, tokens=d_tokens, offsets=d_offsets)
    obj._dev["sizes"] = (d_offsets[1:] - d_offsets[:-1]).to(torch.int32)
    obj._n = n
    obj._ids_checked, obj._ids_ok = (id(obj.source_ids), n), True
    obj._sizes_fn = lambda: obj._dev["sizes"].cpu().numpy().astype(np.int64)
    return obj


def union_embedded(r: EmbeddedDataset, s: EmbeddedDataset) -> EmbeddedDataset:
    """Tagged union of two embeddings sharing a function family (reference
    embed.py:142-169): rows of r first with side 0, rows of s after with
    side 1.  The device arrays are concatenated on the GPU."""
    if r.t != s.t:
        raise ValueError(f"embedding size mismatch: {r.t} vs {s.t}")
    if r.seed != s.seed:
        raise ValueError("inputs were embedded with different seeds")
    torch = _torch()
    from ._native import Context
    ctx = Context.get()
    tr, or_, zr, vr = r.device_inputs(ctx)
    ts, os_, zs, vs = s.device_inputs(ctx)
    n_r, n_s = len(r), len(s)
    wr = r._width if r._width is not None else r._csr_host()[2]
    ws = s._width if s._width is not None else s._csr_host()[2]
    u = EmbeddedDataset(None, None, None, r.t, r.seed, None, np.concatenate([r.sizes, s.sizes]),
                        np.concatenate([np.asarray(r.source_ids), np.asarray(s.source_ids)]),
                        side=np.concatenate([np.zeros(n_r, dtype=np.int8), np.ones(n_s, dtype=np.int8)]))
    u._dev.update(tokens=torch.cat([tr, ts]), offsets=torch.cat([or_, os_[1:] + or_[-1]]),
                  sizes=torch.cat([zr, zs]), values=torch.cat([vr, vs]))
    u._n = n_r + n_s
    u._width = max(int(wr), int(ws))
    if r._csr_arrays is not None and s._csr_arrays is not None or (r._csr is not None and s._csr is not None):
        rt, ro, _ = r._csr_host()
        st, so, _ = s._csr_host()
        u._csr_arrays = (np.concatenate([rt, st]), np.concatenate([ro, so[1:] + ro[-1]]), u._width)
    return u


_PIPELINE_MIN_SETS = 1 << 16


def embed_dataset(params: EmbeddingParams, ds: Dataset, sketch: tuple[int, int] | None = None,
                  chunks: int | None = None) -> EmbeddedDataset:
    """Embed every record with the shared function family (embed.py:117-139)
    on the GPU; the value matrix stays device-resident.

    ``sketch=(ell, seed)`` additionally builds the sketch matrix that
    ``cpsjoin_self(emb, CPSJoinParams(ell=ell, seed=seed))`` will ask for
    (emb.sketches, embed.py:90-98) in the same pass.  Large inputs are
    copied to the device in set-aligned chunks on a side stream while K1
    hashes the chunks already resident (host->device copy overlapped with
    compute; the copy source should be pinned memory for the overlap).
    """
    n = len(ds)
    if n > 0 and ((chunks is None and n >= _PIPELINE_MIN_SETS) or (chunks is not None and chunks > 1)):
        return _embed_pipelined(params, ds, sketch, None if chunks is None else min(chunks, n))
    t = params.t
    tok, off = ds.flat_tokens()
    tok = np.ascontiguousarray(tok, dtype=np.uint32)
    off = np.ascontiguousarray(off, dtype=np.int64)
    if n == 0:
        return EmbeddedDataset(np.zeros((0, t), dtype=np.uint32), np.zeros((0, t), dtype=np.uint32), 0, t,
                               params.seed, verify_csr=ds.csr(), sizes=np.zeros(0, dtype=np.int64),
                               source_ids=np.arange(0, dtype=np.int64), origin=ds)
    if np.any(off[1:] == off[:-1]):
        raise ValueError("cannot embed an empty record")
    torch = _torch()
    from ._native import Context
    ctx = Context.get()
    fam = params.device(ctx)
    dev = torch.device("cuda", ctx.device)
    d_tok = torch.from_numpy(tok.view(np.int32)).to(dev, non_blocking=True)
    d_off = torch.from_numpy(off).to(dev, non_blocking=True)
    d_vals = torch.empty((n, t), dtype=torch.int32, device=dev)
    width = int(getattr(ds, "d", 0) or 0)
    max_token = min(width - 1, 0xFFFFFFFF) if width > 0 else 0xFFFFFFFF
    stream = torch.cuda.current_stream(dev).cuda_stream
    ctx.check(ctx.lib.cpsj_minhash_sketch(ctx.handle, fam.handle, d_tok.data_ptr(), d_off.data_ptr(), n,
                                          max_token, d_vals.data_ptr(), None, stream))
    return EmbeddedDataset._device_backed(d_vals, t, params.seed, tok, off, width, ds, (d_tok, d_off))


def _embed_pipelined(params: EmbeddingParams, ds: Dataset, sketch, chunks: int) -> EmbeddedDataset:
    torch = _torch()
    from ._native import Context
    n = len(ds)
    t = params.t
    tok, off = ds.flat_tokens()
    tok = np.ascontiguousarray(tok, dtype=np.uint32)
    off = np.ascontiguousarray(off, dtype=np.int64)
    # Dataset rows hold >= 2 tokens by construction; other CSR sources are checked
    if not getattr(ds, "rows_nonempty", False) and np.any(off[1:] == off[:-1]):
        raise ValueError("cannot embed an empty record")
    ctx = Context.get()
    efam = params.device(ctx)
    sfam = sketch_family(*sketch).device(ctx) if sketch is not None else None
    dev = torch.device("cuda", ctx.device)
    compute = torch.cuda.current_stream(dev)
    copier = _copy_stream(dev)
    width = int(getattr(ds, "d", 0) or 0)
    max_token = min(width - 1, 0xFFFFFFFF) if width > 0 else 0xFFFFFFFF
    src_tok = torch.from_numpy(tok.view(np.int32))
    src_off = torch.from_numpy(off)
    d_tok = torch.empty(len(tok), dtype=torch.int32, device=dev)
    d_vals = torch.empty((n, t), dtype=torch.int32, device=dev)
    d_sk = torch.empty((n, sketch[0]), dtype=torch.int64, device=dev) if sketch is not None else None
    bounds = _chunk_bounds(n, chunks, nnz=int(off[-1]), t=t, ell=(sketch[0] if sketch is not None else 0))
    chunks = len(bounds) - 1
    d_off = torch.empty(n + 1, dtype=torch.int64, device=dev)
    events = []
    copier.wait_stream(compute)  # destination buffers were allocated on `compute`
    with torch.cuda.stream(copier):
        for c in range(chunks):
            s0, s1 = int(bounds[c]), int(bounds[c + 1])
            t0, t1 = int(off[s0]), int(off[s1])
            d_off[s0 + (c > 0):s1 + 1].copy_(src_off[s0 + (c > 0):s1 + 1], non_blocking=True)
            if t1 > t0:
                d_tok[t0:t1].copy_(src_tok[t0:t1], non_blocking=True)
            ev = torch.cuda.Event(enable_timing=_PIPE_TRACE is not None)
            ev.record(copier)
            events.append(ev)
    h = compute.cuda_stream
    trace = _PIPE_TRACE if _PIPE_TRACE is not None and len(_PIPE_TRACE) == 0 else None
    if trace is not None:
        trace.append(("copies", events))
        kev = []
        trace.append(("k1", kev))
    for c in range(chunks):
        s0, s1 = int(bounds[c]), int(bounds[c + 1])
        compute.wait_event(events[-1] if _PIPE_SERIAL else events[c])
        if trace is not None:
            e = torch.cuda.Event(enable_timing=True)
            e.record(compute)
            kev.append(e)
        if s1 <= s0:
            continue
        offp = d_off.data_ptr() + 8 * s0
        if sfam is not None:
            # values and sketches of the chunk in one K1 launch
            ctx.check(ctx.lib.cpsj_minhash_embed(ctx.handle, efam.handle, sfam.handle, d_tok.data_ptr(), offp,
                                                 s1 - s0, max_token, d_vals.data_ptr() + 4 * t * s0,
                                                 d_sk.data_ptr() + 8 * sketch[0] * s0, h))
        else:
            ctx.check(ctx.lib.cpsj_minhash_sketch(ctx.handle, efam.handle, d_tok.data_ptr(), offp, s1 - s0,
                                                  max_token, d_vals.data_ptr() + 4 * t * s0, None, h))
        if trace is not None:
            e = torch.cuda.Event(enable_timing=True)
            e.record(compute)
            kev.append(e)
    # the copier's work is consumed on `compute`; keep the buffers alive there
    d_tok.record_stream(copier)
    d_off.record_stream(copier)
    emb = EmbeddedDataset._device_backed(d_vals, t, params.seed, tok, off, width, ds, (d_tok, d_off))
    emb._dev["sizes"] = (d_off[1:] - d_off[:-1]).to(torch.int32)
    if sketch is not None:
        emb._dev_sketch[tuple(sketch)] = d_sk
    return emb


# Chunk schedule of the pipelined embed.  The first copy is exposed, every
# later chunk must arrive while K1 hashes the chunks before it, and every
# chunk costs a fixed overhead (length order + two K1 launches and their
# tails).  With cumulative fractions S_c, copy time T_copy and K1 time T_k1
# for the whole input, chunk c + 1 has arrived when chunk c is done iff
#   T_copy S_{c+1} <= T_copy S_0 + T_k1 S_c,
# so S_{c+1} = S_0 + rho S_c with rho = T_k1 / T_copy (taken with a 10%
# margin) is the fastest-growing stall-free schedule; S_0 is the candidate
# that minimises  S_0 T_copy + chunks x overhead.  Rates measured on the B200
# boxes: ~50 GB/s pinned H2D; K1 values 4.1e12 and sketches 5.5e12 hash
# evaluations/s on Zipf sets (tools/k1_probe.py).  A copy-bound input
# (rho < 1.3) keeps a geometric growth of 1.3 instead.
_H2D_BYTES_PER_S = 50e9
_K1_VALUES_EVALS_PER_S = 4.1e12
_K1_SKETCH_EVALS_PER_S = 5.5e12
_CHUNK_OVERHEAD_S = 0.15e-3
_FIRST_CHUNKS = (1.0 / 64, 1.0 / 32, 1.0 / 16, 1.0 / 8, 1.0 / 4, 1.0 / 2)
_MIN_GROWTH = 1.3
_MIN_CHUNK_SETS = 20_000


def _chunk_fractions(t_copy: float, t_k1: float, n: int = 0) -> list:
    rho = 0.9 * t_k1 / max(t_copy, 1e-12)
    best = None
    # a K1 launch needs about two set pairs per warp (148 SMs x 32 warps x 2
    # sets x 2) to keep every warp busy -- long sets (c4: 300 tokens, 1024
    # sketch functions) otherwise run a small chunk at a fraction of the
    # kernel's rate: no first chunk smaller than _MIN_CHUNK_SETS
    s_min = min(1.0, _MIN_CHUNK_SETS / n) if n > 0 else 0.0
    for s0 in _FIRST_CHUNKS + (1.0,):
        if s0 < s_min and s0 < 1.0:
            continue
        S = [s0]
        while S[-1] < 1.0 - 1e-9 and len(S) < 64:
            S.append(max(s0 + rho * S[-1], _MIN_GROWTH * S[-1]))
        S = [x / S[-1] for x in S]  # scaled to end at 1 (the recurrence is linear, so it still holds)
        S[-1] = 1.0
        cost = S[0] * t_copy + len(S) * _CHUNK_OVERHEAD_S
        if best is None or cost < best[0]:
            best = (cost, S)
    return best[1]


def _chunk_bounds(n: int, chunks: int | None, nnz: int | None = None, t: int = 128, ell: int = 8) -> np.ndarray:
    """Set-aligned chunk boundaries: an explicit count uses doubling chunks
    (1/2^(c-1), ..., 1/4, 1/2); None uses the rate-based schedule above
    (nnz = tokens of the input, t / 64 ell = values / sketch functions)."""
    if chunks is not None:
        frac = np.array([0.0] + [2.0 ** -(chunks - 1)] + [2.0 ** -(chunks - k) for k in range(1, chunks)])
        cum = np.cumsum(frac)
    else:
        nnz = 100 * n if nnz is None else nnz
        t_copy = (4.0 * nnz + 8.0 * n) / _H2D_BYTES_PER_S
        t_k1 = nnz * (t / _K1_VALUES_EVALS_PER_S + 64.0 * ell / _K1_SKETCH_EVALS_PER_S)
        cum = np.array([0.0] + _chunk_fractions(t_copy, t_k1, n))
    bounds = np.minimum(np.round(cum * n), n).astype(np.int64)
    bounds[-1] = n
    return bounds


_COPY_STREAMS: dict = {}
_PIPE_TRACE = None  # diagnostics (tools/embed_probe.py): an empty list collects one call's events
_PIPE_SERIAL = False  # diagnostics: every chunk waits for the whole copy


def _copy_stream(dev):
    torch = _torch()
    s = _COPY_STREAMS.get(dev.index)
    if s is None:
        s = _COPY_STREAMS[dev.index] = torch.cuda.Stream(dev)
    return s
