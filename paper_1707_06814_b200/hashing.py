"""Seed plumbing, hash families and the sketch threshold (host side), plus
the GPU MinHash/sketch entry points.

Mirrors the reference's simjoin.hashing interface.  Table generation stays
on the host with numpy's PCG64 exactly as the reference draws it
(hashing.py:43-46, :168-178), so tables -- and everything downstream -- are
identical by construction; the per-token hashing runs in the sm_100a
kernel K1 (csrc/minhash.cu).
"""
from __future__ import annotations

import functools

import numpy as np

_U64 = np.uint64

KIND_EMBED = 1
KIND_SKETCH = 2
KIND_CPS_TREE = 3
KIND_MINHASH_REP = 4
KIND_GENERATOR = 5

_GAMMA = _U64(0x9E3779B97F4A7C15)
_M1 = _U64(0xBF58476D1CE4E5B9)
_M2 = _U64(0x94D049BB133111EB)


def derive_rng(master_seed: int, *path: int) -> np.random.Generator:
    """Independent numpy generator for (master seed, namespace path)."""
    return np.random.default_rng(np.random.SeedSequence(master_seed, spawn_key=tuple(path)))


def mix64(x) -> np.ndarray:
    """SplitMix64 finaliser, vectorised (device twin: cpsj_common.cuh)."""
    z = np.asarray(x, dtype=_U64)
    with np.errstate(over="ignore"):
        z = z + _GAMMA
        z = (z ^ (z >> _U64(30))) * _M1
        z = (z ^ (z >> _U64(27))) * _M2
        return z ^ (z >> _U64(31))


def word_stream(seed: int, n: int, offset: int = 0) -> np.ndarray:
    ks = np.arange(offset, offset + n, dtype=_U64)
    return mix64(_U64(seed) ^ mix64(ks))


def uniform_stream(seed: int, n: int, offset: int = 0) -> np.ndarray:
    return word_stream(seed, n, offset) / 2.0 ** 64


class SketchFamily:
    """64*ell MinHash tables followed by 64*ell one-bit hash tables, drawn
    from one derive_rng(seed, KIND_SKETCH) stream (hashing.py:160-184)."""

    def __init__(self, ell: int, seed: int):
        if ell < 1:
            raise ValueError("sketch length must be at least one word")
        self.ell = ell
        self.seed = seed
        self.bits = 64 * ell
        rng = derive_rng(seed, KIND_SKETCH)
        self.minhash_tables = rng.integers(0, 2 ** 64, size=(self.bits, 4, 256), dtype=_U64)
        self.bit_tables = rng.integers(0, 2 ** 64, size=(self.bits, 4, 256), dtype=_U64)
        self._device = {}

    def device(self, ctx):
        fam = self._device.get(ctx.device)
        if fam is None:
            from ._native import Family
            fam = self._device[ctx.device] = Family(ctx, self.minhash_tables, self.bit_tables)
        return fam


@functools.lru_cache(maxsize=16)
def sketch_family(ell: int, seed: int) -> SketchFamily:
    """Families are a pure function of (ell, seed); cache them per process
    so repeated joins do not redraw and re-upload 2 x 4 MiB of tables."""
    return SketchFamily(ell, seed)


def match_threshold(lam: float, delta: float, m: int) -> int:
    """Smallest accepted matching-bit count k* = binom.ppf(delta, m, (1+lam)/2)
    (hashing.py:234-247)."""
    if not (0.0 < delta < 1.0):
        raise ValueError("delta must be in (0, 1)")
    if m <= 0 or m % 64 != 0:
        raise ValueError("sketch bit count must be a positive multiple of 64")
    from scipy.stats import binom
    return int(binom.ppf(delta, m, (1.0 + lam) / 2.0))


def calibrate_threshold(lam: float, delta: float, m: int) -> float:
    return 2.0 * match_threshold(lam, delta, m) / m - 1.0


def _max_token_of(tokens: np.ndarray, d: int | None) -> int:
    if d is not None and d > 0:
        return min(int(d) - 1, 0xFFFFFFFF)
    return int(tokens.max()) if len(tokens) else 0


def minhash_segments_many(tables: np.ndarray, flat_tokens: np.ndarray, offsets: np.ndarray,
                          d: int | None = None) -> np.ndarray:
    """(n, F) MinHash tokens of every segment under every table, on the GPU
    (minhash_segments, hashing.py:129-146, for all F tables at once)."""
    import torch

    from ._native import Context, Family
    ctx = Context.get()
    fam = Family(ctx, tables)
    n = len(offsets) - 1
    dev = torch.device("cuda", ctx.device)
    tok = torch.from_numpy(np.ascontiguousarray(flat_tokens, dtype=np.uint32).view(np.int32)).to(dev)
    off = torch.from_numpy(np.ascontiguousarray(offsets, dtype=np.int64)).to(dev)
    out = torch.empty((n, fam.F), dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    ctx.check(ctx.lib.cpsj_minhash_sketch(ctx.handle, fam.handle, tok.data_ptr(), off.data_ptr(), n,
                                          _max_token_of(flat_tokens, d), out.data_ptr(), None, stream))
    return out.cpu().numpy().view(np.uint32)


def minhash_segments(table: np.ndarray, flat_tokens: np.ndarray, offsets: np.ndarray,
                     byte_cols=None, sizes=None) -> np.ndarray:
    """MinHash token per segment for one (4, 256) table (hashing.py:129-146)."""
    return minhash_segments_many(np.asarray(table, dtype=_U64)[None], flat_tokens, offsets)[:, 0]


def build_sketch_matrix(family: SketchFamily, flat_tokens: np.ndarray, offsets: np.ndarray) -> np.ndarray:
    """(n, ell) sketch matrix on the GPU (hashing.py:197-211)."""
    import torch

    from ._native import Context
    n = len(offsets) - 1
    if n == 0 or len(flat_tokens) == 0:
        return np.zeros((n, family.ell), dtype=_U64)
    ctx = Context.get()
    fam = family.device(ctx)
    dev = torch.device("cuda", ctx.device)
    tok = torch.from_numpy(np.ascontiguousarray(flat_tokens, dtype=np.uint32).view(np.int32)).to(dev)
    off = torch.from_numpy(np.ascontiguousarray(offsets, dtype=np.int64)).to(dev)
    out = torch.empty((n, family.ell), dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    ctx.check(ctx.lib.cpsj_minhash_sketch(ctx.handle, fam.handle, tok.data_ptr(), off.data_ptr(), n,
                                          _max_token_of(flat_tokens, None), None, out.data_ptr(), stream))
    return out.cpu().numpy().view(_U64)
