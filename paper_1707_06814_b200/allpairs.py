"""Exact set-similarity joins on the GPU: AllPairs and the naive join.

SPEC.md module ``allpairs`` -- specified by the reference
but not shipped by it -- built over the same CSR and result arena as the
CPSJoin path (csrc/exact.cu).  Besides being the exact baseline the paper
compares against (PAPER section 5.3), AllPairs is the recall oracle of the
CPSJoin bench at full BASELINE sizes, where the CPU restatement
(oracle/cpsj_oracle.c) takes too long.

Surface (SPEC names):
  frequency_order(ds)            -> tokens sorted by (frequency, id)
  prefix_length(size, lambda_)   -> |x| - ceil(lambda |x|) + 1
  allpairs_join(ds, lambda_)     -> (list[ResultPair], Counters)
  naive_join(ds, lambda_)        -> list[ResultPair]
"""
from __future__ import annotations

import ctypes
import math

import numpy as np

from .core import Counters, Dataset, ResultPair, check_threshold


def prefix_length(size: int, lambda_: float) -> int:
    """AllPairs Jaccard prefix |x| - ceil(lambda |x|) + 1.

    The product is taken with a 1e-7 margin below the ceiling so that the
    f64 rounding of lambda can only lengthen a prefix (exactness is kept:
    a longer prefix adds candidates, never loses a pair).  Same formula as
    the kernel (exact.cu ap_prefix_len)."""
    lam = check_threshold(lambda_)
    s = int(size)
    if s < 1:
        raise ValueError("size must be >= 1")
    o = max(0, math.ceil(lam * s - 1e-7))
    return min(s, max(0, s - o + 1))


def _device_csr(ds: Dataset):
    import torch

    from ._native import Context
    ctx = Context.get()
    dev = torch.device("cuda", ctx.device)
    tok, off = ds.flat_tokens()
    d_tok = torch.from_numpy(np.ascontiguousarray(tok, dtype=np.uint32).view(np.int32)).to(dev)
    d_off = torch.from_numpy(np.ascontiguousarray(off, dtype=np.int64)).to(dev)
    d = int(ds.d)
    if len(tok):
        d = max(d, int(tok.max()) + 1)
    return ctx, dev, d_tok, d_off, max(d, 1)


def frequency_order(ds: Dataset) -> np.ndarray:
    """Permutation of the token universe [0, d) sorted ascending by token
    frequency, ties by token id."""
    import torch
    ctx, dev, d_tok, _, d = _device_csr(ds)
    rank = torch.empty(d, dtype=torch.int32, device=dev)
    order = torch.empty(d, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    ctx.check(ctx.lib.cpsj_frequency_order(ctx.handle, d_tok.data_ptr(), int(d_tok.numel()), d, rank.data_ptr(),
                                           order.data_ptr(), stream))
    return order.cpu().numpy().view(np.uint32).astype(np.int64)


def exact_join_device(d_tokens, d_offsets, n: int, d: int, lambda_: float, naive: bool = False):
    """Run the exact join on a device-resident CSR (torch tensors); returns
    (keys u64 numpy, sims f64 numpy, stats dict)."""
    import torch

    from ._native import Context, JoinStats
    lam = check_threshold(lambda_)
    ctx = Context.get()
    dev = torch.device("cuda", ctx.device)
    stream = torch.cuda.current_stream(dev).cuda_stream
    st = JoinStats()
    ctx.check(ctx.lib.cpsj_exact_join(ctx.handle, d_tokens.data_ptr() if n else None,
                                      d_offsets.data_ptr() if n else None, int(n), int(max(d, 1)), float(lam),
                                      1 if naive else 0, ctypes.byref(st), stream))
    keys = np.empty(st.n_pairs, dtype=np.uint64)
    sims = np.empty(st.n_pairs, dtype=np.float64)
    ctx.check(ctx.lib.cpsj_join_copy_result(ctx.handle, keys.ctypes.data, sims.ctypes.data, st.n_pairs, None, 0,
                                            stream))
    stats = {f: int(getattr(st, f)) for f, _ in JoinStats._fields_}
    return keys, sims, stats


def allpairs_join_arrays(ds: Dataset, lambda_: float, naive: bool = False):
    """allpairs_join returning arrays (a < b rows, exact similarity)."""
    from .cpsjoin import JoinArrays
    check_threshold(lambda_)
    n = len(ds)
    if n < 2:
        z = np.zeros(0, dtype=np.int64)
        return JoinArrays(z, z.copy(), np.zeros(0), Counters(), z.copy(), {})
    _, _, d_tok, d_off, d = _device_csr(ds)
    keys, sims, stats = exact_join_device(d_tok, d_off, n, d, lambda_, naive)
    a = (keys >> np.uint64(32)).astype(np.int64)
    b = (keys & np.uint64(0xFFFFFFFF)).astype(np.int64)
    counters = Counters(stats["pre_candidates"], stats["candidates"], stats["results"], 0, 0)
    return JoinArrays(a, b, sims, counters, np.zeros(0, dtype=np.int64), stats)


def _pairs(res) -> list[ResultPair]:
    return [ResultPair(int(x), int(y), float(s))
            for x, y, s in zip(res.a.tolist(), res.b.tolist(), res.similarity.tolist())]


def allpairs_join(ds: Dataset, lambda_: float) -> tuple[list[ResultPair], Counters]:
    """Exact join by AllPairs prefix filtering: prefixes under
    the frequency order, pre-candidates from the prefix postings with the
    size filter, every distinct candidate verified exactly.  Counters:
    pre_candidates = posting pairs enumerated (with multiplicity),
    candidates = distinct pairs verified, results = pairs kept."""
    res = allpairs_join_arrays(ds, lambda_)
    return _pairs(res), res.counters


def naive_join(ds: Dataset, lambda_: float) -> list[ResultPair]:
    """All C(n, 2) pairs verified exactly."""
    return _pairs(allpairs_join_arrays(ds, lambda_, naive=True))
