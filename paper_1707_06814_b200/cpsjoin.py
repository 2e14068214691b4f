"""CPSJoin self-join on the GPU (drop-in for the reference's simjoin.cpsjoin).

``cpsjoin_self(emb, CPSJoinParams(...))`` keeps the reference's signature,
parameters, validation messages, warnings (logger "simjoin.cpsjoin") and
return types.  Underneath, every repetition tree runs in one
level-synchronous frontier of sm_100a kernels (csrc/join.cu) behind the C
ABI; the host only derives the plan:

* k* = binom.ppf(delta, 64 ell, (1 + lambda) / 2)       (hashing.py:247)
* accept_dist = 64 ell - k*: popcount(xor) <= accept_dist  <=>  matches >= k*
* flag_dist: the largest popcount distance whose estimate
  2 (m - dist) / m - 1 exceeds (1 - eps) lambda, evaluated with numpy's own
  float64 arithmetic for every dist in [0, m] (cpsjoin.py:206,268)
* split_p = 1.0 / (lambda * t)                           (cpsjoin.py:234)
* repetition seeds from derive_rng(seed, KIND_CPS_TREE)   (cpsjoin.py:346)
"""
from __future__ import annotations

import ctypes
import logging
import math
from dataclasses import dataclass

import numpy as np

from .core import Counters, ResultPair, check_threshold
from .embed import EmbeddedDataset
from .hashing import KIND_CPS_TREE, derive_rng, match_threshold

# same logger name as the reference so existing handlers/caplog filters work
logger = logging.getLogger("simjoin.cpsjoin")


@dataclass
class CPSJoinParams:
    """Tuning knobs; defaults are the reference's (cpsjoin.py:52-78)."""

    lambda_: float
    limit: int = 250
    epsilon: float = 0.1
    ell: int = 8
    delta: float = 0.05
    t: int = 128
    repetitions: int = 10
    seed: int = 0
    use_count_table: bool = False
    depth_cap: int = 64

    def __post_init__(self):
        check_threshold(self.lambda_)
        if self.limit < 1:
            raise ValueError("limit must be at least 1")
        if not (0.0 <= self.epsilon < 1.0):
            raise ValueError("epsilon must lie in [0, 1)")
        if not (0.0 < self.delta < 1.0):
            raise ValueError("delta must lie in (0, 1)")
        if self.repetitions < 1:
            raise ValueError("repetitions must be positive")
        if self.ell < 1:
            raise ValueError("ell must be at least 1")


@dataclass
class JoinPlan:
    kstar: int
    accept_dist: int
    flag_dist: int
    split_p: float
    rep_seeds: np.ndarray


def flag_distance(lam: float, epsilon: float, mbits: int) -> int:
    """Largest dist with est(dist) > (1 - eps) lam, in numpy float64."""
    dist = np.arange(mbits + 1, dtype=np.uint64)
    est = 2.0 * (mbits - dist) / mbits - 1.0
    cond = est > (1.0 - epsilon) * lam
    hits = np.nonzero(cond)[0]
    d = int(hits[-1]) if len(hits) else -1
    # the estimate is monotone in dist, so the rule is a prefix
    assert np.array_equal(cond, dist <= d) if d >= 0 else not cond.any()
    return d


def make_plan(params: CPSJoinParams, t: int) -> JoinPlan:
    mbits = 64 * params.ell
    kstar = match_threshold(params.lambda_, params.delta, mbits)
    return JoinPlan(
        kstar=kstar,
        accept_dist=int(mbits - kstar),
        flag_dist=flag_distance(params.lambda_, params.epsilon, mbits),
        split_p=1.0 / (params.lambda_ * t),
        rep_seeds=derive_rng(params.seed, KIND_CPS_TREE).integers(0, 2 ** 64, size=params.repetitions,
                                                                  dtype=np.uint64),
    )


@dataclass
class JoinArrays:
    """Array form of a join result: rows a < b, exact similarity."""

    a: np.ndarray
    b: np.ndarray
    similarity: np.ndarray
    counters: Counters
    depth_cap_sizes: np.ndarray
    stats: dict


def _run(emb: EmbeddedDataset, params: CPSJoinParams, rep_indices=None, map_ids: bool = True,
         frontier=None) -> JoinArrays:
    import torch

    from ._native import Context, Inputs, JoinStats, Plan
    vals = emb.values if emb._values is not None else None
    t = emb.t
    if vals is not None and vals.shape[1] != t:
        raise ValueError("embedded dataset is inconsistent")
    n = len(emb)
    plan = make_plan(params, t)
    ctx = Context.get()
    dev = torch.device("cuda", ctx.device)
    stream = torch.cuda.current_stream(dev).cuda_stream
    if n >= 2:
        tok, off, sizes, dvals = emb.device_inputs(ctx)
        if dvals.shape[1] != t:
            raise ValueError("embedded dataset is inconsistent")
        sk = emb.sketches_device(params.ell, params.seed)
        side = emb.device_side(ctx)
        inputs = Inputs(tok.data_ptr(), off.data_ptr(), sizes.data_ptr(), n, dvals.data_ptr(), t,
                        sk.data_ptr(), params.ell, None if side is None else side.data_ptr())
    else:
        inputs = Inputs(None, None, None, n, None, t, None, params.ell, None)
    seeds = plan.rep_seeds if rep_indices is None else plan.rep_seeds[np.asarray(rep_indices, dtype=np.int64)]
    seeds = np.ascontiguousarray(seeds)
    cplan = Plan(float(params.lambda_), int(params.limit), int(params.depth_cap), plan.accept_dist,
                 plan.flag_dist, float(plan.split_p), seeds.ctypes.data, int(len(seeds)), _value_bits(emb),
                 1 if params.use_count_table else 0, (1.0 - params.epsilon) * params.lambda_,
                 *(frontier if frontier is not None else (0, 1, 0)))
    st = JoinStats()
    ctx.check(ctx.lib.cpsj_self_join(ctx.handle, ctypes.byref(inputs), ctypes.byref(cplan), ctypes.byref(st),
                                     stream))
    keys = np.empty(st.n_pairs, dtype=np.uint64)
    sims = np.empty(st.n_pairs, dtype=np.float64)
    caps = np.empty(st.n_depth_cap_events, dtype=np.int64)
    ctx.check(ctx.lib.cpsj_join_copy_result(ctx.handle, keys.ctypes.data, sims.ctypes.data, st.n_pairs,
                                            caps.ctypes.data, st.n_depth_cap_events, stream))
    a = (keys >> np.uint64(32)).astype(np.int64)
    b = (keys & np.uint64(0xFFFFFFFF)).astype(np.int64)
    src = emb.source_ids
    if map_ids and src is not None and not emb.ids_are_rows():
        # map rows to source ids, re-orient and re-dedup (cpsjoin.py:313-318)
        ia, ib = np.asarray(src)[a], np.asarray(src)[b]
        lo, hi = np.minimum(ia, ib).astype(np.uint64), np.maximum(ia, ib).astype(np.uint64)
        k2 = (lo << np.uint64(32)) | hi
        _, first = np.unique(k2, return_index=True)
        a, b, sims = lo[first].astype(np.int64), hi[first].astype(np.int64), sims[first]
    counters = Counters(int(st.pre_candidates), int(st.candidates), int(st.results), int(st.max_depth),
                        int(st.peak_live_members))
    stats = {f: int(getattr(st, f)) for f, _ in JoinStats._fields_}
    return JoinArrays(a, b, sims, counters, caps, stats)


def _value_bits(emb: EmbeddedDataset) -> int:
    """Bits of the largest MinHash value: every value is a token of the
    CSR, so the token universe bounds it; host-provided values are checked
    directly.  0 means "use all 32 bits"."""
    if emb._width and "values" in emb._dev and not getattr(emb, "_values_host_set", False):
        vmax = int(emb._width) - 1          # values computed by K1 from this CSR
    elif emb._values is not None:
        # host-provided values: recomputed every call (an in-place change of
        # the array must not leave a stale bound; the split kernels also
        # reject any value >= 2^value_bits on the device)
        vmax = int(emb._values.max()) if emb._values.size else 0
    else:
        return 0
    return max(1, vmax.bit_length())


def _emit_warnings(res: JoinArrays, params: CPSJoinParams, n: int) -> None:
    for m in res.depth_cap_sizes.tolist():
        logger.warning("depth cap %d reached with %d members; branch aborted", params.depth_cap, m)
    eps_eff = max(params.epsilon, 0.05)
    if n > 1:
        bound = 12.0 * math.log(n) / eps_eff
        if res.counters.max_depth > bound:
            logger.warning("observed recursion depth %d exceeds advisory bound %.1f for n=%d",
                           res.counters.max_depth, bound, n)


def cpsjoin_self_arrays(emb: EmbeddedDataset, params: CPSJoinParams, rep_indices=None,
                        frontier: tuple[int, int, int] | None = None) -> JoinArrays:
    """cpsjoin_self returning numpy arrays instead of ResultPair objects.
    ``rep_indices`` restricts the run to a subset of the repetition trees;
    ``frontier=(rank, ranks, depth)`` keeps this rank's share of the nodes at
    ``depth`` (both used to shard the join across GPUs, distributed.py)."""
    if frontier is not None:
        rank, ranks, depth = (int(x) for x in frontier)
        if not (0 <= rank < ranks and depth >= 0):
            raise ValueError("frontier must be (rank, ranks, depth) with 0 <= rank < ranks and depth >= 0")
        frontier = (rank, ranks, depth)
    res = _run(emb, params, rep_indices, frontier=frontier)
    _emit_warnings(res, params, len(emb))
    return res


def cpsjoin_self(emb: EmbeddedDataset, params: CPSJoinParams) -> tuple[list[ResultPair], Counters]:
    """Self-join: all pairs with exact similarity >= lambda, found by
    ``repetitions`` independent Chosen Path trees (cpsjoin.py:331-351)."""
    res = cpsjoin_self_arrays(emb, params)
    pairs = [ResultPair(int(x), int(y), float(s))
             for x, y, s in zip(res.a.tolist(), res.b.tolist(), res.similarity.tolist())]
    return pairs, res.counters


def join_rs_arrays(r: EmbeddedDataset, s: EmbeddedDataset, params: CPSJoinParams) -> JoinArrays:
    """join_rs returning arrays: a = record id in r, b = record id in s."""
    from .embed import union_embedded
    union = union_embedded(r, s)
    res = _run(union, params, map_ids=False)
    n = len(union)
    _emit_warnings(res, params, n)
    if len(res.a):
        # same-side pairs never reach verification, and r rows precede s
        # rows, so the smaller row of every pair is the r side
        src = np.asarray(union.source_ids)
        ids_r = src[res.a].astype(np.uint64)
        ids_s = src[res.b].astype(np.uint64)
        keys = (ids_r << np.uint64(32)) | ids_s
        _, first = np.unique(keys, return_index=True)      # cpsjoin.py:381-384
        res.a = ids_r[first].astype(np.int64)
        res.b = ids_s[first].astype(np.int64)
        res.similarity = res.similarity[first]
    return res


def join_rs(r: EmbeddedDataset, s: EmbeddedDataset, params: CPSJoinParams
            ) -> tuple[list[ResultPair], Counters]:
    """Cross join of two embeddings sharing a function family
    (cpsjoin.py:354-385): a self-join over the tagged union whose BruteForce
    suppresses same-side pairs before verification; ``a`` is a record id of
    r and ``b`` one of s."""
    res = join_rs_arrays(r, s, params)
    pairs = [ResultPair(int(x), int(y), float(v))
             for x, y, v in zip(res.a.tolist(), res.b.tolist(), res.similarity.tolist())]
    return pairs, res.counters
