"""MinHash LSH similarity join on the GPU (SPEC.md module ``minhash_join``,
SPEC:381-438; Algorithm 3 of the paper, the baseline CPSJoin is compared
against in section 5.2).  The reference reserves its RNG namespace
(KIND_MINHASH_REP = 4, hashing.py:35) but ships no code, so the definitions
below are this package's, chosen to follow the SPEC's stated properties:

* repetition r has a seed from derive_rng(seed, KIND_MINHASH_REP) (prefix
  stable, like the CPSJoin repetition seeds, cpsjoin.py:346) and k embedded
  positions drawn WITH replacement, pos_j = floor(u_j t) with u the seed's
  uniform_stream -- so a pair whose embeddings agree on a fraction s of the
  t positions collides with probability s^k exactly;
* the bucket of record x is the k-tuple of its embedded values chained
  through mix64 from the repetition seed, keeping the top
  64 - ceil(log2 L) bits (tuple collisions only add candidates);
* every bucket of >= 2 records goes through the CPSJoin BruteForce: sketch
  filter, size filter, exact verification, then sort + unique.

The buckets, the BruteForce and the verification are the sm_100a kernels
of csrc/join.cu (cpsj_lsh_join); the host derives positions and seeds.
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from .core import Counters, ResultPair, check_threshold
from .embed import EmbeddedDataset
from .hashing import KIND_MINHASH_REP, derive_rng, match_threshold, uniform_stream

K_RANGE = range(2, 11)          # SPEC:392, "values of k in the range {2, 3, ..., 10}"
C_EST, C_HASH = 1.0, 1.0        # cost-model constants
PROBE_REPS = 3                  # repetitions choose_k averages the bucket cost over


@dataclass
class MinHashJoinParams:
    """threshold, target recall phi, concatenation length k
    (None = choose_k), repetitions L (None = repetitions_for_recall), sketch
    settings shared with cpsjoin, seed."""

    lambda_: float
    phi: float = 0.9
    k: int | None = None
    L: int | None = None
    ell: int = 8
    delta: float = 0.05
    seed: int = 0

    def __post_init__(self):
        check_threshold(self.lambda_)
        if not (0.0 < self.phi < 1.0):
            raise ValueError("phi must lie in (0, 1)")
        if self.k is not None and self.k < 1:
            raise ValueError("k must be at least 1")
        if self.L is not None and self.L < 1:
            raise ValueError("L must be at least 1")
        if self.ell < 1:
            raise ValueError("ell must be at least 1")
        if not (0.0 < self.delta < 1.0):
            raise ValueError("delta must lie in (0, 1)")


def repetitions_for_recall(lambda_: float, k: int, phi: float) -> int:
    """L = ceil(ln(1 / (1 - phi)) / lambda^k), at least 1."""
    check_threshold(lambda_)
    if not (0.0 < phi < 1.0):
        raise ValueError("phi must lie in (0, 1)")
    return max(1, math.ceil(math.log(1.0 / (1.0 - phi)) / lambda_ ** k))


def rep_plan(seed: int, reps: int, k: int, t: int, path: tuple = ()) -> tuple[np.ndarray, np.ndarray]:
    """(positions (reps, k) int16, seeds (reps,) u64) of the first ``reps``
    repetitions; prefix-stable in ``reps``."""
    seeds = derive_rng(seed, KIND_MINHASH_REP, *path).integers(0, 2 ** 64, size=reps, dtype=np.uint64)
    pos = np.empty((reps, k), dtype=np.int16)
    for r in range(reps):
        u = uniform_stream(int(seeds[r]), k)
        pos[r] = np.minimum((u * t).astype(np.int64), t - 1)   # u == 1.0 is possible (~2^-54)
    return pos, seeds


def _run(emb: EmbeddedDataset, lam: float, ell: int, delta: float, sketch_seed: int, k: int, pos: np.ndarray,
         seeds: np.ndarray, cost_only: bool):
    import torch

    from ._native import Context, Inputs, JoinStats, LshPlan
    n = len(emb)
    t = emb.t
    mbits = 64 * ell
    accept = int(mbits - match_threshold(lam, delta, mbits))
    ctx = Context.get()
    dev = torch.device("cuda", ctx.device)
    stream = torch.cuda.current_stream(dev).cuda_stream
    if n >= 2:
        tok, off, sizes, dvals = emb.device_inputs(ctx)
        # bucketing alone (choose_k) needs no sketches
        sk = None if cost_only else emb.sketches_device(ell, sketch_seed)
        side = emb.device_side(ctx)
        inputs = Inputs(tok.data_ptr(), off.data_ptr(), sizes.data_ptr(), n, dvals.data_ptr(), t,
                        None if sk is None else sk.data_ptr(), ell, None if side is None else side.data_ptr())
    else:
        inputs = Inputs(None, None, None, n, None, t, None, ell, None)
    pos = np.ascontiguousarray(pos, dtype=np.int16)
    seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
    plan = LshPlan(float(lam), accept, int(k), int(len(seeds)), pos.ctypes.data, seeds.ctypes.data,
                   1 if cost_only else 0)
    st = JoinStats()
    ctx.check(ctx.lib.cpsj_lsh_join(ctx.handle, ctypes.byref(inputs), ctypes.byref(plan), ctypes.byref(st), stream))
    return ctx, st, stream


def choose_k(emb: EmbeddedDataset, lambda_: float, phi: float = 0.9, seed: int = 0, ks=K_RANGE) -> int:
    """for each k, only the splitting step (bucketing) of
    PROBE_REPS probe repetitions; estimated cost of the join at target
    recall phi = L(k) * (mean sum_b C(|b|, 2) * c_est + n k c_hash); the
    argmin (ties -> smallest k)."""
    check_threshold(lambda_)
    n = len(emb)
    kmax = max(ks)
    pos_all, seeds = rep_plan(seed, PROBE_REPS, kmax, emb.t, path=(1,))
    best, best_cost = None, None
    for k in ks:
        if n >= 2:
            _, st, _ = _run(emb, lambda_, 8, 0.05, seed, k, pos_all[:, :k], seeds, cost_only=True)
            bucket = st.pre_candidates / PROBE_REPS
        else:
            bucket = 0.0
        cost = repetitions_for_recall(lambda_, k, phi) * (bucket * C_EST + n * k * C_HASH)
        if best_cost is None or cost < best_cost:
            best, best_cost = k, cost
    return int(best)


def minhash_join_arrays(emb: EmbeddedDataset, params: MinHashJoinParams):
    """minhash_join returning arrays (rows a < b, exact similarity) plus the
    k and L used (in ``stats``).  Sketches are emb.sketches(ell, seed), the
    same family cpsjoin_self uses for the same seed."""
    from .cpsjoin import JoinArrays
    n = len(emb)
    k = params.k if params.k is not None else choose_k(emb, params.lambda_, params.phi, params.seed)
    L = params.L if params.L is not None else repetitions_for_recall(params.lambda_, k, params.phi)
    if n < 2:
        z = np.zeros(0, dtype=np.int64)
        return JoinArrays(z, z.copy(), np.zeros(0), Counters(), z.copy(), {"k": k, "L": L})
    pos, seeds = rep_plan(params.seed, L, k, emb.t)
    ctx, st, stream = _run(emb, params.lambda_, params.ell, params.delta, params.seed, k, pos, seeds,
                           cost_only=False)
    from ._native import JoinStats
    keys = np.empty(st.n_pairs, dtype=np.uint64)
    sims = np.empty(st.n_pairs, dtype=np.float64)
    ctx.check(ctx.lib.cpsj_join_copy_result(ctx.handle, keys.ctypes.data, sims.ctypes.data, st.n_pairs, None, 0,
                                            stream))
    a = (keys >> np.uint64(32)).astype(np.int64)
    b = (keys & np.uint64(0xFFFFFFFF)).astype(np.int64)
    src = emb.source_ids
    if src is not None and not emb.ids_are_rows():
        ia, ib = np.asarray(src)[a], np.asarray(src)[b]
        lo, hi = np.minimum(ia, ib).astype(np.uint64), np.maximum(ia, ib).astype(np.uint64)
        _, first = np.unique((lo << np.uint64(32)) | hi, return_index=True)
        a, b, sims = lo[first].astype(np.int64), hi[first].astype(np.int64), sims[first]
    counters = Counters(int(st.pre_candidates), int(st.candidates), int(st.results), 0, 0)
    stats = {f: int(getattr(st, f)) for f, _ in JoinStats._fields_}
    stats.update(k=int(k), L=int(L))
    return JoinArrays(a, b, sims, counters, np.zeros(0, dtype=np.int64), stats)


def minhash_join(emb: EmbeddedDataset, params: MinHashJoinParams) -> tuple[list[ResultPair], Counters]:
    """MinHash LSH self-join: L repetitions of k-wise
    bucketing + BruteForce inside buckets; 100% precision."""
    res = minhash_join_arrays(emb, params)
    pairs = [ResultPair(int(x), int(y), float(s))
             for x, y, s in zip(res.a.tolist(), res.b.tolist(), res.similarity.tolist())]
    return pairs, res.counters
