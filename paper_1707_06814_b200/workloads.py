"""Seeded synthetic workloads for BASELINE.json's five configurations.

The Mann et al. benchmark datasets the paper uses are not
available here, so these generators stand in for them with the shapes,
size laws and token laws BASELINE.json names:

* background sets first, planted near-duplicates appended;
* per-set sizes from the config's size law;
* tokens drawn WITHOUT replacement per set, from a bounded Zipf law
  (P(rank r) ~ r^-s, token id = r - 1) or uniformly over [0, d), by
  sequential rejection of repeats;
* a planted pair copies a uniformly chosen background set of size s, draws
  J* ~ U[lo, hi], sets r = max(1, round(s (1 - J*) / (1 + J*))), drops r
  random tokens and adds r fresh tokens from the same law, so the pair's
  exact Jaccard is (s - r) / (s + r).

Output is a cleaned CSR (tokens sorted and unique per set, duplicate records
and records with < 2 tokens dropped, exactly as Dataset.from_token_lists
with a given universe d; core.py:60-95 of the reference).

Random streams are split per batch of sets, so a workload is a pure
function of (config, scale).  ``scale`` < 1 shrinks both the background and
the planted counts proportionally (used for the bounded CPU baseline and
parity samples).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

_BATCH = 1 << 15


@dataclass(frozen=True)
class WorkloadConfig:
    name: str
    n_background: int
    n_planted: int
    d: int
    size_law: tuple            # ("uniform", lo, hi) | ("lognormal", mean, sigma, lo, hi)
    token_law: tuple           # ("zipf", s) | ("uniform",)
    j_range: tuple
    lambdas: tuple
    recall: float
    ell: int
    data_seed: int
    emb_seed: int = 7
    join_seed: int = 7
    gpus: tuple = (1,)
    notes: str = ""


CONFIGS = {
    1: WorkloadConfig("c1-zipf-20k", 19_500, 500, 10_000, ("uniform", 50, 150), ("zipf", 1.0),
                      (0.5, 0.9), (0.5,), 0.9, 8, data_seed=1),
    2: WorkloadConfig("c2-zipf-1M", 990_000, 10_000, 1_000_000, ("uniform", 80, 120), ("zipf", 1.0),
                      (0.5, 0.95), (0.5,), 0.9, 8, data_seed=2),
    3: WorkloadConfig("c3-uniform-1M", 980_000, 20_000, 1 << 17, ("uniform", 10, 25), ("uniform",),
                      (0.5, 0.9), (0.5, 0.7), 0.9, 8, data_seed=3, gpus=(1, 8)),
    4: WorkloadConfig("c4-lognormal-500k", 495_000, 5_000, 100_000, ("lognormal", 300.0, 0.5, 50, 2000),
                      ("zipf", 0.8), (0.5, 0.9), (0.5, 0.6, 0.7, 0.8, 0.9), 0.9, 16, data_seed=4),
    5: WorkloadConfig("c5-zipf-10M", 9_900_000, 100_000, 4_000_000, ("uniform", 30, 70), ("zipf", 1.1),
                      (0.6, 0.95), (0.6,), 0.95, 8, data_seed=5, gpus=(1, 2, 4, 8)),
}


@dataclass
class Workload:
    config: WorkloadConfig
    tokens: np.ndarray      # uint32, CSR column indices
    offsets: np.ndarray     # int64, len n + 1
    d: int
    n_background: int = 0
    n_planted: int = 0
    planted_pairs: np.ndarray = field(default_factory=lambda: np.zeros((0, 2), np.int64))

    @property
    def n(self) -> int:
        return len(self.offsets) - 1

    @property
    def sizes(self) -> np.ndarray:
        return np.diff(self.offsets)


class _TokenLaw:
    def __init__(self, law: tuple, d: int):
        self.kind = law[0]
        self.d = d
        if self.kind == "zipf":
            w = np.arange(1, d + 1, dtype=np.float64) ** (-float(law[1]))
            cdf = np.cumsum(w)
            self.cdf = cdf / cdf[-1]
            self.cdf[-1] = 1.0

    def draw(self, rng: np.random.Generator, shape) -> np.ndarray:
        if self.kind == "uniform":
            return rng.integers(0, self.d, size=shape, dtype=np.int64)
        u = rng.random(shape)
        return np.minimum(np.searchsorted(self.cdf, u, side="right"), self.d - 1).astype(np.int64)


def _sizes(rng: np.random.Generator, law: tuple, n: int) -> np.ndarray:
    if law[0] == "uniform":
        return rng.integers(law[1], law[2] + 1, size=n, dtype=np.int64)
    mean, sigma, lo, hi = law[1:]
    mu = np.log(mean) - sigma * sigma / 2.0
    return np.clip(np.rint(rng.lognormal(mu, sigma, size=n)), lo, hi).astype(np.int64)


def _rows_without_replacement(rng, law: _TokenLaw, sizes: np.ndarray) -> list[np.ndarray]:
    """First sizes[i] distinct tokens of a sequential draw, per row."""
    n = len(sizes)
    out: list = [None] * n
    todo = np.arange(n)
    factor = 1.6
    while len(todo):
        s = sizes[todo]
        k = int(np.ceil(s.max() * factor)) + 8
        draws = law.draw(rng, (len(todo), k))
        order = np.argsort(draws, axis=1, kind="stable")
        srt = np.take_along_axis(draws, order, axis=1)
        first_sorted = np.ones_like(srt, dtype=bool)
        first_sorted[:, 1:] = srt[:, 1:] != srt[:, :-1]
        first = np.empty_like(first_sorted)
        np.put_along_axis(first, order, first_sorted, axis=1)
        rank = np.cumsum(first, axis=1)
        keep = first & (rank <= s[:, None])
        got = keep.sum(axis=1)
        done = got >= s
        for j in np.nonzero(done)[0]:
            out[todo[j]] = np.sort(draws[j][keep[j]])
        todo = todo[~done]
        factor *= 2.0
    return out


def generate(cfg: WorkloadConfig | int, scale: float = 1.0) -> Workload:
    if isinstance(cfg, int):
        cfg = CONFIGS[cfg]
    n_bg = max(2, int(round(cfg.n_background * scale)))
    n_pl = int(round(cfg.n_planted * scale))
    law = _TokenLaw(cfg.token_law, cfg.d)
    rows: list[np.ndarray] = []
    for b, lo in enumerate(range(0, n_bg, _BATCH)):
        rng = np.random.default_rng([cfg.data_seed, 0, b])
        cnt = min(_BATCH, n_bg - lo)
        sizes = np.minimum(_sizes(rng, cfg.size_law, cnt), cfg.d)
        rows.extend(_rows_without_replacement(rng, law, sizes))
    prng = np.random.default_rng([cfg.data_seed, 1])
    src = prng.integers(0, n_bg, size=n_pl)
    jstar = prng.uniform(cfg.j_range[0], cfg.j_range[1], size=n_pl)
    for k in range(n_pl):
        base = rows[src[k]]
        s = len(base)
        r = max(1, int(round(s * (1.0 - jstar[k]) / (1.0 + jstar[k]))))
        r = min(r, s - 1)
        keep = np.delete(base, prng.choice(s, size=r, replace=False))
        fresh: list[int] = []
        have = set(base.tolist())
        while len(fresh) < r:
            for v in law.draw(prng, 2 * r).tolist():
                if v not in have:
                    have.add(v)
                    fresh.append(v)
                    if len(fresh) == r:
                        break
        rows.append(np.sort(np.concatenate([keep, np.asarray(fresh, dtype=np.int64)])))
    planted = np.stack([src, np.arange(n_bg, n_bg + n_pl)], axis=1) if n_pl else np.zeros((0, 2), np.int64)
    tokens, offsets, kept = clean_rows(rows)
    # re-index planted pairs after cleaning (dropped rows shift ids)
    newid = np.full(len(rows), -1, dtype=np.int64)
    newid[kept] = np.arange(len(kept))
    if len(planted):
        planted = newid[planted]
        planted = planted[(planted >= 0).all(axis=1)]
    return Workload(cfg, tokens, offsets, cfg.d, n_bg, n_pl, planted)


def clean_rows(rows: list[np.ndarray]):
    """Dataset.from_token_lists(lists, d) semantics on sorted unique rows:
    drop rows with < 2 tokens, then drop duplicate rows (first kept)."""
    lens = np.fromiter((len(r) for r in rows), dtype=np.int64, count=len(rows))
    keep = lens >= 2
    seen: dict = {}
    kept = []
    for i in np.nonzero(keep)[0]:
        key = rows[i].tobytes()
        if key in seen:
            continue
        seen[key] = i
        kept.append(i)
    kept = np.asarray(kept, dtype=np.int64)
    offsets = np.zeros(len(kept) + 1, dtype=np.int64)
    np.cumsum(lens[kept], out=offsets[1:])
    tokens = np.concatenate([rows[i] for i in kept]).astype(np.uint32) if len(kept) else \
        np.zeros(0, np.uint32)
    return tokens, offsets, kept
