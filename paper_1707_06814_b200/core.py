"""Data model of the drop-in: records, datasets, result pairs, counters.

Mirrors the reference's simjoin.core (core.py) interface -- same class and
function names, argument meaning and errors -- with a CSR-first Dataset so
that million-set inputs never materialise per-record Python objects unless
asked (``Dataset.records`` is built lazily).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass(frozen=True, eq=False)
class Record:
    """One set: an ordinal id and a strictly increasing uint32 token array
    (reference core.py:24-32)."""

    id: int
    tokens: np.ndarray

    def __len__(self) -> int:
        return len(self.tokens)


class Dataset:
    """Sets over the token universe [0, d), stored as CSR (reference
    core.py:35-112).  Immutable after construction."""

    def __init__(self, records: list[Record] | None = None, d: int = 0,
                 source_lines: list[int] | None = None, *, _csr: tuple | None = None):
        if _csr is not None:
            tokens, offsets = _csr
        else:
            records = records or []
            offsets = np.zeros(len(records) + 1, dtype=np.int64)
            if records:
                np.cumsum([len(r) for r in records], out=offsets[1:])
                tokens = np.concatenate([np.asarray(r.tokens, dtype=np.uint32) for r in records])
            else:
                tokens = np.zeros(0, dtype=np.uint32)
        self.tokens = np.ascontiguousarray(tokens, dtype=np.uint32)
        self.offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        self.d = int(d)
        self.source_lines = source_lines
        self._records = records if _csr is None else None
        self._csr = None
        self._freq = None
        self._nonempty = True if _csr is not None else None

    # -- construction ---------------------------------------------------
    @classmethod
    def from_token_lists(cls, token_lists, d: int | None = None,
                         source_lines: list[int] | None = None) -> "Dataset":
        """Sort + dedup tokens per record, drop records with < 2 tokens,
        drop duplicate records (first kept), and, when ``d`` is None, remap
        tokens to dense ids by ascending value (reference core.py:60-95)."""
        rows, kept_lines, seen = [], [], set()
        for idx, toks in enumerate(token_lists):
            arr = np.unique(np.fromiter((int(v) for v in toks), dtype=np.int64))
            if arr.size < 2:
                continue
            key = arr.tobytes()
            if key in seen:
                continue
            seen.add(key)
            rows.append(arr)
            if source_lines is not None:
                kept_lines.append(source_lines[idx])
        lines = kept_lines if source_lines is not None else None
        if not rows:
            return cls([], d if d is not None else 0, source_lines=[] if source_lines is not None else None)
        flat = np.concatenate(rows)
        if d is None:
            universe, flat = np.unique(flat, return_inverse=True)
            d = len(universe)
        elif flat.min() < 0 or flat.max() >= d:
            # the reference fails the same way when it builds the CSR (core.py:97-107)
            raise ValueError("column index exceeds matrix dimensions")
        offsets = np.zeros(len(rows) + 1, dtype=np.int64)
        np.cumsum([len(r) for r in rows], out=offsets[1:])
        return cls(d=d, source_lines=lines, _csr=(flat.astype(np.uint32), offsets))

    @classmethod
    def from_csr(cls, tokens: np.ndarray, offsets: np.ndarray, d: int) -> "Dataset":
        """Trusted fast path: rows already sorted, unique, >= 2 tokens and
        pairwise distinct (what from_token_lists would produce with ``d``)."""
        return cls(d=d, _csr=(tokens, offsets))

    @property
    def rows_nonempty(self) -> bool:
        """Every record is non-empty (guaranteed by from_token_lists and the
        trusted from_csr; checked once for hand-built record lists)."""
        if self._nonempty is None:
            self._nonempty = bool(np.all(np.diff(self.offsets) > 0))
        return self._nonempty

    # -- reference surface ----------------------------------------------
    def __len__(self) -> int:
        return len(self.offsets) - 1

    @property
    def sizes(self) -> np.ndarray:
        return np.diff(self.offsets)

    @property
    def records(self) -> list[Record]:
        if self._records is None:
            t, o = self.tokens, self.offsets
            self._records = [Record(i, t[o[i]:o[i + 1]]) for i in range(len(self))]
        return self._records

    @property
    def token_frequency(self) -> np.ndarray:
        if self._freq is None:
            self._freq = np.bincount(self.tokens, minlength=self.d).astype(np.int64)
        return self._freq

    def csr(self):
        """Record-by-token incidence matrix (int32 CSR), built lazily."""
        if self._csr is None:
            from scipy.sparse import csr_matrix
            data = np.ones(len(self.tokens), dtype=np.int32)
            self._csr = csr_matrix((data, self.tokens.astype(np.int32), self.offsets),
                                   shape=(len(self), self.d))
        return self._csr

    def flat_tokens(self) -> tuple[np.ndarray, np.ndarray]:
        return self.tokens, self.offsets


@dataclass(frozen=True)
class ResultPair:
    """Output pair of record ids with its exact similarity; a < b for
    self-joins (reference core.py:115-136)."""

    a: int
    b: int
    similarity: float = field(compare=False)

    @classmethod
    def canonical(cls, a: int, b: int, similarity: float) -> "ResultPair":
        if a == b:
            raise ValueError("self-pairs are never reported")
        return cls(min(a, b), max(a, b), similarity)

    def key(self) -> tuple[int, int]:
        return (self.a, self.b)


@dataclass
class Counters:
    """Candidate-pipeline tallies (reference core.py:139-162)."""

    pre_candidates: int = 0
    candidates: int = 0
    results: int = 0
    max_depth: int = 0
    peak_live_members: int = 0

    def merge(self, other: "Counters") -> None:
        self.pre_candidates += other.pre_candidates
        self.candidates += other.candidates
        self.results += other.results
        self.max_depth = max(self.max_depth, other.max_depth)
        self.peak_live_members = max(self.peak_live_members, other.peak_live_members)


def check_threshold(lam: float) -> float:
    if not (0.0 < lam < 1.0):
        raise ValueError(f"threshold must be in (0, 1), got {lam}")
    return float(lam)


# scalar host helpers (not on the kernel path; reference core.py:172-242)

def intersection_size(x: Record, y: Record) -> int:
    return int(np.intersect1d(x.tokens, y.tokens, assume_unique=True).size)


def jaccard(x: Record, y: Record) -> float:
    if len(x) == 0 and len(y) == 0:
        raise ValueError("jaccard of two empty records is undefined")
    inter = intersection_size(x, y)
    return inter / (len(x) + len(y) - inter)


def braun_blanquet(x: Record, y: Record, t: int) -> float:
    if len(x) != t or len(y) != t:
        raise ValueError(f"braun_blanquet requires |x| = |y| = {t}, got {len(x)} and {len(y)}")
    return intersection_size(x, y) / t


def verify_pair(x: Record, y: Record, lam: float) -> float | None:
    if len(x) == 0 and len(y) == 0:
        raise ValueError("cannot verify two empty records")
    inter = intersection_size(x, y)
    sim = inter / (len(x) + len(y) - inter)
    return sim if sim >= lam else None


def dedup_pairs(pairs: list[ResultPair]) -> list[ResultPair]:
    out: list[ResultPair] = []
    for p in sorted(pairs, key=ResultPair.key):
        if not out or out[-1].key() != p.key():
            out.append(p)
    return out

