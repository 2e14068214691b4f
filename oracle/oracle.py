"""ctypes front-end of the C oracle (cpsj_oracle.c) -- TEST INFRASTRUCTURE ONLY.

Restates the reference's host-side parameter derivation with the same
numpy/scipy calls (hashing.py:43-46 seed plumbing, :168-178 table draw
order, embed.py:39-45, cpsjoin.py:346-347 repetition seeds,
hashing.py:234-247 k*), and drives the C restatement of the hot path.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "libcpsj_oracle.so")
_lib = None

KIND_EMBED, KIND_SKETCH, KIND_CPS_TREE = 1, 2, 3


def build() -> str:
    src = os.path.join(_HERE, "cpsj_oracle.c")
    if not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


def lib():
    global _lib
    if _lib is None:
        build()  # rebuilds only when the source is newer than the library
        L = ctypes.CDLL(_SO)
        P = ctypes.c_void_p
        i64, i32, u64, dbl = ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64, ctypes.c_double
        L.orc_mix64.restype = u64
        L.orc_mix64.argtypes = [u64]
        L.orc_word_stream.argtypes = [u64, i64, u64, P]
        L.orc_minhash.argtypes = [P, P, i64, P, i32, P, ctypes.c_int]
        L.orc_sketch.argtypes = [P, P, i64, P, P, i32, P, ctypes.c_int]
        L.orc_self_join.restype = ctypes.c_int
        L.orc_self_join.argtypes = [P, P, P, i64, P, i32, P, i32, dbl, dbl, i32, i32, i32,
                                    P, i32, ctypes.c_int,
                                    ctypes.POINTER(P), ctypes.POINTER(P), ctypes.POINTER(i64),
                                    P, ctypes.POINTER(P), ctypes.POINTER(i64)]
        L.orc_self_join_ct.restype = ctypes.c_int
        L.orc_self_join_ct.argtypes = L.orc_self_join.argtypes + [ctypes.c_int]
        L.orc_self_join_frontier.restype = ctypes.c_int
        L.orc_self_join_frontier.argtypes = L.orc_self_join.argtypes[:16] + [i32, i32, i32] + \
            L.orc_self_join.argtypes[16:]
        L.orc_exact_join.restype = ctypes.c_int
        L.orc_exact_join.argtypes = [P, P, i64, ctypes.c_uint32, dbl, ctypes.c_int,
                                     ctypes.POINTER(P), ctypes.POINTER(P), ctypes.POINTER(i64)]
        L.orc_free.argtypes = [P]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


# ---------------------------------------------------------------- host params

def derive_rng(master_seed: int, *path: int) -> np.random.Generator:
    # hashing.py:43-46
    return np.random.default_rng(np.random.SeedSequence(master_seed, spawn_key=tuple(path)))


def embedding_tables(t: int, seed: int) -> np.ndarray:
    # embed.py:44-45
    return derive_rng(seed, KIND_EMBED).integers(0, 2**64, size=(t, 4, 256), dtype=np.uint64)


def sketch_tables(ell: int, seed: int) -> tuple[np.ndarray, np.ndarray]:
    # hashing.py:174-178: minhash tables first, then bit tables, one stream
    rng = derive_rng(seed, KIND_SKETCH)
    bits = 64 * ell
    mh = rng.integers(0, 2**64, size=(bits, 4, 256), dtype=np.uint64)
    bt = rng.integers(0, 2**64, size=(bits, 4, 256), dtype=np.uint64)
    return mh, bt


def rep_seeds(seed: int, reps: int) -> np.ndarray:
    # cpsjoin.py:346-347
    return derive_rng(seed, KIND_CPS_TREE).integers(0, 2**64, size=reps, dtype=np.uint64)


def kstar(lam: float, delta: float, mbits: int) -> int:
    # hashing.py:246-247
    from scipy.stats import binom
    return int(binom.ppf(delta, mbits, (1.0 + lam) / 2.0))


# ---------------------------------------------------------------- kernels

def mix64(x: int) -> int:
    return int(lib().orc_mix64(x))


def word_stream(seed: int, n: int, offset: int = 0) -> np.ndarray:
    out = np.empty(n, dtype=np.uint64)
    lib().orc_word_stream(seed, n, offset, _p(out))
    return out


def _csr(tokens, offsets):
    return (np.ascontiguousarray(tokens, dtype=np.uint32),
            np.ascontiguousarray(offsets, dtype=np.int64))


def minhash(tokens, offsets, tables, threads: int = 0) -> np.ndarray:
    tok, off = _csr(tokens, offsets)
    tables = np.ascontiguousarray(tables, dtype=np.uint64)
    n, F = len(off) - 1, tables.shape[0]
    out = np.zeros((n, F), dtype=np.uint32)
    lib().orc_minhash(_p(tok), _p(off), n, _p(tables), F, _p(out), threads)
    return out


def sketch(tokens, offsets, mh_tables, bit_tables, threads: int = 0) -> np.ndarray:
    tok, off = _csr(tokens, offsets)
    mh = np.ascontiguousarray(mh_tables, dtype=np.uint64)
    bt = np.ascontiguousarray(bit_tables, dtype=np.uint64)
    n, ell = len(off) - 1, mh.shape[0] // 64
    out = np.zeros((n, ell), dtype=np.uint64)
    lib().orc_sketch(_p(tok), _p(off), n, _p(mh), _p(bt), ell, _p(out), threads)
    return out


@dataclass
class JoinOut:
    keys: np.ndarray      # u64 (lo << 32) | hi, ascending, unique
    sims: np.ndarray      # f64
    pre_candidates: int
    candidates: int
    results: int
    max_depth: int
    peak_live_members: int
    cap_events: np.ndarray
    error: int

    @property
    def a(self):
        return (self.keys >> np.uint64(32)).astype(np.int64)

    @property
    def b(self):
        return (self.keys & np.uint64(0xFFFFFFFF)).astype(np.int64)


def _take(ptr, n, dtype):
    L = lib()
    if n:
        buf = (ctypes.c_char * (n * np.dtype(dtype).itemsize)).from_address(ptr.value)
        arr = np.frombuffer(bytes(buf), dtype=dtype).copy()
    else:
        arr = np.zeros(0, dtype=dtype)
    L.orc_free(ptr)
    return arr


def self_join(tokens, offsets, sizes, values, sketches, lam: float, *, epsilon=0.1, limit=250,
              delta=0.05, repetitions=10, seed=0, depth_cap=64, threads: int = 0,
              use_count_table: bool = False, frontier=None, rep_seed_list=None) -> JoinOut:
    """cpsjoin.py:331-351 on explicit arrays (self-join, source_ids = arange).
    ``frontier=(rank, ranks, depth)``: this rank's share of a frontier-sharded
    join (orc_self_join_frontier; the union over ranks is the join itself).
    ``rep_seed_list`` replaces the derived repetition seeds."""
    tok, off = _csr(tokens, offsets)
    sizes = np.ascontiguousarray(sizes, dtype=np.int64)
    values = np.ascontiguousarray(values, dtype=np.uint32)
    sk = np.ascontiguousarray(sketches, dtype=np.uint64)
    n, t = values.shape
    ell = sk.shape[1]
    ks = kstar(lam, delta, 64 * ell)
    seeds = rep_seeds(seed, repetitions) if rep_seed_list is None else \
        np.ascontiguousarray(rep_seed_list, dtype=np.uint64)
    repetitions = len(seeds)
    kp, sp, cp = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
    nk, nc = ctypes.c_int64(), ctypes.c_int64()
    counters = np.zeros(5, dtype=np.int64)
    if frontier is not None:
        if use_count_table:
            raise ValueError("frontier mode has no count-table rule")
        rank, ranks, fdepth = (int(x) for x in frontier)
        err = lib().orc_self_join_frontier(_p(tok), _p(off), _p(sizes), n, _p(values), t, _p(sk), ell,
                                           float(lam), float(epsilon), int(limit), ks, int(depth_cap),
                                           _p(seeds), int(repetitions), threads, rank, ranks, fdepth,
                                           ctypes.byref(kp), ctypes.byref(sp), ctypes.byref(nk),
                                           _p(counters), ctypes.byref(cp), ctypes.byref(nc))
        return JoinOut(_take(kp, nk.value, np.uint64), _take(sp, nk.value, np.float64), int(counters[0]),
                       int(counters[1]), int(counters[2]), int(counters[3]), int(counters[4]),
                       _take(cp, nc.value, np.int64), int(err))
    err = lib().orc_self_join_ct(_p(tok), _p(off), _p(sizes), n, _p(values), t, _p(sk), ell,
                                 float(lam), float(epsilon), int(limit), ks, int(depth_cap),
                                 _p(seeds), int(repetitions), threads,
                                 ctypes.byref(kp), ctypes.byref(sp), ctypes.byref(nk),
                                 _p(counters), ctypes.byref(cp), ctypes.byref(nc), int(bool(use_count_table)))
    keys = _take(kp, nk.value, np.uint64)
    sims = _take(sp, nk.value, np.float64)
    ev = _take(cp, nc.value, np.int64)
    return JoinOut(keys, sims, int(counters[0]), int(counters[1]), int(counters[2]),
                   int(counters[3]), int(counters[4]), ev, int(err))


def exact_join(tokens, offsets, d: int, lam: float, threads: int = 0):
    """All pairs with J >= lam (recall ground truth).  Returns (keys, sims)."""
    tok, off = _csr(tokens, offsets)
    n = len(off) - 1
    kp, sp = ctypes.c_void_p(), ctypes.c_void_p()
    nk = ctypes.c_int64()
    lib().orc_exact_join(_p(tok), _p(off), n, int(d), float(lam), threads,
                         ctypes.byref(kp), ctypes.byref(sp), ctypes.byref(nk))
    return _take(kp, nk.value, np.uint64), _take(sp, nk.value, np.float64)


def full_pipeline(tokens, offsets, sizes, *, lam, t=128, emb_seed=0, ell=8, seed=0,
                  repetitions=10, epsilon=0.1, limit=250, delta=0.05, depth_cap=64,
                  threads: int = 0):
    """embed_dataset + sketches + cpsjoin_self, as the reference runs them."""
    values = minhash(tokens, offsets, embedding_tables(t, emb_seed), threads)
    mh, bt = sketch_tables(ell, seed)
    sk = sketch(tokens, offsets, mh, bt, threads)
    out = self_join(tokens, offsets, sizes, values, sk, lam, epsilon=epsilon, limit=limit,
                    delta=delta, repetitions=repetitions, seed=seed, depth_cap=depth_cap,
                    threads=threads)
    return values, sk, out


# ---------------------------------------------------------------- LSH join
# SPEC.md minhash_join: the reference specifies it but ships
# no code; this numpy restatement follows the definitions stated in
# paper_1707_06814_b200/lsh.py and the shared
# BruteForce semantics (cpsjoin.py:139-157).  Small n only.

KIND_MINHASH_REP = 4
_U = np.uint64


def _mix64_vec(z):
    z = np.asarray(z, dtype=_U)
    with np.errstate(over="ignore"):
        z = z + _U(0x9E3779B97F4A7C15)
        z = (z ^ (z >> _U(30))) * _U(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> _U(27))) * _U(0x94D049BB133111EB)
        return z ^ (z >> _U(31))


def lsh_rep_plan(seed: int, reps: int, k: int, t: int, path=()):
    seeds = derive_rng(seed, KIND_MINHASH_REP, *path).integers(0, 2 ** 64, size=reps, dtype=np.uint64)
    pos = np.zeros((reps, k), dtype=np.int64)
    for r in range(reps):
        w = _mix64_vec(_U(int(seeds[r])) ^ _mix64_vec(np.arange(k, dtype=_U)))
        u = w / 2.0 ** 64
        pos[r] = np.minimum((u * t).astype(np.int64), t - 1)
    return pos, seeds


def lsh_join(tokens, offsets, sizes, values, sketches, lam: float, accept: int, pos, seeds, cost_only=False):
    """Returns (keys, sims, pre, cand, res) -- keys sorted unique."""
    tokens = np.asarray(tokens)
    offsets = np.asarray(offsets)
    sizes = np.asarray(sizes, dtype=np.int64)
    values = np.asarray(values, dtype=np.uint32)
    n = len(sizes)
    L = len(seeds)
    rbits = 0
    while ((L - 1) >> rbits) > 0:
        rbits += 1
    pre = cand = res = 0
    found = {}
    rows = [set(tokens[offsets[i]:offsets[i + 1]].tolist()) for i in range(n)]
    for r in range(L):
        h = np.full(n, int(seeds[r]), dtype=_U)
        for j in range(pos.shape[1]):
            h = _mix64_vec(h ^ values[:, pos[r, j]].astype(_U))
        key = h >> _U(rbits) if rbits else h
        order = np.argsort(key, kind="stable")
        ks = key[order]
        starts = np.flatnonzero(np.r_[True, ks[1:] != ks[:-1]])
        ends = np.r_[starts[1:], n]
        for s, e in zip(starts, ends):
            m = e - s
            if m < 2:
                continue
            pre += m * (m - 1) // 2
            if cost_only:
                continue
            mem = order[s:e]
            for a in range(m):
                x = int(mem[a])
                for b in range(a + 1, m):
                    y = int(mem[b])
                    dist = int(np.bitwise_count(sketches[x] ^ sketches[y]).sum())
                    if dist > accept:
                        continue
                    mn, mx = min(sizes[x], sizes[y]), max(sizes[x], sizes[y])
                    if not (float(mn) >= lam * float(mx) - 1e-9):
                        continue
                    cand += 1
                    inter = len(rows[x] & rows[y])
                    sim = inter / float(sizes[x] + sizes[y] - inter)
                    if sim >= lam:
                        res += 1
                        found[(min(x, y) << 32) | max(x, y)] = sim
    keys = np.array(sorted(found), dtype=np.uint64)
    sims = np.array([found[int(k)] for k in keys], dtype=np.float64)
    return keys, sims, pre, cand, res


def first_seen_dense(values: np.ndarray) -> tuple[np.ndarray, int]:
    """EmbeddedDataset.dense / .d (embed.py:108-114, 129-132) restated in
    numpy: keys (i << 32) | values[r, i] numbered by first appearance in
    row-major order.  Test infrastructure (the GPU remap's checker)."""
    n, t = values.shape
    if n == 0:
        return np.zeros((0, t), dtype=np.uint32), 0
    keys = (np.arange(t, dtype=np.uint64)[None, :] << np.uint64(32)) | values.astype(np.uint64)
    uniq, first, inverse = np.unique(keys.ravel(), return_index=True, return_inverse=True)
    rank = np.empty(len(uniq), dtype=np.int64)
    rank[np.argsort(first, kind="stable")] = np.arange(len(uniq))
    return rank[inverse].reshape(n, t).astype(np.uint32), len(uniq)
