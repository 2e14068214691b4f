"""Generate golden vectors by running the REFERENCE itself (in this container).

    PYTHONPATH=/root/reference/pkg/src python oracle/gen_golden.py

Writes tests/golden/*.npz.  Each file holds the CSR input, the parameters,
the reference's outputs (pairs, similarities, counters, depth-cap warning
count) and sha256 digests of its `values` and sketch matrices, plus the
numpy/scipy versions they were made with.  These pin both the C oracle
(tests/test_oracle_golden.py, CPU) and the CUDA path (tests/test_gpu_*.py).
/root/reference is never read at test time; only these files are.
"""
from __future__ import annotations

import hashlib
import logging
import os
import sys

import numpy as np
import scipy

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from simjoin import hashing as H  # noqa: E402
from simjoin.core import Dataset  # noqa: E402
from simjoin.cpsjoin import CPSJoinParams, cpsjoin_self  # noqa: E402
from simjoin.embed import EmbeddedDataset, EmbeddingParams, embed_dataset, _first_seen_dense  # noqa: E402

from paper_1707_06814_b200.workloads import generate  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


class _Count(logging.Handler):
    def __init__(self):
        super().__init__()
        self.n = 0
        self.msgs = []

    def emit(self, record):
        self.n += 1
        self.msgs.append(record.getMessage())


def run_join(emb, lam, *, ell=8, seed=0, reps=10, limit=250, eps=0.1, delta=0.05, depth_cap=64, ct=False):
    h = _Count()
    lg = logging.getLogger("simjoin.cpsjoin")
    lg.addHandler(h)
    lg.setLevel(logging.WARNING)
    try:
        pairs, c = cpsjoin_self(emb, CPSJoinParams(lambda_=lam, ell=ell, seed=seed, repetitions=reps,
                                                   limit=limit, epsilon=eps, delta=delta,
                                                   depth_cap=depth_cap, use_count_table=ct))
    finally:
        lg.removeHandler(h)
    cap_msgs = [m for m in h.msgs if "depth cap" in m]
    return dict(
        pair_a=np.array([p.a for p in pairs], dtype=np.int64),
        pair_b=np.array([p.b for p in pairs], dtype=np.int64),
        pair_sim=np.array([p.similarity for p in pairs], dtype=np.float64),
        counters=np.array([c.pre_candidates, c.candidates, c.results, c.max_depth,
                           c.peak_live_members], dtype=np.int64),
        n_depth_cap_warnings=np.int64(len(cap_msgs)),
        n_warnings=np.int64(h.n),
        params=np.array([lam, ell, seed, reps, limit, eps, delta, depth_cap], dtype=np.float64),
    )


def save(name: str, **kw):
    kw["numpy_version"] = np.array(np.__version__)
    kw["scipy_version"] = np.array(scipy.__version__)
    path = os.path.join(OUT, name + ".npz")
    np.savez_compressed(path, **kw)
    print(f"wrote {path} ({os.path.getsize(path)} B)")


def csr_of(ds):
    tok, off = ds.flat_tokens()
    return dict(tokens=tok.astype(np.uint32), offsets=off.astype(np.int64),
                sizes=ds.sizes.astype(np.int64), d=np.int64(ds.d))


def planted_lists(n_background, n_planted, seed, size=17, overlap=14):
    """Random 17-token background sets plus planted J = 0.7 pairs (the shape
    of the reference's own test fixture, tests/test_cpsjoin.py:35-48)."""
    rng = np.random.default_rng(seed)
    lists = []
    for k in range(n_planted):
        lo = 10_000 + k * (2 * size - overlap)
        common = list(range(lo, lo + overlap))
        lists.append(common + list(range(lo + overlap, lo + size)))
        lists.append(common + list(range(lo + size, lo + 2 * size - overlap)))
    for _ in range(n_background):
        lists.append(rng.choice(5000, size=size, replace=False))
    return lists


def kat_minhash():
    rng = np.random.default_rng(2024)
    lists = []
    for _ in range(60):
        k = int(rng.integers(1, 40))
        lists.append(np.unique(rng.integers(0, 600, size=k)))
    # wide tokens exercise all four key bytes
    for _ in range(20):
        k = int(rng.integers(2, 30))
        lists.append(np.unique(rng.integers(0, 2**32, size=k, dtype=np.uint64)))
    flat = np.concatenate(lists).astype(np.uint32)
    offsets = np.concatenate([[0], np.cumsum([len(x) for x in lists])]).astype(np.int64)
    tables = H.derive_rng(99, 7).integers(0, 2**64, size=(8, 4, 256), dtype=np.uint64)
    zero = np.zeros((1, 4, 256), dtype=np.uint64)
    ident = np.zeros((1, 4, 256), dtype=np.uint64)
    for b in range(4):
        ident[0, b] = np.arange(256, dtype=np.uint64) << np.uint64(8 * b)
    # hi 32 bits constant, lo bits distinguish: exercises the tie path on
    # the high word
    hi_tie = tables[:2].copy()
    hi_tie &= np.uint64(0x00000000FFFFFFFF)
    all_t = np.concatenate([tables, zero, ident, hi_tie])
    outs = np.stack([H.minhash_segments(all_t[i], flat, offsets) for i in range(len(all_t))], axis=1)
    fam = H.SketchFamily(2, 31)
    sk = H.build_sketch_matrix(fam, flat, offsets)
    save("kat_minhash", tokens=flat, offsets=offsets, tables=all_t, minhash=outs.astype(np.uint32),
         sketch_ell=np.int64(2), sketch_seed=np.int64(31), sketch=sk)


def emb_fixture(name, ds, t, emb_seed, joins):
    emb = embed_dataset(EmbeddingParams(t=t, seed=emb_seed), ds)
    out = csr_of(ds)
    out.update(t=np.int64(t), emb_seed=np.int64(emb_seed), values_sha=np.array(sha(emb.values)),
               values_head=emb.values[:8].copy())
    for k, kw in enumerate(joins):
        res = run_join(emb, **kw)
        sk = emb.sketches(kw.get("ell", 8), kw.get("seed", 0))
        res["sketch_sha"] = np.array(sha(sk))
        res["sketch_head"] = sk[:8].copy()
        res["use_count_table"] = np.int64(1 if kw.get("ct") else 0)
        for key, v in res.items():
            out[f"j{k}_{key}"] = v
    out["n_joins"] = np.int64(len(joins))
    save(name, **out)


def synthetic_fixture(name, values, lists, d_origin, joins, patch_rows=None):
    values = np.asarray(values, dtype=np.uint32)
    ds = Dataset.from_token_lists(lists, d=d_origin)
    t = values.shape[1]
    keys = (np.arange(t, dtype=np.uint64)[None, :] << np.uint64(32) | values.astype(np.uint64))
    dense_flat, d_dense = _first_seen_dense(keys.ravel())
    emb = EmbeddedDataset(values, dense_flat.reshape(values.shape).astype(np.uint32), d_dense, t, 0,
                          verify_csr=ds.csr(), sizes=ds.sizes.copy(),
                          source_ids=np.arange(len(ds), dtype=np.int64), origin=ds)
    out = csr_of(ds)
    out["values"] = values
    for k, kw in enumerate(joins):
        res = run_join(emb, **kw)
        sk = emb.sketches(kw.get("ell", 8), kw.get("seed", 0))
        res["sketch"] = sk
        for key, v in res.items():
            out[f"j{k}_{key}"] = v
    out["n_joins"] = np.int64(len(joins))
    save(name, **out)


def rs_fixture(name, r_lists, s_lists, d, t, emb_seed, joins):
    """join_rs (cpsjoin.py:354-385) on two datasets over a shared universe."""
    from simjoin.cpsjoin import join_rs
    ds_r = Dataset.from_token_lists(r_lists, d=d)
    ds_s = Dataset.from_token_lists(s_lists, d=d)
    params = EmbeddingParams(t=t, seed=emb_seed)
    er, es = embed_dataset(params, ds_r), embed_dataset(params, ds_s)
    out = {}
    for side, ds in (("r", ds_r), ("s", ds_s)):
        c = csr_of(ds)
        for k, v in c.items():
            out[f"{side}_{k}"] = v
    out.update(t=np.int64(t), emb_seed=np.int64(emb_seed))
    for k, kw in enumerate(joins):
        h = _Count()
        lg = logging.getLogger("simjoin.cpsjoin")
        lg.addHandler(h)
        try:
            pairs, c = join_rs(er, es, CPSJoinParams(lambda_=kw["lam"], seed=kw["seed"],
                                                     repetitions=kw.get("reps", 10), ell=kw.get("ell", 8)))
        finally:
            lg.removeHandler(h)
        out[f"j{k}_pair_a"] = np.array([p.a for p in pairs], dtype=np.int64)
        out[f"j{k}_pair_b"] = np.array([p.b for p in pairs], dtype=np.int64)
        out[f"j{k}_pair_sim"] = np.array([p.similarity for p in pairs], dtype=np.float64)
        out[f"j{k}_counters"] = np.array([c.pre_candidates, c.candidates, c.results, c.max_depth,
                                          c.peak_live_members], dtype=np.int64)
        out[f"j{k}_params"] = np.array([kw["lam"], kw.get("ell", 8), kw["seed"], kw.get("reps", 10), 250, 0.1,
                                        0.05, 64], dtype=np.float64)
    out["n_joins"] = np.int64(len(joins))
    save(name, **out)


def rs_main():
    # planted halves (tests/test_cpsjoin.py:434-452 shape)
    size, overlap = 17, 14
    r_lists, s_lists = [], []
    for k in range(40):
        lo = k * (2 * size - overlap)
        common = list(range(lo, lo + overlap))
        r_lists.append(common + list(range(lo + overlap, lo + size)))
        s_lists.append(common + list(range(lo + size, lo + 2 * size - overlap)))
    rng = np.random.default_rng(12)
    r_lists += [rng.choice(np.arange(2000, 6000), size=17, replace=False) for _ in range(300)]
    s_lists += [rng.choice(np.arange(2000, 6000), size=17, replace=False) for _ in range(250)]
    rs_fixture("rs_planted", r_lists, s_lists, 6000, 128, 4, [dict(lam=0.5, seed=4), dict(lam=0.6, seed=9, reps=3)])
    # same input on both sides (tests/test_cpsjoin.py:412-424 shape)
    lists = planted_lists(100, 10, 81)
    ds = Dataset.from_token_lists(lists)
    rows = [ds.records[i].tokens.tolist() for i in range(len(ds))]
    rs_fixture("rs_same", rows, rows, ds.d, 128, 15, [dict(lam=0.5, seed=15)])
    # a config-1 sample split into halves
    w1 = generate(1, scale=0.05)
    rows = [w1.tokens[w1.offsets[i]:w1.offsets[i + 1]].tolist() for i in range(w1.n)]
    rs_fixture("rs_c1_sample", rows[::2], rows[1::2], w1.d, 128, 7, [dict(lam=0.5, seed=7, reps=3)])


def ct_main():
    """use_count_table=True (cpsjoin.py:209-219,262-263): exact token-count
    flag rule; the dense cluster and a small limit make it fire."""
    emb_fixture("ct_planted", Dataset.from_token_lists(planted_lists(420, 40, 41)), 128, 7,
                [dict(lam=0.5, seed=7, ct=True, reps=4), dict(lam=0.5, seed=11, limit=40, reps=3, ct=True)])
    rng = np.random.default_rng(5)
    dense = [list(range(180)) + list(range(1000 + 10 * i, 1010 + 10 * i)) for i in range(300)]
    dense += [rng.choice(np.arange(5000, 20000), size=30, replace=False) for _ in range(300)]
    emb_fixture("ct_dense", Dataset.from_token_lists(dense), 128, 8,
                [dict(lam=0.5, seed=8, reps=3, ct=True), dict(lam=0.8, seed=4, reps=2, eps=0.3, ct=True)])
    w1 = generate(1, scale=0.1)
    ds1 = Dataset.from_token_lists([w1.tokens[w1.offsets[i]:w1.offsets[i + 1]] for i in range(w1.n)], d=w1.d)
    emb_fixture("ct_c1_sample", ds1, 128, 7, [dict(lam=0.5, seed=7, reps=3, ct=True)])


def ingest_lists_case(seed, n, d_src, dup_rate, short_rate, neg=False, big=False):
    """Raw token lists with in-record repeats, short and duplicate records."""
    rng = np.random.default_rng(seed)
    lists = []
    for _ in range(n):
        u = rng.random()
        if u < short_rate:
            k = int(rng.integers(0, 2))
            row = rng.integers(0, d_src, size=k).tolist() * int(rng.integers(1, 3))
        elif u < short_rate + dup_rate and lists:
            row = list(lists[int(rng.integers(0, len(lists)))])
            rng.shuffle(row)
        else:
            row = rng.integers(0, d_src, size=int(rng.integers(2, 40))).tolist()
            row += row[: int(rng.integers(0, 4))]       # repeats inside the record
            rng.shuffle(row)
        lists.append(row)
    if neg:
        lists = [[v - d_src // 2 for v in row] for row in lists]
    if big:
        lists = [[v * 1_000_003_777 + 12_345 for v in row] for row in lists]
    return lists


def ingest_fixture(name, lists, d):
    """Input lists and the reference's Dataset.from_token_lists output
    (core.py:60-95), with source_lines = the input index."""
    ds = Dataset.from_token_lists(lists, d=d, source_lines=list(range(len(lists))))
    vals = np.array([v for row in lists for v in row], dtype=np.int64)
    offs = np.zeros(len(lists) + 1, dtype=np.int64)
    np.cumsum([len(r) for r in lists], out=offs[1:])
    out = csr_of(ds) if len(ds) else dict(tokens=np.zeros(0, np.uint32), offsets=np.zeros(1, np.int64),
                                          sizes=np.zeros(0, np.int64), d=np.int64(ds.d))
    # the text form of the same records (one line per record)
    text = "".join(" ".join(str(v) for v in row) + "\n" for row in lists) if not np.any(vals < 0) else ""
    save(name, in_values=vals, in_offsets=offs, in_d=np.int64(-1 if d is None else d),
         out_tokens=out["tokens"], out_offsets=out["offsets"], out_d=np.int64(ds.d),
         out_source=np.asarray(ds.source_lines, dtype=np.int64), text=np.frombuffer(text.encode(), dtype=np.uint8))


def ingest_main():
    ingest_fixture("ingest_dense_remap", ingest_lists_case(1, 1500, 500, 0.1, 0.1), None)
    ingest_fixture("ingest_given_d", ingest_lists_case(2, 1500, 800, 0.15, 0.05), 800)
    ingest_fixture("ingest_negative", ingest_lists_case(3, 1000, 300, 0.1, 0.1, neg=True), None)
    ingest_fixture("ingest_big_values", ingest_lists_case(4, 1000, 5000, 0.05, 0.05, big=True), None)
    ingest_fixture("ingest_all_short", [[1], [], [2, 2, 2], [7]], None)


def dense_fixture(name: str, ds, t: int, seed: int, full: bool):
    """EmbeddedDataset.dense / .d made by the reference (_first_seen_dense,
    embed.py:108-114,129-132) -- pins the GPU remap (csrc/dense.cu)."""
    emb = embed_dataset(EmbeddingParams(t=t, seed=seed), ds)
    flat, off = ds.flat_tokens()
    kw = dict(tokens=flat.astype(np.uint32), offsets=off.astype(np.int64), d_universe=np.int64(ds.d),
              t=np.int64(t), emb_seed=np.int64(seed), values_sha=np.array(sha(emb.values)),
              dense_sha=np.array(sha(emb.dense)), dense_head=emb.dense[:16].copy(), d=np.int64(emb.d))
    if full:
        kw["values"] = emb.values
        kw["dense"] = emb.dense
    save(name, **kw)


def dense_main():
    # tests/test_embed.py:84-88,112-124 shape (make_dataset(n=10), t=8, seed 4)
    rng = np.random.default_rng(3)
    lists = [rng.choice(200, size=rng.integers(2, 25), replace=False) for _ in range(10)]
    dense_fixture("dense_small", Dataset.from_token_lists(lists), 8, 4, True)
    # heavy value sharing (a near-duplicate cluster): first-seen order matters
    rng = np.random.default_rng(5)
    dense = [list(range(180)) + list(range(1000 + 10 * i, 1010 + 10 * i)) for i in range(300)]
    dense += [rng.choice(np.arange(5000, 20000), size=30, replace=False) for _ in range(300)]
    dense_fixture("dense_cluster_remap", Dataset.from_token_lists(dense), 128, 8, False)
    w1 = generate(1, scale=0.05)
    ds1 = Dataset.from_token_lists([w1.tokens[w1.offsets[i]:w1.offsets[i + 1]] for i in range(w1.n)], d=w1.d)
    dense_fixture("dense_c1_sample", ds1, 128, 7, False)


def main():
    os.makedirs(OUT, exist_ok=True)
    if "--dense-only" in sys.argv:
        dense_main()
        return
    if "--ingest-only" in sys.argv:
        ingest_main()
        return
    if "--rs-only" in sys.argv:
        rs_main()
        return
    if "--ct-only" in sys.argv:
        ct_main()
        return
    rs_main()
    ct_main()
    dense_main()
    kat_minhash()
    # reference-fixture shapes (planted J = 0.7 pairs)
    emb_fixture("planted_small", Dataset.from_token_lists(planted_lists(60, 12, 31)), 128, 3,
                [dict(lam=0.5, seed=3)])
    emb_fixture("planted_880", Dataset.from_token_lists(planted_lists(420, 40, 41)), 128, 7,
                [dict(lam=0.5, seed=7), dict(lam=0.6, seed=9, reps=3),
                 dict(lam=0.7, seed=7, ell=16, reps=4), dict(lam=0.5, seed=11, limit=40, reps=5)])
    # dense cluster: drives the flagged brute_force_point path (cps:268-275)
    rng = np.random.default_rng(5)
    dense = [list(range(180)) + list(range(1000 + 10 * i, 1010 + 10 * i)) for i in range(300)]
    dense += [rng.choice(np.arange(5000, 20000), size=30, replace=False) for _ in range(300)]
    emb_fixture("dense_cluster", Dataset.from_token_lists(dense), 128, 8,
                [dict(lam=0.5, seed=8, reps=3), dict(lam=0.8, seed=4, reps=2, eps=0.3)])
    # BASELINE configs, scaled samples
    w1 = generate(1, scale=0.1)
    ds1 = Dataset.from_token_lists([w1.tokens[w1.offsets[i]:w1.offsets[i + 1]] for i in range(w1.n)], d=w1.d)
    emb_fixture("c1_sample", ds1, 128, 7, [dict(lam=0.5, seed=7, reps=3), dict(lam=0.5, seed=7, reps=10)])
    w3 = generate(3, scale=0.003)
    ds3 = Dataset.from_token_lists([w3.tokens[w3.offsets[i]:w3.offsets[i + 1]] for i in range(w3.n)], d=w3.d)
    emb_fixture("c3_sample", ds3, 128, 7, [dict(lam=0.5, seed=7, reps=3), dict(lam=0.7, seed=7, reps=3)])
    w4 = generate(4, scale=0.002)
    ds4 = Dataset.from_token_lists([w4.tokens[w4.offsets[i]:w4.offsets[i + 1]] for i in range(w4.n)], d=w4.d)
    emb_fixture("c4_sample", ds4, 128, 7, [dict(lam=lam, seed=7, ell=16, reps=2)
                                           for lam in (0.5, 0.6, 0.7, 0.8, 0.9)])
    # depth cap (tests/test_cpsjoin.py:373-385 shape): identical embeddings
    n = 260
    row = np.arange(128, dtype=np.uint32)
    synthetic_fixture("depth_cap", [row] * n, [[3 * i, 3 * i + 1, 3 * i + 2] for i in range(n)], 3 * n,
                      [dict(lam=0.9, seed=3, reps=10, depth_cap=6)])
    # identical-values + near-identical rows: every member flagged
    vals = np.tile(np.arange(128, dtype=np.uint32), (300, 1))
    vals[::7, :5] = 9999
    synthetic_fixture("synthetic_flags", vals, [[i, i + 1, 1000, 1001, 1002] for i in range(0, 600, 2)],
                      2000, [dict(lam=0.5, seed=2, reps=2)])


if __name__ == "__main__":
    main()
