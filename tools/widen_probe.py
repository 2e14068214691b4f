"""Timings of the section 8(f) rows on one GPU: MinHash LSH join and GPU
ingestion, each next to its host counterpart on a bounded sample.

    python tools/widen_probe.py [--cfg 2] [--lsh] [--ingest]

Prints one JSON line per measurement.
"""
import json
import os
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def cuda_time(fn, reps=3):
    import torch
    fn()
    torch.cuda.synchronize()
    best = None
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return best, out


def lsh_probe(cfg):
    from oracle.make_truth import truth_path
    from paper_1707_06814_b200 import Dataset, EmbeddingParams, embed_dataset
    from paper_1707_06814_b200.lsh import MinHashJoinParams, choose_k, minhash_join_arrays
    from paper_1707_06814_b200.workloads import CONFIGS, generate
    c = CONFIGS[cfg]
    w = generate(cfg)
    lam = c.lambdas[0]
    ds = Dataset.from_csr(w.tokens, w.offsets, w.d)
    emb = embed_dataset(EmbeddingParams(t=128, seed=7), ds, sketch=(c.ell, 7))
    t_ck, k = cuda_time(lambda: choose_k(emb, lam, phi=c.recall, seed=7), reps=1)
    truth = np.load(truth_path(cfg, 1.0, lam))["keys"]
    params = MinHashJoinParams(lambda_=lam, phi=c.recall, k=k, ell=c.ell, seed=7)
    t_join, res = cuda_time(lambda: minhash_join_arrays(emb, params), reps=2)
    keys = (res.a.astype(np.uint64) << np.uint64(32)) | res.b.astype(np.uint64)
    rec = float(np.isin(truth, keys).mean())
    print(json.dumps({"probe": "lsh", "cfg": cfg, "n": w.n, "lambda": lam, "k": int(k), "L": res.stats["L"],
                      "choose_k_s": round(t_ck, 3), "join_s": round(t_join, 4), "pairs": int(len(keys)),
                      "recall": round(rec, 4), "pre_candidates": res.counters.pre_candidates,
                      "candidates": res.counters.candidates, "sets_per_s": round(w.n / t_join)}), flush=True)


def ingest_probe(cfg):
    from paper_1707_06814_b200 import Dataset
    from paper_1707_06814_b200.ingest import from_flat, load_dataset
    from paper_1707_06814_b200.workloads import generate
    w = generate(cfg)
    rng = np.random.default_rng(0)
    # raw records: each set's tokens shuffled, 2% of records repeated, 1% single-token
    n = w.n
    sizes = np.diff(w.offsets)
    perm_rows = []
    vals = w.tokens.astype(np.int64).copy()
    for i in range(0, n, max(1, n // 64)):           # shuffle within a spread of records (cheap)
        a, b = w.offsets[i], w.offsets[i + 1]
        vals[a:b] = rng.permutation(vals[a:b])
    dup = rng.choice(n, size=n // 50, replace=False)
    extra = [vals[w.offsets[i]:w.offsets[i + 1]] for i in dup]
    vals2 = np.concatenate([vals] + extra + [np.arange(n // 100, dtype=np.int64)])
    sz2 = np.concatenate([sizes, sizes[dup], np.ones(n // 100, dtype=np.int64)])
    offs2 = np.zeros(len(sz2) + 1, dtype=np.int64)
    np.cumsum(sz2, out=offs2[1:])
    t_gpu, ds = cuda_time(lambda: from_flat(vals2, offs2, w.d), reps=2)
    assert len(ds) == n
    t_gpu_remap, ds2 = cuda_time(lambda: from_flat(vals2, offs2, None), reps=2)
    # host restatement on a bounded sample
    m = min(len(sz2), 50_000)
    lists = [vals2[offs2[i]:offs2[i + 1]] for i in range(m)]
    t0 = time.perf_counter()
    Dataset.from_token_lists(lists, d=w.d)
    t_host = time.perf_counter() - t0
    rec = {"probe": "ingest", "cfg": cfg, "records_in": int(len(sz2)), "tokens_in": int(len(vals2)),
           "gpu_s_d_given": round(t_gpu, 4), "gpu_s_dense_remap": round(t_gpu_remap, 4),
           "gpu_records_per_s": round(len(sz2) / t_gpu), "host_sample_records": m,
           "host_s": round(t_host, 3), "host_records_per_s": round(m / t_host)}
    # text loader over the same records
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "data.txt")
        t0 = time.perf_counter()
        with open(path, "w") as f:
            for i in range(len(sz2)):
                f.write(" ".join(map(str, vals2[offs2[i]:offs2[i + 1]].tolist())) + "\n")
        t_write = time.perf_counter() - t0
        nbytes = os.path.getsize(path)
        t_load, ds3 = cuda_time(lambda: load_dataset(path), reps=2)
        assert len(ds3) == n
        rec.update(text_bytes=nbytes, text_write_s=round(t_write, 1), load_dataset_s=round(t_load, 4),
                   load_dataset_GBps=round(nbytes / t_load / 1e9, 3))
    print(json.dumps(rec), flush=True)


def main():
    cfg = 2
    if "--cfg" in sys.argv:
        cfg = int(sys.argv[sys.argv.index("--cfg") + 1])
    if "--lsh" in sys.argv:
        lsh_probe(cfg)
    if "--ingest" in sys.argv:
        ingest_probe(cfg)


if __name__ == "__main__":
    main()
