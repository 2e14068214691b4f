"""Pin the C oracle against golden vectors produced by the reference itself
(oracle/gen_golden.py).  CPU only."""
import glob
import hashlib
import os

import numpy as np
import pytest

from oracle import oracle as O

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def load(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


def test_numpy_stream_matches_golden_version():
    # tables and repetition seeds are drawn on the host with numpy's PCG64;
    # the fixtures record the numpy version they were made with
    z = load("kat_minhash")
    assert str(z["numpy_version"]).split(".")[0] == np.__version__.split(".")[0]


def test_minhash_kat():
    z = load("kat_minhash")
    got = O.minhash(z["tokens"], z["offsets"], z["tables"])
    assert np.array_equal(got, z["minhash"])


def test_sketch_kat():
    z = load("kat_minhash")
    mh, bt = O.sketch_tables(int(z["sketch_ell"]), int(z["sketch_seed"]))
    got = O.sketch(z["tokens"], z["offsets"], mh, bt)
    assert np.array_equal(got, z["sketch"])


def test_mix64_word_stream_known_values():
    # SplitMix64 finaliser of 0 (a published constant of the generator)
    assert O.mix64(0) == 0xE220A8397B1DCDAF
    w = O.word_stream(9, 100)
    assert np.array_equal(w[60:], O.word_stream(9, 40, offset=60))


@pytest.mark.parametrize("lam,m,expect", [(0.5, 512, 368), (0.6, 512, 395), (0.7, 512, 422),
                                          (0.8, 512, 449), (0.9, 512, 478), (0.5, 1024, 745),
                                          (0.9, 1024, 961)])
def test_kstar_table(lam, m, expect):
    assert O.kstar(lam, 0.05, m) == expect


EMB_FIXTURES = ["planted_small", "planted_880", "dense_cluster", "c1_sample", "c3_sample", "c4_sample",
                "ct_planted", "ct_dense", "ct_c1_sample"]


def use_ct(z, k):
    key = f"j{k}_use_count_table"
    return bool(int(z[key])) if key in z.files else False


def fixture_joins(name):
    z = load(name)
    for k in range(int(z["n_joins"])):
        yield z, k


@pytest.mark.parametrize("name", EMB_FIXTURES)
def test_oracle_matches_reference_join(name):
    z = load(name)
    tok, off, sizes = z["tokens"], z["offsets"], z["sizes"]
    t, emb_seed = int(z["t"]), int(z["emb_seed"])
    values = O.minhash(tok, off, O.embedding_tables(t, emb_seed))
    assert sha(values) == str(z["values_sha"])
    for k in range(int(z["n_joins"])):
        lam, ell, seed, reps, limit, eps, delta, cap = z[f"j{k}_params"].tolist()
        mh, bt = O.sketch_tables(int(ell), int(seed))
        sk = O.sketch(tok, off, mh, bt)
        assert sha(sk) == str(z[f"j{k}_sketch_sha"])
        out = O.self_join(tok, off, sizes, values, sk, lam, epsilon=eps, limit=int(limit), delta=delta,
                          repetitions=int(reps), seed=int(seed), depth_cap=int(cap), use_count_table=use_ct(z, k))
        assert np.array_equal(out.a, z[f"j{k}_pair_a"])
        assert np.array_equal(out.b, z[f"j{k}_pair_b"])
        assert np.array_equal(out.sims, z[f"j{k}_pair_sim"])  # bit-exact f64
        got = [out.pre_candidates, out.candidates, out.results, out.max_depth, out.peak_live_members]
        assert got == z[f"j{k}_counters"].tolist()
        assert len(out.cap_events) == int(z[f"j{k}_n_depth_cap_warnings"])


@pytest.mark.parametrize("name", ["depth_cap", "synthetic_flags"])
def test_oracle_matches_reference_synthetic(name):
    z = load(name)
    tok, off, sizes, values = z["tokens"], z["offsets"], z["sizes"], z["values"]
    for k in range(int(z["n_joins"])):
        lam, ell, seed, reps, limit, eps, delta, cap = z[f"j{k}_params"].tolist()
        mh, bt = O.sketch_tables(int(ell), int(seed))
        sk = O.sketch(tok, off, mh, bt)
        assert np.array_equal(sk, z[f"j{k}_sketch"])
        out = O.self_join(tok, off, sizes, values, sk, lam, epsilon=eps, limit=int(limit), delta=delta,
                          repetitions=int(reps), seed=int(seed), depth_cap=int(cap))
        assert np.array_equal(out.a, z[f"j{k}_pair_a"])
        assert np.array_equal(out.sims, z[f"j{k}_pair_sim"])
        got = [out.pre_candidates, out.candidates, out.results, out.max_depth, out.peak_live_members]
        assert got == z[f"j{k}_counters"].tolist()
        assert len(out.cap_events) == int(z[f"j{k}_n_depth_cap_warnings"])


def brute_exact(tok, off, lam):
    n = len(off) - 1
    rows = [set(tok[off[i]:off[i + 1]].tolist()) for i in range(n)]
    out = []
    for i in range(n):
        for j in range(i + 1, n):
            inter = len(rows[i] & rows[j])
            sim = inter / (len(rows[i]) + len(rows[j]) - inter)
            if sim >= lam:
                out.append(((i << 32) | j, sim))
    return out


@pytest.mark.parametrize("lam", [0.3, 0.5, 0.7])
def test_exact_join_matches_bruteforce(lam):
    z = load("planted_880")
    tok, off = z["tokens"], z["offsets"]
    sel = 300
    off_s = off[:sel + 1]
    tok_s = tok[:off_s[-1]]
    keys, sims = O.exact_join(tok_s, off_s, int(z["d"]), lam)
    bf = brute_exact(tok_s, off_s, lam)
    assert keys.tolist() == [k for k, _ in bf]
    assert sims.tolist() == [s for _, s in bf]


def test_exact_join_c1_sample_contains_found_pairs():
    z = load("c1_sample")
    keys, _ = O.exact_join(z["tokens"], z["offsets"], int(z["d"]), 0.5)
    found = (z["j1_pair_a"].astype(np.uint64) << np.uint64(32)) | z["j1_pair_b"].astype(np.uint64)
    assert np.isin(found, keys).all()  # 100% precision of the reference output
    assert len(found) >= 0.9 * len(keys)


@pytest.mark.parametrize("name", ["dense_small", "dense_cluster_remap", "dense_c1_sample"])
def test_first_seen_dense_restatement_matches_reference(name):
    """oracle.first_seen_dense (the GPU remap's checker) reproduces the
    reference's EmbeddedDataset.dense / .d on its own fixtures."""
    import hashlib

    from oracle import oracle as O
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    if "values" in z.files:
        values = z["values"]
    else:
        values = O.minhash(z["tokens"], z["offsets"], O.embedding_tables(int(z["t"]), int(z["emb_seed"])), 1)
    assert hashlib.sha256(np.ascontiguousarray(values).tobytes()).hexdigest() == str(z["values_sha"])
    dense, d = O.first_seen_dense(values)
    assert d == int(z["d"])
    assert hashlib.sha256(np.ascontiguousarray(dense).tobytes()).hexdigest() == str(z["dense_sha"])
    assert np.array_equal(dense[:16], z["dense_head"])
