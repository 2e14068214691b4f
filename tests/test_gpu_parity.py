"""Bit-exact parity of the sm_100a path against golden vectors made by the
reference itself (tests/golden, oracle/gen_golden.py) and against the C
oracle on seeded inputs.  Every call goes through the C ABI."""
import hashlib
import logging
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def load(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1707_06814_b200 import _native
    _native.load()


def _params(z, k):
    from paper_1707_06814_b200 import CPSJoinParams
    lam, ell, seed, reps, limit, eps, delta, cap = z[f"j{k}_params"].tolist()
    ct_key = f"j{k}_use_count_table"
    ct = bool(int(z[ct_key])) if ct_key in z.files else False
    return CPSJoinParams(lambda_=lam, ell=int(ell), seed=int(seed), repetitions=int(reps), limit=int(limit),
                         epsilon=eps, delta=delta, depth_cap=int(cap), use_count_table=ct)


def _check_join(res, z, k):
    assert np.array_equal(res.a, z[f"j{k}_pair_a"])
    assert np.array_equal(res.b, z[f"j{k}_pair_b"])
    assert np.array_equal(res.similarity, z[f"j{k}_pair_sim"])  # bit-exact f64
    c = res.counters
    assert [c.pre_candidates, c.candidates, c.results, c.max_depth, c.peak_live_members] == \
        z[f"j{k}_counters"].tolist()
    assert len(res.depth_cap_sizes) == int(z[f"j{k}_n_depth_cap_warnings"])


def test_minhash_kat_tables():
    from paper_1707_06814_b200.hashing import minhash_segments_many
    z = load("kat_minhash")
    got = minhash_segments_many(z["tables"], z["tokens"], z["offsets"])
    assert np.array_equal(got, z["minhash"])


def test_sketch_kat():
    from paper_1707_06814_b200.hashing import SketchFamily, build_sketch_matrix
    z = load("kat_minhash")
    fam = SketchFamily(int(z["sketch_ell"]), int(z["sketch_seed"]))
    assert np.array_equal(build_sketch_matrix(fam, z["tokens"], z["offsets"]), z["sketch"])


@pytest.mark.parametrize("L", [1, 2, 3, 4, 5])
def test_minhash_every_key_width_matches_oracle(L):
    # L = 5: a 17-bit universe, the folded T1/T2 table layout (minhash.cu: LW)
    from oracle import oracle as O
    from paper_1707_06814_b200.hashing import minhash_segments_many
    rng = np.random.default_rng(L)
    hi = (1 << 17) - 1 if L == 5 else (1 << (8 * L)) - 1
    rows = [np.unique(rng.integers(0, hi + 1, size=int(rng.integers(1, 300)), dtype=np.uint64)) for _ in range(400)]
    tok = np.concatenate(rows).astype(np.uint32)
    off = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int64)
    tables = O.derive_rng(5, L).integers(0, 2 ** 64, size=(70, 4, 256), dtype=np.uint64)
    got = minhash_segments_many(tables, tok, off, d=hi + 1)
    assert np.array_equal(got, O.minhash(tok, off, tables))


def test_minhash_high_word_ties_resolved_on_full_hash():
    # tables whose high 32 bits are constant: every token ties on the
    # compared word, the lane must fall back to the full 64-bit hash
    from oracle import oracle as O
    from paper_1707_06814_b200.hashing import minhash_segments_many
    rng = np.random.default_rng(3)
    rows = [np.unique(rng.integers(0, 5000, size=50)) for _ in range(200)]
    tok = np.concatenate(rows).astype(np.uint32)
    off = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int64)
    tables = O.derive_rng(8).integers(0, 2 ** 64, size=(40, 4, 256), dtype=np.uint64)
    tables[:20] &= np.uint64(0xFFFFFFFF)
    tables[20:30] = 0  # full ties: smallest token wins
    got = minhash_segments_many(tables, tok, off, d=5000)
    assert np.array_equal(got, O.minhash(tok, off, tables))


@pytest.mark.parametrize("env", [{}, {"CPSJ_K1_NO_PFX": "1"}, {"CPSJ_K1_FUSE": "1"}, {"CPSJ_K1_NO_SPLIT": "1"},
                                 {"CPSJ_K1_NO_WIDE": "1"}, {"CPSJ_K1_NO_ORDER": "1"}])
@pytest.mark.parametrize("cfg,scale,ell", [(2, 0.01, 8), (3, 0.02, 8), (4, 0.004, 16), (1, 0.3, 4)])
def test_k1_alternate_paths_match_oracle(cfg, scale, ell, env, monkeypatch):
    """Every K1 A/B switch (cached upper-byte entries off, the fused launch,
    every CTA looping over the chunks, three lookups on a 17-bit universe, no
    length order) gives the oracle's values and sketches: Zipf sets over 2^20
    tokens, uniform sets over 2^17 (the folded-table layout), long sets with
    1024 sketch functions, a 2-byte universe."""
    from oracle import oracle as O
    from paper_1707_06814_b200 import Dataset, EmbeddingParams, embed_dataset
    from paper_1707_06814_b200.workloads import generate
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    w = generate(cfg, scale=scale)
    ds = Dataset.from_csr(w.tokens, w.offsets, w.d)
    emb = embed_dataset(EmbeddingParams(t=128, seed=7), ds, sketch=(ell, 9))
    values = O.minhash(w.tokens, w.offsets, O.embedding_tables(128, 7))
    mh, bt = O.sketch_tables(ell, 9)
    sk = O.sketch(w.tokens, w.offsets, mh, bt)
    assert np.array_equal(emb.values, values)
    assert np.array_equal(emb.sketches(ell, 9), sk)
    emb2 = embed_dataset(EmbeddingParams(t=128, seed=7), ds)  # separate values and sketch launches
    assert np.array_equal(emb2.values, values)
    assert np.array_equal(emb2.sketches(ell, 9), sk)


def _sketch_gpu(mh, bt, tok, off, max_token):
    import torch

    from paper_1707_06814_b200._native import Context, Family
    ctx = Context.get()
    fam = Family(ctx, mh, bt)
    n = len(off) - 1
    dev = torch.device("cuda", ctx.device)
    t = torch.from_numpy(np.ascontiguousarray(tok, dtype=np.uint32).view(np.int32)).to(dev)
    o = torch.from_numpy(np.ascontiguousarray(off, dtype=np.int64)).to(dev)
    out = torch.full((n, mh.shape[0] // 64), -1, dtype=torch.int64, device=dev)
    ctx.check(ctx.lib.cpsj_minhash_sketch(ctx.handle, fam.handle, t.data_ptr(), o.data_ptr(), n, max_token, None,
                                          out.data_ptr(), torch.cuda.current_stream(dev).cuda_stream))
    return out.cpu().numpy().view(np.uint64)


@pytest.mark.parametrize("L", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("n_sets", [5, 3000])
def test_sketch_15bit_ties_and_bit_disagreement(L, n_sets):
    # the sketch kernel compares (top 15 hash bits, sketch bit) keys; tables
    # with few distinct top-15 values force ties on the compared bits whose
    # tied tokens carry different sketch bits, plus full high-word ties and
    # full 64-bit ties (smallest token), empty and single-token sets
    from oracle import oracle as O
    rng = np.random.default_rng(100 + L)
    hi = (1 << 17) - 1 if L == 5 else (1 << (8 * L)) - 1  # L = 5: the folded T1/T2 layout (LW)
    lens = rng.integers(0, 400, size=n_sets)
    lens[:3] = [0, 1, 2]
    rows = [np.unique(rng.integers(0, hi + 1, size=int(k), dtype=np.uint64)) for k in lens]
    tok = np.concatenate(rows).astype(np.uint32)
    off = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int64)
    g = O.derive_rng(11, L)
    mh = g.integers(0, 2 ** 64, size=(128, 4, 256), dtype=np.uint64)
    bt = g.integers(0, 2 ** 64, size=(128, 4, 256), dtype=np.uint64)
    mask17 = np.uint64((1 << 49) - 1)  # keep the low 49 bits: top 15 bits come from `few`
    few = g.integers(0, 3, size=(40, 4, 256), dtype=np.uint64) << np.uint64(49)
    mh[:40] = (mh[:40] & mask17) | few
    mh[40:60] &= np.uint64(0xFFFFFFFF)  # high word 0: every token ties on the high word
    mh[60:70] = 0  # full ties: the smallest token wins
    got = _sketch_gpu(mh, bt, tok, off, hi)
    assert np.array_equal(got, O.sketch(tok, off, mh, bt))


@pytest.mark.parametrize("L", [1, 2, 3])
def test_fused_embed_launch_matches_oracle(L):
    # cpsj_minhash_embed: values of one family and sketches of another in one
    # K1 launch (the pipelined embed's per-chunk call)
    import torch

    from oracle import oracle as O
    from paper_1707_06814_b200._native import Context, Family
    rng = np.random.default_rng(200 + L)
    hi = (1 << (8 * L)) - 1
    rows = [np.unique(rng.integers(0, hi + 1, size=int(rng.integers(1, 300)), dtype=np.uint64))
            for _ in range(700)]
    tok = np.concatenate(rows).astype(np.uint32)
    off = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int64)
    g = O.derive_rng(21, L)
    et = g.integers(0, 2 ** 64, size=(128, 4, 256), dtype=np.uint64)
    mh = g.integers(0, 2 ** 64, size=(256, 4, 256), dtype=np.uint64)
    bt = g.integers(0, 2 ** 64, size=(256, 4, 256), dtype=np.uint64)
    ctx = Context.get()
    efam, sfam = Family(ctx, et), Family(ctx, mh, bt)
    dev = torch.device("cuda", ctx.device)
    n = len(off) - 1
    t = torch.from_numpy(tok.view(np.int32)).to(dev)
    o = torch.from_numpy(off).to(dev)
    vals = torch.empty((n, 128), dtype=torch.int32, device=dev)
    sk = torch.empty((n, 4), dtype=torch.int64, device=dev)
    ctx.check(ctx.lib.cpsj_minhash_embed(ctx.handle, efam.handle, sfam.handle, t.data_ptr(), o.data_ptr(), n, hi,
                                         vals.data_ptr(), sk.data_ptr(), torch.cuda.current_stream(dev).cuda_stream))
    assert np.array_equal(vals.cpu().numpy().view(np.uint32), O.minhash(tok, off, et))
    assert np.array_equal(sk.cpu().numpy().view(np.uint64), O.sketch(tok, off, mh, bt))


EMB_FIXTURES = ["planted_small", "planted_880", "dense_cluster", "c1_sample", "c3_sample", "c4_sample",
                "ct_planted", "ct_dense", "ct_c1_sample"]


@pytest.mark.parametrize("name", EMB_FIXTURES)
def test_join_matches_reference_golden(name):
    from paper_1707_06814_b200 import Dataset, EmbeddingParams, cpsjoin_self_arrays, embed_dataset
    z = load(name)
    ds = Dataset.from_csr(z["tokens"], z["offsets"], int(z["d"]))
    emb = embed_dataset(EmbeddingParams(t=int(z["t"]), seed=int(z["emb_seed"])), ds)
    assert sha(emb.values) == str(z["values_sha"])
    for k in range(int(z["n_joins"])):
        p = _params(z, k)
        assert sha(emb.sketches(p.ell, p.seed)) == str(z[f"j{k}_sketch_sha"])
        _check_join(cpsjoin_self_arrays(emb, p), z, k)


@pytest.mark.parametrize("env", [{"CPSJ_NO_SUBTREE": "1"}, {"CPSJ_K7_TINY_SCRATCH": "1"},
                                 {"CPSJ_NO_SMALL_LEAF": "1", "CPSJ_NO_LEAF_OVERLAP": "1"},
                                 {"CPSJ_TINY_CAND_CAP": "1"}, {"CPSJ_BLOCK_LEAF": "1"}, {"CPSJ_SPLIT_OWN_SORT": "1"},
                                 {"CPSJ_DEVICE_LEVELS": "1"}, {"CPSJ_DEVICE_LEVELS": "1", "CPSJ_NO_SUBTREE": "1"}])
@pytest.mark.parametrize("name", ["planted_880", "dense_cluster", "c1_sample"])
def test_join_alternate_paths_match_reference_golden(name, env, monkeypatch):
    """The same trees through the level kernels only (no K7 handoff), through
    K7 with scratch small enough to overflow and retry, through the
    pair-packed small-leaf kernel on the main stream, with a candidate
    buffer small enough that the call re-runs, and through the opt-in
    device-driven level engine (csrc/dle.cuh): identical results."""
    from paper_1707_06814_b200 import Dataset, EmbeddingParams, cpsjoin_self_arrays, embed_dataset
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    z = load(name)
    ds = Dataset.from_csr(z["tokens"], z["offsets"], int(z["d"]))
    emb = embed_dataset(EmbeddingParams(t=int(z["t"]), seed=int(z["emb_seed"])), ds)
    for k in range(int(z["n_joins"])):
        _check_join(cpsjoin_self_arrays(emb, _params(z, k)), z, k)


@pytest.mark.parametrize("no_k7", [False, True])
@pytest.mark.parametrize("ranks,depth", [(2, 1), (3, 1), (3, 2)])
@pytest.mark.parametrize("name", ["dense_cluster", "c1_sample", "c4_sample"])
def test_frontier_sharding_equals_unsharded(name, ranks, depth, no_k7, monkeypatch):
    """Frontier sharding (distributed.shard_frontier): the ranks' pair union
    and counter sums equal the unsharded join, simulated in one process."""
    from paper_1707_06814_b200 import Dataset, EmbeddingParams, cpsjoin_self_arrays, embed_dataset
    if no_k7:
        monkeypatch.setenv("CPSJ_NO_SUBTREE", "1")
    z = load(name)
    ds = Dataset.from_csr(z["tokens"], z["offsets"], int(z["d"]))
    emb = embed_dataset(EmbeddingParams(t=int(z["t"]), seed=int(z["emb_seed"])), ds)
    p = _params(z, 0)
    ref = cpsjoin_self_arrays(emb, p)
    parts = [cpsjoin_self_arrays(emb, p, frontier=(r, ranks, depth)) for r in range(ranks)]
    keys = np.concatenate([(x.a.astype(np.uint64) << np.uint64(32)) | x.b.astype(np.uint64) for x in parts])
    sims = np.concatenate([x.similarity for x in parts])
    uk, first = np.unique(keys, return_index=True)
    assert np.array_equal(uk, (ref.a.astype(np.uint64) << np.uint64(32)) | ref.b.astype(np.uint64))
    assert np.array_equal(sims[first], ref.similarity)
    c = ref.counters
    assert sum(x.counters.pre_candidates for x in parts) == c.pre_candidates
    assert sum(x.counters.candidates for x in parts) == c.candidates
    assert sum(x.counters.results for x in parts) == c.results
    assert max(x.counters.max_depth for x in parts) == c.max_depth
    assert max(x.counters.peak_live_members for x in parts) == c.peak_live_members
    assert sum(len(x.depth_cap_sizes) for x in parts) == len(ref.depth_cap_sizes)


@pytest.mark.parametrize("no_k7", [False, True])
@pytest.mark.parametrize("ranks,depth", [(2, 1), (3, 2), (5, 1)])
@pytest.mark.parametrize("name", ["c1_sample", "c4_sample", "dense_cluster"])
def test_frontier_rank_share_matches_oracle_rank(name, ranks, depth, no_k7, monkeypatch):
    """Every rank's share of a frontier-sharded join (the size-balanced cut
    of cpsj_plan) equals the C oracle's frontier mode for that rank: same
    pairs, f64 similarities and counters, rank by rank."""
    from oracle import oracle as O
    from paper_1707_06814_b200 import Dataset, EmbeddingParams, cpsjoin_self_arrays, embed_dataset
    if no_k7:
        monkeypatch.setenv("CPSJ_NO_SUBTREE", "1")
    z = load(name)
    ds = Dataset.from_csr(z["tokens"], z["offsets"], int(z["d"]))
    emb = embed_dataset(EmbeddingParams(t=int(z["t"]), seed=int(z["emb_seed"])), ds)
    p = _params(z, 0)
    sizes = np.diff(z["offsets"]).astype(np.int64)
    for r in range(ranks):
        got = cpsjoin_self_arrays(emb, p, frontier=(r, ranks, depth))
        ref = O.self_join(z["tokens"], z["offsets"], sizes, emb.values, emb.sketches(p.ell, p.seed), p.lambda_,
                          epsilon=p.epsilon, limit=p.limit, delta=p.delta, repetitions=p.repetitions, seed=p.seed,
                          depth_cap=p.depth_cap, frontier=(r, ranks, depth))
        assert np.array_equal(got.a, ref.a) and np.array_equal(got.b, ref.b), r
        assert np.array_equal(got.similarity, ref.sims), r
        c = got.counters
        assert [c.pre_candidates, c.candidates, c.results, c.max_depth, c.peak_live_members] == \
            [ref.pre_candidates, ref.candidates, ref.results, ref.max_depth, ref.peak_live_members], r
        assert sorted(got.depth_cap_sizes.tolist()) == sorted(ref.cap_events.tolist()), r


def _synthetic_emb(z):
    from scipy.sparse import csr_matrix

    from paper_1707_06814_b200 import EmbeddedDataset
    n = len(z["offsets"]) - 1
    csr = csr_matrix((np.ones(len(z["tokens"]), np.int32), z["tokens"].astype(np.int32), z["offsets"]),
                     shape=(n, int(z["d"])))
    return EmbeddedDataset(z["values"], None, None, z["values"].shape[1], 0, verify_csr=csr, sizes=z["sizes"],
                           source_ids=np.arange(n, dtype=np.int64))


@pytest.mark.parametrize("name", ["depth_cap", "synthetic_flags"])
def test_join_synthetic_matches_reference_golden(name, caplog):
    from paper_1707_06814_b200 import cpsjoin_self_arrays
    z = load(name)
    emb = _synthetic_emb(z)
    for k in range(int(z["n_joins"])):
        p = _params(z, k)
        assert np.array_equal(emb.sketches(p.ell, p.seed), z[f"j{k}_sketch"])
        with caplog.at_level(logging.WARNING, logger="simjoin.cpsjoin"):
            caplog.clear()
            res = cpsjoin_self_arrays(emb, p)
        _check_join(res, z, k)
        n_cap = sum("depth cap" in r.getMessage() for r in caplog.records)
        assert n_cap == int(z[f"j{k}_n_depth_cap_warnings"])


@pytest.mark.parametrize("cfg,scale,lam,ell,reps", [(1, 1.0, 0.5, 8, 3), (3, 0.01, 0.7, 8, 4),
                                                    (4, 0.004, 0.6, 16, 2), (5, 0.002, 0.6, 8, 3),
                                                    (2, 0.01, 0.5, 8, 2)])
def test_join_matches_oracle_on_workloads(cfg, scale, lam, ell, reps):
    from oracle import oracle as O
    from paper_1707_06814_b200 import CPSJoinParams, Dataset, EmbeddingParams, cpsjoin_self_arrays, embed_dataset
    from paper_1707_06814_b200.workloads import generate
    w = generate(cfg, scale=scale)
    ds = Dataset.from_csr(w.tokens, w.offsets, w.d)
    emb = embed_dataset(EmbeddingParams(t=128, seed=7), ds)
    p = CPSJoinParams(lambda_=lam, ell=ell, seed=7, repetitions=reps)
    res = cpsjoin_self_arrays(emb, p)
    values, sk, ref = O.full_pipeline(w.tokens, w.offsets, w.sizes, lam=lam, emb_seed=7, ell=ell, seed=7,
                                      repetitions=reps)
    assert np.array_equal(emb.values, values)
    assert np.array_equal(emb.sketches(ell, 7), sk)
    assert np.array_equal(res.a, ref.a) and np.array_equal(res.b, ref.b)
    assert np.array_equal(res.similarity, ref.sims)
    c = res.counters
    assert [c.pre_candidates, c.candidates, c.results, c.max_depth, c.peak_live_members] == \
        [ref.pre_candidates, ref.candidates, ref.results, ref.max_depth, ref.peak_live_members]


def _csr_rows(rows):
    tok = np.concatenate([np.asarray(r, dtype=np.uint32) for r in rows])
    off = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int64)
    return tok, off


@pytest.mark.parametrize("t,ell,lam,limit,eps", [(16, 1, 0.5, 30, 0.1), (64, 3, 0.6, 5, 0.2), (128, 2, 0.7, 1, 0.0),
                                                 (33, 5, 0.55, 100, 0.5), (128, 16, 0.9, 60, 0.1)])
def test_edge_parameters_match_oracle(t, ell, lam, limit, eps):
    """Odd t (partial 128-function chunks), ell not a power of two (the
    generic BruteForce path), limit = 1, epsilon 0 / 0.5."""
    from oracle import oracle as O
    from paper_1707_06814_b200 import CPSJoinParams, Dataset, EmbeddingParams, cpsjoin_self_arrays, embed_dataset
    from paper_1707_06814_b200.workloads import generate
    w = generate(1, scale=0.03)
    emb = embed_dataset(EmbeddingParams(t=t, seed=3), Dataset.from_csr(w.tokens, w.offsets, w.d))
    p = CPSJoinParams(lambda_=lam, ell=ell, seed=5, repetitions=3, limit=limit, epsilon=eps)
    res = cpsjoin_self_arrays(emb, p)
    assert np.array_equal(emb.values, O.minhash(w.tokens, w.offsets, O.embedding_tables(t, 3)))
    ref = O.self_join(w.tokens, w.offsets, w.sizes, emb.values, emb.sketches(ell, 5), lam, epsilon=eps, limit=limit,
                      repetitions=3, seed=5)
    assert np.array_equal(emb.sketches(ell, 5), O.sketch(w.tokens, w.offsets, *O.sketch_tables(ell, 5)))
    assert np.array_equal(res.a, ref.a) and np.array_equal(res.similarity, ref.sims)
    c = res.counters
    assert [c.pre_candidates, c.candidates, c.results, c.max_depth, c.peak_live_members] == \
        [ref.pre_candidates, ref.candidates, ref.results, ref.max_depth, ref.peak_live_members]


def test_long_sets_and_wide_tokens_match_oracle():
    """Sets beyond the 16-bit position field (> 65536 tokens) and 4-byte
    token ids (the 32-function K1 path), joined through the full pipeline."""
    from oracle import oracle as O
    from paper_1707_06814_b200 import CPSJoinParams, Dataset, EmbeddingParams, cpsjoin_self_arrays, embed_dataset
    rng = np.random.default_rng(9)
    base = np.unique(rng.integers(0, 2 ** 32 - 1, size=70000, dtype=np.uint64)).astype(np.int64)
    rows = [base, np.sort(np.concatenate([base[:60000], np.unique(rng.integers(0, 2 ** 32 - 1, 12000))]))]
    rows += [np.unique(rng.integers(0, 2 ** 32 - 1, size=int(rng.integers(2, 3000)))) for _ in range(60)]
    rows = [np.unique(r) for r in rows]
    tok, off = _csr_rows(rows)
    ds = Dataset.from_csr(tok, off, 2 ** 32)
    emb = embed_dataset(EmbeddingParams(t=64, seed=1), ds)
    assert np.array_equal(emb.values, O.minhash(tok, off, O.embedding_tables(64, 1)))
    p = CPSJoinParams(lambda_=0.5, seed=2, repetitions=2, limit=20)
    res = cpsjoin_self_arrays(emb, p)
    ref = O.self_join(tok, off, np.diff(off), emb.values, emb.sketches(8, 2), 0.5, limit=20, repetitions=2, seed=2)
    assert np.array_equal(res.a, ref.a) and np.array_equal(res.similarity, ref.sims)
    assert res.counters.results == ref.results


def test_long_set_three_byte_tokens_matches_oracle():
    """A > 65536-token set with 3-byte tokens (16-bit K1's long-set path)."""
    from oracle import oracle as O
    from paper_1707_06814_b200.hashing import minhash_segments_many, sketch_family, build_sketch_matrix
    rng = np.random.default_rng(4)
    rows = [np.unique(rng.integers(0, 1 << 20, size=90000)), np.unique(rng.integers(0, 1 << 20, size=50))]
    tok, off = _csr_rows(rows)
    tables = O.derive_rng(3, 9).integers(0, 2 ** 64, size=(130, 4, 256), dtype=np.uint64)
    assert np.array_equal(minhash_segments_many(tables, tok, off, d=1 << 20), O.minhash(tok, off, tables))
    fam = sketch_family(1, 4)
    assert np.array_equal(build_sketch_matrix(fam, tok, off), O.sketch(tok, off, *O.sketch_tables(1, 4)))


def test_two_sets_and_identical_rows():
    """n = 2 (root is a leaf), a pair of identical rows (J = 1) and the
    empty result, through the C ABI."""
    from paper_1707_06814_b200 import CPSJoinParams, Dataset, EmbeddingParams, cpsjoin_self_arrays, embed_dataset
    tok, off = _csr_rows([[1, 2, 3, 4], [1, 2, 3, 5]])
    emb = embed_dataset(EmbeddingParams(seed=1), Dataset.from_csr(tok, off, 10))
    res = cpsjoin_self_arrays(emb, CPSJoinParams(lambda_=0.5, repetitions=3))
    assert res.a.tolist() == [0] and res.b.tolist() == [1] and res.similarity.tolist() == [3 / 5]
    assert res.counters.pre_candidates == 3 and res.counters.max_depth == 0
    res = cpsjoin_self_arrays(emb, CPSJoinParams(lambda_=0.9, repetitions=3))
    assert len(res.a) == 0 and res.counters.pre_candidates == 3


def test_small_limit_deep_tree_matches_oracle():
    # limit=8 forces many internal nodes and deep frontiers
    from oracle import oracle as O
    from paper_1707_06814_b200 import CPSJoinParams, Dataset, EmbeddingParams, cpsjoin_self_arrays, embed_dataset
    from paper_1707_06814_b200.workloads import generate
    w = generate(1, scale=0.1)
    ds = Dataset.from_csr(w.tokens, w.offsets, w.d)
    emb = embed_dataset(EmbeddingParams(t=64, seed=1), ds)
    p = CPSJoinParams(lambda_=0.5, seed=2, repetitions=4, limit=8, epsilon=0.3)
    res = cpsjoin_self_arrays(emb, p)
    ref = O.self_join(w.tokens, w.offsets, w.sizes, emb.values, emb.sketches(8, 2), 0.5, epsilon=0.3, limit=8,
                      repetitions=4, seed=2)
    assert np.array_equal(res.a, ref.a) and np.array_equal(res.similarity, ref.sims)
    c = res.counters
    assert [c.pre_candidates, c.candidates, c.results, c.max_depth, c.peak_live_members] == \
        [ref.pre_candidates, ref.candidates, ref.results, ref.max_depth, ref.peak_live_members]


# ---- reference test strategy through the drop-in (tests/test_cpsjoin.py shapes)

def _planted(n_background, n_planted, seed):
    from paper_1707_06814_b200 import Dataset
    rng = np.random.default_rng(seed)
    size, overlap, lists = 17, 14, []
    for k in range(n_planted):
        lo = 10_000 + k * (2 * size - overlap)
        common = list(range(lo, lo + overlap))
        lists.append(common + list(range(lo + overlap, lo + size)))
        lists.append(common + list(range(lo + size, lo + 2 * size - overlap)))
    for _ in range(n_background):
        lists.append(rng.choice(5000, size=size, replace=False))
    return Dataset.from_token_lists(lists)


def _naive(ds, lam):
    recs = [set(r.tokens.tolist()) for r in ds.records]
    out = set()
    for i in range(len(recs)):
        for j in range(i + 1, len(recs)):
            inter = len(recs[i] & recs[j])
            if inter / (len(recs[i]) + len(recs[j]) - inter) >= lam:
                out.add((i, j))
    return out


def test_small_dataset_equals_naive():
    from paper_1707_06814_b200 import CPSJoinParams, EmbeddingParams, cpsjoin_self, embed_dataset
    ds = _planted(60, 12, 31)
    pairs, c = cpsjoin_self(embed_dataset(EmbeddingParams(seed=3), ds), CPSJoinParams(lambda_=0.5, seed=3))
    assert {p.key() for p in pairs} == _naive(ds, 0.5)
    assert c.max_depth == 0


def test_recall_precision_and_exact_similarity():
    from paper_1707_06814_b200 import CPSJoinParams, EmbeddingParams, cpsjoin_self, embed_dataset, jaccard
    ds = _planted(420, 40, 41)
    pairs, c = cpsjoin_self(embed_dataset(EmbeddingParams(seed=7), ds), CPSJoinParams(lambda_=0.5, seed=7))
    truth = _naive(ds, 0.5)
    got = {p.key() for p in pairs}
    assert got <= truth and len(got) >= 0.9 * len(truth)
    for p in pairs:
        assert jaccard(ds.records[p.a], ds.records[p.b]) == p.similarity
    assert c.results <= c.candidates <= c.pre_candidates


def test_no_pairs_and_degenerate_sizes():
    from paper_1707_06814_b200 import CPSJoinParams, Dataset, EmbeddingParams, cpsjoin_self, embed_dataset
    rng = np.random.default_rng(17)
    ds = Dataset.from_token_lists([rng.choice(4000, size=10, replace=False) for _ in range(120)])
    pairs, _ = cpsjoin_self(embed_dataset(EmbeddingParams(seed=5), ds), CPSJoinParams(lambda_=0.5, seed=5))
    assert pairs == []
    one = Dataset.from_token_lists([[1, 2, 3]])
    pairs, c = cpsjoin_self(embed_dataset(EmbeddingParams(seed=1), one), CPSJoinParams(lambda_=0.5))
    assert pairs == [] and c.pre_candidates == 0 and c.peak_live_members == 0
    empty = Dataset.from_token_lists([])
    pairs, _ = cpsjoin_self(embed_dataset(EmbeddingParams(seed=1), empty), CPSJoinParams(lambda_=0.5))
    assert pairs == []


def test_deterministic_given_seed():
    from paper_1707_06814_b200 import CPSJoinParams, EmbeddingParams, cpsjoin_self, embed_dataset
    ds = _planted(300, 25, 51)
    for ct in (False, True):
        p1, c1 = cpsjoin_self(embed_dataset(EmbeddingParams(seed=9), ds),
                              CPSJoinParams(lambda_=0.6, seed=9, use_count_table=ct))
        p2, c2 = cpsjoin_self(embed_dataset(EmbeddingParams(seed=9), ds),
                              CPSJoinParams(lambda_=0.6, seed=9, use_count_table=ct))
        assert [(p.a, p.b, p.similarity) for p in p1] == [(p.a, p.b, p.similarity) for p in p2]
        assert c1 == c2


@pytest.mark.parametrize("cfg,scale,limit", [(1, 0.2, 250), (3, 0.01, 60), (1, 0.05, 20)])
def test_count_table_flag_rule_matches_oracle(cfg, scale, limit):
    from oracle import oracle as O
    from paper_1707_06814_b200 import CPSJoinParams, Dataset, EmbeddingParams, cpsjoin_self_arrays, embed_dataset
    from paper_1707_06814_b200.workloads import generate
    w = generate(cfg, scale=scale)
    emb = embed_dataset(EmbeddingParams(t=128, seed=7), Dataset.from_csr(w.tokens, w.offsets, w.d))
    p = CPSJoinParams(lambda_=0.5, seed=3, repetitions=3, limit=limit, use_count_table=True)
    res = cpsjoin_self_arrays(emb, p)
    ref = O.self_join(w.tokens, w.offsets, w.sizes, emb.values, emb.sketches(8, 3), 0.5, limit=limit,
                      repetitions=3, seed=3, use_count_table=True)
    assert np.array_equal(res.a, ref.a) and np.array_equal(res.similarity, ref.sims)
    c = res.counters
    assert [c.pre_candidates, c.candidates, c.results, c.max_depth, c.peak_live_members] == \
        [ref.pre_candidates, ref.candidates, ref.results, ref.max_depth, ref.peak_live_members]


def test_full_config1_against_oracle_and_exact_truth():
    """Config 1 at full size (n = 20,000, R = 10): bit-exact vs the oracle;
    100% precision and recall >= 0.9 against the exact join."""
    from oracle import oracle as O
    from paper_1707_06814_b200 import CPSJoinParams, Dataset, EmbeddingParams, cpsjoin_self_arrays, embed_dataset
    from paper_1707_06814_b200.workloads import generate
    w = generate(1)
    ds = Dataset.from_csr(w.tokens, w.offsets, w.d)
    emb = embed_dataset(EmbeddingParams(t=128, seed=7), ds)
    res = cpsjoin_self_arrays(emb, CPSJoinParams(lambda_=0.5, seed=7, repetitions=10))
    values, sk, ref = O.full_pipeline(w.tokens, w.offsets, w.sizes, lam=0.5, emb_seed=7, seed=7, repetitions=10)
    assert np.array_equal(res.a, ref.a) and np.array_equal(res.similarity, ref.sims)
    truth, _ = O.exact_join(w.tokens, w.offsets, w.d, 0.5)
    keys = (res.a.astype(np.uint64) << np.uint64(32)) | res.b.astype(np.uint64)
    assert np.isin(keys, truth).all()
    assert len(keys) >= 0.9 * len(truth)


@pytest.mark.parametrize("chunks", [1, 3, 8])
def test_pipelined_embed_with_sketch_hint_matches_oracle(chunks):
    from oracle import oracle as O
    from paper_1707_06814_b200 import CPSJoinParams, Dataset, EmbeddingParams, cpsjoin_self_arrays, embed_dataset
    from paper_1707_06814_b200.workloads import generate
    w = generate(1, scale=0.25)
    ds = Dataset.from_csr(w.tokens, w.offsets, w.d)
    emb = embed_dataset(EmbeddingParams(t=128, seed=7), ds, sketch=(8, 7), chunks=chunks)
    values, sk, ref = O.full_pipeline(w.tokens, w.offsets, w.sizes, lam=0.5, emb_seed=7, seed=7, repetitions=2)
    assert np.array_equal(emb.values, values)
    assert np.array_equal(emb.sketches(8, 7), sk)
    res = cpsjoin_self_arrays(emb, CPSJoinParams(lambda_=0.5, seed=7, repetitions=2))
    assert np.array_equal(res.a, ref.a) and np.array_equal(res.similarity, ref.sims)


@pytest.mark.parametrize("cfg,scale", [(2, 0.07), (3, 0.4)])
def test_default_pipelined_embed_matches_oracle(cfg, scale):
    """The DEFAULT chunk schedule (chunks=None: the rate-based schedule of
    embed._chunk_fractions, used by embed_dataset for n >= 65,536 and by the
    bench's e2e leg) gives the oracle's values, sketches and join bit for bit."""
    from oracle import oracle as O
    from paper_1707_06814_b200 import CPSJoinParams, Dataset, EmbeddingParams, cpsjoin_self_arrays, embed_dataset
    from paper_1707_06814_b200.embed import _PIPELINE_MIN_SETS, _chunk_bounds
    from paper_1707_06814_b200.workloads import generate
    w = generate(cfg, scale=scale)
    assert w.n >= _PIPELINE_MIN_SETS and len(_chunk_bounds(w.n, None, nnz=len(w.tokens), t=128, ell=8)) > 2
    ds = Dataset.from_csr(w.tokens, w.offsets, w.d)
    emb = embed_dataset(EmbeddingParams(t=128, seed=7), ds, sketch=(8, 7))
    values, sk, ref = O.full_pipeline(w.tokens, w.offsets, w.sizes, lam=0.5, emb_seed=7, seed=7, repetitions=2)
    assert np.array_equal(emb.values, values)
    assert np.array_equal(emb.sketches(8, 7), sk)
    res = cpsjoin_self_arrays(emb, CPSJoinParams(lambda_=0.5, seed=7, repetitions=2))
    assert np.array_equal(res.a, ref.a) and np.array_equal(res.b, ref.b)
    assert np.array_equal(res.similarity, ref.sims)
    c = res.counters
    assert [c.pre_candidates, c.candidates, c.results, c.max_depth, c.peak_live_members] == \
        [ref.pre_candidates, ref.candidates, ref.results, ref.max_depth, ref.peak_live_members]


# ---- R x S join, against reference-made fixtures

@pytest.mark.parametrize("name", ["rs_planted", "rs_same", "rs_c1_sample"])
def test_join_rs_matches_reference_golden(name):
    from paper_1707_06814_b200 import Dataset, EmbeddingParams, embed_dataset, join_rs_arrays
    z = load(name)
    params = EmbeddingParams(t=int(z["t"]), seed=int(z["emb_seed"]))
    er = embed_dataset(params, Dataset.from_csr(z["r_tokens"], z["r_offsets"], int(z["r_d"])))
    es = embed_dataset(params, Dataset.from_csr(z["s_tokens"], z["s_offsets"], int(z["s_d"])))
    for k in range(int(z["n_joins"])):
        res = join_rs_arrays(er, es, _params(z, k))
        assert np.array_equal(res.a, z[f"j{k}_pair_a"])
        assert np.array_equal(res.b, z[f"j{k}_pair_b"])
        assert np.array_equal(res.similarity, z[f"j{k}_pair_sim"])
        c = res.counters
        assert [c.pre_candidates, c.candidates, c.results, c.max_depth, c.peak_live_members] == \
            z[f"j{k}_counters"].tolist()


def test_join_rs_same_input_is_self_join_plus_diagonal():
    from paper_1707_06814_b200 import CPSJoinParams, EmbeddingParams, cpsjoin_self, embed_dataset, join_rs
    ds = _planted(100, 10, 81)
    params = EmbeddingParams(t=128, seed=15)
    jp = CPSJoinParams(lambda_=0.5, seed=15)
    cross, _ = join_rs(embed_dataset(params, ds), embed_dataset(params, ds), jp)
    self_pairs, _ = cpsjoin_self(embed_dataset(params, ds), jp)
    cross_keys = {(min(p.a, p.b), max(p.a, p.b)) for p in cross}
    assert cross_keys == {p.key() for p in self_pairs} | {(i, i) for i in range(len(ds))}


def test_join_rs_rejects_mismatched_embeddings():
    from paper_1707_06814_b200 import CPSJoinParams, Dataset, EmbeddingParams, embed_dataset, join_rs
    ds = Dataset.from_token_lists([[0, 1], [1, 2]], d=10)
    a = embed_dataset(EmbeddingParams(t=16, seed=1), ds)
    b = embed_dataset(EmbeddingParams(t=32, seed=1), ds)
    c = embed_dataset(EmbeddingParams(t=16, seed=2), ds)
    with pytest.raises(ValueError):
        join_rs(a, b, CPSJoinParams(lambda_=0.5, seed=1))
    with pytest.raises(ValueError):
        join_rs(a, c, CPSJoinParams(lambda_=0.5, seed=1))
