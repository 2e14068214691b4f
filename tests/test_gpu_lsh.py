"""MinHash LSH join (SPEC minhash_join; lsh.py + cpsj_lsh_join) against the
numpy restatement in oracle/oracle.py: same pairs, bit-exact similarities,
same counters; plus the SPEC's stated properties."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1707_06814_b200 import _native
    _native.load()


def _planted(seed, n_bg=900, n_pl=150, d=3000, lo=20, hi=60):
    from paper_1707_06814_b200 import Dataset
    rng = np.random.default_rng(seed)
    rows = [np.sort(rng.choice(d, size=int(rng.integers(lo, hi + 1)), replace=False)) for _ in range(n_bg)]
    for _ in range(n_pl):
        src = rows[int(rng.integers(0, n_bg))]
        r = max(1, int(len(src) * rng.uniform(0.02, 0.3)))
        keep = rng.choice(len(src), size=len(src) - r, replace=False)
        rows.append(np.unique(np.concatenate([src[keep], rng.integers(0, d, size=r)])))
    return Dataset.from_token_lists(rows, d=d)


def _embed(ds, ell=8, seed=7):
    from paper_1707_06814_b200 import EmbeddingParams, embed_dataset
    emb = embed_dataset(EmbeddingParams(t=128, seed=7), ds)
    return emb, emb.values, emb.sketches(ell, seed)


def _oracle(ds, values, sk, lam, ell, k, L, seed, delta=0.05):
    from oracle import oracle as O
    pos, seeds = O.lsh_rep_plan(seed, L, k, 128)
    mbits = 64 * ell
    accept = mbits - O.kstar(lam, delta, mbits)
    return O.lsh_join(ds.tokens, ds.offsets, ds.sizes, values, sk, lam, accept, pos, seeds)


@pytest.mark.parametrize("k,L,lam", [(3, 8, 0.5), (2, 4, 0.5), (4, 12, 0.6), (1, 2, 0.7)])
def test_lsh_matches_oracle(k, L, lam):
    from oracle import oracle as O
    from paper_1707_06814_b200.lsh import MinHashJoinParams, minhash_join_arrays, rep_plan
    ds = _planted(k)
    emb, values, sk = _embed(ds)
    # the host plan is the oracle's restatement
    pos, seeds = rep_plan(7, L, k, 128)
    opos, oseeds = O.lsh_rep_plan(7, L, k, 128)
    assert np.array_equal(pos, opos) and np.array_equal(seeds, oseeds)
    res = minhash_join_arrays(emb, MinHashJoinParams(lambda_=lam, k=k, L=L, seed=7))
    keys, sims, pre, cand, nres = _oracle(ds, values, sk, lam, 8, k, L, 7)
    got = (res.a.astype(np.uint64) << np.uint64(32)) | res.b.astype(np.uint64)
    assert len(keys) > 0
    assert np.array_equal(got, keys)
    assert np.array_equal(res.similarity, sims)
    c = res.counters
    assert (c.pre_candidates, c.candidates, c.results) == (pre, cand, nres)
    assert res.stats["k"] == k and res.stats["L"] == L


def test_lsh_large_bucket_tiles():
    """One bucket of 600 identical records: 32x32 tiles beyond the CPSJoin
    leaf limit (closed-form tile index), all C(600, 2) pairs at 1.0."""
    from paper_1707_06814_b200 import Dataset
    from paper_1707_06814_b200.lsh import MinHashJoinParams, minhash_join_arrays
    n, row = 600, np.arange(5, 25, dtype=np.uint32)
    ds = Dataset.from_csr(np.tile(row, n), np.arange(n + 1, dtype=np.int64) * len(row), 40)
    emb, _, _ = _embed(ds)
    res = minhash_join_arrays(emb, MinHashJoinParams(lambda_=0.9, k=3, L=1, seed=1))
    assert len(res.a) == n * (n - 1) // 2 and np.all(res.similarity == 1.0)
    assert res.counters.pre_candidates == n * (n - 1) // 2 == res.counters.candidates


def test_lsh_edge_cases():
    from paper_1707_06814_b200 import Dataset
    from paper_1707_06814_b200.lsh import MinHashJoinParams, minhash_join
    ds = Dataset.from_token_lists([[1, 2, 3]], d=5)
    emb, _, _ = _embed(ds)
    pairs, c = minhash_join(emb, MinHashJoinParams(lambda_=0.5, k=2, L=3))
    assert pairs == [] and c.pre_candidates == 0
    # all-identical records -> all pairs in the first repetition
    n, row = 30, np.arange(3, 12, dtype=np.uint32)
    ds = Dataset.from_csr(np.tile(row, n), np.arange(n + 1, dtype=np.int64) * len(row), 20)
    emb, _, _ = _embed(ds)
    pairs, c = minhash_join(emb, MinHashJoinParams(lambda_=0.5, k=5, L=1))
    assert len(pairs) == n * (n - 1) // 2


def test_choose_k_matches_cost_model():
    """choose_k = argmin over k of L(k) * (mean bucket cost + n k), with the
    bucket cost recomputed by the oracle's restatement."""
    from oracle import oracle as O
    from paper_1707_06814_b200.lsh import PROBE_REPS, choose_k, repetitions_for_recall
    ds = _planted(3, n_bg=600, n_pl=100, d=400, lo=10, hi=30)
    emb, values, sk = _embed(ds)
    lam = 0.5
    pos, seeds = O.lsh_rep_plan(0, PROBE_REPS, 10, 128, path=(1,))
    costs = {}
    for k in range(2, 11):
        _, _, pre, _, _ = O.lsh_join(ds.tokens, ds.offsets, ds.sizes, values, sk, lam, 0, pos[:, :k], seeds,
                                     cost_only=True)
        costs[k] = repetitions_for_recall(lam, k, 0.9) * (pre / PROBE_REPS + len(ds) * k)
    want = min(costs, key=lambda k: (costs[k], k))
    assert choose_k(emb, lam) == want
    # pairwise-disjoint records: singleton buckets, smallest k wins
    from paper_1707_06814_b200 import Dataset
    disj = Dataset.from_csr(np.arange(400, dtype=np.uint32), np.arange(0, 401, 4, dtype=np.int64), 400)
    emb2, _, _ = _embed(disj)
    assert choose_k(emb2, 0.5) == 2


def test_collision_probability_is_braun_blanquet_to_the_k():
    """per-repetition collision probability of a pair whose
    embeddings agree on a fraction s of the positions is s^k (Monte Carlo,
    3 sigma), measured through the device bucketing (cost_only)."""
    from paper_1707_06814_b200 import Dataset
    from paper_1707_06814_b200.lsh import _run, rep_plan
    x = np.arange(0, 40, dtype=np.uint32)
    y = np.concatenate([np.arange(0, 30), np.arange(100, 110)]).astype(np.uint32)
    ds = Dataset.from_csr(np.concatenate([x, y]), np.array([0, 40, 80]), 200)
    emb, values, _ = _embed(ds)
    s = float(np.mean(values[0] == values[1]))
    k, L = 2, 4000
    pos, seeds = rep_plan(11, L, k, 128)
    _, st, _ = _run(emb, 0.5, 8, 0.05, 0, k, pos, seeds, cost_only=True)
    p = s ** k
    freq = st.pre_candidates / L
    assert abs(freq - p) <= 3 * np.sqrt(p * (1 - p) / L) + 1e-9


def test_lsh_recall_target():
    """With L = repetitions_for_recall(lambda, k, phi) the measured recall on
    planted data is >= phi - 0.05."""
    from oracle import oracle as O
    from paper_1707_06814_b200.lsh import MinHashJoinParams, minhash_join_arrays
    ds = _planted(21, n_bg=1500, n_pl=300)
    emb, _, _ = _embed(ds)
    res = minhash_join_arrays(emb, MinHashJoinParams(lambda_=0.5, phi=0.9, k=3, seed=3))
    truth, _ = O.exact_join(ds.tokens, ds.offsets, ds.d, 0.5)
    got = (res.a.astype(np.uint64) << np.uint64(32)) | res.b.astype(np.uint64)
    assert np.isin(got, truth).all()
    assert np.isin(truth, got).mean() >= 0.85
