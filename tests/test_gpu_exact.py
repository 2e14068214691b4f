"""GPU exact joins (SPEC allpairs module, csrc/exact.cu) against the C
oracle's exact join (oracle/cpsj_oracle.c orc_exact_join, itself checked
against brute force in test_oracle_golden.py) and the committed exact-join
truth files (tests/golden/truth_*.npz).  Bit-exact: same pair keys, same
f64 similarities."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1707_06814_b200 import _native
    _native.load()


def _keys(res):
    return (res.a.astype(np.uint64) << np.uint64(32)) | res.b.astype(np.uint64)


def _random_ds(seed, n, d, lo, hi, zipf=None, dup_frac=0.0):
    from paper_1707_06814_b200 import Dataset
    rng = np.random.default_rng(seed)
    rows = []
    p = None
    if zipf is not None:
        p = 1.0 / np.arange(1, d + 1) ** zipf
        p /= p.sum()
    for _ in range(n):
        s = int(rng.integers(lo, hi + 1))
        rows.append(np.unique(rng.choice(d, size=min(s, d), replace=False, p=p)))
    # near-duplicates so that there is something to find
    for _ in range(int(dup_frac * n)):
        src = rows[int(rng.integers(0, len(rows)))]
        r = max(1, len(src) // 6)
        keep = rng.choice(len(src), size=len(src) - r, replace=False)
        extra = rng.integers(0, d, size=r)
        rows.append(np.unique(np.concatenate([src[keep], extra])))
    return Dataset.from_token_lists(rows, d=d)


def _oracle(ds, lam):
    from oracle import oracle as O
    return O.exact_join(ds.tokens, ds.offsets, ds.d, lam)


@pytest.mark.parametrize("seed,lam,zipf", [(1, 0.5, None), (2, 0.7, 1.0), (3, 0.3, 0.8), (4, 0.9, None),
                                           (5, 0.6, 1.1)])
def test_allpairs_matches_oracle(seed, lam, zipf):
    from paper_1707_06814_b200.allpairs import allpairs_join_arrays
    ds = _random_ds(seed, 1500, 400, 5, 60, zipf=zipf, dup_frac=0.3)
    res = allpairs_join_arrays(ds, lam)
    keys, sims = _oracle(ds, lam)
    assert len(keys) > 0
    assert np.array_equal(_keys(res), keys)
    assert np.array_equal(res.similarity, sims)
    c = res.counters
    assert c.pre_candidates >= c.candidates >= c.results == len(keys)


@pytest.mark.parametrize("lam", [0.5, 0.8])
def test_naive_equals_allpairs(lam):
    from paper_1707_06814_b200.allpairs import allpairs_join_arrays
    ds = _random_ds(11, 1200, 300, 2, 40, zipf=1.0, dup_frac=0.4)
    ap = allpairs_join_arrays(ds, lam)
    nv = allpairs_join_arrays(ds, lam, naive=True)
    assert np.array_equal(_keys(ap), _keys(nv))
    assert np.array_equal(ap.similarity, nv.similarity)
    n = len(ds)
    assert nv.counters.pre_candidates == n * (n - 1) // 2


def test_allpairs_edge_cases():
    from paper_1707_06814_b200 import Dataset, allpairs_join, naive_join
    # paper section 1: two 3-token sets with J = 1/2
    ds = Dataset.from_token_lists([[1, 2, 3], [2, 3, 4]], d=5)
    pairs, c = allpairs_join(ds, 0.5)
    assert [(p.a, p.b, p.similarity) for p in pairs] == [(0, 1, 0.5)]
    assert naive_join(ds, 0.5) == pairs
    # no pair above the threshold
    ds = Dataset.from_token_lists([[0, 1], [2, 3], [4, 5, 6]], d=7)
    assert allpairs_join(ds, 0.5)[0] == [] and naive_join(ds, 0.5) == []
    # n = 0 and 1
    assert allpairs_join(Dataset.from_token_lists([], d=3), 0.5)[0] == []
    assert allpairs_join(Dataset.from_token_lists([[0, 1]], d=3), 0.5)[0] == []
    assert naive_join(Dataset.from_token_lists([[0, 1]], d=3), 0.5) == []
    with pytest.raises(ValueError):
        allpairs_join(ds, 1.0)


def test_allpairs_identical_records_all_pairs():
    """All-identical records (built with from_csr; from_token_lists would drop
    the duplicates) -> C(n, 2) pairs at similarity 1.0."""
    from paper_1707_06814_b200 import Dataset, allpairs_join, naive_join
    n, row = 40, np.arange(3, 13, dtype=np.uint32)
    ds = Dataset.from_csr(np.tile(row, n), np.arange(n + 1, dtype=np.int64) * len(row), 20)
    pairs, c = allpairs_join(ds, 0.9)
    assert len(pairs) == n * (n - 1) // 2 and all(p.similarity == 1.0 for p in pairs)
    assert naive_join(ds, 0.9) == pairs
    # every pair shares the whole prefix: enumerated once per shared token,
    # verified once
    assert c.candidates == n * (n - 1) // 2 < c.pre_candidates


def test_allpairs_threshold_boundaries():
    """Pairs exactly at J = lambda are kept (f64 inter / union >= lambda),
    also for lambdas that are not dyadic."""
    from paper_1707_06814_b200 import Dataset
    from paper_1707_06814_b200.allpairs import allpairs_join_arrays
    rows = []
    base = list(range(100, 110))           # |x| = 10
    for k in range(0, 10):
        rows.append(base[:10 - k] + list(range(200 + 20 * k, 200 + 20 * k + k)))   # J = (10-k)/(10+k)
    ds = Dataset.from_token_lists(rows, d=400)
    for lam in (0.1, 0.2, 0.3, 0.6, 0.7, 0.8, 9 / 11, 0.9):
        got = allpairs_join_arrays(ds, lam)
        keys, sims = _oracle(ds, lam)
        assert np.array_equal(_keys(got), keys), lam
        assert np.array_equal(got.similarity, sims), lam


def test_frequency_order():
    from paper_1707_06814_b200 import Dataset, frequency_order
    # all frequencies equal -> identity by token id
    ds = Dataset.from_csr(np.array([0, 1, 2, 3], dtype=np.uint32), np.array([0, 2, 4]), 4)
    assert frequency_order(ds).tolist() == [0, 1, 2, 3]
    # one token in every record -> last
    ds = Dataset.from_token_lists([[0, 5], [1, 5], [2, 5], [3, 4, 5]], d=6)
    assert frequency_order(ds)[-1] == 5
    # random: agrees with a recount
    ds = _random_ds(7, 800, 500, 3, 30, zipf=1.0)
    freq = np.bincount(ds.tokens, minlength=ds.d)
    want = np.lexsort((np.arange(ds.d), freq))
    assert frequency_order(ds).tolist() == want.tolist()


def test_allpairs_prefix_completeness_randomised():
    """Many small random datasets: AllPairs == oracle exact join."""
    from paper_1707_06814_b200.allpairs import allpairs_join_arrays
    for seed in range(20):
        rng = np.random.default_rng(100 + seed)
        lam = float(rng.choice([0.3, 0.45, 0.5, 0.55, 0.65, 0.75, 0.85]))
        ds = _random_ds(200 + seed, 300, int(rng.integers(30, 200)), 2, 25, dup_frac=0.5)
        got = allpairs_join_arrays(ds, lam)
        keys, sims = _oracle(ds, lam)
        assert np.array_equal(_keys(got), keys), (seed, lam)
        assert np.array_equal(got.similarity, sims), (seed, lam)


@pytest.mark.parametrize("cfg,lam", [(1, 0.5), (2, 0.5), (3, 0.5), (3, 0.7)])
def test_allpairs_matches_committed_truth(cfg, lam):
    """Full-size BASELINE configs: GPU AllPairs reproduces the oracle's
    exact-join truth files bit for bit."""
    from paper_1707_06814_b200.allpairs import exact_join_device
    from paper_1707_06814_b200.workloads import generate
    import torch
    z = np.load(os.path.join(GOLDEN, f"truth_c{cfg}_s1_l{lam:g}.npz"))
    w = generate(cfg)
    tok = torch.from_numpy(w.tokens.view(np.int32)).cuda()
    off = torch.from_numpy(w.offsets).cuda()
    keys, sims, stats = exact_join_device(tok, off, w.n, w.d, lam)
    assert np.array_equal(keys, z["keys"])
    assert np.array_equal(sims, z["sims"])
