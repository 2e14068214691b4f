"""GPU ingestion (csrc/ingest.cu, ingest.py) against golden fixtures made by
the reference's own Dataset.from_token_lists (oracle/gen_golden.py
--ingest-only) and against the host restatement (core.Dataset)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
CASES = ["ingest_dense_remap", "ingest_given_d", "ingest_negative", "ingest_big_values", "ingest_all_short"]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1707_06814_b200 import _native
    _native.load()


def _check(ds, z, source_offset=0):
    assert np.array_equal(ds.tokens, z["out_tokens"])
    assert np.array_equal(ds.offsets, z["out_offsets"])
    assert ds.d == int(z["out_d"])
    assert np.array_equal(np.asarray(ds.source_lines, dtype=np.int64), z["out_source"] + source_offset)


@pytest.mark.parametrize("name", CASES)
def test_from_flat_matches_reference(name):
    from paper_1707_06814_b200.ingest import from_flat
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    d = int(z["in_d"])
    n = len(z["in_offsets"]) - 1
    ds = from_flat(z["in_values"], z["in_offsets"], None if d < 0 else d, source_lines=list(range(n)))
    _check(ds, z)


@pytest.mark.parametrize("name", CASES)
def test_load_dataset_matches_reference(name, tmp_path):
    from paper_1707_06814_b200.ingest import load_dataset
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    if len(z["text"]) == 0:
        pytest.skip("negative tokens have no text form")
    p = tmp_path / "data.txt"
    p.write_bytes(z["text"].tobytes())
    d = int(z["in_d"])
    ds = load_dataset(str(p), None if d < 0 else d)
    _check(ds, z, source_offset=1)     # 1-based line numbers


def test_from_token_lists_matches_host_restatement():
    from paper_1707_06814_b200 import Dataset
    from paper_1707_06814_b200.ingest import from_token_lists
    rng = np.random.default_rng(9)
    lists = []
    for i in range(20000):
        if i % 17 == 0 and lists:
            lists.append(list(lists[int(rng.integers(0, len(lists)))]))
        else:
            lists.append(rng.integers(0, 50000, size=int(rng.integers(0, 60))).tolist())
    for d in (None, 50000):
        want = Dataset.from_token_lists(lists, d=d, source_lines=list(range(len(lists))))
        got = from_token_lists(lists, d=d, source_lines=list(range(len(lists))))
        assert np.array_equal(got.tokens, want.tokens) and np.array_equal(got.offsets, want.offsets)
        assert got.d == want.d and got.source_lines == want.source_lines


def test_ingest_errors_and_text_edges(tmp_path):
    from paper_1707_06814_b200.ingest import from_token_lists, load_dataset
    with pytest.raises(ValueError, match="column index exceeds matrix dimensions"):
        from_token_lists([[1, 2], [3, 9]], d=5)
    with pytest.raises(ValueError, match="column index exceeds matrix dimensions"):
        from_token_lists([[1, 2], [-1, 3]], d=5)
    p = tmp_path / "bad.txt"
    p.write_bytes(b"1 2 3\n4 5\n6 x 7\n")
    with pytest.raises(ValueError, match="line 3"):
        load_dataset(str(p))
    p.write_bytes(b"1 2\n3 -4\n")
    with pytest.raises(ValueError, match="line 2"):
        load_dataset(str(p))
    p.write_bytes(b"1 99999999999999999999\n")
    with pytest.raises(ValueError, match="line 1"):
        load_dataset(str(p))
    # empty file -> empty dataset
    p.write_bytes(b"")
    ds = load_dataset(str(p))
    assert len(ds) == 0 and ds.source_lines == []
    # SPEC examples: "3 1 2 2" -> {1, 2, 3}; "7" dropped; duplicate lines
    # -> one record; CRLF endings; no final newline; blank lines
    p.write_bytes(b"3 1 2 2\r\n7\r\n\r\n1 2 3\n  10\t20  \n3 2 1")
    ds = load_dataset(str(p))
    assert [r.tokens.tolist() for r in ds.records] == [[0, 1, 2], [3, 4]]
    assert ds.d == 5 and ds.source_lines == [1, 5]


def test_ingested_dataset_joins_like_host_built():
    """The GPU-ingested Dataset drives the CPSJoin path to the same result
    as the host-built one."""
    from paper_1707_06814_b200 import CPSJoinParams, Dataset, EmbeddingParams, cpsjoin_self_arrays, embed_dataset
    from paper_1707_06814_b200.ingest import from_token_lists
    rng = np.random.default_rng(4)
    base = [rng.choice(3000, size=int(rng.integers(10, 40)), replace=False).tolist() for _ in range(1500)]
    lists = base + [b[:-2] + [5000 + i, 6000 + i] for i, b in enumerate(base[:300])]
    got = from_token_lists(lists)
    want = Dataset.from_token_lists(lists)
    p = CPSJoinParams(lambda_=0.6, seed=2, repetitions=3)
    ra = cpsjoin_self_arrays(embed_dataset(EmbeddingParams(seed=1), got), p)
    rb = cpsjoin_self_arrays(embed_dataset(EmbeddingParams(seed=1), want), p)
    assert np.array_equal(ra.a, rb.a) and np.array_equal(ra.b, rb.b) and len(ra.a) > 100
