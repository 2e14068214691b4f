"""GPU first-seen dense remap (csrc/dense.cu, cpsj_dense_remap) against the
reference's own EmbeddedDataset.dense / .d (golden fixtures made by
oracle/gen_golden.py --dense-only) and against the numpy restatement in
oracle/oracle.py at sizes the fixtures do not reach."""
import hashlib
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("name", ["dense_small", "dense_cluster_remap", "dense_c1_sample"])
def test_dense_remap_matches_reference(name):
    from paper_1707_06814_b200 import Dataset, EmbeddingParams, embed_dataset
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    ds = Dataset.from_csr(z["tokens"], z["offsets"], int(z["d_universe"]))
    emb = embed_dataset(EmbeddingParams(t=int(z["t"]), seed=int(z["emb_seed"])), ds)
    assert sha(emb.values) == str(z["values_sha"])
    assert emb.d == int(z["d"])
    assert sha(emb.dense) == str(z["dense_sha"])
    assert emb.dense.dtype == np.uint32
    if "dense" in z.files:
        assert np.array_equal(emb.dense, z["dense"])


def test_dense_remap_reference_properties():
    """tests/test_embed.py:112-124 of the reference, through the drop-in."""
    from paper_1707_06814_b200 import Dataset, EmbeddingParams, embed_dataset
    rng = np.random.default_rng(3)
    lists = [rng.choice(200, size=rng.integers(2, 25), replace=False) for _ in range(10)]
    emb = embed_dataset(EmbeddingParams(t=8, seed=4), Dataset.from_token_lists(lists))
    assert emb.dense[0].tolist() == list(range(8))
    seen = {}
    for row in range(len(emb)):
        for pos in range(8):
            key = (pos, emb.values[row, pos])
            assert seen.setdefault(key, emb.dense[row, pos]) == emb.dense[row, pos]
    assert emb.d == len(seen)
    for i in range(len(emb)):
        assert np.array_equal(emb.embedded_record(i), np.sort(emb.dense[i]))


@pytest.mark.parametrize("cfg,scale,t", [(2, 0.05, 128), (3, 0.02, 64), (1, 0.2, 1)])
def test_dense_remap_matches_restatement_at_scale(cfg, scale, t):
    import torch

    from oracle import oracle as O
    from paper_1707_06814_b200 import EmbeddingParams
    from paper_1707_06814_b200.embed import dense_remap_device, embed_device_csr
    from paper_1707_06814_b200.workloads import generate
    w = generate(cfg, scale=scale)
    dev = torch.device("cuda", 0)
    d_tok = torch.from_numpy(w.tokens.view(np.int32)).to(dev)
    d_off = torch.from_numpy(w.offsets).to(dev)
    emb = embed_device_csr(EmbeddingParams(t, 7), d_tok, d_off, w.d)
    dense, d = dense_remap_device(emb._dev["values"], t)
    ref, rd = O.first_seen_dense(emb.values)
    assert d == rd
    assert np.array_equal(dense.cpu().numpy().view(np.uint32), ref)


def test_dense_remap_empty():
    import torch

    from paper_1707_06814_b200.embed import dense_remap_device
    out, d = dense_remap_device(torch.zeros((0, 16), dtype=torch.int32, device="cuda"), 16)
    assert d == 0 and out.shape == (0, 16)
