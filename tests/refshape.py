"""Test helper: an object shaped like the reference's
``simjoin.embed.EmbeddedDataset`` (embed.py:51-98) -- same constructor
arguments, attribute names, dtypes and ``sketches(ell, seed)`` method --
built from a golden fixture, for running the INTEGRATION.md ctypes stub on
the GPU box, where /root/reference does not exist.  The sketches come from
the C oracle (test infrastructure).  ``tests/test_cpu_host.py`` pins every
attribute the stub reads to the real class wherever the reference is
importable."""
from __future__ import annotations

import numpy as np
from scipy.sparse import csr_matrix


class RefShapedEmbeddedDataset:
    def __init__(self, values, dense, d, t, seed, verify_csr, sizes, source_ids, side=None, origin=None):
        self.values = values
        self.dense = dense
        self.d = d
        self.t = t
        self.seed = seed
        self.verify_csr = verify_csr
        self.sizes = sizes
        self.source_ids = source_ids
        self.side = side
        self.origin = origin
        self._sketch_cache: dict = {}

    def __len__(self) -> int:
        return len(self.values)

    def sketches(self, ell: int, seed: int) -> np.ndarray:
        from oracle import oracle as O
        key = (ell, seed)
        if key not in self._sketch_cache:
            mh, bt = O.sketch_tables(ell, seed)
            self._sketch_cache[key] = O.sketch(self.verify_csr.indices.astype(np.uint32), self.verify_csr.indptr,
                                               mh, bt, 1)
        return self._sketch_cache[key]


def from_fixture(z) -> RefShapedEmbeddedDataset:
    """The reference's embed_dataset(EmbeddingParams(t, emb_seed), ds) of a
    golden fixture's CSR (values from the C oracle; ``dense`` is not read by
    the join and is left empty)."""
    from oracle import oracle as O
    tok = z["tokens"].astype(np.uint32)
    off = z["offsets"].astype(np.int64)
    n, t, d = len(off) - 1, int(z["t"]), int(z["d"])
    values = O.minhash(tok, off, O.embedding_tables(t, int(z["emb_seed"])), 1)
    # Dataset.csr() (core.py:97-103): int32 indices, int64 indptr, int32 data
    csr = csr_matrix((np.ones(len(tok), dtype=np.int32), tok.astype(np.int32), off), shape=(n, d))
    return RefShapedEmbeddedDataset(values, np.zeros((n, t), dtype=np.uint32), 0, t, int(z["emb_seed"]), csr,
                                    z["sizes"].astype(np.int64).copy(), np.arange(n, dtype=np.int64))
