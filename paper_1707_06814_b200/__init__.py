"""B200-native CPSJoin (Chosen Path Similarity Join, arXiv 1707.06814).

Drop-in for the reference package's self-join path:

    from paper_1707_06814_b200 import (Dataset, EmbeddingParams, embed_dataset,
                                       CPSJoinParams, cpsjoin_self)

Host code mirrors simjoin's API; the hot path runs in hand-written sm_100a
kernels behind a C ABI (include/cpsjoin_b200.h).  There is no CPU
fallback: without the built library and a CUDA device the entry points
raise.
"""
from .allpairs import allpairs_join, frequency_order, naive_join, prefix_length  # noqa: F401
from .core import Counters, Dataset, Record, ResultPair, check_threshold, jaccard  # noqa: F401
from .cpsjoin import CPSJoinParams, cpsjoin_self, cpsjoin_self_arrays, join_rs, join_rs_arrays  # noqa: F401
from .embed import EmbeddedDataset, EmbeddingParams, embed_dataset, union_embedded  # noqa: F401
from .hashing import SketchFamily, match_threshold  # noqa: F401
from .lsh import MinHashJoinParams, choose_k, minhash_join, repetitions_for_recall  # noqa: F401

__version__ = "0.1.0"
