import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_1707_06814_b200 import CPSJoinParams, Dataset, EmbeddingParams, cpsjoin_self_arrays, embed_dataset
rng = np.random.default_rng(4)
base = [rng.choice(3000, size=int(rng.integers(10, 40)), replace=False).tolist() for _ in range(1500)]
lists = base + [b[:-2] + [5000 + i, 6000 + i] for i, b in enumerate(base[:300])]
want = Dataset.from_token_lists(lists)
p = CPSJoinParams(lambda_=0.6, seed=2, repetitions=3)
for env in ["0", "1"]:
    os.environ["CPSJ_NO_SMALL_LEAF"] = env
    os.environ["CPSJ_JOIN_TRACE"] = "1"
    r = cpsjoin_self_arrays(embed_dataset(EmbeddingParams(seed=1), want), p)
    print(env, len(r.a), r.counters, flush=True)
