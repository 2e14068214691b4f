"""One embed + one CPSJoin call on a BASELINE workload (for ncu launch lists).

    python tools/join_once.py CFG SCALE R
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1707_06814_b200 import CPSJoinParams, EmbeddingParams, cpsjoin_self_arrays  # noqa: E402
from paper_1707_06814_b200.embed import embed_device_csr  # noqa: E402
from paper_1707_06814_b200.workloads import CONFIGS, generate  # noqa: E402

cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 2
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
R = int(sys.argv[3]) if len(sys.argv) > 3 else 2
cfg = CONFIGS[cfg_id]
w = generate(cfg_id, scale=scale)
dev = torch.device("cuda", 0)
d_tok = torch.from_numpy(w.tokens.view(np.int32)).to(dev)
d_off = torch.from_numpy(w.offsets).to(dev)
emb = embed_device_csr(EmbeddingParams(128, cfg.emb_seed), d_tok, d_off, w.d)
emb.sketches_device(cfg.ell, cfg.join_seed)
res = cpsjoin_self_arrays(emb, CPSJoinParams(lambda_=cfg.lambdas[0], ell=cfg.ell, seed=cfg.join_seed, repetitions=R))
torch.cuda.synchronize()
print("pairs", len(res.a), res.stats)
