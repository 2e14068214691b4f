"""One embed + CPSJoin call(s) on a BASELINE workload (for ncu launch lists).

    python tools/join_once.py CFG SCALE R [CALLS]  (CPSJ_JOIN_TRACE=1 traces the last call)
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
calls = int(sys.argv[4]) if len(sys.argv) > 4 else 1
trace = os.environ.pop("CPSJ_JOIN_TRACE", None)
for i in range(calls):
    if i == calls - 1 and trace is not None:
        os.environ["CPSJ_JOIN_TRACE"] = trace  # trace only the last (warm) call
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    res = cpsjoin_self_arrays(emb, CPSJoinParams(lambda_=cfg.lambdas[0], ell=cfg.ell, seed=cfg.join_seed,
                                                 repetitions=R))
    t1.record()
    torch.cuda.synchronize()
    print(f"call {i}: {t0.elapsed_time(t1):.3f} ms", flush=True)
print("pairs", len(res.a), res.stats)
