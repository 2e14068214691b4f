"""One K1 sketch launch (+ one values launch) on a BASELINE workload, for ncu.

    CPSJ_K1_K16=1 python tools/k1_once.py CFG SCALE
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1707_06814_b200 import EmbeddingParams  # noqa: E402
from paper_1707_06814_b200._native import Context  # noqa: E402
from paper_1707_06814_b200.hashing import sketch_family  # noqa: E402
from paper_1707_06814_b200.workloads import CONFIGS, generate  # noqa: E402

cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 2
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
cfg = CONFIGS[cfg_id]
w = generate(cfg_id, scale=scale)
dev = torch.device("cuda", 0)
ctx = Context.get()
d_tok = torch.from_numpy(w.tokens.view(np.int32)).to(dev)
d_off = torch.from_numpy(w.offsets).to(dev)
n = w.n
vals = torch.empty((n, 128), dtype=torch.int32, device=dev)
sk = torch.empty((n, cfg.ell), dtype=torch.int64, device=dev)
efam = EmbeddingParams(128, cfg.emb_seed).device(ctx)
sfam = sketch_family(cfg.ell, cfg.join_seed).device(ctx)
st = torch.cuda.current_stream().cuda_stream
maxtok = int(w.tokens.max())
for fam, v, s in ((efam, vals, None), (sfam, None, sk)):
    ctx.check(ctx.lib.cpsj_minhash_sketch(ctx.handle, fam.handle, d_tok.data_ptr(), d_off.data_ptr(), n, maxtok,
                                          v.data_ptr() if v is not None else None,
                                          s.data_ptr() if s is not None else None, st))
torch.cuda.synchronize()
print("ok")
