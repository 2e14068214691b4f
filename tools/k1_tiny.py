"""One fused K1 launch on the first N sets of config 2 (ncu target)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1707_06814_b200 import EmbeddingParams  # noqa: E402
from paper_1707_06814_b200._native import Context  # noqa: E402
from paper_1707_06814_b200.hashing import sketch_family  # noqa: E402
from paper_1707_06814_b200.workloads import CONFIGS, generate  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
cfg = CONFIGS[2]
w = generate(2, scale=0.05)
dev = torch.device("cuda", 0)
ctx = Context.get()
d_tok = torch.from_numpy(w.tokens.view(np.int32)).to(dev)
d_off = torch.from_numpy(w.offsets).to(dev)
efam = EmbeddingParams(128, cfg.emb_seed).device(ctx)
sfam = sketch_family(cfg.ell, cfg.join_seed).device(ctx)
vals = torch.empty((w.n, 128), dtype=torch.int32, device=dev)
sk = torch.empty((w.n, cfg.ell), dtype=torch.int64, device=dev)
for _ in range(3):
    ctx.check(ctx.lib.cpsj_minhash_embed(ctx.handle, efam.handle, sfam.handle, d_tok.data_ptr(), d_off.data_ptr(),
                                         n, 999999, vals.data_ptr(), sk.data_ptr(),
                                         torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()
print("ok")
