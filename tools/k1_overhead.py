"""Fixed cost of one K1 launch (values + sketch, fused) vs set count (diagnostics)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1707_06814_b200 import EmbeddingParams  # noqa: E402
from paper_1707_06814_b200._native import Context  # noqa: E402
from paper_1707_06814_b200.hashing import sketch_family  # noqa: E402
from paper_1707_06814_b200.workloads import CONFIGS, generate  # noqa: E402

cfg = CONFIGS[2]
w = generate(2, scale=1.0)
dev = torch.device("cuda", 0)
ctx = Context.get()
d_tok = torch.from_numpy(w.tokens.view(np.int32)).to(dev)
d_off = torch.from_numpy(w.offsets).to(dev)
efam = EmbeddingParams(128, cfg.emb_seed).device(ctx)
sfam = sketch_family(cfg.ell, cfg.join_seed).device(ctx)
vals = torch.empty((w.n, 128), dtype=torch.int32, device=dev)
sk = torch.empty((w.n, cfg.ell), dtype=torch.int64, device=dev)
h = torch.cuda.current_stream().cuda_stream


def run(n, env):
    for k in ("CPSJ_K1_NO_ORDER", "CPSJ_K1_FUSE", "CPSJ_K1_NO_SPLIT"):
        os.environ.pop(k, None)
    os.environ.update(env)
    ts = []
    for _ in range(7):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        ctx.check(ctx.lib.cpsj_minhash_embed(ctx.handle, efam.handle, sfam.handle, d_tok.data_ptr(),
                                             d_off.data_ptr(), n, w.d - 1, vals.data_ptr(), sk.data_ptr(), h))
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[3]


import time
t_end = time.time() + 3
while time.time() < t_end:
    run(100000, {})
for n in [1000, 10000, 31250, 100000, 300000, 1000000]:
    print(f"n={n:8d}: default {run(n, {}):.3f} ms  no-order {run(n, {'CPSJ_K1_NO_ORDER': '1'}):.3f} ms  "
          f"fused launch {run(n, {'CPSJ_K1_FUSE': '1'}):.3f} ms  no-split {run(n, {'CPSJ_K1_NO_SPLIT': '1'}):.3f} ms "
          f"  per-set {13.1e-3 * n / 1000:.3f}")
