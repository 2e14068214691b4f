"""Pipelined embed time against the chunk schedule's per-chunk overhead
constant (embed._CHUNK_OVERHEAD_S) and first-chunk candidates."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1707_06814_b200.embed as E  # noqa: E402
from paper_1707_06814_b200 import Dataset, EmbeddingParams, embed_dataset  # noqa: E402
from paper_1707_06814_b200.workloads import CONFIGS, generate  # noqa: E402

cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 2
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
cfg = CONFIGS[cfg_id]
w = generate(cfg_id, scale=scale)
tok_pin = torch.from_numpy(w.tokens.view(np.int32)).pin_memory()
off_pin = torch.from_numpy(w.offsets).pin_memory()
ds = Dataset.from_csr(tok_pin.numpy().view(np.uint32), off_pin.numpy(), w.d)
ep = EmbeddingParams(128, cfg.emb_seed)
skey = (cfg.ell, cfg.join_seed)


def timed(fn, reps=7):
    out = []
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b))
    return sorted(out)[len(out) // 2]


for _ in range(10):
    embed_dataset(ep, ds, sketch=skey)
for ov in [0.03e-3, 0.06e-3, 0.1e-3, 0.15e-3, 0.25e-3, 0.4e-3]:
    E._CHUNK_OVERHEAD_S = ov
    b = E._chunk_bounds(w.n, None, len(w.tokens), 128, cfg.ell)
    ms = timed(lambda: embed_dataset(ep, ds, sketch=skey))
    print(f"overhead {ov * 1e3:.2f} ms: {len(b) - 1} chunks, first {b[1] / w.n:.4f}: pipelined embed {ms:.3f} ms", flush=True)
