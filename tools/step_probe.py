"""Per-phase wall timing of the bench steps (diagnostics only)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1707_06814_b200 import CPSJoinParams, Dataset, EmbeddingParams, cpsjoin_self_arrays, embed_dataset  # noqa
from paper_1707_06814_b200.embed import embed_device_csr  # noqa
from paper_1707_06814_b200.workloads import CONFIGS, generate  # noqa

cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 2
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
R = int(sys.argv[3]) if len(sys.argv) > 3 else 3
cfg = CONFIGS[cfg_id]
w = generate(cfg_id, scale=scale)
dev = torch.device("cuda", 0)
tok_pin = torch.from_numpy(w.tokens.view(np.int32)).pin_memory()
off_pin = torch.from_numpy(w.offsets).pin_memory()
ds = Dataset.from_csr(tok_pin.numpy().view(np.uint32), off_pin.numpy(), w.d)
d_tok, d_off = tok_pin.to(dev), off_pin.to(dev)
ep = EmbeddingParams(128, cfg.emb_seed)
jp = CPSJoinParams(lambda_=cfg.lambdas[0], ell=cfg.ell, seed=cfg.join_seed, repetitions=R)


def sync_t():
    torch.cuda.synchronize()
    return time.perf_counter()


for mode in ["device", "e2e", "device", "e2e"]:
    for it in range(4):
        t0 = sync_t()
        if mode == "device":
            emb = embed_device_csr(ep, d_tok, d_off, w.d)
        else:
            emb = embed_dataset(ep, ds, sketch=(cfg.ell, cfg.join_seed))
        t1 = sync_t()
        emb.sketches_device(cfg.ell, cfg.join_seed)
        t2 = sync_t()
        res = cpsjoin_self_arrays(emb, jp)
        t3 = sync_t()
        del emb
        t4 = sync_t()
        print(f"{mode:6s} it{it}: embed {1e3*(t1-t0):7.2f}  sketch {1e3*(t2-t1):7.2f}  join {1e3*(t3-t2):7.2f}"
              f"  free {1e3*(t4-t3):6.2f}  levels {res.stats['n_levels']} launches {res.stats['gpu_launches']}",
              flush=True)
