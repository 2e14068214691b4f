"""Host/device timing breakdown of one cpsjoin_self call (diagnostics)."""
import cProfile
import os
import pstats
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1707_06814_b200 import CPSJoinParams, EmbeddingParams, cpsjoin_self_arrays  # noqa
from paper_1707_06814_b200._native import Context, load  # noqa

if os.environ.get("CPSJ_LIB"):  # A/B against another build of the library
    load(os.environ["CPSJ_LIB"])
from paper_1707_06814_b200.embed import embed_device_csr  # noqa
from paper_1707_06814_b200.workloads import CONFIGS, generate  # noqa

cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 2
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
R = int(sys.argv[3]) if len(sys.argv) > 3 else 3
cfg = CONFIGS[cfg_id]
w = generate(cfg_id, scale=scale)
dev = torch.device("cuda", 0)
d_tok = torch.from_numpy(w.tokens.view(np.int32)).to(dev)
d_off = torch.from_numpy(w.offsets).to(dev)
emb = embed_device_csr(EmbeddingParams(128, cfg.emb_seed), d_tok, d_off, w.d)
emb.sketches_device(cfg.ell, cfg.join_seed)
jp = CPSJoinParams(lambda_=cfg.lambdas[0], ell=cfg.ell, seed=cfg.join_seed, repetitions=R)
ctx = Context.get()
for _ in range(2):
    cpsjoin_self_arrays(emb, jp)
torch.cuda.synchronize()
times = []
for _ in range(int(os.environ.get("PROBE_REPS", "5"))):
    t0 = time.perf_counter()
    res = cpsjoin_self_arrays(emb, jp)
    times.append(1e3 * (time.perf_counter() - t0))
print("join wall ms:", " ".join(f"{t:.2f}" for t in times), res.stats)
ctx.profile(True)
cpsjoin_self_arrays(emb, jp)
p = ctx.profile_read()
ctx.profile(False)
print("profile:", {k: round(v[0], 3) for k, v in p.items()})
pr = cProfile.Profile()
pr.enable()
for _ in range(3):
    cpsjoin_self_arrays(emb, jp)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(12)
