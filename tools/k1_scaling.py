"""K1 launch time against the number of sets (config 2 prefix): the intercept
is the fixed cost of a launch (table loads, prologue latencies, tails), which
the pipelined embed pays once per chunk."""
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
w = generate(2, scale=float(sys.argv[1]) if len(sys.argv) > 1 else 1.0)
dev = torch.device("cuda", 0)
ctx = Context.get()
d_tok = torch.from_numpy(w.tokens.view(np.int32)).to(dev)
d_off = torch.from_numpy(w.offsets).to(dev)
efam = EmbeddingParams(128, cfg.emb_seed).device(ctx)
sfam = sketch_family(cfg.ell, cfg.join_seed).device(ctx)
vals = torch.empty((w.n, 128), dtype=torch.int32, device=dev)
sk = torch.empty((w.n, cfg.ell), dtype=torch.int64, device=dev)
st = torch.cuda.current_stream().cuda_stream


def run(fam, n, v, s):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    ctx.check(ctx.lib.cpsj_minhash_sketch(ctx.handle, fam.handle, d_tok.data_ptr(), d_off.data_ptr(), n,
                                          w.d - 1, v, s, st))
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b)


for n in [1000, 5000, 10000, 25000, 50000, 100000, 200000, 400000, w.n]:
    n = min(n, w.n)
    tv = sorted(run(efam, n, vals.data_ptr(), None) for _ in range(7))[3]
    ts = sorted(run(sfam, n, None, sk.data_ptr()) for _ in range(7))[3]
    print(f"n={n:8d}: values {tv:7.3f} ms ({tv / n * 1e6:6.2f} ns/set)  sketch {ts:7.3f} ms ({ts / n * 1e6:6.2f} ns/set)",
          flush=True)
