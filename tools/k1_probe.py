"""Time K1 (values, t=128; sketch, 64*ell) alone on a BASELINE workload."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1707_06814_b200 import EmbeddingParams  # noqa: E402
from paper_1707_06814_b200._native import Context  # noqa: E402
from paper_1707_06814_b200.hashing import sketch_family  # noqa: E402
from paper_1707_06814_b200.workloads import CONFIGS, generate  # noqa: E402

cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 2
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
cfg = CONFIGS[cfg_id]
t0 = time.time()
w = generate(cfg_id, scale=scale)
print(f"workload n={w.n} nnz={len(w.tokens)} gen {time.time() - t0:.1f}s", flush=True)
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
maxtok = w.d - 1


def run(fam, vptr, sptr):
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    ctx.check(ctx.lib.cpsj_minhash_sketch(ctx.handle, fam.handle, d_tok.data_ptr(), d_off.data_ptr(), n, maxtok,
                                          vptr, sptr, st))
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b)


for i in range(reps):
    tv = run(efam, vals.data_ptr(), None)
    ts = run(sfam, None, sk.data_ptr())
    print(f"iter {i}: values {tv:.3f} ms  sketch {ts:.3f} ms", flush=True)
import hashlib  # noqa: E402
print("sha values", hashlib.sha256(vals.cpu().numpy().tobytes()).hexdigest()[:16],
      "sketch", hashlib.sha256(sk.cpu().numpy().tobytes()).hexdigest()[:16])
evals_v = len(w.tokens) * 128
evals_s = len(w.tokens) * 64 * cfg.ell
print(f"evals/s values {evals_v / tv * 1e3:.3e} sketch {evals_s / ts * 1e3:.3e}")
