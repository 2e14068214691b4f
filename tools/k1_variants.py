"""A/B the K1 kernel variants on a BASELINE workload: time each and check the
outputs are identical to the full-warp 16-bit kernel's (diagnostics only).

    python tools/k1_variants.py CFG SCALE
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
efam = EmbeddingParams(128, cfg.emb_seed).device(ctx)
sfam = sketch_family(cfg.ell, cfg.join_seed).device(ctx)
st = torch.cuda.current_stream().cuda_stream
maxtok = int(w.tokens.max()) if len(w.tokens) else 0
nnz = len(w.tokens)
print(f"workload c{cfg_id} x{scale}: n={n} nnz={nnz} max_token={maxtok}", flush=True)


def run(fam, vals, sk):
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    ctx.check(ctx.lib.cpsj_minhash_sketch(ctx.handle, fam.handle, d_tok.data_ptr(), d_off.data_ptr(), n, maxtok,
                                          vals.data_ptr() if vals is not None else None,
                                          sk.data_ptr() if sk is not None else None, st))
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b)


VARIANTS = {
    "k16+s16": {"CPSJ_K1_NO_H8": "1"},
    "h8+s16": {},
}
ref_v = ref_s = None
for name, env in VARIANTS.items():
    for k in ("CPSJ_K1_NO_H8", "CPSJ_K1_NO_ORDER", "CPSJ_K1_NO_S16"):
        os.environ.pop(k, None)
    os.environ.update(env)
    vals = torch.zeros((n, 128), dtype=torch.int32, device=dev)
    sk = torch.zeros((n, cfg.ell), dtype=torch.int64, device=dev)
    tv, ts = [], []
    for i in range(6):
        tv.append(run(efam, vals, None))
        ts.append(run(sfam, None, sk))
    tv, ts = sorted(tv[1:])[2], sorted(ts[1:])[2]
    if ref_v is None:
        ref_v, ref_s = vals.clone(), sk.clone()
        same = "ref"
    else:
        same = "same" if torch.equal(vals, ref_v) and torch.equal(sk, ref_s) else "DIFFERENT"
    ev = nnz * (128 + 64 * cfg.ell) / (tv + ts) * 1e3
    print(f"{name:16s} values {tv:7.3f} ms  sketch {ts:7.3f} ms  total {tv + ts:7.3f}  {ev:.3e} evals/s  {same}",
          flush=True)
