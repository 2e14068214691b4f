"""Timeline of the pipelined embed on a BASELINE workload (diagnostics):
H2D alone, K1 alone, and the pipelined embed_dataset, with CUDA events.

    python tools/embed_probe.py CFG SCALE
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1707_06814_b200 import Dataset, EmbeddingParams, embed_dataset  # noqa: E402
from paper_1707_06814_b200.embed import embed_device_csr  # noqa: E402
from paper_1707_06814_b200.workloads import CONFIGS, generate  # noqa: E402

cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 2
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
cfg = CONFIGS[cfg_id]
w = generate(cfg_id, scale=scale)
dev = torch.device("cuda", 0)
tok_pin = torch.from_numpy(w.tokens.view(np.int32)).pin_memory()
off_pin = torch.from_numpy(w.offsets).pin_memory()
ds = Dataset.from_csr(tok_pin.numpy().view(np.uint32), off_pin.numpy(), w.d)
ep = EmbeddingParams(128, cfg.emb_seed)
skey = (cfg.ell, cfg.join_seed)


def timed(fn, reps=5):
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


d_tok = torch.empty(len(w.tokens), dtype=torch.int32, device=dev)
d_off = torch.empty(len(w.offsets), dtype=torch.int64, device=dev)


def h2d():
    d_tok.copy_(tok_pin, non_blocking=True)
    d_off.copy_(off_pin, non_blocking=True)


def k1():
    emb = embed_device_csr(ep, d_tok, d_off, w.d)
    emb.sketches_device(*skey)


def pipe():
    embed_dataset(ep, ds, sketch=skey)


h2d()
import time
t_end = time.time() + 4.0
while time.time() < t_end:  # clocks up
    k1()
torch.cuda.synchronize()
print(f"H2D {tok_pin.numel() * 4 / 1e6:.0f} MB: {timed(h2d):.2f} ms")
print(f"K1 values+sketch (resident): {timed(k1):.2f} ms")
for ch in [None, 5, 3]:
    def p(ch=ch):
        embed_dataset(ep, ds, sketch=skey, chunks=ch)
    print(f"pipelined embed chunks={ch}: {timed(p):.2f} ms")

# timeline of one pipelined call: K1 launches as seen by events on the compute stream
print(f"K1 resident again: {timed(k1):.2f} ms; pipelined None again: {timed(pipe):.2f} ms")

from paper_1707_06814_b200.embed import _chunk_bounds
from paper_1707_06814_b200._native import Context
from paper_1707_06814_b200.hashing import sketch_family
ctx = Context.get()
efam = ep.device(ctx)
sfam = sketch_family(*skey).device(ctx)
d_vals = torch.empty((w.n, 128), dtype=torch.int32, device=dev)
d_sk = torch.empty((w.n, cfg.ell), dtype=torch.int64, device=dev)
h2d()
torch.cuda.synchronize()
for ch in [None, 5, 1]:
    b = _chunk_bounds(w.n, ch) if ch != 1 else np.array([0, w.n])
    def kc(b=b, which="both"):
        h = torch.cuda.current_stream().cuda_stream
        for c in range(len(b) - 1):
            s0, s1 = int(b[c]), int(b[c + 1])
            offp = d_off.data_ptr() + 8 * s0
            if which in ("both", "values"):
                ctx.check(ctx.lib.cpsj_minhash_sketch(ctx.handle, efam.handle, d_tok.data_ptr(), offp, s1 - s0,
                                                      w.d - 1, d_vals.data_ptr() + 4 * 128 * s0, None, h))
            if which in ("both", "sketch"):
                ctx.check(ctx.lib.cpsj_minhash_sketch(ctx.handle, sfam.handle, d_tok.data_ptr(), offp, s1 - s0,
                                                      w.d - 1, None, d_sk.data_ptr() + 8 * cfg.ell * s0, h))
    print(f"chunked K1 resident chunks={ch} ({len(b) - 1}): both {timed(kc):.2f} ms, values "
          f"{timed(lambda: kc(which='values')):.2f}, sketch {timed(lambda: kc(which='sketch')):.2f}")

side = torch.cuda.Stream()
big_src = torch.empty(100_000_000, dtype=torch.int32).pin_memory()
big_dst = torch.empty(100_000_000, dtype=torch.int32, device=dev)
def k1_with_copy():
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        big_dst.copy_(big_src, non_blocking=True)
    kc(b=np.array([0, w.n]))
    torch.cuda.current_stream().wait_stream(side)
print(f"K1 (1 chunk) with a concurrent 400 MB H2D on a side stream: {timed(k1_with_copy):.2f} ms")
b10 = _chunk_bounds(w.n, None)
def h2d_chunks():
    for c in range(len(b10) - 1):
        t0, t1 = int(w.offsets[b10[c]]), int(w.offsets[b10[c + 1]])
        d_tok[t0:t1].copy_(tok_pin[t0:t1], non_blocking=True)
print(f"H2D in {len(b10) - 1} chunks: {timed(h2d_chunks):.2f} ms")

import cProfile, pstats
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    pipe()
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"host time per pipelined embed call: {(t1 - t0) / 5 * 1e3:.2f} ms")
pr = cProfile.Profile()
pr.enable()
for _ in range(3):
    pipe()
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)

import paper_1707_06814_b200.embed as E
E._PIPE_TRACE = []
torch.cuda.synchronize()
st = torch.cuda.Event(enable_timing=True); en = torch.cuda.Event(enable_timing=True)
st.record()
pipe()
en.record()
torch.cuda.synchronize()
cop = dict(E._PIPE_TRACE)["copies"]; kst = dict(E._PIPE_TRACE)["k1"]
print("chunk  copy_done_ms  k1_start_ms  k1_end_ms")
for c in range(len(cop)):
    print(c, f"{st.elapsed_time(cop[c]):8.3f}", f"{st.elapsed_time(kst[2 * c]):8.3f}",
          f"{st.elapsed_time(kst[2 * c + 1]):8.3f}")
print("end", f"{st.elapsed_time(en):.3f}")
E._PIPE_TRACE = None

E._PIPE_SERIAL = True
print(f"pipelined embed, K1 after the whole copy: {timed(pipe):.2f} ms")
E._PIPE_TRACE = []
torch.cuda.synchronize()
st.record()
pipe()
en.record()
torch.cuda.synchronize()
cop = dict(E._PIPE_TRACE)["copies"]; kst = dict(E._PIPE_TRACE)["k1"]
for c in range(len(cop)):
    print("serial", c, f"{st.elapsed_time(cop[c]):8.3f}", f"{st.elapsed_time(kst[2 * c]):8.3f}")
print("serial end", f"{st.elapsed_time(en):.3f}")
E._PIPE_TRACE = None
E._PIPE_SERIAL = False

cs = torch.cuda.Stream()
def pipe_cs():
    with torch.cuda.stream(cs):
        embed_dataset(ep, ds, sketch=skey)
    torch.cuda.current_stream().wait_stream(cs)
print(f"pipelined embed on a non-default compute stream: {timed(pipe_cs):.2f} ms")
print("copier stream", E._copy_stream(dev), "default", torch.cuda.current_stream(), torch.cuda.default_stream())
