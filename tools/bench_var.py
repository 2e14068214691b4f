"""Diagnose per-step timing variance of the bench's device step."""
import os
import subprocess
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1707_06814_b200 import CPSJoinParams, Dataset, EmbeddingParams, cpsjoin_self_arrays, embed_dataset  # noqa
from paper_1707_06814_b200.embed import embed_device_csr  # noqa
from paper_1707_06814_b200.workloads import CONFIGS, generate  # noqa

cfg = CONFIGS[2]
w = generate(2)
dev = torch.device("cuda", 0)
tok_pin = torch.from_numpy(w.tokens.view(np.int32)).pin_memory()
off_pin = torch.from_numpy(w.offsets).pin_memory()
ds = Dataset.from_csr(tok_pin.numpy().view(np.uint32), off_pin.numpy(), w.d)
d_tok, d_off = tok_pin.to(dev), off_pin.to(dev)
ep = EmbeddingParams(128, cfg.emb_seed)
jp = CPSJoinParams(lambda_=0.5, ell=8, seed=7, repetitions=2)
st = torch.cuda.current_stream()


def dev_step(events):
    if events:
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record(st)
    emb = embed_device_csr(ep, d_tok, d_off, w.d)
    if events:
        ev[1].record(st)
    emb.sketches_device(8, 7)
    if events:
        ev[2].record(st)
    return cpsjoin_self_arrays(emb, jp)


def e2e_step():
    emb = embed_dataset(ep, ds, sketch=(8, 7))
    return cpsjoin_self_arrays(emb, jp)


def run(name, fn, k=8):
    ts = []
    for _ in range(k):
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print(f"{name:28s} " + " ".join(f"{t:6.1f}" for t in ts), flush=True)


for _ in range(3):
    dev_step(False)
    e2e_step()
run("device (no events)", lambda: dev_step(False))
run("device (events)", lambda: dev_step(True))
run("e2e", e2e_step)
p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,clocks_event_reasons.active", "--format=csv,noheader",
                      "-lms", "500"], stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
time.sleep(1.0)
run("device + smi500", lambda: dev_step(True))
run("e2e + smi500", e2e_step)
p.terminate()
p.wait()
run("device after smi", lambda: dev_step(True))
