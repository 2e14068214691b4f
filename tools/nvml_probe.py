"""Which NVML query perturbs a busy B200?  A steady stream of identical
kernels (the K1 sketch launch on a c2-sized CSR) is timed per launch with
CUDA events while the host issues one kind of NVML query at a fixed point;
the launch times around the query show the stall (diagnostic, not product).

    python tools/nvml_probe.py
"""
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import pynvml

    from paper_1707_06814_b200.embed import embed_device_csr
    from paper_1707_06814_b200.workloads import generate
    from paper_1707_06814_b200 import EmbeddingParams
    torch.cuda.set_device(0)
    w = generate(2, scale=0.2)
    dev = torch.device("cuda", 0)
    d_tok = torch.from_numpy(w.tokens.view(np.int32)).to(dev)
    d_off = torch.from_numpy(w.offsets).to(dev)
    ep = EmbeddingParams(t=128, seed=7)

    def step():
        emb = embed_device_csr(ep, d_tok, d_off, w.d)
        emb.sketches_device(8, 7)

    for _ in range(5):
        step()
    torch.cuda.synchronize()
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    queries = {
        "none": lambda: None,
        "clock_sm": lambda: pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
        "reasons": lambda: pynvml.nvmlDeviceGetCurrentClocksEventReasons(h),
        "power": lambda: pynvml.nvmlDeviceGetPowerUsage(h),
        "temp": lambda: pynvml.nvmlDeviceGetTemperature(h, pynvml.NVML_TEMPERATURE_GPU),
        "util": lambda: pynvml.nvmlDeviceGetUtilizationRates(h),
    }
    for name, q in list(queries.items()) * 2:
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(41)]
        evs[0].record()
        qt = None
        for i in range(40):
            step()
            evs[i + 1].record()
            if i == 20:
                torch.cuda.synchronize() if name == "sync_first" else None
                t0 = time.perf_counter()
                q()
                qt = (time.perf_counter() - t0) * 1e3
        torch.cuda.synchronize()
        per = [a.elapsed_time(b) for a, b in zip(evs[:-1], evs[1:])]
        base = statistics.median(per)
        print(f"{name:10s} host {qt:7.3f} ms | median {base:.3f} ms, max {max(per):.3f} ms at step "
              f"{per.index(max(per))}, excess {sum(per) - base * len(per):.2f} ms", flush=True)
        time.sleep(1.0)


if __name__ == "__main__":
    main()
