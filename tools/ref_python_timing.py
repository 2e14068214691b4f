"""Time the reference AS SHIPPED (pure-Python numpy/scipy simjoin, one core)
on the BASELINE workloads, beside the C port
(oracle/, 1 thread and all threads) on the same inputs.  Runs only where
/root/reference exists (this container; it does not travel to the GPU box),
so the host differs from the GPU box's -- stated in the output.

    python tools/ref_python_timing.py [CFG:N_SETS ...] > profiles/ref_python_r02.jsonl

Default: config 1 in full and 50,000-set samples of configs 2-5 (the
seeded generator at scale 50k / n).  Phases: embed_dataset, emb.sketches,
cpsjoin_self at R = the bench's repetition count for the config.
"""
import json
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/pkg/src"
sys.path.insert(0, ROOT)
sys.path.insert(0, REF)

# R used by the GPU bench for each config (its recall-target search on the
# full workload); the reference runs the same R
R_BENCH = {1: 3, 2: 2, 3: 2, 4: 3, 5: 3}


def main():
    from simjoin.core import Dataset
    from simjoin.cpsjoin import CPSJoinParams, cpsjoin_self
    from simjoin.embed import EmbeddingParams, embed_dataset

    from oracle import oracle as O
    from paper_1707_06814_b200.workloads import CONFIGS, generate
    specs = sys.argv[1:] or ["1:0", "2:50000", "3:50000", "4:50000", "5:50000"]
    import scipy
    host = {"cpu": platform.processor() or platform.machine(), "cpu_count": os.cpu_count(),
            "numpy": np.__version__, "scipy": scipy.__version__,
            "note": "timed in the build container (the reference cannot travel to the GPU box); 1 core"}
    for spec in specs:
        cfg_id, nsets = (int(x) for x in spec.split(":"))
        cfg = CONFIGS[cfg_id]
        n_full = cfg.n_background + cfg.n_planted
        scale = 1.0 if nsets <= 0 else min(1.0, nsets / n_full)
        w = generate(cfg_id, scale=scale)
        lam, R = cfg.lambdas[0], R_BENCH[cfg_id]
        lists = [w.tokens[w.offsets[i]:w.offsets[i + 1]].astype(np.int64) for i in range(w.n)]
        t0 = time.perf_counter()
        ds = Dataset.from_token_lists(lists, d=w.d)
        t1 = time.perf_counter()
        emb = embed_dataset(EmbeddingParams(t=128, seed=cfg.emb_seed), ds)
        t2 = time.perf_counter()
        emb.sketches(cfg.ell, cfg.join_seed)
        t3 = time.perf_counter()
        pairs, c = cpsjoin_self(emb, CPSJoinParams(lambda_=lam, ell=cfg.ell, seed=cfg.join_seed, repetitions=R))
        t4 = time.perf_counter()
        total = t4 - t1
        # the C port on the same input, 1 thread and all threads
        port = {}
        for th in (1, 0):
            s0 = time.perf_counter()
            _, _, out = O.full_pipeline(w.tokens, w.offsets, w.sizes, lam=lam, t=128, emb_seed=cfg.emb_seed,
                                        ell=cfg.ell, seed=cfg.join_seed, repetitions=R, threads=th)
            port[f"threads_{th or os.cpu_count()}_s"] = round(time.perf_counter() - s0, 3)
            same = (len(out.keys) == len(pairs) and [out.pre_candidates, out.candidates, out.results] ==
                    [c.pre_candidates, c.candidates, c.results])
        rec = {"config": cfg_id, "workload": cfg.name, "scale": scale, "n_sets": int(w.n),
               "nnz": int(len(w.tokens)), "lambda": lam, "ell": cfg.ell, "repetitions": R,
               "reference_python": {"from_token_lists_s": round(t1 - t0, 3), "embed_s": round(t2 - t1, 3),
                                    "sketches_s": round(t3 - t2, 3), "cpsjoin_self_s": round(t4 - t3, 3),
                                    "sets_per_s": w.n / total, "join_only_sets_per_s": w.n / (t4 - t3),
                                    "cores": 1},
               "pairs": len(pairs), "counters": [c.pre_candidates, c.candidates, c.results, c.max_depth,
                                                 c.peak_live_members],
               "c_port": port, "c_port_same_output": bool(same), "host": host}
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
