"""Time the GPU exact join (AllPairs) on BASELINE workloads and optionally
write the exact-join truth file the bench uses for recall.

    python tools/exact_probe.py CFG[:SCALE[:LAMBDA]] ... [--write] [--naive]

--write stores $TRUTH_DIR (default tests/golden)/truth_c{CFG}_s{SCALE}_l{LAMBDA}.npz (same format
as oracle/make_truth.py, provenance "gpu_allpairs"); the GPU AllPairs is
checked bit-exact against the oracle's truth files for c1-c3 in
tests/test_gpu_exact.py.
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def csr_sha(tokens, offsets) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(offsets, dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(tokens, dtype=np.uint32).tobytes())
    return h.hexdigest()


def main():
    import torch

    from paper_1707_06814_b200 import _native
    from paper_1707_06814_b200.allpairs import exact_join_device
    from paper_1707_06814_b200.workloads import CONFIGS, generate
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    write = "--write" in sys.argv
    naive = "--naive" in sys.argv
    ctx = _native.Context.get()
    for spec in args:
        parts = spec.split(":")
        cfg = int(parts[0])
        scale = float(parts[1]) if len(parts) > 1 else 1.0
        lam = float(parts[2]) if len(parts) > 2 else CONFIGS[cfg].lambdas[0]
        t0 = time.time()
        w = generate(cfg, scale=scale)
        t1 = time.time()
        tok = torch.from_numpy(w.tokens.view(np.int32)).cuda()
        off = torch.from_numpy(w.offsets).cuda()
        torch.cuda.synchronize()
        exact_join_device(tok, off, w.n, w.d, lam, naive)   # warm-up (allocator, module load)
        ctx.profile(True)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        keys, sims, stats = exact_join_device(tok, off, w.n, w.d, lam, naive)
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        prof = ctx.profile_read()
        ctx.profile(False)
        rec = {"cfg": cfg, "scale": scale, "lambda": lam, "n": w.n, "nnz": int(len(w.tokens)),
               "pairs": int(len(keys)), "pre_candidates": stats["pre_candidates"],
               "candidates": stats["candidates"], "gen_s": round(t1 - t0, 1), "join_ms": round((t3 - t2) * 1e3, 2),
               "prof_ms": {k: round(v[0], 3) for k, v in prof.items() if v[1]}, "naive": naive}
        print(json.dumps(rec), flush=True)
        if write and not naive:
            out_dir = os.environ.get("TRUTH_DIR", os.path.join(ROOT, "tests", "golden"))
            os.makedirs(out_dir, exist_ok=True)
            path = os.path.join(out_dir, f"truth_c{cfg}_s{scale:g}_l{lam:g}.npz")
            np.savez_compressed(path, keys=keys, sims=sims, csr_sha=np.array(csr_sha(w.tokens, w.offsets)),
                                n=np.int64(w.n), nnz=np.int64(len(w.tokens)),
                                numpy_version=np.array(np.__version__), provenance=np.array("gpu_allpairs"))
            print("wrote", path, flush=True)
        del tok, off


if __name__ == "__main__":
    main()
