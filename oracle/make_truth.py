"""Exact-join ground truth for a BASELINE workload (recall denominators).

    python oracle/make_truth.py CFG [SCALE] [LAMBDA]

Runs the oracle's exact prefix-filter join (cpsj_oracle.c orc_exact_join,
validated against brute force in tests/test_oracle_golden.py) on the seeded
workload and writes tests/golden/truth_c{CFG}_s{SCALE}_l{LAMBDA}.npz with the
sorted pair keys ((a << 32) | b), similarities and a sha256 of the CSR so
bench.py can check it is looking at the same data.  Test/bench
infrastructure only.
"""
import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_1707_06814_b200.workloads import CONFIGS, generate  # noqa: E402


def truth_path(cfg: int, scale: float, lam: float) -> str:
    return os.path.join(ROOT, "tests", "golden", f"truth_c{cfg}_s{scale:g}_l{lam:g}.npz")


def csr_sha(tokens, offsets) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(offsets, dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(tokens, dtype=np.uint32).tobytes())
    return h.hexdigest()


def main():
    cfg = int(sys.argv[1])
    scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
    lam = float(sys.argv[3]) if len(sys.argv) > 3 else CONFIGS[cfg].lambdas[0]
    t0 = time.time()
    w = generate(cfg, scale=scale)
    t1 = time.time()
    keys, sims = O.exact_join(w.tokens, w.offsets, w.d, lam)
    t2 = time.time()
    path = truth_path(cfg, scale, lam)
    np.savez_compressed(path, keys=keys, sims=sims, csr_sha=np.array(csr_sha(w.tokens, w.offsets)),
                        n=np.int64(w.n), nnz=np.int64(len(w.tokens)), numpy_version=np.array(np.__version__))
    print(f"{path}: n={w.n} truth={len(keys)} gen={t1 - t0:.1f}s exact={t2 - t1:.1f}s")


if __name__ == "__main__":
    main()
