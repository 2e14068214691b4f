"""Markdown table of the bench sweep rows (profiles/sweep_rNN_c*_l*.json).

    python tools/sweep_table.py [r02]
"""
import glob
import json
import os
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
root = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles")
print("| Config | λ | n | Σ\\|x\\| | ℓ | R | recall (exact truth) | ms/step | value sets/s | e2e ms | e2e sets/s | K1 ms | K4 INT frac | "
      "bit-exact vs oracle | CPU port sets/s |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|")
for f in sorted(glob.glob(os.path.join(root, f"sweep_{tag}_c*_l*.json"))):
    d = json.load(open(f))
    c, k, p = d["config"], d["kernels_ms_per_step"], d["parity"]
    vs = "full workload" if "device_vs_oracle" in p else "device = e2e (oracle on a sample)"
    cpu = d.get("cpu_baseline") or {}
    print(f"| {c['workload'].split(' ')[0]} | {c['lambda']} | {c['n_sets']:,} | {c['nnz_tokens']:,} | {c['ell']} | "
          f"{c['repetitions']} | {c['recall']:.3f} | {d['ms_per_step']:.2f} | {d['value'] / 1e6:.1f} M | "
          f"{d['e2e']['ms_per_step']:.2f} | {d['e2e']['value'] / 1e6:.1f} M | {k['k1_minhash']:.2f} | "
          f"{d['roofline_int']['frac']:.2f} | {p['bit_exact']} ({vs}) | {cpu.get('value', 0) / 1e3:.0f} k |")
