#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_b.json 2> gpurun_out/bench_b.err; echo "bench rc=$?"; tail -3 gpurun_out/bench_b.err
for cfg in "2 1.0 2" "5 0.2 3" "3 1.0 2"; do for env in "X=1" "CPSJ_NO_LEAF_OVERLAP=1"; do
  echo "== c$cfg $env"; env $env timeout 300 python tools/join_once.py $cfg 6 2>&1 | grep -E "call [45]"
done; done
