#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests.log
grep -E "FAILED|Error" gpurun_out/gpu_tests.log | head -10
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -2 gpurun_out/bench.err
for env in "X=1" "CPSJ_NO_BLOCK_LEAF=1" "CPSJ_DEFER_DEPTH=2" "CPSJ_DEFER_DEPTH=3" "CPSJ_DEFER_DEPTH=1"; do
  echo "== $env"; env $env CPSJ_JOIN_TRACE=1 timeout 300 python tools/join_once.py 2 1.0 2 6 2>&1 | grep -E "call [345]|\[join\]" | tail -14
done
for cfg in 4 2; do for env in "X=1" "CPSJ_K1_NO_FUSE=1"; do
  echo "== c$cfg $env"; env $env timeout 900 python bench.py --config $cfg --steps 4 --warmup 2 --no-cpu-baseline --no-parity 2>&1 >/dev/null | grep -E "step_e2e|device step"
done; done
