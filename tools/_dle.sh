#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests.log
grep -E "^FAILED|Error" gpurun_out/gpu_tests.log | head -5
for cfg in "2 1.0 2" "1 1.0 3" "3 1.0 2"; do for env in "X=1" "CPSJ_DLE_GRID=2" "CPSJ_DLE_GRID=8" "CPSJ_HOST_LEVELS=1"; do
  echo "== c$cfg $env"; env $env timeout 300 python tools/join_once.py $cfg 6 2>&1 | grep -E "call [45]"
done; done
