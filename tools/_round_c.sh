#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/gpu_parity.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/gpu_parity.log
for cfg in "2 1.0 2" "5 0.2 3" "3 1.0 2" "1 1.0 3"; do for env in "X=1" "CPSJ_SPLIT_CUB=1" "CPSJ_NO_BLOCK_LEAF=1"; do
  echo "== c$cfg $env"; env $env timeout 300 python tools/join_once.py $cfg 6 2>&1 | grep -E "call [45]"
done; done
timeout 600 python tools/embed_probe.py 2 1.0 2>&1 | grep -v "^\s*$" | head -60
