#!/bin/bash
# A/B of the K1 sketch kernel: prefix-cached upper entries vs all lookups
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/gpu_parity.log 2>&1; echo "parity rc=$?"; tail -3 gpurun_out/gpu_parity.log
for cfg in ${K1_CFGS:-"2 1.0" "4 0.5" "5 0.2" "3 1.0" "1 1.0"}; do
  for env in "X=1" "CPSJ_K1_NO_PFX=1"; do
    echo "== c$cfg $env"; env $env timeout 300 python tools/k1_probe.py $cfg 4 2>&1 | tail -4
  done
done
