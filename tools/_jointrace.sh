#!/bin/bash
# per-level trace of the c2 join, host-driven and device-driven level loops
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for env in "X=1" "CPSJ_DEVICE_LEVELS=1"; do
  echo "== $env"; env $env CPSJ_JOIN_TRACE=1 timeout 300 python tools/join_once.py ${JT_CFG:-2 1.0 2} 5 2>&1 | grep -E "call [34]|\[join\]" | cut -c1-330
done
