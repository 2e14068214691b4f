#!/bin/bash
# per-launch device times of one warm c2 join (device-driven and host-driven level loops)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python tools/join_once.py 2 1.0 2 2 > gpurun_out/plain_join.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_join_dle.csv python tools/join_once.py 2 1.0 2 2 > gpurun_out/ncu_join_dle.log 2>&1
echo "dle rc=$?"
CPSJ_HOST_LEVELS=1 python tools/join_once.py 2 1.0 2 2 > gpurun_out/plain_join_host.log 2>&1 &&
CPSJ_HOST_LEVELS=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_join_host.csv python tools/join_once.py 2 1.0 2 2 > gpurun_out/ncu_join_host.log 2>&1
echo "host rc=$?"
