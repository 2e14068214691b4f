#!/bin/bash
# Round-2 measurement sweep: every BASELINE (config, lambda) row with the
# full-workload oracle parity check (exact-join truth files are committed
# under tests/golden/; tools/exact_probe.py --write regenerates them).
# Logs in gpurun_out/sweep/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/sweep
for spec in ${SWEEP_SPECS:-"1 0.5" "3 0.5" "3 0.7" "4 0.5" "4 0.6" "4 0.7" "4 0.8" "4 0.9" "5 0.6"}; do
  set -- $spec
  steps=5; [ "$1" = 1 ] && steps=30
  timeout 1800 python bench.py --config $1 --lambda $2 --steps $steps --warmup 3 --full-parity > gpurun_out/sweep/sweep_r02_c$1_l$2.json 2> gpurun_out/sweep/sweep_r02_c$1_l$2.log
  echo "c$1 l$2 rc=$?"; tail -1 gpurun_out/sweep/sweep_r02_c$1_l$2.log | cut -c1-260
done
