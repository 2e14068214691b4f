#!/bin/bash
# Round-2 measurement sweep: exact-join truths for the remaining BASELINE
# (config, lambda) pairs, then every (config, lambda) bench row with the
# full-workload oracle parity check.  Logs in gpurun_out/sweep/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/sweep
export TRUTH_DIR=gpurun_out/truth
timeout 1500 python tools/exact_probe.py 4:1:0.6 4:1:0.7 4:1:0.8 4:1:0.9 5:1:0.6 --write > gpurun_out/sweep/truth.log 2>&1
echo "truth rc=$?"; tail -12 gpurun_out/sweep/truth.log
cp gpurun_out/truth/*.npz tests/golden/ 2>/dev/null
for spec in "1 0.5" "3 0.5" "3 0.7" "4 0.5" "4 0.6" "4 0.7" "4 0.8" "4 0.9" "5 0.6"; do
  set -- $spec
  timeout 1200 python bench.py --config $1 --lambda $2 --steps 5 --warmup 3 > gpurun_out/sweep/c$1_l$2.json 2> gpurun_out/sweep/c$1_l$2.err
  echo "c$1 l$2 rc=$?"; tail -1 gpurun_out/sweep/c$1_l$2.err
done
