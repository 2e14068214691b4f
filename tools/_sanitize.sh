#!/bin/bash
# compute-sanitizer evidence: ONE tool per gpurun call (the
# profiling recipe: four tools in one call have wedged a B200 before), over
# parity tests that drive every join kernel (level path, K7 subtree with its
# persistent queue, K4 leaf kernels, K5, K6, dense remap, K1).
#   bash tools/_sanitize.sh memcheck|racecheck|synccheck|initcheck
cd "${GRAFT_REPO_ROOT:-/root/repo}"
tool=${1:-memcheck}
mkdir -p gpurun_out/sanitizer
SAN=/usr/local/cuda/bin/compute-sanitizer
SEL="join_matches_reference_golden or small_limit_deep_tree or dense_remap_matches_reference or minhash_kat_tables"
python -m pytest tests/test_gpu_parity.py tests/test_gpu_dense.py -q -x -k "$SEL" > gpurun_out/sanitizer/plain.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/sanitizer/plain.log; exit 1; }
timeout 2400 $SAN --tool $tool --target-processes all --print-limit 50 \
  python -m pytest tests/test_gpu_parity.py tests/test_gpu_dense.py -q -x -k "$SEL" \
  > gpurun_out/sanitizer/$tool.log 2>&1
echo "$tool rc=$?"; tail -6 gpurun_out/sanitizer/$tool.log
