#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests.log
for e in "X=1" "CPSJ_K1_FUSE=1"; do
  echo "== bench $e"
  env $e timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$e.json 2> gpurun_out/bench_$e.err; echo "bench rc=$?"; tail -3 gpurun_out/bench_$e.err
done
echo "== c3 k1"; python tools/k1_probe.py 3 1.0 4 2>&1 | tail -3 | head -2
bash tools/_joinab.sh
python tools/k1_once.py 2 1.0 > gpurun_out/plain_pfx.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_sketch_s16 -c 1 -f -o gpurun_out/ncu_k1_s16_r02 python tools/k1_once.py 2 1.0 > gpurun_out/ncu_pfx.log 2>&1
echo "ncu rc=$?"
bash tools/_joinlaunches.sh
