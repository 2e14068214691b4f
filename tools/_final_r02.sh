#!/bin/bash
# Round-2 evidence for profiles/: GPU tests, smoke, the default bench, the
# reference arm, the functional 2-rank bench, then the ncu captures.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/final; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q > $O/gpu_tests_r02.log 2>&1; echo "tests rc=$?"; tail -2 $O/gpu_tests_r02.log
timeout 600 python __graft_entry__.py --smoke > $O/smoke_r02.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke_r02.log
timeout 1200 python bench.py > $O/bench_r02_c2.json 2> $O/bench_r02_c2.log; echo "bench rc=$?"; tail -2 $O/bench_r02_c2.log
timeout 1200 python bench.py --impl reference --steps 2 --warmup 1 > $O/ref_r02_c2.json 2> $O/ref_r02_c2.log; echo "ref rc=$?"; tail -1 $O/ref_r02_c2.log
timeout 900 python bench.py --gpus 2 --dist-backend gloo --steps 2 --warmup 1 --no-cpu-baseline > $O/bench_gloo2_r02.json 2> $O/bench_gloo2_r02.log; echo "gloo2 rc=$?"; tail -1 $O/bench_gloo2_r02.log
# ncu (one tool per call; plain runs first)
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-parity > $O/plain_bench.json 2> $O/plain_bench.log &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file $O/launches_r02_c2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-parity > $O/ncu_bench.log 2>&1
echo "launch list rc=$?"
python tools/k1_once.py 2 1.0 > $O/plain_k1.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:"k_sketch_s16|k_values_h8" -c 2 -f -o $O/ncu_k1_r02 python tools/k1_once.py 2 1.0 > $O/ncu_k1.log 2>&1
echo "ncu k1 rc=$?"
python tools/join_once.py 2 1.0 2 > $O/plain_join.log 2>&1 &&
ncu --set full --clock-control none -k regex:"k_leaf_tiles|k_leaf_small|k_build_keys|Onesweep|k_flags|k_verify|k_children_e|k_survivors|k_subtree|k_rs_scatter" -c 40 -f -o $O/ncu_join_r02 python tools/join_once.py 2 1.0 2 > $O/ncu_join.log 2>&1
echo "ncu join rc=$?"
# gpurun brings back at most 64 MiB: summaries here, the big report stays behind
python tools/ncu_summary.py $O/ncu_join_r02.ncu-rep $O/ncu_join_r02_c2.csv && rm -f $O/ncu_join_r02.ncu-rep
python tools/ncu_summary.py $O/ncu_k1_r02.ncu-rep $O/ncu_k1_r02_c2.csv
du -sh gpurun_out
