cd ${GRAFT_REPO_ROOT:-/root/repo}
mkdir -p gpurun_out
CPSJ_JOIN_TRACE=1 python tools/join_once.py 2 1.0 2 > gpurun_out/join_trace.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_build_keys|k_flags|k_verify|Onesweep|k_children_e|k_survivors|k_node_sketch" -c 24 -o gpurun_out/ncu_join_split python tools/join_once.py 2 1.0 2 > gpurun_out/ncu_join_split.log 2>&1
echo done
