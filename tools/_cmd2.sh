ncu --set full --import-source on --clock-control none -k k_subtree -c 1 -o gpurun_out/subtree2 python tools/join_once.py 2 1.0 2 > gpurun_out/ncu_sub.log 2>&1
