#!/bin/bash
# ncu --set full of the K1 sketch kernel, prefix cache on and off (c2, full size)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python tools/k1_once.py 2 1.0 > gpurun_out/plain_pfx.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_sketch_s16 -c 1 -f -o gpurun_out/ncu_k1_s16_pfx python tools/k1_once.py 2 1.0 > gpurun_out/ncu_pfx.log 2>&1
echo "pfx rc=$?"
CPSJ_K1_NO_PFX=1 python tools/k1_once.py 2 1.0 > gpurun_out/plain_nopfx.log 2>&1 &&
CPSJ_K1_NO_PFX=1 ncu --set full --clock-control none --import-source on -k regex:k_sketch_s16 -c 1 -f -o gpurun_out/ncu_k1_s16_nopfx python tools/k1_once.py 2 1.0 > gpurun_out/ncu_nopfx.log 2>&1
echo "nopfx rc=$?"
