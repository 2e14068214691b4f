cd ${GRAFT_REPO_ROOT:-/root/repo}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/gpu_parity.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/gpu_parity.log
for cfg in "2 1.0" "3 1.0" "5 0.2" "4 0.5" "1 1.0"; do
  for v in default w24 t20 t28 nopfx; do
    lib=paper_1707_06814_b200/_lib/variants/$v.so; e="X=1"
    [ $v = default ] && lib=paper_1707_06814_b200/_lib/libcpsjoin_b200.so
    [ $v = nopfx ] && lib=paper_1707_06814_b200/_lib/libcpsjoin_b200.so && e="CPSJ_K1_NO_PFX=1"
    echo "== $v c$cfg"; env $e CPSJ_LIB=$lib timeout 300 python tools/k1_probe.py $cfg 4 2>&1 | tail -3 | head -2
  done
done
