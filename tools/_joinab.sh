cd ${GRAFT_REPO_ROOT:-/root/repo}
for cfg in "2 1.0 2" "5 0.2 3"; do
  for v in default s4096 s2048 s2048d4 s4096d4; do
    lib=paper_1707_06814_b200/_lib/variants/$v.so
    [ $v = default ] && lib=paper_1707_06814_b200/_lib/libcpsjoin_b200.so
    for e in "X=1" "CPSJ_DEVICE_LEVELS=1"; do
      echo "== $v c$cfg $e"; env $e CPSJ_LIB=$lib timeout 300 python tools/join_once.py $cfg 6 2>&1 | grep -E "call [45]|pairs" | cut -c1-200
    done
  done
done
