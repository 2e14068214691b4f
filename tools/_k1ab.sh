cd ${GRAFT_REPO_ROOT:-/root/repo}
for v in base cache24 cache20 cache16; do
  for cfg in "2 1.0" "4 0.5" "5 0.2" "3 1.0" "1 1.0"; do
    echo "== $v c$cfg"; CPSJ_LIB=paper_1707_06814_b200/_lib/variants/$v.so timeout 300 python tools/k1_probe.py $cfg 4 2>&1 | tail -3
  done
done
