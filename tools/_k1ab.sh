#!/bin/bash
# A/B harness for K1 builds: variants from tools/build_variant.sh NAME - -DFLAG=...
# (paper_1707_06814_b200/_lib/variants/NAME.so) against the default library.
#   K1_VARIANTS="w24 t20" bash tools/_k1ab.sh
cd ${GRAFT_REPO_ROOT:-/root/repo}
for cfg in "2 1.0" "3 1.0" "5 0.2" "4 0.5" "1 1.0"; do
  for v in default ${K1_VARIANTS} nopfx; do
    lib=paper_1707_06814_b200/_lib/variants/$v.so; e="X=1"
    [ $v = default ] && lib=paper_1707_06814_b200/_lib/libcpsjoin_b200.so
    [ $v = nopfx ] && lib=paper_1707_06814_b200/_lib/libcpsjoin_b200.so && e="CPSJ_K1_NO_PFX=1"
    echo "== $v c$cfg"; env $e CPSJ_LIB=$lib timeout 300 python tools/k1_probe.py $cfg 4 2>&1 | tail -3 | head -2
  done
done
