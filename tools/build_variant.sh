#!/bin/bash
# Build an A/B variant of the library: tools/build_variant.sh NAME [GIT_REV] [NVCC defines...]
# GIT_REV (or "-" for the working tree) selects the csrc sources; output
# paper_1707_06814_b200/_lib/variants/NAME.so (load with CPSJ_LIB=...).
set -e
cd "$(dirname "$0")/.."
name=$1; rev=${2:--}; shift 2 || true
out=paper_1707_06814_b200/_lib/variants; mkdir -p $out
src=paper_1707_06814_b200/csrc; tmp=$(mktemp -d)
if [ "$rev" != "-" ]; then git archive "$rev" paper_1707_06814_b200/csrc include | tar -x -C $tmp; src=$tmp/paper_1707_06814_b200/csrc; inc=$tmp/include; else inc=include; fi
objs=""
for f in $(ls $src/*.cu | xargs -n1 basename | sed 's/\.cu$//'); do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr --extended-lambda "$@" -I $inc -c $src/$f.cu -o $tmp/$f.o &
  objs="$objs $tmp/$f.o"
done
wait
/usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a $objs -o $out/$name.so -Xcompiler -fPIC
rm -rf $tmp
echo $out/$name.so
