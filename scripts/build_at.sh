#!/bin/bash
# Build libmuxb200.so of another commit (A/B runs): scripts/build_at.sh <commit> <out.so>
set -e
C=$1; OUT=$2; T=$(mktemp -d)
mkdir -p $T/paper_2605_08962_b200/csrc $T/include
for f in $(git ls-tree --name-only $C paper_2605_08962_b200/csrc/); do git show $C:$f > $T/$f; done
git show $C:include/mux_b200.h > $T/include/mux_b200.h
objs=""
for f in $T/paper_2605_08962_b200/csrc/*.cu; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
    -Xcompiler -fPIC -I $T/include -c $f -o $f.o & objs="$objs $f.o"
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT $objs -Xcompiler -fPIC
rm -rf $T
echo built $OUT
