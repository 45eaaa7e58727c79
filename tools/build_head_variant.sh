#!/bin/bash
# Build the committed (git HEAD or REV) sources as variants/libNAME.so for A/B runs:
#   tools/build_head_variant.sh NAME [REV]
set -e
name=$1; rev=${2:-HEAD}
d=/tmp/variant_$name
rm -rf $d; mkdir -p $d/pkg/csrc $d/include
cd /root/repo
for f in $(git ls-tree --name-only $rev include/); do git show $rev:$f > $d/include/$(basename $f); done
for f in $(git ls-tree --name-only $rev paper_2401_14762_b200/csrc/); do git show $rev:$f > $d/pkg/csrc/$(basename $f); done
mkdir -p variants
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC -I $d/include \
  -o variants/lib$name.so $d/pkg/csrc/*.cu
echo built variants/lib$name.so
