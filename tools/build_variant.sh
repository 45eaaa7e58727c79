#!/bin/bash
# Build an experimental library variant: tools/build_variant.sh NAME 'sed-expr-for-greedy|-' [extra nvcc flags...]
# -> variants/libNAME.so (copies csrc to /tmp so the tree stays clean)
set -e
name=$1; expr=$2; shift 2
d=/tmp/variant_$name
rm -rf $d; mkdir -p $d/pkg/csrc $d/include
cp /root/repo/include/*.h $d/include/
cp /root/repo/paper_2401_14762_b200/csrc/* $d/pkg/csrc/
if [ "$expr" != "-" ]; then sed -i "$expr" $d/pkg/csrc/hcs_greedy.cu; fi
mkdir -p /root/repo/variants
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC -I $d/include "$@" \
  -o /root/repo/variants/lib$name.so $d/pkg/csrc/*.cu
echo built variants/lib$name.so
