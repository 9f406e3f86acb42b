#!/bin/bash
# Build libnmq.so variants (extra -D flags) into tools/variants/ for sweep.sh.
# usage: tools/build_variants.sh name1:"-DFOO=1 -DBAR" name2:"..."
set -e
cd "$(dirname "$0")/.."
mkdir -p tools/variants
C=paper_2305_02678_b200/csrc
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared \
    $flags -o tools/variants/libnmq_$name.so $C/nmq_kernels.cu $C/nmq_fast.cu $C/nmq_warp.cu $C/nmq_lod.cu $C/nmq_train.cu $C/nmq_kl.cu $C/nmq_abi.cu $C/nmq_multi.cu &
done
wait
ls -la tools/variants
