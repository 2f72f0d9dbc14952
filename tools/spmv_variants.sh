#!/bin/bash
# Build libmcr variants (tile pipeline knobs) into build/variants/<name>/libmcr.so
# name: b<batch>m<min blocks>s<stages>t<tile nnz>
set -e
cd "$(dirname "$0")/.."
mkdir -p build/variants
for v in "$@"; do
  b=$(echo $v | sed -E 's/b([0-9]+)m.*/\1/'); m=$(echo $v | sed -E 's/.*m([0-9]+)s.*/\1/')
  s=$(echo $v | sed -E 's/.*s([0-9]+)t.*/\1/'); t=$(echo $v | sed -E 's/.*t([0-9]+)$/\1/')
  mkdir -p build/variants/$v
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -shared -Iinclude \
    -DMCR_SP_BATCH=$b -DMCR_SP_MINB=$m -DMCR_SP_STAGES=$s -DMCR_TILE_NNZ=$t -o build/variants/$v/libmcr.so paper_1210_6412_b200/csrc/mcr.cu paper_1210_6412_b200/csrc/formats.cpp &
done
wait
