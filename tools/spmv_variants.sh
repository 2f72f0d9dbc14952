#!/bin/bash
# Build libmcr variants (tile pipeline knobs) into build/variants/<name>/libmcr.so
set -e
cd "$(dirname "$0")/.."
mkdir -p build/variants
for v in "b8m4s2:-DMCR_SP_BATCH=8 -DMCR_SP_MINB=4 -DMCR_SP_STAGES=2" "b4m4s2:-DMCR_SP_BATCH=4 -DMCR_SP_MINB=4 -DMCR_SP_STAGES=2" "b8m3s2:-DMCR_SP_BATCH=8 -DMCR_SP_MINB=3 -DMCR_SP_STAGES=2" "b8m2s3:-DMCR_SP_BATCH=8 -DMCR_SP_MINB=2 -DMCR_SP_STAGES=3"; do
  name=${v%%:*}; flags=${v#*:}
  mkdir -p build/variants/$name
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -shared -Iinclude $flags -o build/variants/$name/libmcr.so paper_1210_6412_b200/csrc/mcr.cu &
done
wait
