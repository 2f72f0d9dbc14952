#!/bin/bash
# Debug build of libmcr (MCR_XDOT_DEBUG self-checks) next to the release one; run with
# MCR_LIB=paper_1210_6412_b200/libmcr_dbg.so MCR_XDOT_STATS=1.
cd "$(dirname "$0")/.." || exit 1
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo ${MCR_DBG_DEFS:--DMCR_XDOT_DEBUG} \
  -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -shared -I include \
  -o paper_1210_6412_b200/${MCR_DBG_OUT:-libmcr_dbg.so} paper_1210_6412_b200/csrc/mcr.cu paper_1210_6412_b200/csrc/formats.cpp
