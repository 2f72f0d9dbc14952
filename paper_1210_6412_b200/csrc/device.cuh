// device.cuh -- sm_100a kernels of the reachability solver (umbrella header).
//
//   common.cuh   layout structs, SolveState, helpers, BiCGStab scalar steps, row epilogues
//   spmv.cuh     persistent TMA-pipelined CSR SpMV (k_spmv<EPI>) and SELL-32-sigma
//   vector.cuh   BiCGStab vector phases, reference-order dots, row-shard finalisation
//   xdot.cuh     the reference's sequential inner product, bit-exact, in parallel
//   small.cuh    whole-solve cooperative kernels for small systems
//   dense.cuh    dense slab GEMV (k_dense<EPI>)
//   upload.cuh   upload-time kernels
//   staged.cuh   band-staged two-pass SpMV for x far larger than L2
#pragma once

#include "common.cuh"
#include "spmv.cuh"
#include "vector.cuh"
#include "xdot.cuh"
#include "small.cuh"
#include "dense.cuh"
#include "upload.cuh"
#include "staged.cuh"
