// libmsp: the C-ABI of include/msp.h (paper arXiv 2208.08594, PAPER.md "P:n").  One
// translation unit, organised in parts (included in dependency order):
//   msp_handle.cuh   handle state, CUDA error / launch helpers, device level layout
//   setup_host.cuh   config and BSR intake, index checks, SELL level layouts, BILU tables
//   setup_device.cuh GPU SETUP (S1, Galerkin chain, BILU factorization), do_setup
//   dist_setup.cuh   distributed SETUP: partitioned levels, halo plans, localization
//   launch.cuh       hot-path launch sequences (a2-a9, V-cycles, MSP application)
//   gmres.cuh        orthogonalisation, Arnoldi steps / graphs, the GMRES loop
//   capi_*.cuh       the extern "C" entry points
#include "msp_handle.cuh"
#include "setup_host.cuh"
#include "setup_device.cuh"
#include "dist_setup.cuh"
#include "launch.cuh"
#include "gmres.cuh"
#include "capi_core.cuh"
#include "capi_kernels.cuh"
#include "capi_dist.cuh"
#include "capi_host.cuh"
