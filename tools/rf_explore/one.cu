// Single-instantiation TU for fast RF-model exploration (tools/rf_explore/run.sh).
#include "gpp_kernels.cuh"
#ifndef POLICY
#define POLICY gpp::FastPolicy
#endif
#ifndef NWV
#define NWV 3
#endif
#ifndef IGPV
#define IGPV 3
#endif
template __global__ void gpp::gpp_main_kernel<POLICY, NWV, IGPV, false>(gpp::Params);
