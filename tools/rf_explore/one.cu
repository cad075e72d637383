// Single-instantiation TU for fast RF-model exploration (tools/rf_explore/run.sh).
// -DKERNEL=1 selects gpp_main_kernel<POLICY, NWV, IGPV>; default is the
// production gpp_sacc_kernel<NWV, IGPV>.
#include "gpp_kernels.cuh"
#ifndef POLICY
#define POLICY gpp::FastPolicy
#endif
#ifndef NWV
#define NWV 3
#endif
#ifndef IGPV
#define IGPV 2
#endif
#if defined(KERNEL) && KERNEL == 1
template __global__ void gpp::gpp_main_kernel<POLICY, NWV, IGPV, false>(gpp::Params);
#else
template __global__ void gpp::gpp_sacc_kernel<NWV, IGPV, false>(const __grid_constant__ gpp::Params,
                                                              const __grid_constant__ gpp::WxTable);
#endif
