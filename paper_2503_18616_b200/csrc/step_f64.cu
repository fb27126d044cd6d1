// fp64 build of the fused env step: compiled with -fmad=false so every
// expression rounds exactly like the reference's C (-ffp-contract=off),
// giving bitwise parity with the compiled CPU backend.
#include "step_kernel.cuh"

template cudaError_t ts_launch_step<double>(const TsDevProg &, const TsParams &, const TsLaunch &, int, int,
                                            cudaStream_t, bool);
template cudaError_t ts_launch_reset<double>(const TsDevProg &, const TsParams &, const TsLaunch &,
                                             const uint8_t *, int, cudaStream_t);
template cudaError_t ts_launch_cluster_step<double>(const TsDevProg *, int, int, int, const TsParams &, const TsLaunch &,
                                                  int, int, cudaStream_t);
