// fp32 throughput build of the fused env step (compiled -fmad=false like the
// fp64 build; the tool / env logic stays fp64 in both).
#define TS_DEFINE_SCALAR_KERNELS   // the per-env command / epilogue kernels live in this TU
#include "step_kernel.cuh"

template cudaError_t ts_launch_step<float>(const TsDevProg &, const TsParams &, const TsLaunch &, int, int,
                                           cudaStream_t, bool);
template cudaError_t ts_launch_reset<float>(const TsDevProg &, const TsParams &, const TsLaunch &,
                                            const uint8_t *, int, cudaStream_t);
template cudaError_t ts_launch_cluster_step<float>(const TsDevProg *, int, int, int, const TsParams &, const TsLaunch &,
                                                  int, int, cudaStream_t);
