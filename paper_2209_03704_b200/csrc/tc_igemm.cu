// tc_igemm.cu -- placeholder until the tcgen05 implicit GEMM lands.
#include "common.cuh"
#include "kernels.h"
namespace segconv_b200 {
bool tc_igemm_supported(const FusedProblem&, int) { return false; }
bool tc_igemm_available(int, int, int) { return false; }
cudaError_t launch_tc_igemm(const FusedProblem&, int, cudaStream_t) { return cudaErrorNotSupported; }
}  // namespace segconv_b200
