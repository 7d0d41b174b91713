// Generic level kernel (any block sizes, any redirection permutation).
#include "kernel_table.cuh"

namespace bcss {
const KernelCfg kGeneric = make_cfg<GenericLevelKernel<32, 64, 16, 2, 2, 2>>("generic32x64");
const KernelCfg kGenericAlt1 = make_cfg<GenericLevelKernel<64, 64, 16, 2, 2, 3>>("generic64x64s3");
const KernelCfg kGenericAlt2 = make_cfg<GenericLevelKernel<64, 128, 16, 2, 4, 3>>("generic64x128s3");
}  // namespace bcss
