// Generic level kernel (any block sizes, any redirection permutation).
#include "kernel_table.cuh"

namespace bcss {
const KernelCfg kGeneric = make_cfg<GenericLevelKernel<32, 64, 16, 2, 2, 2>>("generic32x64");
}  // namespace bcss
