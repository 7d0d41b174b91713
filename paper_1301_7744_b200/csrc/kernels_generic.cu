// Generic level kernel (any block sizes, any redirection permutation).
#include "kernel_table.cuh"

namespace bcss {
// insertion-form redirection (every level except a reuse=False top level)
const KernelCfg kGeneric = make_cfg<GenericLevelKernel<64, 64, 16, 2, 2, 3, true>>("generic64x64ins");
// any redirection permutation (reuse=False top level: unsorted keys into A)
const KernelCfg kGenericPerm = make_cfg<GenericLevelKernel<64, 64, 16, 2, 2, 3, false>>("generic64x64perm");
}  // namespace bcss
