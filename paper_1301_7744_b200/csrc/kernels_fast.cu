// Fast level kernels for one power-of-two b_a (compile with -DBCSS_BA=4|8|16|32|64).
#include "kernel_table.cuh"

#ifndef BCSS_BA
#error "define BCSS_BA"
#endif

#define BCSS_CAT2(a, b) a##b
#define BCSS_CAT(a, b) BCSS_CAT2(a, b)
#define BCSS_UNPAREN(...) __VA_ARGS__
#define BCSS_ENTRY(K, name) make_cfg<BCSS_UNPAREN K>(name),

namespace bcss {
const KernelCfg BCSS_CAT(kFast, BCSS_BA)[N_SHAPES] = {BCSS_FAST_SHAPES(BCSS_ENTRY, BCSS_BA)};
const KernelCfg BCSS_CAT(kGen, BCSS_BA)[N_GEN] = {BCSS_GEN_SHAPES(BCSS_ENTRY, BCSS_BA)};
}  // namespace bcss
