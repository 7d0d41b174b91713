// Table of compiled level-kernel configurations (one translation unit per
// b_a so the fast kernels build in parallel).
#pragma once

#include <cstddef>

#include "sttsm_kernels.cuh"
#include "sttsm_ws_kernel.cuh"

namespace bcss {

struct KernelCfg {
  int BM, BN, NT;
  size_t smem;
  void (*fn)(LevelArgs);
  const char* name;
};

template <class K>
__global__ void __launch_bounds__(K::NT, 1) level_kernel(const LevelArgs a) { K::run(a); }

template <class K>
KernelCfg make_cfg(const char* name) {
  return KernelCfg{K::BM, K::BN, K::NT, K::SMEM_BYTES, level_kernel<K>, name};
}

// shape 3 (the large levels' 128x128 tile): slice depth and stages can be
// changed for experiments (-DBCSS_S3_BK=16 -DBCSS_S3_ST=5)
#ifndef BCSS_S3_BK
#define BCSS_S3_BK 32
#endif
#ifndef BCSS_S3_ST
#define BCSS_S3_ST 3
#endif
#define BCSS_SHAPE3(BA) WsLevelKernel<128, 128, BCSS_S3_BK, 4, 4, BCSS_S3_ST, BA>

// Fast tile shapes (BM, BN, BK, warps WM x WN, stages), in the order the
// plan's shape policy indexes them.  Every b_a instantiates the same list.
#define BCSS_FAST_SHAPES(X, BA)                                        \
  X((WsLevelKernel<128, 128, 32, 2, 4, 3, BA>), "ws128x128c8")    \
  X((WsLevelKernel<64, 256, 16, 2, 4, 4, BA>), "ws64x256c8")      \
  X((WsLevelKernel<32, 256, 32, 1, 8, 3, BA>), "ws32x256c8")      \
  X((BCSS_SHAPE3(BA)), "ws128x128c16")   \
  X((WsLevelKernel<64, 256, 16, 2, 8, 4, BA>), "ws64x256c16")     \
  X((WsLevelKernel<32, 256, 32, 1, 16, 3, BA>), "ws32x256c16")     \
  X((WsLevelKernel<16, 512, 16, 1, 16, 3, BA>), "ws16x512c16k16") \
  X((WsLevelKernel<64, 256, 16, 2, 8, 5, BA>), "ws64x256c16k16s5") \
  X((WsLevelKernel<96, 128, 32, 3, 4, 3, BA>), "ws96x128c12")      \
  X((WsLevelKernel<48, 256, 16, 3, 4, 4, BA>), "ws48x256c12k16")   \
  X((WsLevelKernel<32, 128, 32, 1, 16, 5, BA>), "ws32x128c16s5")

constexpr int N_SHAPES = 11;
// shapes the calibrated policy chooses from (shape_costs.hpp); the others
// serve special roles (ws32x128c16s5: half-width tiles of a launch's last round)
constexpr int N_POLICY_SHAPES = 10;

// General-redirection variants (reuse=False top level), a subset of the shapes
// above; BCSS_GEN_OF[i] is the fast shape each one mirrors (its measured cost).
#define BCSS_GEN_SHAPES(X, BA)                                                 \
  X((WsLevelKernel<128, 128, 32, 4, 4, 3, BA, 4, true>), "gen128x128c16")     \
  X((WsLevelKernel<64, 256, 16, 2, 8, 4, BA, 4, true>), "gen64x256c16")       \
  X((WsLevelKernel<32, 256, 32, 1, 8, 3, BA, 4, true>), "gen32x256c8")       \
  X((WsLevelKernel<96, 128, 32, 3, 4, 3, BA, 4, true>), "gen96x128c12")

constexpr int N_GEN = 4;
constexpr int BCSS_GEN_OF[N_GEN] = {3, 4, 2, 8};

// Non-power-of-two b_a (multiples of 4): the same kernel with POW2 = false,
// instantiated per row group RG (the largest of 28, 24, 20, 12, 4 dividing
// b_a; BK a multiple of RG) on three tile shapes, 16 consumer warps each; every
// policy shape index maps to one of them (BCSS_NP_SHAPES).
// (PAD: b_a padded up to a multiple of RG, see WsLevelKernel; one more table per RG)
#define BCSS_NP_BIG(RG, BK, PAD) WsLevelKernel<128, 128, BK, 4, 4, 3, RG, 4, false, false, PAD>
// 96x128 tiles, 12 consumer warps, 4 stages (row groups 12 and 24: kernels_np.cu)
#define BCSS_NP_BIG96(RG, BK, PAD) WsLevelKernel<96, 128, BK, 3, 4, 4, RG, 4, false, false, PAD>
#define BCSS_NP_MID(RG, BK, PAD) WsLevelKernel<64, 256, BK, 2, 8, 3, RG, 4, false, false, PAD>
#define BCSS_NP_SMALL(RG, BK, PAD) WsLevelKernel<32, 256, BK, 1, 16, 3, RG, 4, false, false, PAD>
constexpr int N_NP = 5;
constexpr int kNpRg[N_NP] = {4, 12, 20, 24, 28};
extern const KernelCfg kNP4[N_SHAPES];
extern const KernelCfg kNP12[N_SHAPES];
extern const KernelCfg kNP20[N_SHAPES];
extern const KernelCfg kNP24[N_SHAPES];
extern const KernelCfg kNP28[N_SHAPES];
// padded variants (PAD = true): also 8- and 16-row groups, for b_a just below them (6, 14, 15, ...)
constexpr int N_NPP = 7;
constexpr int kNppRg[N_NPP] = {4, 8, 12, 16, 20, 24, 28};
extern const KernelCfg kNPP4[N_SHAPES];
extern const KernelCfg kNPP8[N_SHAPES];
extern const KernelCfg kNPP12[N_SHAPES];
extern const KernelCfg kNPP16[N_SHAPES];
extern const KernelCfg kNPP20[N_SHAPES];
extern const KernelCfg kNPP24[N_SHAPES];
extern const KernelCfg kNPP28[N_SHAPES];

// b_a variants of the fast kernels (one translation unit each): 4, 8, 16, 32, 64
constexpr int N_BA = 5;
extern const KernelCfg kFast4[N_SHAPES];
extern const KernelCfg kFast8[N_SHAPES];
extern const KernelCfg kFast16[N_SHAPES];
extern const KernelCfg kFast32[N_SHAPES];
extern const KernelCfg kFast64[N_SHAPES];
extern const KernelCfg kGen4[N_GEN];
extern const KernelCfg kGen8[N_GEN];
extern const KernelCfg kGen16[N_GEN];
extern const KernelCfg kGen32[N_GEN];
extern const KernelCfg kGen64[N_GEN];
extern const KernelCfg kGeneric;      // other b_a, insertion-form levels
extern const KernelCfg kGenericPerm;  // other b_a, reuse=False top level

}  // namespace bcss
