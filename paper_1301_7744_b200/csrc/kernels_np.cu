// Fast level kernels for non-power-of-two b_a (POW2 = false), one row group
// per translation unit (compile with -DBCSS_NP_RG=4|12|20|24|28 (|8|16 padded), and
// -DBCSS_NP_PAD=1 for the padded-row-group variants).  The table has one
// entry per policy shape index, each one of three tile shapes.
#include "kernel_table.cuh"

#ifndef BCSS_NP_RG
#error "define BCSS_NP_RG"
#endif

#ifndef BCSS_NP_PAD
#define BCSS_NP_PAD 0
#endif
#if BCSS_NP_PAD
#define BCSS_NP_TABLE kNPP
#else
#define BCSS_NP_TABLE kNP
#endif

#define BCSS_CAT2(a, b) a##b
#define BCSS_CAT(a, b) BCSS_CAT2(a, b)

namespace bcss {
namespace {
constexpr int RG = BCSS_NP_RG;
// slice depths: a multiple of RG that keeps the loaders balanced and the ring
// within shared memory (RG 4, 8, 16: 32 / 16 / 32; else RG, or 2 RG for RG 12)
constexpr bool SUB32 = RG == 4 || RG == 8 || RG == 16;  // (8, 16: padded variants only)
constexpr int BK_BIG = SUB32 ? 32 : RG == 12 ? 24 : RG;
constexpr int BK_MID = SUB32 ? 16 : RG == 12 ? 24 : RG;
constexpr int BK_SMALL = SUB32 ? 32 : RG == 12 ? 24 : RG;
// 32-row tiles need BK a multiple of 8 (loader balance); else the 64-row one
constexpr bool SMALL_OK = BK_SMALL % 8 == 0;
constexpr bool PADDED = BCSS_NP_PAD != 0;
using Big = BCSS_NP_BIG(RG, BK_BIG, PADDED);
// 96x128 tiles with 12 consumer warps and a 4-deep ring for the policy's
// 96-row shape: row groups 12, 20 and 24 (BK <= 24; the X loader's last round
// is partial for BK = 20), unpadded kernels only (measured: b_a = 24 top level
// 27.7 -> 29.4 TF at m = 3, 24.5 -> 32.4 TF at m = 4; b_a = 20 29.6 -> 30.5 TF
// at m = 4, 23.3 -> 24.9 at m = 3; row group 28 loses 4 %, the padded
// variants 2 %)
template <bool OK>
struct Big96Sel { using type = BCSS_NP_BIG96(RG, BK_BIG, PADDED); };
template <>
struct Big96Sel<false> { using type = Big; };
using Big96 = Big96Sel<(!PADDED && BK_BIG <= 24)>::type;
using Mid = BCSS_NP_MID(RG, BK_MID, PADDED);
template <bool OK>
struct SmallSel { using type = BCSS_NP_SMALL(RG, BK_SMALL, PADDED); };
template <>
struct SmallSel<false> { using type = Mid; };
using Small = SmallSel<SMALL_OK>::type;
}  // namespace

// policy shape index -> tile shape (kernel_table.cuh BCSS_FAST_SHAPES order)
const KernelCfg BCSS_CAT(BCSS_NP_TABLE, BCSS_NP_RG)[N_SHAPES] = {
    make_cfg<Big>("np128x128"),   // 0 ws128x128c8
    make_cfg<Mid>("np64x256"),    // 1 ws64x256c8
    make_cfg<Small>("np32x256"),  // 2 ws32x256c8
    make_cfg<Big>("np128x128"),   // 3 ws128x128c16
    make_cfg<Mid>("np64x256"),    // 4 ws64x256c16
    make_cfg<Small>("np32x256"),  // 5 ws32x256c16
    make_cfg<Small>("np32x256"),  // 6 ws16x512c16k16
    make_cfg<Mid>("np64x256"),    // 7 ws64x256c16k16s5
    make_cfg<Big96>(Big96::BM == 96 ? "np96x128" : "np128x128"),  // 8 ws96x128c12
    make_cfg<Mid>("np64x256"),    // 9 ws48x256c12k16
    make_cfg<Small>("np32x256"),  // 10 ws32x128c16s5
};
}  // namespace bcss
