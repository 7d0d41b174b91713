// Warp-specialized FP64 DMMA level kernel (sm_100a).
//
// Same contraction as FastLevelKernel (see sttsm_kernels.cuh for the algebra:
// one level of _level_product, change_of_basis.py:185-236, with the jb loop
// fused into M), but the roles are split:
//   * NPROD producer warps walk the CTA's work items and stage operands with
//     16-byte cp.async into a STAGES-deep ring; completion is signalled per
//     slot on a "full" mbarrier (cp.async.mbarrier.arrive.noinc);
//   * WM x WN consumer warps only load DMMA fragments from shared memory and
//     issue mma.sync m8n8k4 f64 (SASS DMMA.8x8x4), release each slot on an
//     "empty" mbarrier and write finished tiles straight from registers.
// Consumers never execute address arithmetic or wait on global loads, so the
// FP64 tensor pipe stays fed while producers run ahead by up to STAGES slots.
#pragma once

#include "sttsm_kernels.cuh"


namespace bcss {

constexpr long long kNoRow = (long long)(~0ull >> 1) * -1 - 1;  // padding row (row offsets may be negative)

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("{\n.reg .b64 st;\nmbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cp_async(uint64_t* bar) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(a) : "memory");
}
// Bulk (TMA-engine) copy global -> shared of `bytes` (multiple of 16), which
// completes on `bar`; the issuing thread must have raised the barrier's
// expected transaction count (mbar_expect_tx) by the bytes it issues.
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;\n" ::"r"(b), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_copy_g2s(void* smem, const void* gmem, unsigned bytes, uint64_t* bar) {
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(d),
               "l"(gmem), "r"(bytes), "r"(b)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}\n" ::"r"(a), "r"(parity) : "memory");
}

template <int R>
__device__ __forceinline__ void regs_dec() { asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(R)); }
template <int R>
__device__ __forceinline__ void regs_inc() { asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(R)); }

// NPROD producer warps form whole warpgroups (setmaxnreg acts per warpgroup):
// they shrink to PROD_REGS registers and the consumers grow into the rest.
// GEN = true: general redirection permutations (reuse=False top level, whose
// unsorted keys map to A's canonical blocks by arbitrary mode permutations).
// POW2 = false: b_a is not a power of two (a multiple of 4); BA is then the
// row group RG (a multiple of 4 dividing b_a and BK) and b_a comes from the
// launch arguments: stored-block offsets use b_a^p multiplications and
// divisions instead of shifts, every row group is staged [e][col], and the
// epilogue splits columns by division.
// PAD (with POW2 = false): b_a is not a multiple of the row group; the
// contraction index runs over blocks padded to b_a' = a.bAp rows (X is
// padded with zero columns, run.cu), rows e >= b_a of a group are zero-filled,
// and an odd b_a (odd strides, 8-byte alignment only) moves 8 bytes at a time.
template <int BM_, int BN_, int BK_, int WM, int WN, int STAGES, int BA, int NPROD = 4, bool GEN = false,
          bool POW2 = true, bool PAD = false>
struct WsLevelKernel {
  static_assert(!PAD || !POW2, "padded row groups are a non-power-of-two variant");
  static constexpr int BM = BM_, BN = BN_, BK = BK_;
  static constexpr int NCW = WM * WN;               // consumer warps
  static_assert(NPROD % 4 == 0 && NCW % 4 == 0, "roles must be whole warpgroups");
  static constexpr int NT = (NCW + NPROD) * 32;     // threads per CTA
  // setmaxnreg.inc blocks until the CTA's launch-time pool has the registers,
  // so the consumers' share is what the producers give back from that pool.
  static constexpr int LAUNCH_REGS = (65536 / NT) / 8 * 8 > 255 ? 248 : (65536 / NT) / 8 * 8;
  static constexpr int PROD_REGS = 56;
  static constexpr int CONS_REGS_RAW = (LAUNCH_REGS * NT - NPROD * 32 * PROD_REGS) / (NCW * 32);
  static constexpr int CONS_REGS = (CONS_REGS_RAW > 256 ? 256 : CONS_REGS_RAW) / 8 * 8;
  static constexpr int PT = NPROD * 32;             // producer threads
  static constexpr int WTM = BM / WM, WTN = BN / WN;
  static constexpr int FM = WTM / 8, FN = WTN / 8;
  static constexpr int LBA = (BA == 2) ? 1 : (BA == 4) ? 2 : (BA == 8) ? 3 : (BA == 16) ? 4 : (BA == 32) ? 5 : 6;
  static constexpr int RG = !POW2 ? BA : BA < BK ? BA : BK;  // rows per group (one ib)
  static constexpr int G = BK / RG;             // groups per stage
  static constexpr int LDA = BK + 4;
  static constexpr int LDR = BN + 4;            // row-major group stride ([e][col])
  // [col][e] staging (e-contiguous blocks): column stride CS; power-of-two row
  // groups use RG with an XOR swizzle, the others pad to CS = RG+4 or RG+8
  // (CS/4 odd: the fragment loads' rows fall in distinct banks, no swizzle)
  static constexpr int CS = POW2 ? RG : (((RG + 4) / 4) % 2 ? RG + 4 : RG + 8);
  static constexpr int GR_ROW = RG * LDR;
  static constexpr int GR_COL = BN * CS;
  // !POW2: the [col][e] layout only where its larger groups keep the ring in
  // shared memory (else those groups are gathered 8 bytes at a time, [e][col])
  static constexpr bool NP_EC =
      !POW2 && (size_t)STAGES * (BM * LDA + (BK / RG) * (GR_ROW > GR_COL ? GR_ROW : GR_COL)) * 8 + 8192 <= 232448;
  static constexpr int GR_SIZE = NP_EC && GR_COL > GR_ROW ? GR_COL : GR_ROW;  // POW2: >= BN*RG
  static constexpr int SW_SHIFT = RG >= 16 ? 0 : 1;
  static constexpr int SW_MASK = RG >= 16 ? 3 : (RG == 8 ? 1 : 0);
  static constexpr int A_STAGE = BM * LDA, B_STAGE = G * GR_SIZE;
  static constexpr int NA = (BM * BK / 2 + PT - 1) / PT;  // X pairs per producer thread per stage
  static constexpr bool NA_EXACT = (BM * BK / 2) % PT == 0;  // (else the last round is partial)
  static constexpr int GP = RG * BN / 2;         // B pairs per group
  // column runs of at least 2^BULK_MIN_LG doubles go through bulk copies
  // (measured after the producer's addressing was hoisted: >= 512 B runs pay
  // off for b_a >= 16, >= 4 KB runs for b_a <= 8; shorter runs lose to cp.async)
#ifdef BCSS_BULK_LG_SMALL  // experiments: thresholds for b_a <= 8 / b_a >= 16
  static constexpr int BULK_MIN_LG = BA >= 16 ? BCSS_BULK_LG_LARGE : BCSS_BULK_LG_SMALL;
#else
  static constexpr int BULK_MIN_LG = BA >= 16 ? 6 : 9;
#endif
  static constexpr int NB = (BK * BN / 2) / PT;  // B pairs per producer thread per stage
  static constexpr int CSTEP_ = PT / (RG / 2);
  static constexpr int GPAD = (G + 3) / 4 * 4;   // modes per slot, int4-aligned
  static constexpr size_t SMEM_BYTES = (size_t)STAGES * (A_STAGE + B_STAGE) * sizeof(double) +
                                       (size_t)STAGES * BM * sizeof(long long) +  // output row offsets
                                       STAGES * sizeof(int4) + STAGES * 2 * sizeof(uint64_t) +
                                       STAGES * GPAD * sizeof(int) +
                                       (BN / CSTEP_) * sizeof(int);  // mirrored level 0: digit_rev(i * CSTEP)
  static_assert(BM <= PT, "one producer thread per output row");
  static_assert(WTM % 8 == 0 && WTN % 8 == 0, "tile shape");
  static_assert((BK * BN / 2) % PT == 0 && GP % 32 == 0, "loader balance");
  static_assert(POW2 ? ((1 << LBA) == BA && RG % 4 == 0) : (RG % 4 == 0 && BK % RG == 0 && !GEN),
                "BA must be a power of two in 4..64 (or, !POW2, a row group dividing BK)");
  static_assert(SMEM_BYTES <= 232448, "shared memory per CTA");

  static __device__ __forceinline__ int swz(int col) { return ((col >> SW_SHIFT) & SW_MASK) << 2; }

  // reverse the order of `digits` base-2^lbc digits of v
  static __device__ __forceinline__ long long digit_rev(int v, int digits, int lbc) {
    long long r = 0;
    const int mask = (1 << lbc) - 1;
    for (int d = 0; d < digits; ++d) {
      r = (r << lbc) | (v & mask);
      v >>= lbc;
    }
    return r;
  }


  // ---- producer: one stage of cp.async (PT threads) ----------------------------
  // Addressing is hoisted per thread: a thread's columns (and, for
  // e-contiguous blocks, its e pair and swizzle) are fixed within a group, so
  // every copy after the first is one add on each side.
  static constexpr int HP = RG / 2;          // e pairs per column (e-contiguous blocks)
  static constexpr int CSTEP = PT / HP;      // column stride of a thread (e-contiguous blocks)
  static constexpr int CPR = BN / 2;         // column pairs per row (column-contiguous blocks)
  static constexpr int ESTEP = PT >= CPR ? PT / CPR : 1;   // row stride of a thread
  static constexpr int NCOL = PT >= CPR ? 1 : CPR / PT;    // column pairs per thread
  static_assert(!POW2 || (PT % HP == 0 && BN % CSTEP == 0 && CSTEP % 4 == 0), "e-contiguous loader");
  static_assert((PT >= CPR ? PT % CPR == 0 && RG % ESTEP == 0 : CPR % PT == 0), "column loader");

  static __device__ __forceinline__ void cp16(unsigned sdst, const double* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sdst), "l"(src));
  }
  static __device__ __forceinline__ void cp8z(unsigned sdst, const double* src, bool ok) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sdst), "l"(src), "r"(ok ? 8 : 0));
  }
  static __device__ __forceinline__ void cp16z(unsigned sdst, const double* src, bool ok) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sdst), "l"(src), "r"(ok ? 16 : 0));
  }

  // neighbour entries of the G groups of stage `kstep` of tile t (loaded a stage ahead)
  static __device__ __forceinline__ void load_nb(const LevelArgs& a, const TileInfo& t, int kstep, int2 (&nb)[G]) {
    const int2* nrow = a.nbr + (long long)t.key * a.nbar;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int i0 = kstep * BK + g * RG;
      nb[g] = __ldg(nrow + (i0 < a.n ? (POW2 ? (i0 >> LBA) : i0 / a.bAp) : 0));
    }
  }

  // General redirection: logical mode d < k of the block (K, ib) sits at stored
  // position code_map(code, d), the contracted mode k at code_map(code, k), the
  // tail behind the b_a digits.  For power-of-two b_a the column -> stored
  // offset map is a bit permutation, so it distributes over disjoint bit fields.
  static __device__ __forceinline__ long long perm_col(int col, int code, int k) {
    long long r = 0;
    for (int d = 0; d < k; ++d) r |= (long long)((col >> (d * LBA)) & (BA - 1)) << (code_map(code, d) * LBA);
    return r | ((long long)(col >> (k * LBA)) << ((k + 1) * LBA));
  }
  static constexpr int LOG_NI = (BN / CSTEP_ >= 64) ? 6 : (BN / CSTEP_ >= 32) ? 5 : (BN / CSTEP_ >= 16) ? 4
                              : (BN / CSTEP_ >= 8) ? 3 : (BN / CSTEP_ >= 4) ? 2 : (BN / CSTEP_ >= 2) ? 1 : 0;
  static __device__ __forceinline__ void produce_group_gen(const LevelArgs& a, int code, const double* base, int e0,
                                                        bool grp_ok, bool full_n, int n0, unsigned dst, int* mode,
                                                        int ptid) {
    const int k = a.k;
    const int se = code_map(code, k) * LBA;  // log2 of the e stride
    if (ptid == 0) *mode = se == 0;
    if (se == 0) {  // e-contiguous: pairs along e, staged [col][e ^ swz]
      const int e2 = (ptid % HP) * 2, c = ptid / HP;
      const unsigned d = dst + (unsigned)(c * RG + (e2 ^ swz(c))) * 8u;
      const long long pb = perm_col(n0 + c, code, k);
      long long basis[LOG_NI > 0 ? LOG_NI : 1];
#pragma unroll
      for (int j = 0; j < LOG_NI; ++j) basis[j] = perm_col(CSTEP << j, code, k);
      const double* src0 = base + (e0 + e2);
#pragma unroll 4
      for (int i = 0; i < BN / CSTEP; ++i) {
        long long off = pb;
#pragma unroll
        for (int j = 0; j < LOG_NI; ++j)
          if ((i >> j) & 1) off |= basis[j];
        const bool ok = grp_ok && (full_n || n0 + c + i * CSTEP < a.rest);
        cp16z(d + (unsigned)(i * CSTEP * RG) * 8u, ok ? src0 + off : a.X, ok);
      }
    } else {  // column-contiguous or scattered columns: staged [e][col]
      const bool pair = code_map(code, 0) == 0 || k == 0;  // columns c2, c2+1 adjacent
      const int et = PT >= CPR ? ptid / CPR : 0;
#pragma unroll
      for (int j = 0; j < NCOL; ++j) {
        const int c2 = 2 * ((PT >= CPR ? ptid % CPR : ptid) + j * PT);
        const int cg = n0 + c2;
        const bool ok = grp_ok && (full_n || cg < a.rest);
        const bool ok1 = grp_ok && (full_n || cg + 1 < a.rest);
        const long long sstep = (long long)ESTEP << se;
        const double* src = base + perm_col(cg, code, k) + ((long long)(e0 + et) << se);
        const double* src1 = base + perm_col(cg + 1, code, k) + ((long long)(e0 + et) << se);
        const unsigned d = dst + (unsigned)(et * LDR + c2) * 8u;
#pragma unroll 4
        for (int i = 0; i < RG / ESTEP; ++i) {
          const unsigned di = d + (unsigned)(i * ESTEP * LDR) * 8u;
          if (pair) {
            cp16z(di, ok ? src + i * sstep : a.X, ok);
          } else {
            cp8z(di, ok ? src + i * sstep : a.X, ok);
            cp8z(di + 8u, ok1 ? src1 + i * sstep : a.X, ok1);
          }
        }
      }
    }
  }

  // !POW2: one row group staged [e][col].  Contracted digit at stored
  // position 0 (e-contiguous in HBM, every level-0 block): element (e, col)
  // at e + b_a * col' (col' = col, or digit-reversed on mirrored level 0),
  // copied 8 bytes at a time; position p > 0: column pairs are contiguous
  // (b_a^p is even), element (e, col) at lo + hi * b_a^(p+1) + e * b_a^p with
  // lo = col mod b_a^p, hi = col div b_a^p.
  static __device__ __forceinline__ void produce_group_np(const LevelArgs& a, const double* base, int e0, int pos,
                                                        bool grp_ok, bool full_n, int n0, unsigned dst, int ptid) {
    const int et = PT >= CPR ? ptid / CPR : 0;
    const int ev = PAD ? a.bA - e0 - et : RG;  // row et + i*ESTEP of the group is real while i*ESTEP < ev
    const bool odd = PAD && (a.bA & 1);
#pragma unroll
    for (int j = 0; j < NCOL; ++j) {
      const int c2 = 2 * ((PT >= CPR ? ptid % CPR : ptid) + j * PT);
      const int cg = n0 + c2;
      const bool ok = grp_ok && (full_n || cg < a.rest);
      const bool ok1 = grp_ok && (full_n || cg + 1 < a.rest);
      const unsigned d = dst + (unsigned)(et * LDR + c2) * 8u;
      if (pos == 0 && NP_EC) {
        return;  // staged [col][e] by produce_group_np_ec
      } else if (pos == 0) {
        long long c0 = cg, c1 = cg + 1;
        if (a.mirror_digits) {
          c0 = digit_rev(cg, a.mirror_digits, a.lbc);
          c1 = digit_rev(cg + 1, a.mirror_digits, a.lbc);
        }
        const double* s0 = base + e0 + et + (long long)a.bA * c0;
        const double* s1 = base + e0 + et + (long long)a.bA * c1;
#pragma unroll 4
        for (int i = 0; i < RG / ESTEP; ++i) {
          const unsigned di = d + (unsigned)(i * ESTEP * LDR) * 8u;
          const bool r = !PAD || i * ESTEP < ev;
          cp8z(di, ok && r ? s0 + i * ESTEP : a.X, ok && r);
          cp8z(di + 8u, ok1 && r ? s1 + i * ESTEP : a.X, ok1 && r);
        }
      } else {
        const int bp = (int)a.pw[pos];  // b_a^p <= rest < 2^31: 32-bit division
        const int hi = cg / bp, lo = cg - hi * bp;
        const double* src = base + lo + (long long)hi * bp * a.bA + (long long)(e0 + et) * bp;
        const long long sstep = (long long)ESTEP * bp;
        if (!odd) {
#pragma unroll 4
          for (int i = 0; i < RG / ESTEP; ++i) {
            const unsigned di = d + (unsigned)(i * ESTEP * LDR) * 8u;
            const bool r = ok && (!PAD || i * ESTEP < ev);
            cp16z(di, r ? src + i * sstep : a.X, r);
          }
        } else {  // odd b_a^p: columns cg, cg+1 may sit in different runs, and nothing is 16-byte aligned
          const int hi1 = (cg + 1) / bp, lo1 = cg + 1 - hi1 * bp;
          const double* src1 = base + lo1 + (long long)hi1 * bp * a.bA + (long long)(e0 + et) * bp;
#pragma unroll 4
          for (int i = 0; i < RG / ESTEP; ++i) {
            const unsigned di = d + (unsigned)(i * ESTEP * LDR) * 8u;
            const bool r = i * ESTEP < ev;
            cp8z(di, ok && r ? src + i * sstep : a.X, ok && r);
            cp8z(di + 8u, ok1 && r ? src1 + i * sstep : a.X, ok1 && r);
          }
        }
      }
    }
  }

  // !POW2, contracted digit at stored position 0 (e-contiguous in HBM):
  // 16-byte e pairs into the padded [col][e] layout (column stride CS)
  static __device__ __forceinline__ void produce_group_np_ec(const LevelArgs& a, const double* base, int e0,
                                                           bool grp_ok, bool full_n, int n0, unsigned dst, int ptid) {
    constexpr int NP_PAIRS = BN * (RG / 2);
    static_assert(NP_PAIRS % PT == 0, "e-pair loader balance");
    const bool odd = PAD && (a.bA & 1);
#pragma unroll 4
    for (int j = 0; j < NP_PAIRS / PT; ++j) {
      const int q = ptid + j * PT;
      const int col = q / (RG / 2), e2 = 2 * (q - col * (RG / 2));
      const int cg = n0 + col;
      const bool ok = grp_ok && (full_n || cg < a.rest);
      const long long cc = a.mirror_digits ? digit_rev(cg, a.mirror_digits, a.lbc) : (long long)cg;
      const double* src = base + e0 + e2 + (long long)a.bA * cc;
      const unsigned d = dst + (unsigned)(col * CS + e2) * 8u;
      if (!PAD) {
        cp16z(d, ok ? src : a.X, ok);
      } else {
        const int er = a.bA - (e0 + e2);  // real rows left from this pair on (even for an even b_a)
        if (!odd) {
          const bool r = ok && er >= 2;
          cp16z(d, r ? src : a.X, r);
        } else {
          const bool r0 = ok && er >= 1, r1 = ok && er >= 2;
          cp8z(d, r0 ? src : a.X, r0);
          cp8z(d + 8u, r1 ? src + 1 : a.X, r1);
        }
      }
    }
  }

  static __device__ __forceinline__ void produce(const LevelArgs& a, const TileInfo& t, int kstep,
                                                 const int2 (&nb)[G], unsigned As_s, unsigned Bs_s, int* modes,
                                                 const int* srev, int ptid, uint64_t* fullbar) {
    const int k0 = kstep * BK;
#pragma unroll
    for (int u = 0; u < NA; ++u) {
      const int idx = ptid + u * PT;
      if (!NA_EXACT && idx >= BM * BK / 2) break;
      const int r = idx / (BK / 2), c = (idx % (BK / 2)) * 2;
      const int rr = t.mt * BM + r;
      const bool ok = (rr < t.rows) && (k0 + c < a.n);
      const double* src = ok ? a.X + (long long)(t.row0 + rr) * a.ldx + k0 + c : a.X;
      cp16z(As_s + (unsigned)(r * LDA + c) * 8u, src, ok);
    }
    const int n0 = t.nt * BN;
    const bool full_n = n0 + BN <= a.rest;
    const double* tin_call = a.Tin + (long long)t.in_call * a.keys_in * a.blk_in;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int i0 = k0 + g * RG;
      const bool grp_ok = i0 < a.n;
      const int pos = code_p(nb[g].y);
      const double* base = tin_call + (long long)nb[g].x * a.blk_in;
      const int e0 = POW2 ? (i0 & (BA - 1)) : i0 % a.bAp;
      const unsigned dst = Bs_s + (unsigned)(g * GR_SIZE) * 8u;
      if constexpr (GEN) {
        produce_group_gen(a, nb[g].y, base, e0, grp_ok, full_n, n0, dst, modes + g, ptid);
        continue;
      }
      if constexpr (!POW2) {
        if (ptid == 0) modes[g] = NP_EC && pos == 0;
        if (NP_EC && pos == 0) produce_group_np_ec(a, base, e0, grp_ok, full_n, n0, dst, ptid);
        else produce_group_np(a, base, e0, pos, grp_ok, full_n, n0, dst, ptid);
        continue;
      }
      if (ptid == 0) modes[g] = pos == 0;
      if (pos == 0 && a.mirror_digits) {
        // mirrored level 0: GEMM column g reads T(1) column digit_rev(g), so the
        // output (element digits reversed) is written in GEMM column order
        const int e2 = (ptid % HP) * 2, c = ptid / HP;
        const unsigned d = dst + (unsigned)(c * RG + (e2 ^ swz(c))) * 8u;
        // digit reversal is a bit permutation and n0, c, i*CSTEP have disjoint bits
        const long long rb = digit_rev(n0 + c, a.mirror_digits, a.lbc);
        const double* src0 = base + (e0 + e2);
#pragma unroll 4
        for (int i = 0; i < BN / CSTEP; ++i) {
          const bool ok = grp_ok && n0 + c + i * CSTEP < a.rest;
          const double* src = src0 + ((rb | srev[i]) << LBA);
          cp16z(d + (unsigned)(i * CSTEP * RG) * 8u, ok ? src : a.X, ok);
        }
      } else if (pos == 0) {  // e-contiguous block: pairs along e, staged [col][e ^ swz]
        const int e2 = (ptid % HP) * 2, c = ptid / HP;
        const double* src = base + (e0 + e2) + ((long long)(n0 + c) << LBA);
        const unsigned d = dst + (unsigned)(c * RG + (e2 ^ swz(c))) * 8u;
        if (full_n && grp_ok) {
#pragma unroll 8
          for (int i = 0; i < BN / CSTEP; ++i) cp16(d + (unsigned)(i * CSTEP * RG) * 8u, src + ((long long)(i * CSTEP) << LBA));
        } else {
#pragma unroll 4
          for (int i = 0; i < BN / CSTEP; ++i) {
            const bool ok = grp_ok && n0 + c + i * CSTEP < a.rest;
            cp16z(d + (unsigned)(i * CSTEP * RG) * 8u, ok ? src + ((long long)(i * CSTEP) << LBA) : a.X, ok);
          }
        }
      } else if (pos * LBA >= BULK_MIN_LG && grp_ok && full_n) {
        // long column runs: one bulk copy per run into the padded [e][col]
        // layout (the copy engine does the addressing)
        const int sh = pos * LBA;
        const int L = (1 << sh) < BN ? (1 << sh) : BN;   // contiguous doubles per run
        const int runs_per_row = BN / L;
        const int mine = ptid < RG * runs_per_row ? (RG * runs_per_row - 1 - ptid) / PT + 1 : 0;
        if (mine) mbar_expect_tx(fullbar, (unsigned)(mine * L * 8));
        const unsigned bar = (unsigned)__cvta_generic_to_shared(fullbar);
        for (int r = ptid; r < RG * runs_per_row; r += PT) {
          const int e = r / runs_per_row, c0 = (r % runs_per_row) * L;
          const int cg = n0 + c0;
          const long long off = (long long)(cg & ((1 << sh) - 1)) + ((long long)(cg >> sh) << (sh + LBA)) +
                                ((long long)(e0 + e) << sh);
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                  dst + (unsigned)(e * LDR + c0) * 8u),
              "l"(base + off), "r"((unsigned)L * 8u), "r"(bar)
              : "memory");
        }
      } else {  // column-contiguous block: pairs along col, staged [e][col]
        const int sh = pos * LBA;
        const int lomask = (1 << sh) - 1;
        const int et = PT >= CPR ? ptid / CPR : 0;
#pragma unroll
        for (int j = 0; j < NCOL; ++j) {
          const int c2 = 2 * ((PT >= CPR ? ptid % CPR : ptid) + j * PT);
          const int cg = n0 + c2;
          const bool ok = grp_ok && (full_n || cg < a.rest);
          const double* src =
              base + ((long long)(cg & lomask) + ((long long)(cg >> sh) << (sh + LBA)) + ((long long)(e0 + et) << sh));
          const long long sstep = (long long)ESTEP << sh;
          const unsigned d = dst + (unsigned)(et * LDR + c2) * 8u;
          if (ok) {
#pragma unroll 8
            for (int i = 0; i < RG / ESTEP; ++i) cp16(d + (unsigned)(i * ESTEP * LDR) * 8u, src + i * sstep);
          } else {
#pragma unroll 4
            for (int i = 0; i < RG / ESTEP; ++i) cp16z(d + (unsigned)(i * ESTEP * LDR) * 8u, a.X, false);
          }
        }
      }
    }
  }

  // ---- consumer: DMMA over one staged slice -------------------------------------
  // Warp wm owns the 8-row fragments fm*WM + wm of the tile (interleaved, so a
  // partial tile's valid fragments spread evenly over the warps); only the
  // first NF of its FM fragments hold valid rows, the rest are skipped.
  // one row group (one ib) of the slice, for a compile-time staging mode
  // (CM: e-contiguous block staged [col][e ^ swz]; else [e][col])
  // (MODE 1: e-contiguous, 0: column-contiguous, -1: select at run time from cm)
  template <int NF, int MODE>
  static __device__ __forceinline__ void consume_group(const double* ap, const double* Bg, int colw, int sw, int g,
                                                       bool cm_rt, double (&acc)[FM][FN][2]) {
    const int lane = threadIdx.x & 31;
    const bool cm = MODE < 0 ? cm_rt : MODE == 1;
    const double* bp = Bg + (cm ? colw * CS + (lane & 3) : (lane & 3) * LDR + colw);
    const int SN = cm ? 8 * CS : 8;
#pragma unroll
    for (int kk = 0; kk < RG / 4; ++kk) {
      const int ko = cm ? (POW2 ? ((kk * 4) ^ sw) : kk * 4) : kk * 4 * LDR;
      double af[NF], bf[FN];
#pragma unroll
      for (int fm = 0; fm < NF; ++fm) af[fm] = ap[fm * 8 * WM * LDA + (g * RG + kk * 4)];
#pragma unroll
      for (int fn = 0; fn < FN; ++fn) bf[fn] = bp[ko + fn * SN];
#pragma unroll
      for (int fm = 0; fm < NF; ++fm)
#pragma unroll
        for (int fn = 0; fn < FN; ++fn) dmma(acc[fm][fn][0], acc[fm][fn][1], af[fm], bf[fn]);
    }
  }

  template <int NF>
  static __device__ __forceinline__ void consume(const double* As, const double* Bs, const int* modes, int cw,
                                                 double (&acc)[FM][FN][2]) {
    const int lane = threadIdx.x & 31;
    const int wm = cw / WN, wn = cw % WN;
    const double* ap = As + (wm * 8 + (lane >> 2)) * LDA + (lane & 3);
    const int colw = wn * WTN + (lane >> 2);
    const int sw = swz(colw);
    int md[GPAD];
#pragma unroll
    for (int g4 = 0; g4 < GPAD; g4 += 4) {
      const int4 v = *reinterpret_cast<const int4*>(modes + g4);
      md[g4] = v.x; md[g4 + 1] = v.y; md[g4 + 2] = v.z; md[g4 + 3] = v.w;
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
      if constexpr (!POW2) {  // [col][e] (position-0 groups, where it fits) or [e][col]
        if (NP_EC && md[g]) consume_group<NF, 1>(ap, Bs + g * GR_SIZE, colw, sw, g, true, acc);
        else consume_group<NF, 0>(ap, Bs + g * GR_SIZE, colw, sw, g, false, acc);
      } else if constexpr (RG >= 16) {  // the mode is CTA-uniform per group: branch to a specialized body
        if (md[g]) consume_group<NF, 1>(ap, Bs + g * GR_SIZE, colw, sw, g, true, acc);
        else consume_group<NF, 0>(ap, Bs + g * GR_SIZE, colw, sw, g, false, acc);
      } else {  // short groups (b_a <= 8): selects are cheaper than the branches (measured)
        consume_group<NF, -1>(ap, Bs + g * GR_SIZE, colw, sw, g, md[g] != 0, acc);
      }
    }
  }
  template <int NF>
  static __device__ __forceinline__ void consume_valid(int nf, const double* As, const double* Bs, const int* modes,
                                                       int cw, double (&acc)[FM][FN][2]) {
    if constexpr (NF > 0) {
      if (nf >= NF) consume<NF>(As, Bs, modes, cw, acc);
      else consume_valid<NF - 1>(nf, As, Bs, modes, cw, acc);
    }
  }

  // Output offset (in doubles, relative to Tout) of row r of the tile, or -1:
  // the inverse fronting puts row (jb, c) of call `child_call[...]`, key K at
  // (call*keys_out + K)*blk_out + b_A^k*c (change_of_basis.py:231-235).
  static __device__ __forceinline__ long long row_offset(const LevelArgs& a, const TileInfo& t, int r_local) {
    const int r = t.mt * BM + r_local;
    if (r >= t.rows) return kNoRow;
    const int xrow = t.row0 + r;
    const int jb = xrow / a.bC, c = xrow - jb * a.bC;
    const int call = __ldg(a.child_call + t.child_off + (jb - t.row0 / a.bC));
    long long base = (long long)call * a.keys_out * a.blk_out;
    if (a.call_out) {  // per-call destination (a peer GPU's receive slot): offset from Tout in the flat address space
      const double* dst = a.call_out[call];
      if (dst) base = (long long)(reinterpret_cast<uintptr_t>(dst) - reinterpret_cast<uintptr_t>(a.Tout)) / 8;
    }
    return base + (long long)t.key * a.blk_out + a.row_mul * c;
  }

  static __device__ __forceinline__ void epilogue(const LevelArgs& a, const long long (&roff)[FM], int nt, int cw,
                                                  double (&acc)[FM][FN][2]) {
    const int lane = threadIdx.x & 31;
    const int wn = cw % WN;
    const int kl = a.k * LBA;
#ifdef BCSS_NO_EPILOGUE  // timing experiments only: results are not written
    if (a.k >= 0) return;
#endif
    const long long tstride = (long long)a.bAk * a.bC;
    if constexpr (!POW2) {
      if (PAD && a.bAk >= 2 && (a.bAk & 1)) {
        // odd b_a: col and col + 1 may sit in different runs of b_a^k columns,
        // and rows are only 8-byte aligned (a loop of its own, so the common
        // case keeps its code)
#pragma unroll
        for (int fm = 0; fm < FM; ++fm) {
          if (roff[fm] == kNoRow) continue;
          double* base = a.Tout + roff[fm];
#pragma unroll
          for (int fn = 0; fn < FN; ++fn) {
            const int col = nt * BN + (cw % WN) * WTN + fn * 8 + 2 * (lane & 3);
            if (col >= a.rest) continue;
            const int q = col / a.bAk;
            base[(col - q * a.bAk) + tstride * q] = acc[fm][fn][0];
            if (col + 1 < a.rest) {
              const int q1 = (col + 1) / a.bAk;
              base[(col + 1 - q1 * a.bAk) + tstride * q1] = acc[fm][fn][1];
            }
          }
        }
        return;
      }
#pragma unroll
      for (int fm = 0; fm < FM; ++fm) {
        if (roff[fm] == kNoRow) continue;
        double* base = a.Tout + roff[fm];
#pragma unroll
        for (int fn = 0; fn < FN; ++fn) {
          const int col = nt * BN + (cw % WN) * WTN + fn * 8 + 2 * (lane & 3);
          if (col >= a.rest) continue;
          if (a.bAk >= 2) {  // b_a^k even: col, col + 1 in one run
            const long long q = col / a.bAk;
            *reinterpret_cast<double2*>(base + (col - q * a.bAk) + tstride * q) =
                make_double2(acc[fm][fn][0], acc[fm][fn][1]);
          } else if (a.mirror_digits) {
            if (col + 1 < a.rest) *reinterpret_cast<double2*>(base + col) = make_double2(acc[fm][fn][0], acc[fm][fn][1]);
            else base[col] = acc[fm][fn][0];
          } else {
            base[tstride * col] = acc[fm][fn][0];
            if (col + 1 < a.rest) base[tstride * (col + 1)] = acc[fm][fn][1];
          }
        }
      }
      return;
    }
#ifndef BCSS_EPI_GENERAL
    // (only where the consumers have register headroom beyond the
    // accumulators and ptxas does not spill for it: not in the 104-register
    // 16-warp 64x256 / 128x128 shapes, nor in 16x512)
    const long long c0 = (long long)nt * BN + wn * WTN;  // this warp's first column
    if (CONS_REGS - FM * FN * 4 >= 64 && BM > 16 && a.bAk >= WTN && c0 + WTN <= a.rest) {
      // The warp's WTN columns lie inside one run of b_A^k contiguous output
      // columns (b_A^k and WTN are powers of two, c0 is WTN-aligned): one
      // base address per fragment row, immediate column offsets.
      const long long tb = (c0 & (a.bAk - 1)) + tstride * (c0 >> kl) + 2 * (lane & 3);
#pragma unroll
      for (int fm = 0; fm < FM; ++fm) {
        if (roff[fm] == kNoRow) continue;
        double* p = a.Tout + roff[fm] + tb;
#pragma unroll
        for (int fn = 0; fn < FN; ++fn)
          *reinterpret_cast<double2*>(p + fn * 8) = make_double2(acc[fm][fn][0], acc[fm][fn][1]);
      }
      return;
    }
#ifndef BCSS_EPI_MID_OFF  // (A/B switch)
    if (CONS_REGS - FM * FN * 4 >= 64 && BM > 16 && a.bAk >= 8 && c0 + WTN <= a.rest) {
      // 8 <= b_A^k < WTN: each 8-column fragment lies inside one run and c0
      // is run-aligned, so fragment fn's offset only depends on fn
      const long long tb = tstride * (c0 >> kl) + 2 * (lane & 3);
      long long fo[FN];
#pragma unroll
      for (int fn = 0; fn < FN; ++fn) fo[fn] = ((fn * 8) & (a.bAk - 1)) + tstride * ((fn * 8) >> kl);
#pragma unroll
      for (int fm = 0; fm < FM; ++fm) {
        if (roff[fm] == kNoRow) continue;
        double* p = a.Tout + roff[fm] + tb;
#pragma unroll
        for (int fn = 0; fn < FN; ++fn)
          *reinterpret_cast<double2*>(p + fo[fn]) = make_double2(acc[fm][fn][0], acc[fm][fn][1]);
      }
      return;
    }
#endif
#ifndef BCSS_EPI_L0_OFF  // (A/B switch)
    if (CONS_REGS - FM * FN * 4 >= 64 && BM > 16 && a.bAk == 1 && !a.mirror_digits && c0 + WTN <= a.rest) {
      // level 0: GEMM columns are the tail modes at stride b_c
      const long long ts = tstride;
      const long long tb = ts * (c0 + 2 * (lane & 3));
#pragma unroll
      for (int fm = 0; fm < FM; ++fm) {
        if (roff[fm] == kNoRow) continue;
        double* p = a.Tout + roff[fm] + tb;
#pragma unroll
        for (int fn = 0; fn < FN; ++fn) {
          p[ts * (fn * 8)] = acc[fm][fn][0];
          p[ts * (fn * 8 + 1)] = acc[fm][fn][1];
        }
      }
      return;
    }
#endif
#endif
#pragma unroll
    for (int fm = 0; fm < FM; ++fm) {
      if (roff[fm] == kNoRow) continue;
      double* base = a.Tout + roff[fm];
#pragma unroll
      for (int fn = 0; fn < FN; ++fn) {
        const int col = nt * BN + wn * WTN + fn * 8 + 2 * (lane & 3);
        if (col >= a.rest) continue;
        if (a.bAk >= 2) {
          const long long off = (col & (a.bAk - 1)) + tstride * (col >> kl);
          *reinterpret_cast<double2*>(base + off) = make_double2(acc[fm][fn][0], acc[fm][fn][1]);
        } else if (a.mirror_digits) {  // mirrored level 0: GEMM column = element offset
          if (col + 1 < a.rest) *reinterpret_cast<double2*>(base + col) = make_double2(acc[fm][fn][0], acc[fm][fn][1]);
          else base[col] = acc[fm][fn][0];
        } else {  // level 0: columns are the tail modes, stride b_c (rest is odd iff b_c = 1)
          base[tstride * col] = acc[fm][fn][0];
          if (col + 1 < a.rest) base[tstride * (col + 1)] = acc[fm][fn][1];
        }
      }
    }
  }

  static __device__ __forceinline__ void producer_main(const LevelArgs& a, double* As, double* Bs, long long* rowoff,
                                                       int4* tiles, uint64_t* full, uint64_t* empty, int* modes,
                                                       int* srev, long long first, long long total_steps, int ksteps) {
    const int ptid = threadIdx.x - NCW * 32;
    if (a.mirror_digits) {  // producers only: named barrier 1 over the PT producer threads
      if (ptid < BN / CSTEP) srev[ptid] = (int)digit_rev(ptid * CSTEP, a.mirror_digits, a.lbc);
      asm volatile("bar.sync 1, %0;\n" ::"n"(PT) : "memory");
    }
    TileInfo t = decode_item(a, first, BM);
    long long my_roff = ptid < BM ? row_offset(a, t, ptid) : kNoRow;  // fetched a tile ahead of use
    int2 nb[G];
    load_nb(a, t, 0, nb);
    const unsigned As_s = (unsigned)__cvta_generic_to_shared(As);
    const unsigned Bs_s = (unsigned)__cvta_generic_to_shared(Bs);
    int k = 0, slot = 0;
    unsigned phase = 0;
    for (long long step = 0; step < total_steps; ++step) {
      // next stage's position and neighbour entries, loaded before this stage's copies
      TileInfo tn = t;
      int kn = k + 1;
      const bool more = step + 1 < total_steps;
      if (kn == ksteps) {
        kn = 0;
        if (more) tn = decode_item(a, t.item + gridDim.x, BM);
      }
      int2 nbn[G];
      if (more) load_nb(a, tn, kn, nbn);
      if (step >= STAGES) mbar_wait(empty + slot, phase ^ 1);
      produce(a, t, k, nb, As_s + (unsigned)(slot * A_STAGE) * 8u, Bs_s + (unsigned)(slot * B_STAGE) * 8u,
              modes + slot * GPAD, srev, ptid, full + slot);
      mbar_arrive_cp_async(full + slot);
      const bool last = (k == ksteps - 1);
      if (last && ptid < BM) rowoff[slot * BM + ptid] = my_roff;
      if (ptid == 0) {
        const int vrows = t.rows - t.mt * BM;
        tiles[slot] = make_int4(t.nt, ((vrows < BM ? vrows : BM) + 7) >> 3, 0, 0);
      }
      mbar_arrive(full + slot);  // release this thread's modes / rowoff / tiles writes
      if (++slot == STAGES) { slot = 0; phase ^= 1; }
      if (last && more && ptid < BM) my_roff = row_offset(a, tn, ptid);
      t = tn;
      k = kn;
#pragma unroll
      for (int g = 0; g < G; ++g) nb[g] = nbn[g];
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
  }

  static __device__ void run(const LevelArgs& a) {
    extern __shared__ __align__(16) double smem[];
    double* As = smem;
    double* Bs = smem + STAGES * A_STAGE;
    long long* rowoff = reinterpret_cast<long long*>(Bs + STAGES * B_STAGE);
    int4* tiles = reinterpret_cast<int4*>(rowoff + STAGES * BM);
    uint64_t* full = reinterpret_cast<uint64_t*>(tiles + STAGES);
    uint64_t* empty = full + STAGES;
    int* modes = reinterpret_cast<int*>(empty + STAGES);
    int* srev = modes + STAGES * GPAD;  // mirrored level 0: digit_rev(i * CSTEP), i < BN / CSTEP
    const long long first = blockIdx.x;
    if (first >= a.total_items) return;
    const long long my_items = (a.total_items - 1 - first) / gridDim.x + 1;
    const int ksteps = (a.n + BK - 1) / BK;
    const long long total_steps = my_items * ksteps;
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
      for (int s = 0; s < STAGES; ++s) {
        mbar_init(full + s, 2 * PT);   // every producer thread: its cp.async batch + a release arrive
        mbar_init(empty + s, NCW);     // one arrive per consumer warp
      }
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();

    if (warp >= NCW) {
      // ---------------- producer warps ----------------
      regs_dec<PROD_REGS>();
      producer_main(a, As, Bs, rowoff, tiles, full, empty, modes, srev, first, total_steps, ksteps);
      return;
    }
    // ---------------- consumer warps ----------------
    regs_inc<CONS_REGS>();
    const int lane = threadIdx.x & 31;
    const int wm = warp / WN;
    double acc[FM][FN][2];
#pragma unroll
    for (int fm = 0; fm < FM; ++fm)
#pragma unroll
      for (int fn = 0; fn < FN; ++fn) acc[fm][fn][0] = acc[fm][fn][1] = 0.0;
    int k = 0, slot = 0;
    unsigned phase = 0;
#ifdef BCSS_SKEW
    // the second half of the consumer warps starts SKEW slices behind the
    // first, so one half's epilogue overlaps the other half's DMMA
    // (at most STAGES: the leading half cannot get further ahead without the
    // lagging half releasing slots)
    constexpr int SKEW = BCSS_SKEW < STAGES ? BCSS_SKEW : STAGES;
    const bool lag = warp >= NCW / 2;
    const long long skew_at = (SKEW < total_steps ? SKEW : total_steps) - 1;
    if (lag) asm volatile("bar.sync 2, %0;\n" ::"n"(NCW * 32) : "memory");
#endif
    for (long long step = 0; step < total_steps; ++step) {
      mbar_wait(full + slot, phase);
      const int4 tl = tiles[slot];
      const int nf = tl.y > wm ? (tl.y - wm + WM - 1) / WM : 0;  // this warp's valid fragments
      consume_valid<FM>(nf, As + slot * A_STAGE, Bs + slot * B_STAGE, modes + slot * GPAD, warp, acc);
      const bool last = (++k == ksteps);
      long long roff[FM];
      if (last) {  // read the tile's output rows before the slot is released
#pragma unroll
        for (int fm = 0; fm < FM; ++fm) roff[fm] = rowoff[slot * BM + (fm * WM + wm) * 8 + (lane >> 2)];
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + slot);
#ifdef BCSS_SKEW
      if (!lag && step == skew_at) asm volatile("bar.arrive 2, %0;\n" ::"n"(NCW * 32) : "memory");
#endif
      if (++slot == STAGES) { slot = 0; phase ^= 1; }
      if (last) {
        k = 0;
        epilogue(a, roff, tl.x, warp, acc);
#pragma unroll
        for (int fm = 0; fm < FM; ++fm)
#pragma unroll
          for (int fn = 0; fn < FN; ++fn) acc[fm][fn][0] = acc[fm][fn][1] = 0.0;
      }
    }
  }
};

}  // namespace bcss
