// FP64 tensor-core (DMMA) level-contraction kernel for BCSS sttsm on sm_100a.
//
// One launch computes one level of the algorithm-by-blocks
// (_level_product, /root/reference/pkg/src/blocksym/change_of_basis.py:185-236)
// for every call of that level in the current wave, with the jb loop fused:
// all output block rows jb_k = 0..J that share the parent temporary T(k+1)
// form the M dimension of one GEMM.
//
//   T(k)[jb, s'][K] (b_c rows x rest cols) = sum_ib X[jb-rows, ib-cols] @ front(S_ib)
//   S_ib = stored block sorted(K u {ib}) of T(k+1)[s'],  contracted at its
//          insertion position p (storage redirection, storage.py:123-129 +
//          canonicalize, indexing.py:34-54)
//
// GEMM view per (parent, key): M = rows of X (jb fused), N = rest =
// b_a^k*b_c^(m-1-k) columns, K = n (nbar chunks of b_a).  The B operand is a
// gather: each reduction row i = ib*b_a + e reads block S_ib with its own
// stride pattern (lo, e, hi, t).  FP64 tensor cores on Blackwell are the
// warp-level DMMA (mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4); tcgen05 has no
// f64 kind.  Operands are staged by cp.async (LDGSTS) through a STAGES-deep
// shared-memory ring; a persistent CTA walks its work items and keeps the
// ring running across item boundaries.
#pragma once

#include <cstdint>

namespace bcss {

struct LevelArgs {
  const double* X;          // p x n, row-major
  const double* Tin;        // [calls_in][keys_in][blk_in]   (A at the top level)
  double* Tout;             // [calls_out][keys_out][blk_out] (packed C at level 0)
  const int4* parents;      // {in_call, row0, rows, child_off}
  const long long* item_off;  // n_parents + 1 prefix sums of work items
  const int* child_call;    // output call index of (parent child_off + jb - row0/b_c)
  const int2* nbr;          // [keys_out * nbar] {rank in T(k+1) keys, code}
  long long total_items;
  long long keys_in, keys_out, blk_in, blk_out;
  int n_parents;
  int n, ldx, p_rows;
  int nbar, bA, bC, lbA;
  int k;
  int rest, bAk;
  int n_tiles;
  long long pw[10];         // bA^i
};

// nbr code word: bits 0..3 = insertion position p (fast path); bits 4.. =
// 3-bit stored position of every logical mode d = 0..k (generic path).
__host__ __device__ inline int code_p(int code) { return code & 15; }
__host__ __device__ inline int code_map(int code, int d) { return (code >> (4 + 3 * d)) & 7; }

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

struct TileInfo {
  long long item;
  int key, nt, mt;
  int in_call, row0, rows, child_off;
};

__device__ __forceinline__ TileInfo decode_item(const LevelArgs& a, long long item, int BM) {
  TileInfo t;
  t.item = item;
  int lo = 0, hi = a.n_parents - 1;  // largest P with item_off[P] <= item
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (__ldg(a.item_off + mid) <= item) lo = mid; else hi = mid - 1;
  }
  const int4 par = __ldg(a.parents + lo);
  t.in_call = par.x;
  t.row0 = par.y;
  t.rows = par.z;
  t.child_off = par.w;
  const long long local = item - __ldg(a.item_off + lo);
  const int mtiles = (t.rows + BM - 1) / BM;
  t.mt = (int)(local % mtiles);
  const long long q = local / mtiles;
  t.nt = (int)(q % a.n_tiles);
  t.key = (int)(q / a.n_tiles);
  return t;
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool FAST>
struct LevelKernel {
  static constexpr int NT = WM * WN * 32;
  static constexpr int WTM = BM / WM, WTN = BN / WN;
  static constexpr int FM = WTM / 8, FN = WTN / 8;
  static constexpr int LDA = BK + 4;   // 8 mod 32 banks per row: conflict-free A fragments
  static constexpr int LDB = BN + 4;   // same for B fragments
  static constexpr int A_STAGE = BM * LDA, B_STAGE = BK * LDB;
  static constexpr size_t SMEM_BYTES = (size_t)STAGES * (A_STAGE + B_STAGE) * sizeof(double);
  static_assert(WTM % 8 == 0 && WTN % 8 == 0 && BK % 4 == 0, "tile shape");
  static_assert((BM * BK) % NT == 0 && (BK * BN) % NT == 0, "loader balance");

  // ---- operand staging --------------------------------------------------------
  static __device__ __forceinline__ void load_stage(const LevelArgs& a, const TileInfo& t, int kstep,
                                                    double* As, double* Bs) {
    const int tid = threadIdx.x;
    const int k0 = kstep * BK;
    // A = X[row0 + mt*BM + r, k0 + c]: rows beyond the parent's range are zero.
    const int rbase = t.mt * BM;
    if (FAST) {
#pragma unroll
      for (int it = 0; it < (BM * BK / 2) / NT; ++it) {
        const int idx = tid + it * NT;
        const int r = idx / (BK / 2), c = (idx % (BK / 2)) * 2;
        const bool ok = (rbase + r < t.rows) && (k0 + c < a.n);
        const double* src = ok ? a.X + (long long)(t.row0 + rbase + r) * a.ldx + k0 + c : a.X;
        cp_async16(As + r * LDA + c, src, ok);
      }
    } else {
#pragma unroll
      for (int it = 0; it < (BM * BK) / NT; ++it) {
        const int idx = tid + it * NT;
        const int r = idx / BK, c = idx % BK;
        const bool ok = (rbase + r < t.rows) && (k0 + c < a.n);
        const double* src = ok ? a.X + (long long)(t.row0 + rbase + r) * a.ldx + k0 + c : a.X;
        cp_async8(As + r * LDA + c, src, ok);
      }
    }
    // B = logical T(k+1) block (K, ib) rows e, columns [n0, n0+BN).
    const int n0 = t.nt * BN;
    const int2* nrow = a.nbr + (long long)t.key * a.nbar;
    const double* tin_call = a.Tin + (long long)t.in_call * a.keys_in * a.blk_in;
    if (FAST) {
      // Row groups share one ib (one stored block, one contracted position).
      const int RG = a.bA < BK ? a.bA : BK;
      const int lgRG = a.bA < BK ? a.lbA : __ffs(BK) - 1;
      const int kl = a.k * a.lbA;
#pragma unroll 4
      for (int it = 0; it < (BK * BN) / NT; ++it) {
        const int idx = tid + it * NT;
        const int g = idx >> (lgRG + __ffs(BN) - 1);        // / (RG*BN)
        const int j = idx & ((RG * BN) - 1);
        const int i = k0 + (g << lgRG);                     // first reduction row of the group
        const int ib = i >> a.lbA;
        const int e0 = i & (a.bA - 1);
        const int2 nb = __ldg(nrow + (ib < a.nbar ? ib : 0));
        const int pos = code_p(nb.y);
        int e, col;
        if (pos == 0) { e = j & (RG - 1); col = j >> lgRG; }   // stored block is e-contiguous
        else { col = j & (BN - 1); e = j >> (__ffs(BN) - 1); }  // lo-contiguous
        const int cg = n0 + col;
        const bool ok = (i + e < a.n) && (cg < a.rest);
        const int af = cg & (a.bAk - 1);
        const int tt = cg >> kl;
        const int sh = pos * a.lbA;
        const long long off = (long long)(af & ((1 << sh) - 1)) + ((long long)(e0 + e) << sh) +
                              ((long long)(af >> sh) << (sh + a.lbA)) + ((long long)tt << (kl + a.lbA));
        const double* src = ok ? tin_call + (long long)nb.x * a.blk_in + off : a.X;
        cp_async8(Bs + ((g << lgRG) + e) * LDB + col, src, ok);
      }
    } else {
#pragma unroll 1
      for (int it = 0; it < (BK * BN) / NT; ++it) {
        const int idx = tid + it * NT;
        const int r = idx / BN, col = idx % BN;
        const int i = k0 + r, cg = n0 + col;
        const bool ok = (i < a.n) && (cg < a.rest);
        const double* src = a.X;
        if (ok) {
          const int ib = i / a.bA, e = i - ib * a.bA;
          const int2 nb = __ldg(nrow + ib);
          int af = cg % a.bAk;
          const int tt = cg / a.bAk;
          long long off = (long long)tt * a.pw[a.k + 1] + (long long)e * a.pw[code_map(nb.y, a.k)];
          for (int d = 0; d < a.k; ++d) {
            const int dig = af % a.bA;
            af /= a.bA;
            off += (long long)dig * a.pw[code_map(nb.y, d)];
          }
          src = tin_call + (long long)nb.x * a.blk_in + off;
        }
        cp_async8(Bs + r * LDB + col, src, ok);
      }
    }
  }

  // ---- DMMA on one staged slice ----------------------------------------------
  static __device__ __forceinline__ void compute_stage(const double* As, const double* Bs,
                                                       double (&acc)[FM][FN][2]) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wm = warp / WN, wn = warp % WN;
    const double* ap = As + (wm * WTM + (lane >> 2)) * LDA + (lane & 3);
    const double* bp = Bs + (lane & 3) * LDB + wn * WTN + (lane >> 2);
#pragma unroll
    for (int kk = 0; kk < BK / 4; ++kk) {
      double af[FM], bf[FN];
#pragma unroll
      for (int fm = 0; fm < FM; ++fm) af[fm] = ap[fm * 8 * LDA + kk * 4];
#pragma unroll
      for (int fn = 0; fn < FN; ++fn) bf[fn] = bp[kk * 4 * LDB + fn * 8];
#pragma unroll
      for (int fm = 0; fm < FM; ++fm)
#pragma unroll
        for (int fn = 0; fn < FN; ++fn) dmma(acc[fm][fn][0], acc[fm][fn][1], af[fm], bf[fn]);
    }
  }

  // ---- write-back of the finished tile (inverse fronting folded in) ----------
  static __device__ __forceinline__ void epilogue(const LevelArgs& a, const TileInfo& t,
                                                  double (&acc)[FM][FN][2]) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wm = warp / WN, wn = warp % WN;
    const int jb0 = t.row0 / a.bC;
    const long long tstride = (long long)a.bAk * a.bC;
#pragma unroll
    for (int fm = 0; fm < FM; ++fm) {
      const int r = t.mt * BM + wm * WTM + fm * 8 + (lane >> 2);
      if (r >= t.rows) continue;
      const int xrow = t.row0 + r;
      const int jb = xrow / a.bC, c = xrow - jb * a.bC;
      const int call = __ldg(a.child_call + t.child_off + (jb - jb0));
      double* base = a.Tout + ((long long)call * a.keys_out + t.key) * a.blk_out + (long long)a.bAk * c;
#pragma unroll
      for (int fn = 0; fn < FN; ++fn) {
        const int col = t.nt * BN + wn * WTN + fn * 8 + 2 * (lane & 3);
        if (FAST && a.bAk >= 2) {
          if (col < a.rest) {
            const int af = col & (a.bAk - 1);
            const long long off = af + tstride * (col >> (a.k * a.lbA));
            *reinterpret_cast<double2*>(base + off) = make_double2(acc[fm][fn][0], acc[fm][fn][1]);
          }
        } else {
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int cq = col + q;
            if (cq < a.rest) {
              const int tt = cq / a.bAk, af = cq - tt * a.bAk;
              base[af + tstride * tt] = acc[fm][fn][q];
            }
          }
        }
      }
    }
  }

  static __device__ void run(const LevelArgs& a) {
    extern __shared__ __align__(16) double smem[];
    double* As = smem;
    double* Bs = smem + STAGES * A_STAGE;
    const long long first = blockIdx.x;
    if (first >= a.total_items) return;
    const long long my_items = (a.total_items - 1 - first) / gridDim.x + 1;
    const int ksteps = (a.n + BK - 1) / BK;
    const long long total_steps = my_items * ksteps;

    TileInfo ld = decode_item(a, first, BM);
    TileInfo cp = ld;
    int ld_k = 0;
    long long ld_step = 0;

    double acc[FM][FN][2];
#pragma unroll
    for (int fm = 0; fm < FM; ++fm)
#pragma unroll
      for (int fn = 0; fn < FN; ++fn) acc[fm][fn][0] = acc[fm][fn][1] = 0.0;

    auto advance_load = [&]() {
      ++ld_step;
      if (++ld_k == ksteps) {
        ld_k = 0;
        if (ld_step < total_steps) ld = decode_item(a, ld.item + gridDim.x, BM);
      }
    };
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
      if (ld_step < total_steps) {
        load_stage(a, ld, ld_k, As + s * A_STAGE, Bs + s * B_STAGE);
        advance_load();
      }
      cp_async_commit();
    }
    int cp_k = 0;
    for (long long step = 0; step < total_steps; ++step) {
      cp_async_wait<STAGES - 2>();
      __syncthreads();
      if (ld_step < total_steps) {
        const int slot = (int)(ld_step % STAGES);
        load_stage(a, ld, ld_k, As + slot * A_STAGE, Bs + slot * B_STAGE);
        advance_load();
      }
      cp_async_commit();
      const int slot = (int)(step % STAGES);
      compute_stage(As + slot * A_STAGE, Bs + slot * B_STAGE, acc);
      if (++cp_k == ksteps) {
        cp_k = 0;
        epilogue(a, cp, acc);
#pragma unroll
        for (int fm = 0; fm < FM; ++fm)
#pragma unroll
          for (int fn = 0; fn < FN; ++fn) acc[fm][fn][0] = acc[fm][fn][1] = 0.0;
        if (step + 1 < total_steps) cp = decode_item(a, cp.item + gridDim.x, BM);
      }
    }
    cp_async_wait<0>();
  }
};

}  // namespace bcss
