// Shared device definitions of the BCSS sttsm level kernels (sm_100a) and the
// generic (any block size) level kernel; the fast warp-specialized kernel is
// in sttsm_ws_kernel.cuh.
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
  const int4* items;        // per work item {parent, key, n-tile, m-tile}
  const int* child_call;    // output call index of (parent child_off + jb - row0/b_c)
  const int2* nbr;          // [keys_out * nbar] {rank in T(k+1) keys, code}
  long long total_items;
  long long keys_in, keys_out, blk_in, blk_out;
  int n_parents;
  int n, ldx, p_rows;
  int nbar, bA, bC, lbA;
  int bAp;                  // fast kernels: rows per block of the contraction index (b_a, or b_a padded
                            // up to a multiple of the row group: n and ldx then count padded columns of X)
  int k;
  int rest, bAk;
  int n_tiles;
  const double* const* call_out;  // stop level: per-call output slice (e.g. a peer GPU's buffer) or null
  long long row_mul;        // output offset of tile row c: bAk, or b_c^(m-1) (mirrored level 0)
  int mirror_digits;        // mirrored level 0: reverse the m-1 column digits (lbc bits each), else 0
  int lbc;
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

__device__ __forceinline__ TileInfo decode_item(const LevelArgs& a, long long item, int /*BM*/) {
  TileInfo t;
  t.item = item;
  const int4 it = __ldg(a.items + item);
  const int4 par = __ldg(a.parents + it.x);
  t.key = it.y;
  t.nt = it.z;
  t.mt = it.w;
  t.in_call = par.x;
  t.row0 = par.y;
  t.rows = par.z;
  t.child_off = par.w;
  return t;
}

// ---------------------------------------------------------------------------
// Generic kernel: any block sizes (including odd b_a / b_c, b = 1), either
// reuse mode, any redirection permutation.  Per-element addressing with
// div/mod and zero-filled bounds.  Its GEMM columns run over (key, column)
// pairs of the whole level (item key field unused, n-tiles over
// keys_out * rest), so small blocks - whose keys have only b_a^k b_c^(m-1-k)
// columns each - still fill the tile.
// ---------------------------------------------------------------------------
// INS = true: the redirection is the insertion form (every reuse=True level and
// the reuse=False levels below the top): the stored offset of logical column c
// = (a-digits c_a < b_a^k, tail t) with the contracted digit e at stored
// position p is lo_p + e b_a^p + b_a (c_a - lo_p) + t b_a^(k+1), lo_p = c_a mod
// b_a^p, so a thread's column terms are computed once per tile and each
// element costs one neighbour lookup and a few multiply-adds.
template <int BM_, int BN_, int BK_, int WM, int WN, int STAGES, bool INS = false>
struct GenericLevelKernel {
  static constexpr int BM = BM_, BN = BN_, BK = BK_;
  static constexpr int NT = WM * WN * 32;
  static_assert(!INS || (NT % BN == 0 && (BK * BN) % NT == 0), "INS: one fixed column per thread");
  static constexpr int RSTEP = NT / BN;  // INS: a thread's rows are r0 + i * RSTEP

  // INS: per-thread column terms of the current load tile
  struct ColInfo {
    long long key_nbar;   // key * n/b_a (neighbour-table row), -1 = past the level's columns
    long long tbase;      // t * b_a^(k+1)
    long long q[8];       // q[p] = lo_p + b_a (c_a - lo_p)
  };
  static __device__ __forceinline__ void col_info(const LevelArgs& a, const TileInfo& t, ColInfo& ci) {
    const long long j = (long long)t.nt * BN + (threadIdx.x % BN);
    if (j >= a.keys_out * a.rest) { ci.key_nbar = -1; return; }
    const long long key = j / a.rest;
    const int c = (int)(j - key * a.rest);
    const int ca = c % a.bAk, tt = c / a.bAk;
    ci.key_nbar = key * a.nbar;
    ci.tbase = (long long)tt * a.pw[a.k + 1];
#pragma unroll
    for (int p = 0; p < 8; ++p) {
      const long long lo = p <= a.k ? ca % a.pw[p] : 0;
      ci.q[p] = lo + (long long)a.bA * (ca - lo);
    }
  }
  static __device__ __forceinline__ void load_stage_ins(const LevelArgs& a, const TileInfo& t, const ColInfo& ci,
                                                        int kstep, double* As, double* Bs) {
    const int tid = threadIdx.x;
    const int k0 = kstep * BK;
    const int rbase = t.mt * BM;
#pragma unroll
    for (int it = 0; it < (BM * BK) / NT; ++it) {
      const int idx = tid + it * NT;
      const int r = idx / BK, c = idx % BK;
      const bool ok = (rbase + r < t.rows) && (k0 + c < a.n);
      const double* src = ok ? a.X + (long long)(t.row0 + rbase + r) * a.ldx + k0 + c : a.X;
      cp_async8(As + r * LDA + c, src, ok);
    }
    const double* tin_call = a.Tin + (long long)t.in_call * a.keys_in * a.blk_in;
    const int col = tid % BN;
    int i = k0 + tid / BN;
    int ib = i / a.bA, e = i - ib * a.bA;
#pragma unroll 4
    for (int it = 0; it < (BK * BN) / NT; ++it) {
      const int r = tid / BN + it * RSTEP;
      const bool ok = ci.key_nbar >= 0 && i < a.n;
      const double* src = a.X;
      if (ok) {
        const int2 nb = __ldg(a.nbr + ci.key_nbar + ib);
        const int pos = code_p(nb.y);
        long long q = ci.q[0];
#pragma unroll
        for (int p = 1; p < 8; ++p)
          if (pos == p) q = ci.q[p];
        src = tin_call + (long long)nb.x * a.blk_in + ci.tbase + q + (long long)e * a.pw[pos];
      }
      cp_async8(Bs + r * LDB + col, src, ok);
      i += RSTEP;
      e += RSTEP;
      while (e >= a.bA) { e -= a.bA; ++ib; }
    }
  }
  static constexpr int WTM = BM / WM, WTN = BN / WN;
  static constexpr int FM = WTM / 8, FN = WTN / 8;
  static constexpr int LDA = BK + 4;
  static constexpr int LDB = BN + 4;
  static constexpr int A_STAGE = BM * LDA, B_STAGE = BK * LDB;
  static constexpr size_t SMEM_BYTES = (size_t)STAGES * (A_STAGE + B_STAGE) * sizeof(double);
  static_assert(WTM % 8 == 0 && WTN % 8 == 0 && BK % 4 == 0, "tile shape");
  static_assert((BM * BK) % NT == 0 && (BK * BN) % NT == 0, "loader balance");

  static __device__ __forceinline__ void load_stage(const LevelArgs& a, const TileInfo& t, int kstep,
                                                    double* As, double* Bs) {
    const int tid = threadIdx.x;
    const int k0 = kstep * BK;
    const int rbase = t.mt * BM;
#pragma unroll
    for (int it = 0; it < (BM * BK) / NT; ++it) {
      const int idx = tid + it * NT;
      const int r = idx / BK, c = idx % BK;
      const bool ok = (rbase + r < t.rows) && (k0 + c < a.n);
      const double* src = ok ? a.X + (long long)(t.row0 + rbase + r) * a.ldx + k0 + c : a.X;
      cp_async8(As + r * LDA + c, src, ok);
    }
    // flat columns: GEMM column j of the parent is (key, c) = divmod(j, rest),
    // so a tile spans several keys when a key's block has few columns (small b)
    const long long n0 = (long long)t.nt * BN;
    const long long ncols = a.keys_out * a.rest;
    const double* tin_call = a.Tin + (long long)t.in_call * a.keys_in * a.blk_in;
#pragma unroll 1
    for (int it = 0; it < (BK * BN) / NT; ++it) {
      const int idx = tid + it * NT;
      const int r = idx / BN, col = idx % BN;
      const int i = k0 + r;
      const long long j = n0 + col;
      const bool ok = (i < a.n) && (j < ncols);
      const double* src = a.X;
      if (ok) {
        const long long key = j / a.rest;
        const int cg = (int)(j - key * a.rest);
        const int ib = i / a.bA, e = i - ib * a.bA;
        const int2 nb = __ldg(a.nbr + key * a.nbar + ib);
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

  static __device__ __forceinline__ void epilogue(const LevelArgs& a, const TileInfo& t,
                                                  double (&acc)[FM][FN][2]) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wm = warp / WN, wn = warp % WN;
    const int jb0 = t.row0 / a.bC;
    const long long tstride = (long long)a.bAk * a.bC;
    const long long ncols = a.keys_out * a.rest;
#pragma unroll
    for (int fm = 0; fm < FM; ++fm) {
      const int r = t.mt * BM + wm * WTM + fm * 8 + (lane >> 2);
      if (r >= t.rows) continue;
      const int xrow = t.row0 + r;
      const int jb = xrow / a.bC, c = xrow - jb * a.bC;
      const int call = __ldg(a.child_call + t.child_off + (jb - jb0));
      double* base = (a.call_out && a.call_out[call] ? const_cast<double*>(a.call_out[call])
                                                     : a.Tout + (long long)call * a.keys_out * a.blk_out) +
                     (long long)a.bAk * c;
#pragma unroll
      for (int fn = 0; fn < FN; ++fn) {
        const long long col = (long long)t.nt * BN + wn * WTN + fn * 8 + 2 * (lane & 3);
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const long long j = col + q;
          if (j < ncols) {  // flat column -> (key, column of the key's block)
            const long long key = j / a.rest;
            const int cq = (int)(j - key * a.rest);
            const int tt = cq / a.bAk, af = cq - tt * a.bAk;
            base[key * a.blk_out + af + tstride * tt] = acc[fm][fn][q];
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
    ColInfo ci;
    if constexpr (INS) col_info(a, ld, ci);
    double acc[FM][FN][2];
#pragma unroll
    for (int fm = 0; fm < FM; ++fm)
#pragma unroll
      for (int fn = 0; fn < FN; ++fn) acc[fm][fn][0] = acc[fm][fn][1] = 0.0;
    auto advance_load = [&]() {
      ++ld_step;
      if (++ld_k == ksteps) {
        ld_k = 0;
        if (ld_step < total_steps) {
          ld = decode_item(a, ld.item + gridDim.x, BM);
          if constexpr (INS) col_info(a, ld, ci);
        }
      }
    };
    auto load = [&](double* As_, double* Bs_) {
      if constexpr (INS) load_stage_ins(a, ld, ci, ld_k, As_, Bs_);
      else load_stage(a, ld, ld_k, As_, Bs_);
    };
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
      if (ld_step < total_steps) {
        load(As + s * A_STAGE, Bs + s * B_STAGE);
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
        load(As + slot * A_STAGE, Bs + slot * B_STAGE);
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
