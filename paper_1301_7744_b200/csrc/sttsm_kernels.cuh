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
  const int4* items;        // per work item {parent, key, n-tile, m-tile}
  const int* child_call;    // output call index of (parent child_off + jb - row0/b_c)
  const int2* nbr;          // [keys_out * nbar] {rank in T(k+1) keys, code}
  unsigned* counter;        // dynamic work queue (zeroed before the launch) or null = static stride
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
// div/mod and zero-filled bounds; correctness path for small/odd problems.
// ---------------------------------------------------------------------------
template <int BM_, int BN_, int BK_, int WM, int WN, int STAGES>
struct GenericLevelKernel {
  static constexpr int BM = BM_, BN = BN_, BK = BK_;
  static constexpr int NT = WM * WN * 32;
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
    const int n0 = t.nt * BN;
    const int2* nrow = a.nbr + (long long)t.key * a.nbar;
    const double* tin_call = a.Tin + (long long)t.in_call * a.keys_in * a.blk_in;
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

// ---------------------------------------------------------------------------
// Fast kernel: power-of-two b_a = BA (compile time) and b_c, reuse=True
// (insertion redirection).  Per stage (BK reduction rows) the B tile is
// G = BK/RG row groups, one stored block S_ib each.  The element (e, col) of
// the logical block sits at
//     off = insert_bits(col, at = p*lg(BA), value = e, width = lg(BA))
// inside S_ib (the contracted digit is spliced into the column index at the
// insertion position p).  Groups with p == 0 are e-contiguous in HBM and are
// staged column-major ([col][e], XOR-swizzled quads); the others are
// column-contiguous and staged row-major ([e][col], padded stride); both with
// 16-byte cp.async and bank-conflict-free DMMA fragment loads.
// ---------------------------------------------------------------------------
template <int BM_, int BN_, int BK_, int WM, int WN, int STAGES, int BA>
struct FastLevelKernel {
  static constexpr int BM = BM_, BN = BN_, BK = BK_;
  static constexpr int NT = WM * WN * 32;
  static constexpr int WTM = BM / WM, WTN = BN / WN;
  static constexpr int FM = WTM / 8, FN = WTN / 8;
  static constexpr int LBA = (BA == 2) ? 1 : (BA == 4) ? 2 : (BA == 8) ? 3 : (BA == 16) ? 4 : (BA == 32) ? 5 : 6;
  static constexpr int RG = BA < BK ? BA : BK;  // rows per group (one ib)
  static constexpr int G = BK / RG;             // groups per stage
  static constexpr int LDA = BK + 4;
  static constexpr int LDR = BN + 4;            // row-major group stride ([e][col])
  static constexpr int GR_SIZE = RG * LDR;      // >= BN*RG, the col-major footprint
  // col-major swizzle: element (col, e) at col*RG + (e ^ swz(col)); spreads the
  // four columns a fragment touches over distinct 4-double bank quads.
  static constexpr int SW_SHIFT = RG >= 16 ? 0 : 1;
  static constexpr int SW_MASK = RG >= 16 ? 3 : (RG == 8 ? 1 : 0);
  static __device__ __forceinline__ int swz(int col) { return ((col >> SW_SHIFT) & SW_MASK) << 2; }
  static constexpr int A_STAGE = BM * LDA, B_STAGE = G * GR_SIZE;
  static constexpr size_t SMEM_BYTES = (size_t)STAGES * (A_STAGE + B_STAGE) * sizeof(double) +
                                       STAGES * G * sizeof(int) + STAGES * 2 * sizeof(int4);
  static_assert(WTM % 8 == 0 && WTN % 8 == 0, "tile shape");
  static_assert((BM * BK / 2) % NT == 0 && (BK * BN / 2) % NT == 0 && (RG * BN / 2) % 32 == 0,
                "loader balance");
  static_assert((1 << LBA) == BA && RG % 4 == 0, "BA must be a power of two >= 4");
  static_assert(BK == 16 || BK == 32, "stage depth");
  static_assert(SMEM_BYTES <= 232448, "shared memory per CTA");

  // ---- operand staging ---------------------------------------------------------
  // One stage = NA cp.async.cg of the X tile plus NB of the B tile per thread.
  // They are issued in KP slices, one after each k4 step of the DMMA loop of
  // the previous stage, so address arithmetic overlaps the tensor pipe.
  static constexpr int NA = (BM * BK / 2) / NT;
  static constexpr int GP = RG * BN / 2;          // 16-byte pairs per group
  static constexpr int NB = (BK * BN / 2) / NT;    // B pairs per thread per stage
  static constexpr int NU = NA + NB;
  static constexpr int KP = BK / 4;              // k4 steps per stage = slices

  static __device__ __forceinline__ void load_unit(const LevelArgs& a, const TileInfo& t, int kstep,
                                                   double* As, double* Bs, int* modes, int u) {
    const int tid = threadIdx.x;
    const int k0 = kstep * BK;
    if (u < NA) {
      const int idx = tid + u * NT;
      const int r = idx / (BK / 2), c = (idx % (BK / 2)) * 2;
      const int rr = t.mt * BM + r;
      const bool ok = (rr < t.rows) && (k0 + c < a.n);
      const double* src = ok ? a.X + (long long)(t.row0 + rr) * a.ldx + k0 + c : a.X;
      cp_async16(As + r * LDA + c, src, ok);
      return;
    }
    const int qs = tid + (u - NA) * NT;  // pair index within the stage
    const int g = qs / GP, q = qs % GP;  // group (warp-uniform: GP >= 32), pair within group
    const int i0 = k0 + g * RG;  // first reduction row of the group
    const bool grp_ok = i0 < a.n;
    const int2 nb = __ldg(a.nbr + (long long)t.key * a.nbar + (grp_ok ? (i0 >> LBA) : 0));
    const int pos = code_p(nb.y);
    const double* base = a.Tin + ((long long)t.in_call * a.keys_in + nb.x) * a.blk_in;
    const int e0 = i0 & (BA - 1);
    const int n0 = t.nt * BN;
    double* dst = Bs + g * GR_SIZE;
    if (q == 0) modes[g] = pos == 0;
    if (pos == 0) {
      // e-contiguous: pairs along e, staged [col][e ^ swz]
      const int e2 = (q % (RG / 2)) * 2, col = q / (RG / 2);
      const int cg = n0 + col;
      const bool ok = grp_ok && cg < a.rest;
      const double* src = ok ? base + (e0 + e2) + ((long long)cg << LBA) : a.X;
      cp_async16(dst + col * RG + (e2 ^ swz(col)), src, ok);
    } else {
      // column-contiguous: pairs along col, staged [e][col]
      const int sh = pos * LBA;
      const int c2 = (q % (BN / 2)) * 2, e = q / (BN / 2);
      const int cg = n0 + c2;
      const bool ok = grp_ok && cg < a.rest;
      const long long off = (long long)(cg & ((1 << sh) - 1)) + ((long long)(cg >> sh) << (sh + LBA)) +
                            ((long long)(e0 + e) << sh);
      const double* src = ok ? base + off : a.X;
      cp_async16(dst + e * LDR + c2, src, ok);
    }
  }

  // slice `part` of a stage's loads (compile-time after unrolling)
  static __device__ __forceinline__ void load_part(const LevelArgs& a, const TileInfo& t, int kstep,
                                                   double* As, double* Bs, int* modes, bool on, int part) {
    if (!on) return;
#pragma unroll
    for (int u = (part * NU) / KP; u < ((part + 1) * NU) / KP; ++u) load_unit(a, t, kstep, As, Bs, modes, u);
  }

  static __device__ __forceinline__ void load_stage(const LevelArgs& a, const TileInfo& t, int kstep,
                                                    double* As, double* Bs, int* modes) {
#pragma unroll
    for (int u = 0; u < NU; ++u) load_unit(a, t, kstep, As, Bs, modes, u);
  }

  // DMMA over one staged slice, with the next stage's loads interleaved.
  static __device__ __forceinline__ void compute_stage(const double* As, const double* Bs, const int* modes,
                                                       double (&acc)[FM][FN][2], const LevelArgs& a,
                                                       const TileInfo& lt, int lk, double* lAs, double* lBs,
                                                       int* lmodes, bool lon) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wm = warp / WN, wn = warp % WN;
    const double* ap = As + (wm * WTM + (lane >> 2)) * LDA + (lane & 3);
    const int colw = wn * WTN + (lane >> 2);
    const int sw = swz(colw);  // same for colw + 8*fn
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const bool cm = modes[g] != 0;
      // element (e, col) of group g: cm ? col*RG + (e ^ swz(col)) : e*LDR + col
      const double* bp = Bs + g * GR_SIZE + (cm ? colw * RG + (lane & 3) : (lane & 3) * LDR + colw);
      const int sn = cm ? 8 * RG : 8;      // next n fragment
#pragma unroll
      for (int kk = 0; kk < RG / 4; ++kk) {
        const int ko = cm ? ((kk * 4) ^ sw) : kk * 4 * LDR;
        double af[FM], bf[FN];
#pragma unroll
        for (int fm = 0; fm < FM; ++fm) af[fm] = ap[fm * 8 * LDA + (g * RG + kk * 4)];
#pragma unroll
        for (int fn = 0; fn < FN; ++fn) bf[fn] = bp[ko + fn * sn];
#pragma unroll
        for (int fm = 0; fm < FM; ++fm)
#pragma unroll
          for (int fn = 0; fn < FN; ++fn) dmma(acc[fm][fn][0], acc[fm][fn][1], af[fm], bf[fn]);
        load_part(a, lt, lk, lAs, lBs, lmodes, lon, g * (RG / 4) + kk);
      }
    }
  }

  static __device__ __forceinline__ void epilogue(const LevelArgs& a, const TileInfo& t,
                                                  double (&acc)[FM][FN][2]) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wm = warp / WN, wn = warp % WN;
    const int jb0 = t.row0 / a.bC;
    const int kl = a.k * LBA;
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
        if (col >= a.rest) continue;
        if (a.bAk >= 2) {
          const long long off = (col & (a.bAk - 1)) + tstride * (col >> kl);
          *reinterpret_cast<double2*>(base + off) = make_double2(acc[fm][fn][0], acc[fm][fn][1]);
        } else {  // level 0: columns are the tail modes, stride b_c
          base[tstride * col] = acc[fm][fn][0];
          base[tstride * (col + 1)] = acc[fm][fn][1];
        }
      }
    }
  }

  static __device__ void run(const LevelArgs& a) {
    extern __shared__ __align__(16) double smem[];
    double* As = smem;
    double* Bs = smem + STAGES * A_STAGE;
    int4* tiles = reinterpret_cast<int4*>(Bs + STAGES * B_STAGE);  // per slot: tile of the staged data
    int* modes = reinterpret_cast<int*>(tiles + 2 * STAGES);
    const long long first = blockIdx.x;
    if (first >= a.total_items) return;
    const long long my_items = (a.total_items - 1 - first) / gridDim.x + 1;
    const int ksteps = (a.n + BK - 1) / BK;
    const long long total_steps = my_items * ksteps;
    TileInfo ld = decode_item(a, first, BM);
    int ld_k = 0;
    long long ld_step = 0;
    double acc[FM][FN][2];
#pragma unroll
    for (int fm = 0; fm < FM; ++fm)
#pragma unroll
      for (int fn = 0; fn < FN; ++fn) acc[fm][fn][0] = acc[fm][fn][1] = 0.0;
    auto note_tile = [&](int slot) {  // remember which tile a slot belongs to (for the epilogue)
      if (threadIdx.x == 0) {
        tiles[2 * slot] = make_int4(ld.key, ld.nt, ld.mt, (int)(ld.item & 0x7fffffff));
        tiles[2 * slot + 1] = make_int4(ld.in_call, ld.row0, ld.rows, ld.child_off);
      }
    };
    auto advance_ld = [&]() {
      ++ld_step;
      if (++ld_k == ksteps) {
        ld_k = 0;
        if (ld_step < total_steps) ld = decode_item(a, ld.item + gridDim.x, BM);
      }
    };
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
      if (ld_step < total_steps) {
        note_tile(s);
        load_stage(a, ld, ld_k, As + s * A_STAGE, Bs + s * B_STAGE, modes + s * G);
        advance_ld();
      }
      cp_async_commit();
    }
    int cp_k = 0;
    for (long long step = 0; step < total_steps; ++step) {
      cp_async_wait<STAGES - 2>();
      __syncthreads();
      const bool lon = ld_step < total_steps;
      const int lslot = (int)(ld_step % STAGES);
      if (lon) note_tile(lslot);
      const int slot = (int)(step % STAGES);
      compute_stage(As + slot * A_STAGE, Bs + slot * B_STAGE, modes + slot * G, acc, a, ld, ld_k,
                    As + lslot * A_STAGE, Bs + lslot * B_STAGE, modes + lslot * G, lon);
      cp_async_commit();
      if (lon) advance_ld();
      if (++cp_k == ksteps) {
        cp_k = 0;
        const int4 t0 = tiles[2 * slot], t1 = tiles[2 * slot + 1];
        TileInfo cp;
        cp.key = t0.x; cp.nt = t0.y; cp.mt = t0.z; cp.item = t0.w;
        cp.in_call = t1.x; cp.row0 = t1.y; cp.rows = t1.z; cp.child_off = t1.w;
        epilogue(a, cp, acc);
#pragma unroll
        for (int fm = 0; fm < FM; ++fm)
#pragma unroll
          for (int fn = 0; fn < FN; ++fn) acc[fm][fn][0] = acc[fm][fn][1] = 0.0;
      }
    }
    cp_async_wait<0>();
  }
};

}  // namespace bcss
