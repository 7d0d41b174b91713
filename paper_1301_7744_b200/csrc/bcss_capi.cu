// C ABI of the B200-native BCSS sttsm (declared in include/bcss_sttsm.h).
//
// Host side: problem validation (change_of_basis.py:54-63, 259-266), the
// level/work-list plan that replaces the reference's depth-first `descend`
// (change_of_basis.py:269-283) by breadth-first levels over "waves" of
// top-level units, workspace management and kernel launches.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/bcss_sttsm.h"
#include "combinatorics.hpp"
#include "kernel_table.cuh"

namespace {

thread_local std::string g_last_error;

int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

#define CUDA_TRY(expr)                                                                   \
  do {                                                                                   \
    cudaError_t _e = (expr);                                                             \
    if (_e != cudaSuccess)                                                               \
      return fail(BCSS_ERR_CUDA, "%s failed: %s", #expr, cudaGetErrorString(_e));        \
  } while (0)

bool is_pow2(int64_t v) { return v > 0 && (v & (v - 1)) == 0; }
int ilog2(int64_t v) { int r = 0; while ((int64_t(1) << r) < v) ++r; return r; }
int64_t ipow(int64_t b, int e) { int64_t r = 1; while (e-- > 0) r *= b; return r; }

// ---- kernel configurations ----------------------------------------------------
using bcss::KernelCfg;
using bcss::N_SHAPES;

// The fast tile shapes' BM (bcss::BCSS_FAST_SHAPES order).
int shape_bm(int shape) { return bcss::kFast32[shape].BM; }

const KernelCfg& kernel_cfg(int cfg) {
  if (cfg == 0) return bcss::kGeneric;
  const int shape = (cfg - 1) / 4, ba = (cfg - 1) % 4;
  const KernelCfg* t = ba == 0 ? bcss::kFast4 : ba == 1 ? bcss::kFast8 : ba == 2 ? bcss::kFast16 : bcss::kFast32;
  return t[shape];
}
constexpr int N_CFGS = 1 + 4 * N_SHAPES;
enum { CFG_GENERIC = 0 };
// fast configuration of tile shape `shape` for power-of-two b_a in {4, 8, 16, 32}, else -1
int fast_cfg(int64_t bA, int shape) {
  int i;
  switch (bA) {
    case 4: i = 0; break;
    case 8: i = 1; break;
    case 16: i = 2; break;
    case 32: i = 3; break;
    default: return -1;
  }
  return 1 + shape * 4 + i;
}

// Relative DMMA efficiency of each tile shape (larger tiles reuse operands
// more); the plan picks, per parent, the shape minimizing padded work / eff.
// BCSS_SHAPE_EFF="e128,e64,e32" overrides, BCSS_FORCE_SHAPE=i forces one.
struct ShapePolicy {
  // Measured full-tile FP64 TFLOP/s of each shape (BCSS_FAST_SHAPES order) per
  // b_a in {4, 8, 16, 32} on B200 (tools/calibrate_shapes.py: top level of configs 2/3/4, padding
  // corrected); b_a = 4 borrows the b_a = 8 row.
  double eff[4][N_SHAPES] = {
      {32.52, 29.87, 29.28, 31.85, 31.28, 28.90, 19.83, 31.09, 31.91, 29.94},
      {32.52, 29.87, 29.28, 31.85, 31.28, 28.90, 19.83, 31.09, 31.91, 29.94},
      {32.80, 31.61, 30.58, 32.51, 31.64, 30.48, 23.06, 31.47, 32.96, 31.15},
      {33.11, 32.26, 31.74, 32.62, 32.04, 30.95, 21.70, 31.99, 33.08, 31.32},
  };
  int force = -1;
  ShapePolicy() {
    // BCSS_SHAPE_EFF="e0,e1,...,e5" overrides every b_a's row; BCSS_FORCE_SHAPE=i forces one
    if (const char* e = getenv("BCSS_SHAPE_EFF")) {
      double v[N_SHAPES];
      int got = 0;
      const char* q = e;
      while (got < N_SHAPES) {
        int used = 0;
        if (sscanf(q, "%lf%n", &v[got], &used) != 1) break;
        ++got;
        q += used;
        if (*q == ',') ++q;
      }
      if (got == N_SHAPES)
        for (auto& row : eff)
          for (int i = 0; i < N_SHAPES; ++i) row[i] = v[i];
    }
    if (const char* f = getenv("BCSS_FORCE_SHAPE")) force = atoi(f);
  }
  // shape minimizing padded rows / throughput for a parent with `rows` rows
  int pick(int rows, int64_t bA) const {
    if (force >= 0 && force < N_SHAPES) return force;
    const int bi = bA <= 4 ? 0 : bA == 8 ? 1 : bA == 16 ? 2 : 3;
    int best = 0;
    double bt = 1e300;
    for (int sidx = 0; sidx < N_SHAPES; ++sidx) {
      if (eff[bi][sidx] <= 0) continue;
      const int bm = shape_bm(sidx);
      const double t = (double)((rows + bm - 1) / bm * bm) / eff[bi][sidx];
      if (t < bt - 1e-9) { bt = t; best = sidx; }
    }
    return best;
  }
  // Row decomposition of a parent with `rows` rows into contiguous pieces, one
  // tile shape each (largest tiles first), minimizing padded rows / throughput
  // (knapsack over row counts): e.g. 160 rows -> 128 + 32.
  std::vector<std::pair<int, int>> split(int rows, int64_t bA) const {
    if (force >= 0 && force < N_SHAPES) return {{force, rows}};
    const int bi = bA <= 4 ? 0 : bA == 8 ? 1 : bA == 16 ? 2 : 3;
    std::vector<double> cost(rows + 1, 1e300);
    std::vector<int> choice(rows + 1, -1);
    cost[0] = 0;
    for (int r = 1; r <= rows; ++r)
      for (int sidx = 0; sidx < N_SHAPES; ++sidx) {
        if (eff[bi][sidx] <= 0) continue;
        const int bm = shape_bm(sidx);
        const double c = cost[std::max(0, r - bm)] + bm / eff[bi][sidx];
        if (c < cost[r] - 1e-12) { cost[r] = c; choice[r] = sidx; }
      }
    std::map<int, int, std::greater<int>> tiles_by_bm;  // bm -> (shape, count) via two maps
    std::map<int, int> shape_of_bm, count_of_bm;
    for (int r = rows; r > 0;) {
      const int sidx = choice[r];
      const int bm = shape_bm(sidx);
      shape_of_bm[bm] = sidx;
      count_of_bm[bm] += 1;
      r = std::max(0, r - bm);
    }
    std::vector<std::pair<int, int>> out;
    int left = rows;
    for (auto it = count_of_bm.rbegin(); it != count_of_bm.rend(); ++it) {
      const int take = std::min(left, it->first * it->second);
      if (take > 0) out.push_back({shape_of_bm[it->first], take});
      left -= take;
    }
    return out;
  }
};

// Register-resident DMMA loop: 16 independent m8n8k4 accumulators per warp.
__global__ void dmma_peak_kernel(double* sink, int iters) {
  const double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[16][2];
#pragma unroll
  for (int i = 0; i < 16; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) bcss::dmma(c[i][0], c[i][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) sink[threadIdx.x] = s;
}

}  // namespace

// ---- plan ----------------------------------------------------------------------
// One kernel launch: the parents of a level that share a tile configuration.
struct LaunchHost {
  int cfg = 0;
  int n_tiles = 0;
  uint64_t flops = 0;
  std::vector<int4> parents;       // {in_call, row0, rows, child_off}
  std::vector<long long> item_off; // prefix sums of work items, size parents+1
  std::vector<int4> items;         // per work item {parent, key, n-tile, m-tile}
  size_t off_parents = 0, off_items = 0;  // into the device table buffer
};

struct LevelHost {
  int k = 0;
  int64_t keys_out = 0, keys_in = 0, blk_out = 0, blk_in = 0, rest = 0, bAk = 0;
  int64_t n_calls = 0;
  uint64_t flops = 0;
  std::vector<LaunchHost> launches;
  std::vector<int> child_call;
  std::vector<int32_t> suffixes;  // n_calls x (m-k)
  size_t off_child = 0;
};

struct WaveHost {
  std::vector<int> units;          // top-level units whose lower levels this wave computes
  std::vector<LevelHost> levels;   // k = m-1 (if top_units is non-empty) down to 0
  std::vector<size_t> level_off;   // byte offset of T(k)'s region in the workspace
  std::vector<int> top_units;      // units of the top level computed in this wave (may be a superset)
  std::vector<int> top_call;       // per unit of `units`: its call index in the T(m-1) buffer
};

struct bcss_plan {
  int m = 0;
  int64_t n = 0, p = 0, bA = 0, bC = 0, nbar = 0, pbar = 0;
  bool reuse = true;
  std::vector<int> units;
  bool units_set = false;
  size_t ws_limit = 0;
  bool keep_temps = false;

  bool built = false;
  std::vector<WaveHost> waves;
  std::vector<std::vector<int2>> nbr;  // per k
  std::vector<size_t> nbr_off;         // per k, into the table buffer
  size_t ws_bytes = 0;
  uint64_t flops = 0;
  int64_t c_blocks = 0;

  int device = -1;
  void* d_tables = nullptr;
  size_t tables_bytes = 0;
  void* d_ws = nullptr;
  size_t ws_capacity = 0;
  bool own_ws = false;
  double *hA = nullptr, *hX = nullptr, *hC = nullptr;  // device buffers for run_host
  size_t hA_bytes = 0, hX_bytes = 0, hC_bytes = 0;
  cudaStream_t host_stream = nullptr;
  int64_t last_launches = 0;
  bool timing = false;
  bool dynamic = false;             // dynamic work queues (kernels use the static stride today)
  bool concurrent = true;           // concurrent launches per level (BCSS_SERIAL_LAUNCH=1 disables)
  int pipeline_waves = 0;           // run_host: overlap H2D / compute / D2H over this many waves
  bool top_first = false;           // first wave computes T(m-1) for all units
  int start_level = 0;              // 0 = from A; else compute below caller-provided T(start_level)
  std::vector<int32_t> start_suffixes;  // their calls (m - start_level entries each)
  int stop_level = 0;               // last level computed; its T goes to the caller's output buffer
  cudaStream_t copy_in = nullptr, copy_out = nullptr, copy_out2 = nullptr;
  cudaEvent_t out2_done = nullptr;
  std::vector<cudaEvent_t> chunk_ev;  // A chunk (first block index a) landed
  std::vector<cudaEvent_t> wave_ev;   // a wave's C blocks are final
  unsigned* d_counters = nullptr;
  size_t counters_n = 0;
  std::vector<cudaStream_t> side;   // concurrent launches of one level
  std::vector<cudaEvent_t> join;
  cudaEvent_t fork = nullptr;
  std::vector<cudaEvent_t> events;  // 2 per timed level
  std::vector<int> launch_level;
  std::vector<uint64_t> launch_flops;
  cudaStream_t timed_stream = nullptr;
};

namespace {

int64_t keys_at(const bcss_plan& P, int k) {
  if (k == 0) return 1;
  if (k == P.m) return bcss::simplex_count(P.nbar, P.m);  // A is always BCSS
  return P.reuse ? bcss::simplex_count(P.nbar, k) : ipow(P.nbar, k);
}
int64_t blk_at(const bcss_plan& P, int k) { return ipow(P.bA, k) * ipow(P.bC, P.m - k); }

// Neighbour table of level k: for every output key K and every ib, the rank of
// the stored block of T(k+1) that holds the logical block (K, ib) and the
// redirection (stored position of each logical mode).  Reuse: K sorted,
// stored = sorted(K u {ib}) with the canonicalize mapping (insertion).
// No reuse: K runs over all k-tuples; T(k+1) below the top is itself a dense
// block table (identity mapping), the top level redirects through A's BCSS.
void build_nbr(bcss_plan& P, int k, std::vector<int2>& out) {
  const int64_t nkeys = keys_at(P, k);
  out.assign((size_t)(nkeys * P.nbar), int2{0, 0});
  std::vector<int32_t> key(k), idx(k + 1), canon(k + 1), map(k + 1);
  std::vector<int64_t> canon64(k + 1);
  for (int64_t kr = 0; kr < nkeys; ++kr) {
    if (k > 0) {
      if (P.reuse) {
        std::vector<int64_t> tmp(k);
        bcss::hypertriangle_unrank(kr, k, P.nbar, tmp.data());
        for (int d = 0; d < k; ++d) key[d] = (int32_t)tmp[d];
      } else {
        int64_t r = kr;
        for (int d = k - 1; d >= 0; --d) { key[d] = (int32_t)(r % P.nbar); r /= P.nbar; }
      }
    }
    for (int64_t ib = 0; ib < P.nbar; ++ib) {
      for (int d = 0; d < k; ++d) idx[d] = key[d];
      idx[k] = (int32_t)ib;
      int64_t rank;
      int pos;
      if (P.reuse || k + 1 == P.m) {
        bcss::canonical_mapping(idx.data(), k + 1, canon.data(), map.data());
        for (int d = 0; d <= k; ++d) canon64[d] = canon[d];
        rank = bcss::hypertriangle_rank(canon64.data(), k + 1, P.nbar);
        pos = map[k];
      } else {
        rank = kr * P.nbar + ib;
        for (int d = 0; d <= k; ++d) map[d] = d;
        pos = k;
      }
      int code = pos;
      for (int d = 0; d <= k; ++d) code |= map[d] << (4 + 3 * d);
      out[(size_t)(kr * P.nbar + ib)] = int2{(int)rank, code};
    }
  }
}

// Calls (suffixes) of level k generated by the units in `units`:
// number of nondecreasing (m-1-k)-tuples over [0, u] per unit u.
int64_t calls_for(const bcss_plan& P, const std::vector<int>& units, int k) {
  int64_t c = 0;
  for (int u : units) c += (P.m - 1 - k == 0) ? 1 : bcss::simplex_count(u + 1, P.m - 1 - k);
  return c;
}

std::vector<size_t> level_bytes(const bcss_plan& P, const std::vector<int>& units) {
  std::vector<size_t> b(P.m, 0);
  for (int k = 1; k < P.m; ++k)
    b[k] = (size_t)calls_for(P, units, k) * keys_at(P, k) * blk_at(P, k) * sizeof(double);
  return b;
}

size_t peak_for(const bcss_plan& P, const std::vector<int>& units) {
  const auto b = level_bytes(P, units);
  if (P.keep_temps) { size_t s = 0; for (auto v : b) s += v; return s; }
  size_t r[2] = {0, 0};
  for (int k = 1; k < P.m; ++k) r[(P.m - 1 - k) % 2] = std::max(r[(P.m - 1 - k) % 2], b[k]);
  return r[0] + r[1];
}

void build_wave_levels(bcss_plan& P, WaveHost& W) {
  const bool fast = P.reuse && is_pow2(P.bC) && fast_cfg(P.bA, 0) >= 0;
  static const ShapePolicy policy;
  W.levels.clear();
  std::vector<int32_t> prev_suffix;  // suffixes of level k+1 calls
  std::vector<int> prev_call;        // their call index in the T(k+1) buffer
  int64_t prev_calls = 0;
  const bool has_top = !W.top_units.empty();
  int k_first = has_top ? P.m - 1 : P.m - 2;
  if (P.start_level > 0) {  // start below caller-provided temporaries T(start_level)
    k_first = P.start_level - 1;
    prev_suffix = P.start_suffixes;
    prev_calls = (int64_t)(P.start_suffixes.size() / (P.m - P.start_level));
    for (int64_t c = 0; c < prev_calls; ++c) prev_call.push_back((int)c);
  } else if (!has_top) {  // the top level was computed by an earlier wave
    for (size_t i = 0; i < W.units.size(); ++i) {
      prev_suffix.push_back(W.units[i]);
      prev_call.push_back(W.top_call[i]);
    }
    prev_calls = (int64_t)W.units.size();
  }
  for (int k = k_first; k >= P.stop_level; --k) {
    LevelHost L;
    L.k = k;
    L.keys_out = keys_at(P, k);
    L.keys_in = keys_at(P, k + 1);
    L.blk_out = blk_at(P, k);
    L.blk_in = blk_at(P, k + 1);
    L.bAk = ipow(P.bA, k);
    L.rest = L.bAk * ipow(P.bC, P.m - 1 - k);
    const int sl = P.m - k;  // suffix length of this level's calls
    std::vector<int4> parents;
    if (k == P.m - 1 && P.start_level == 0) {
      const std::vector<int>& tu = W.top_units;
      for (size_t i = 0; i < tu.size(); ++i) {
        L.suffixes.push_back(tu[i]);
        L.child_call.push_back((int)i);
      }
      size_t s = 0;
      while (s < tu.size()) {
        size_t e = s + 1;
        while (e < tu.size() && tu[e] == tu[e - 1] + 1) ++e;
        parents.push_back(int4{0, (int)(tu[s] * P.bC), (int)((e - s) * P.bC), (int)s});
        s = e;
      }
      L.n_calls = (int64_t)tu.size();
      // the lower levels of this wave start from its own units
      prev_call.assign(W.top_call.begin(), W.top_call.end());
    } else {
      int64_t running = 0;
      std::vector<int64_t> full(P.m);
      for (int64_t c = 0; c < prev_calls; ++c) {
        const int32_t* sp = &prev_suffix[(size_t)(c * (sl - 1))];
        const int J = sp[0];
        parents.push_back(int4{prev_call[(size_t)c], 0, (int)((J + 1) * P.bC), (int)running});
        for (int jb = 0; jb <= J; ++jb) {
          L.suffixes.push_back(jb);
          for (int q = 0; q < sl - 1; ++q) L.suffixes.push_back(sp[q]);
          if (k == 0) {
            full[0] = jb;
            for (int q = 0; q < sl - 1; ++q) full[q + 1] = sp[q];
            L.child_call.push_back((int)bcss::hypertriangle_rank(full.data(), P.m, P.pbar));
          } else {
            L.child_call.push_back((int)running);
          }
          ++running;
        }
      }
      L.n_calls = running;
    }
    // group parents into launches by tile configuration
    std::map<int, LaunchHost> by_cfg;
    for (const int4& whole : parents) {
      // a parent's rows may be split into pieces of different tile shapes; a
      // piece is a parent with a later row0 (its child index follows from
      // child_off + (jb - row0/b_c) in the epilogue)
      std::vector<std::pair<int, int>> pieces;
      if (fast) pieces = policy.split(whole.z, P.bA);
      else pieces = {{-1, whole.z}};
      int r0 = 0;
      for (const auto& pc : pieces) {
        const int cfg = fast ? fast_cfg(P.bA, pc.first) : CFG_GENERIC;
        int4 par = whole;
        par.y = whole.y + r0;
        par.z = pc.second;
        par.w = whole.w + r0 / (int)P.bC;
        r0 += pc.second;
        LaunchHost& X = by_cfg[cfg];
        const KernelCfg& C = kernel_cfg(cfg);
        if (X.parents.empty()) {
          X.cfg = cfg;
          X.n_tiles = (int)((L.rest + C.BN - 1) / C.BN);
          X.item_off.push_back(0);
        }
        X.parents.push_back(par);
        X.item_off.push_back(X.item_off.back() +
                             (long long)L.keys_out * X.n_tiles * ((par.z + C.BM - 1) / C.BM));
        X.flops += (uint64_t)2 * par.z * P.n * L.keys_out * L.rest;
      }
    }
    for (auto& kv : by_cfg) {
      // flat work list: parent-major, then key, n-tile, m-tile (adjacent CTAs
      // share the B tile of one (key, n-tile))
      LaunchHost& X = kv.second;
      const int BM = kernel_cfg(X.cfg).BM;
      X.items.reserve((size_t)X.item_off.back());
      for (size_t pi = 0; pi < X.parents.size(); ++pi) {
        const int mtiles = (X.parents[pi].z + BM - 1) / BM;
        for (int64_t key = 0; key < L.keys_out; ++key)
          for (int nt = 0; nt < X.n_tiles; ++nt)
            for (int mt = 0; mt < mtiles; ++mt) X.items.push_back(int4{(int)pi, (int)key, nt, mt});
      }
      L.flops += kv.second.flops;
      L.launches.push_back(std::move(kv.second));
    }
    if (k == P.m - 1 && P.start_level == 0) {
      prev_suffix.clear();
      for (int u : W.units) prev_suffix.push_back(u);
      prev_calls = (int64_t)W.units.size();
    } else {
      prev_suffix = L.suffixes;
      prev_call.resize((size_t)L.n_calls);
      for (int64_t c = 0; c < L.n_calls; ++c) prev_call[(size_t)c] = (int)c;
      prev_calls = L.n_calls;
    }
    W.levels.push_back(std::move(L));
  }
}

// Exact flops of top-level subtree u: sum over levels of (calls of the
// subtree at level k) x 2*b_c*n*keys(k)*rest(k).
double unit_cost(const bcss_plan& P, int u) {
  double f = 0;
  for (int k = P.m - 1; k >= 0; --k)
    f += (double)calls_for(P, {u}, k) * 2.0 * P.bC * P.n * keys_at(P, k) *
         (double)(ipow(P.bA, k) * ipow(P.bC, P.m - 1 - k));
  return f;
}

int build_plan(bcss_plan& P) {
  if (P.built) return BCSS_OK;
  try {
    std::vector<int> units = P.units;
    if (!P.units_set)
      for (int u = 0; u < P.pbar; ++u) units.push_back(u);
    std::sort(units.begin(), units.end());
    units.erase(std::unique(units.begin(), units.end()), units.end());
    // pipeline groups: contiguous units with ~equal flops, largest units first
    // (run_host downloads one group's C while later groups compute, so the
    // last group - the one whose download is not overlapped - is the smallest)
    std::vector<std::vector<int>> groups;
    if (P.pipeline_waves > 1 && !P.keep_temps && units.size() > 1) {
      double tot = 0;
      for (int u : units) tot += unit_cost(P, u);
      const double target = tot / P.pipeline_waves;
      double acc = 0;
      groups.emplace_back();
      for (auto it = units.rbegin(); it != units.rend(); ++it) {
        const double c = unit_cost(P, *it);
        if (!groups.back().empty() && acc + c / 2 > target * groups.size() &&
            (int)groups.size() < P.pipeline_waves)
          groups.emplace_back();
        groups.back().push_back(*it);
        acc += c;
      }
      for (auto& g : groups) std::sort(g.begin(), g.end());
    } else {
      groups.push_back(units);
    }
    // waves: greedy groups of units whose live temporaries fit the limit
    P.waves.clear();
    for (const auto& grp : groups) {
      std::vector<int> cur;
      for (int u : grp) {
        std::vector<int> trial = cur;
        trial.push_back(u);
        if (!cur.empty() && !P.keep_temps && P.ws_limit > 0 && peak_for(P, trial) > P.ws_limit) {
          P.waves.push_back(WaveHost{cur, {}, {}, {}, {}});
          cur = {u};
        } else {
          cur = trial;
        }
      }
      if (!cur.empty()) P.waves.push_back(WaveHost{cur, {}, {}, {}, {}});
    }
    if (!P.keep_temps && P.ws_limit > 0) {
      for (auto& W : P.waves)
        if (peak_for(P, W.units) > P.ws_limit)
          return fail(BCSS_ERR_NOMEM, "one top-level unit needs %zu workspace bytes > limit %zu",
                      peak_for(P, W.units), P.ws_limit);
    }
    if (P.start_level > 0 || P.stop_level > 0) {
      // partial runs (multi-GPU exchange points): one wave, regions from the built levels
      P.waves.clear();
      P.waves.push_back(WaveHost{units, {}, {}, {}, {}});
      WaveHost& W = P.waves[0];
      if (P.start_level == 0) {
        W.top_units = units;
        for (size_t i = 0; i < units.size(); ++i) W.top_call.push_back((int)i);
      }
      build_wave_levels(P, W);
      auto al = [](size_t v) { return (v + 255) / 256 * 256; };
      size_t r[2] = {0, 0};
      const int k_first = W.levels.empty() ? 0 : W.levels.front().k;
      for (auto& L : W.levels)
        if (L.k > P.stop_level && L.k >= 1)
          r[(k_first - L.k) % 2] = std::max(r[(k_first - L.k) % 2],
                                            al((size_t)L.n_calls * L.keys_out * L.blk_out * sizeof(double)));
      W.level_off.assign(P.m + 1, 0);
      for (auto& L : W.levels)
        if (L.k > P.stop_level && L.k >= 1) W.level_off[L.k] = (k_first - L.k) % 2 == 0 ? 0 : r[0];
      P.ws_bytes = r[0] + r[1];
      P.top_first = false;
    } else {
    // Top level: with a pipeline, the first wave computes T(m-1) for every
    // unit (it overlaps the chunked upload of A) and later waves only run the
    // levels below; otherwise every wave computes its own units' top level.
    P.top_first = P.pipeline_waves > 1 && P.waves.size() > 1 && !P.keep_temps;
    {
      std::vector<int> all;
      for (auto& W : P.waves) all.insert(all.end(), W.units.begin(), W.units.end());
      std::sort(all.begin(), all.end());
      for (size_t wi = 0; wi < P.waves.size(); ++wi) {
        WaveHost& W = P.waves[wi];
        W.top_units = P.top_first ? (wi == 0 ? all : std::vector<int>{}) : W.units;
        const std::vector<int>& ref = P.top_first ? all : W.units;
        W.top_call.clear();
        for (int u : W.units)
          W.top_call.push_back((int)(std::lower_bound(ref.begin(), ref.end(), u) - ref.begin()));
      }
    }
    // Workspace layout per wave: keep_temps gives every level its own region;
    // otherwise levels alternate between two regions (T(k+1) is read while
    // T(k) is written); with top_first, T(m-1) of all units has its own
    // region and the lower levels alternate behind it.
    P.ws_bytes = 0;
    auto al = [](size_t v) { return (v + 255) / 256 * 256; };
    size_t top_bytes = 0;
    if (P.top_first) top_bytes = al(level_bytes(P, P.waves[0].top_units)[P.m - 1]);
    for (auto& W : P.waves) {
      auto b = level_bytes(P, W.units);
      W.level_off.assign(P.m + 1, 0);
      size_t end = 0;
      if (P.keep_temps) {
        for (int k = 1; k < P.m; ++k) { W.level_off[k] = end; end += al(b[k]); }
      } else if (P.top_first) {
        size_t r[2] = {0, 0};
        for (int k = 1; k < P.m - 1; ++k) r[(P.m - 2 - k) % 2] = std::max(r[(P.m - 2 - k) % 2], al(b[k]));
        W.level_off[P.m - 1] = 0;
        for (int k = 1; k < P.m - 1; ++k) W.level_off[k] = top_bytes + ((P.m - 2 - k) % 2 == 0 ? 0 : r[0]);
        end = top_bytes + r[0] + r[1];
      } else {
        size_t r[2] = {0, 0};
        for (int k = 1; k < P.m; ++k) r[(P.m - 1 - k) % 2] = std::max(r[(P.m - 1 - k) % 2], al(b[k]));
        for (int k = 1; k < P.m; ++k) W.level_off[k] = (P.m - 1 - k) % 2 == 0 ? 0 : r[0];
        end = r[0] + r[1];
      }
      P.ws_bytes = std::max(P.ws_bytes, end);
    }
    }  // full run
    // tables
    P.nbr.assign(P.m, {});
    P.nbr_off.assign(P.m, 0);
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 255) / 256 * 256; return o; };
    for (int k = 0; k < P.m; ++k) {
      build_nbr(P, k, P.nbr[k]);
      P.nbr_off[k] = take(P.nbr[k].size() * sizeof(int2));
    }
    P.flops = 0;
    P.c_blocks = 0;
    const bool partial = P.start_level > 0 || P.stop_level > 0;
    for (auto& W : P.waves) {
      if (!partial) build_wave_levels(P, W);
      for (auto& L : W.levels) {
        for (auto& X : L.launches) {
          X.off_parents = take(X.parents.size() * sizeof(int4));
          X.off_items = take(X.items.size() * sizeof(int4));
        }
        L.off_child = take(L.child_call.size() * sizeof(int));
        P.flops += L.flops;
        if (L.k == 0) P.c_blocks += L.n_calls;
      }
    }
    P.tables_bytes = off;
    P.built = true;
    return BCSS_OK;
  } catch (const std::exception& e) {
    return fail(BCSS_ERR_PARAMETER, "plan construction failed: %s", e.what());
  }
}

// Upload the device tables once per plan.  The copy is stream-ordered on the
// run's stream and synchronized: a plain cudaMemcpy from pageable memory can
// return before its DMA lands, and kernels on a non-blocking stream would
// then race it.
int upload_tables(bcss_plan& P, cudaStream_t stream) {
  int dev;
  CUDA_TRY(cudaGetDevice(&dev));
  if (P.d_tables && P.device == dev) return BCSS_OK;
  if (P.d_tables) { cudaFree(P.d_tables); P.d_tables = nullptr; }
  std::vector<char> host(P.tables_bytes, 0);
  for (int k = 0; k < P.m; ++k)
    if (!P.nbr[k].empty()) memcpy(&host[P.nbr_off[k]], P.nbr[k].data(), P.nbr[k].size() * sizeof(int2));
  for (auto& W : P.waves)
    for (auto& L : W.levels) {
      for (auto& X : L.launches) {
        memcpy(&host[X.off_parents], X.parents.data(), X.parents.size() * sizeof(int4));
        memcpy(&host[X.off_items], X.items.data(), X.items.size() * sizeof(int4));
      }
      memcpy(&host[L.off_child], L.child_call.data(), L.child_call.size() * sizeof(int));
    }
  CUDA_TRY(cudaMalloc(&P.d_tables, std::max<size_t>(P.tables_bytes, 256)));
  CUDA_TRY(cudaMemcpyAsync(P.d_tables, host.data(), P.tables_bytes, cudaMemcpyHostToDevice, stream));
  CUDA_TRY(cudaStreamSynchronize(stream));
  P.device = dev;
  static bool attr_done[64] = {false};
  if (dev < 64 && !attr_done[dev]) {
    for (int c = 0; c < N_CFGS; ++c) {
      const KernelCfg& C = kernel_cfg(c);
      CUDA_TRY(cudaFuncSetAttribute(C.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C.smem));
    }
    attr_done[dev] = true;
  }
  return BCSS_OK;
}

int ensure_workspace(bcss_plan& P) {
  if (P.ws_bytes == 0) return BCSS_OK;
  if (P.d_ws && P.ws_capacity >= P.ws_bytes) return BCSS_OK;
  if (P.d_ws && !P.own_ws)
    return fail(BCSS_ERR_STATE, "caller workspace of %zu bytes < required %zu", P.ws_capacity, P.ws_bytes);
  if (P.d_ws) cudaFree(P.d_ws);
  P.d_ws = nullptr;
  cudaError_t e = cudaMalloc(&P.d_ws, P.ws_bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(BCSS_ERR_NOMEM, "cudaMalloc of %zu workspace bytes failed: %s", P.ws_bytes, cudaGetErrorString(e));
  }
  P.ws_capacity = P.ws_bytes;
  P.own_ws = true;
  return BCSS_OK;
}

double* region_for(bcss_plan& P, const WaveHost& W, int k) {
  return reinterpret_cast<double*>(static_cast<char*>(P.d_ws) + W.level_off[k]);
}

int validate_problem(int m, int64_t n, int64_t p, int64_t b_a, int64_t b_c) {
  if (m < 2) return fail(BCSS_ERR_PARAMETER, "change of basis is defined for order >= 2");
  if (m > 8) return fail(BCSS_ERR_PARAMETER, "order %d > 8 is not supported", m);
  if (n < 1 || p < 1 || b_a < 1 || b_c < 1)
    return fail(BCSS_ERR_PARAMETER, "dimensions and block dimensions must be positive");
  if (n % b_a != 0) return fail(BCSS_ERR_BLOCK_DIVISIBILITY, "block dimension %lld does not divide %lld", (long long)b_a, (long long)n);
  if (p % b_c != 0) return fail(BCSS_ERR_BLOCK_DIVISIBILITY, "output block dimension %lld does not divide %lld", (long long)b_c, (long long)p);
  // int32 limits of the device tables and per-block offsets
  const double blk = std::pow((double)std::max(b_a, b_c), m);
  if (blk >= 2147483647.0) return fail(BCSS_ERR_PARAMETER, "block of %g elements exceeds the int32 block offset range", blk);
  if (n > (1 << 30) || p > (1 << 30)) return fail(BCSS_ERR_PARAMETER, "dimension too large");
  return BCSS_OK;
}

}  // namespace

// ---- C ABI -----------------------------------------------------------------------
extern "C" {

const char* bcss_last_error(void) { return g_last_error.c_str(); }
int bcss_abi_version(void) { return 100; }

int64_t bcss_simplex_count(int64_t extent, int m) {
  if (extent < 1 || m < 1) return -1;
  try { return bcss::simplex_count(extent, m); } catch (...) { return -1; }
}

int bcss_hypertriangle_rank(const int64_t* idx, int m, int64_t extent, int64_t* out_rank) {
  if (!idx || !out_rank || m < 1 || extent < 1) return fail(BCSS_ERR_PARAMETER, "bad arguments");
  for (int t = 0; t < m; ++t) {
    if (idx[t] < 0 || idx[t] >= extent)
      return fail(BCSS_ERR_RANGE, "index %lld outside grid %lld", (long long)idx[t], (long long)extent);
    if (t > 0 && idx[t] < idx[t - 1]) return fail(BCSS_ERR_SHAPE, "index is not nondecreasing");
  }
  try { *out_rank = bcss::hypertriangle_rank(idx, m, extent); } catch (const std::exception& e) {
    return fail(BCSS_ERR_PARAMETER, "%s", e.what());
  }
  return BCSS_OK;
}

int bcss_hypertriangle_unrank(int64_t rank, int m, int64_t extent, int64_t* out_idx) {
  if (!out_idx || m < 1 || extent < 1) return fail(BCSS_ERR_PARAMETER, "bad arguments");
  try {
    if (rank < 0 || rank >= bcss::simplex_count(extent, m)) return fail(BCSS_ERR_RANGE, "rank out of range");
    bcss::hypertriangle_unrank(rank, m, extent, out_idx);
  } catch (const std::exception& e) {
    return fail(BCSS_ERR_PARAMETER, "%s", e.what());
  }
  return BCSS_OK;
}

int bcss_blocked_flops(int m, int64_t n, int64_t p, int64_t b_a, int64_t b_c, int reuse, uint64_t* out_flops) {
  if (!out_flops) return fail(BCSS_ERR_PARAMETER, "null output");
  if (m < 2) return fail(BCSS_ERR_PARAMETER, "cost model is defined for order >= 2");
  if (n < 1 || p < 1 || b_a < 1 || b_c < 1) return fail(BCSS_ERR_PARAMETER, "dimensions must be positive");
  if (n % b_a || p % b_c) return fail(BCSS_ERR_PARAMETER, "block dimensions must divide the dimensions");
  try { *out_flops = bcss::blocked_flops(m, n, p, b_a, b_c, reuse != 0); } catch (const std::exception& e) {
    return fail(BCSS_ERR_PARAMETER, "%s", e.what());
  }
  return BCSS_OK;
}

int bcss_plan_create(int m, int64_t n, int64_t p, int64_t b_a, int64_t b_c, int reuse, bcss_plan** out_plan) {
  if (!out_plan) return fail(BCSS_ERR_PARAMETER, "null plan output");
  *out_plan = nullptr;
  int st = validate_problem(m, n, p, b_a, b_c);
  if (st) return st;
  bcss_plan* P = new (std::nothrow) bcss_plan();
  if (!P) return fail(BCSS_ERR_NOMEM, "out of host memory");
  P->m = m; P->n = n; P->p = p; P->bA = b_a; P->bC = b_c;
  P->nbar = n / b_a; P->pbar = p / b_c; P->reuse = reuse != 0;
  if (const char* e = getenv("BCSS_DYNAMIC_SCHEDULE")) P->dynamic = atoi(e) != 0;
  if (const char* e = getenv("BCSS_SERIAL_LAUNCH")) P->concurrent = atoi(e) == 0;
  *out_plan = P;
  return BCSS_OK;
}

int bcss_plan_destroy(bcss_plan* P) {
  if (!P) return BCSS_OK;
  if (P->d_tables) cudaFree(P->d_tables);
  if (P->d_ws && P->own_ws) cudaFree(P->d_ws);
  if (P->hA) cudaFree(P->hA);
  if (P->hX) cudaFree(P->hX);
  if (P->hC) cudaFree(P->hC);
  if (P->host_stream) cudaStreamDestroy(P->host_stream);
  for (auto ev : P->events) cudaEventDestroy(ev);
  for (auto ev : P->join) cudaEventDestroy(ev);
  for (auto ss : P->side) cudaStreamDestroy(ss);
  if (P->fork) cudaEventDestroy(P->fork);
  for (auto ev : P->chunk_ev) cudaEventDestroy(ev);
  for (auto ev : P->wave_ev) cudaEventDestroy(ev);
  if (P->copy_in) cudaStreamDestroy(P->copy_in);
  if (P->copy_out) cudaStreamDestroy(P->copy_out);
  if (P->copy_out2) cudaStreamDestroy(P->copy_out2);
  if (P->out2_done) cudaEventDestroy(P->out2_done);
  if (P->d_counters) cudaFree(P->d_counters);
  delete P;
  return BCSS_OK;
}

static void invalidate(bcss_plan* P) {
  P->built = false;
  if (P->d_tables) { cudaFree(P->d_tables); P->d_tables = nullptr; }
}

int bcss_plan_set_units(bcss_plan* P, const int32_t* units, int n_units) {
  if (!P) return fail(BCSS_ERR_STATE, "null plan");
  if (n_units < 0 || (n_units > 0 && !units)) return fail(BCSS_ERR_PARAMETER, "bad unit list");
  for (int i = 0; i < n_units; ++i)
    if (units[i] < 0 || units[i] >= P->pbar) return fail(BCSS_ERR_RANGE, "unit %d outside 0..%lld", units[i], (long long)P->pbar - 1);
  P->units.assign(units, units + n_units);
  P->units_set = true;
  invalidate(P);
  return BCSS_OK;
}

int bcss_plan_set_workspace_limit(bcss_plan* P, size_t bytes) {
  if (!P) return fail(BCSS_ERR_STATE, "null plan");
  P->ws_limit = bytes;
  invalidate(P);
  return BCSS_OK;
}

int bcss_plan_set_keep_temps(bcss_plan* P, int keep) {
  if (!P) return fail(BCSS_ERR_STATE, "null plan");
  P->keep_temps = keep != 0;
  invalidate(P);
  return BCSS_OK;
}

int bcss_plan_workspace_bytes(bcss_plan* P, size_t* out_bytes) {
  if (!P || !out_bytes) return fail(BCSS_ERR_STATE, "null argument");
  int st = build_plan(*P);
  if (st) return st;
  *out_bytes = P->ws_bytes;
  return BCSS_OK;
}

int bcss_plan_set_workspace(bcss_plan* P, void* dev_ptr, size_t bytes) {
  if (!P) return fail(BCSS_ERR_STATE, "null plan");
  if (P->d_ws && P->own_ws) cudaFree(P->d_ws);
  P->d_ws = dev_ptr;
  P->ws_capacity = dev_ptr ? bytes : 0;
  P->own_ws = false;
  return BCSS_OK;
}

int bcss_plan_stats(bcss_plan* P, int64_t* waves, int64_t* launches, uint64_t* flops, int64_t* c_blocks) {
  if (!P) return fail(BCSS_ERR_STATE, "null plan");
  int st = build_plan(*P);
  if (st) return st;
  int64_t nl = 0;
  for (auto& W : P->waves)
    for (auto& L : W.levels)
      for (auto& X : L.launches) nl += X.item_off.back() > 0 ? 1 : 0;
  if (waves) *waves = (int64_t)P->waves.size();
  if (launches) *launches = nl;
  if (flops) *flops = P->flops;
  if (c_blocks) *c_blocks = P->c_blocks;
  return BCSS_OK;
}

}  // extern "C"

namespace {

// Host-transfer pipeline of run_host: A arrives in chunks (blocks whose first
// index is a, a contiguous range of the packed payload), wave 0's top level
// is split by key ranges that need only the chunks already landed, and each
// wave's C blocks are downloaded while later waves compute.
struct Pipe {
  double* c_host = nullptr;
  // BCSS_TRACE=1: timing events (name, event) printed after the run
  std::vector<std::pair<std::string, cudaEvent_t>>* trace = nullptr;
};

void trace_mark(const Pipe* pipe, const std::string& name, cudaStream_t s) {
  if (!pipe || !pipe->trace) return;
  cudaEvent_t ev;
  cudaError_t e1 = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  cudaError_t e2 = cudaEventRecord(ev, s);
  if (e1 != cudaSuccess || e2 != cudaSuccess)
    fprintf(stderr, "[bcss trace] %s: %s / %s\n", name.c_str(), cudaGetErrorString(e1), cudaGetErrorString(e2));
  pipe->trace->emplace_back(name, ev);
}

int launch_one(bcss_plan* P, const WaveHost& W, const LevelHost& L, const LaunchHost& X, const double* A,
               const double* X_, double* C, long long item_lo, long long item_hi, unsigned* counter,
               cudaStream_t ls, int sms) {
  const long long total = item_hi - item_lo;
  if (total <= 0) return BCSS_OK;
  const KernelCfg& K = kernel_cfg(X.cfg);
  char* tbl = static_cast<char*>(P->d_tables);
  bcss::LevelArgs a;
  memset(&a, 0, sizeof(a));
  a.X = X_;
  const bool from_input = (P->start_level == 0 && L.k == P->m - 1) || (P->start_level > 0 && L.k == P->start_level - 1);
  a.Tin = from_input ? A : region_for(*P, W, L.k + 1);
  a.Tout = (L.k == P->stop_level) ? C : region_for(*P, W, L.k);
  a.parents = reinterpret_cast<const int4*>(tbl + X.off_parents);
  a.items = reinterpret_cast<const int4*>(tbl + X.off_items) + item_lo;
  a.child_call = reinterpret_cast<const int*>(tbl + L.off_child);
  a.nbr = reinterpret_cast<const int2*>(tbl + P->nbr_off[L.k]);
  a.counter = P->dynamic ? counter : nullptr;
  a.total_items = total;
  a.keys_in = L.keys_in; a.keys_out = L.keys_out;
  a.blk_in = L.blk_in; a.blk_out = L.blk_out;
  a.n_parents = (int)X.parents.size();
  a.n = (int)P->n; a.ldx = (int)P->n; a.p_rows = (int)P->p;
  a.nbar = (int)P->nbar; a.bA = (int)P->bA; a.bC = (int)P->bC;
  a.lbA = is_pow2(P->bA) ? ilog2(P->bA) : -1;
  a.k = L.k;
  a.rest = (int)L.rest; a.bAk = (int)L.bAk;
  a.n_tiles = X.n_tiles;
  for (int i = 0; i < 10; ++i) a.pw[i] = (long long)std::min<double>(std::pow((double)P->bA, i), 9.0e18);
  int occ = 1;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, K.fn, K.NT, K.smem));
  const long long grid = std::min<long long>(total, (long long)sms * std::max(occ, 1));
  K.fn<<<(unsigned)grid, K.NT, K.smem, ls>>>(a);
  CUDA_TRY(cudaGetLastError());
  return BCSS_OK;
}

int ensure_side(bcss_plan* P, int n) {
  while ((int)P->side.size() < n) {
    cudaStream_t ss;
    CUDA_TRY(cudaStreamCreateWithFlags(&ss, cudaStreamNonBlocking));
    P->side.push_back(ss);
    cudaEvent_t ev;
    CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    P->join.push_back(ev);
  }
  if (!P->fork) CUDA_TRY(cudaEventCreateWithFlags(&P->fork, cudaEventDisableTiming));
  return BCSS_OK;
}

// first packed rank of the m-tuples over `extent` whose first index is a
int64_t first_rank_with(int64_t a, int m, int64_t extent) {
  if (a >= extent) return bcss::simplex_count(extent, m);
  std::vector<int64_t> t(m, a);
  return bcss::hypertriangle_rank(t.data(), m, extent);
}

int run_impl(bcss_plan* P, const double* A, const double* X_, double* C, cudaStream_t s, const Pipe* pipe) {
  int st = build_plan(*P);
  if (st) return st;
  if ((st = upload_tables(*P, s))) return st;
  if ((st = ensure_workspace(*P))) return st;
  int dev, sms;
  CUDA_TRY(cudaGetDevice(&dev));
  CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  int64_t launches = 0;
  if (P->timing) {
    P->launch_level.clear();
    P->launch_flops.clear();
    P->timed_stream = s;
  }
  // Launches of one level (one per tile shape) are independent: they run
  // concurrently on side streams, so one launch's tail overlaps the next
  // launch's CTAs instead of idling SMs.
  size_t n_launch_total = 0;
  for (auto& W : P->waves)
    for (auto& L : W.levels) n_launch_total += L.launches.size();
  if (P->counters_n < n_launch_total) {
    if (P->d_counters) cudaFree(P->d_counters);
    P->d_counters = nullptr;
    CUDA_TRY(cudaMalloc(&P->d_counters, n_launch_total * sizeof(unsigned)));
    P->counters_n = n_launch_total;
  }
  CUDA_TRY(cudaMemsetAsync(P->d_counters, 0, n_launch_total * sizeof(unsigned), s));
  size_t counter_idx = 0;
  int level_idx = 0;
  const size_t blk_c = (size_t)ipow(P->bC, P->m);
  for (size_t wi = 0; wi < P->waves.size(); ++wi) {
    const WaveHost& W = P->waves[wi];
    for (const LevelHost& L : W.levels) {
      const int nl = (int)L.launches.size();
      // chunk-gated top level of the first wave (pipelined host run)
      const bool gate = pipe && wi == 0 && L.k == P->m - 1;
      const bool gate_split = gate && nl == 1 && L.launches[0].parents.size() == 1;
      if (gate && !gate_split) CUDA_TRY(cudaStreamWaitEvent(s, P->chunk_ev.back(), 0));
      const bool conc = (P->concurrent && nl > 1) || gate_split;
      if (conc && (st = ensure_side(P, std::max(nl - 1, 1)))) return st;
      if (P->timing) {
        while (P->events.size() < (size_t)(2 * (level_idx + 1))) {
          cudaEvent_t ev;
          CUDA_TRY(cudaEventCreate(&ev));
          P->events.push_back(ev);
        }
        CUDA_TRY(cudaEventRecord(P->events[2 * level_idx], s));
      }
      if (conc) {
        CUDA_TRY(cudaEventRecord(P->fork, s));
        for (int i = 1; i < std::max(nl, 2); ++i) CUDA_TRY(cudaStreamWaitEvent(P->side[i - 1], P->fork, 0));
      }
      if (gate_split) {
        // keys with first index <= a need only A chunks 0..a; ~8 sub-launches
        // alternate between two streams, each waiting for its last chunk
        const LaunchHost& X = L.launches[0];
        const int64_t per_key = X.item_off.back() / L.keys_out;
        const int64_t nb = P->nbar;
        const int groups = (int)std::min<int64_t>(8, nb);
        int64_t a0 = 0;
        unsigned* counter = P->d_counters + counter_idx++;
        for (int g = 0; g < groups; ++g) {
          int64_t a1 = (g == groups - 1) ? nb : std::max(a0 + 1, (nb * (g + 1)) / groups);
          const int64_t k_lo = first_rank_with(a0, P->m - 1, nb), k_hi = first_rank_with(a1, P->m - 1, nb);
          cudaStream_t ls = (g % 2 == 0) ? s : P->side[0];
          CUDA_TRY(cudaStreamWaitEvent(ls, P->chunk_ev[a1 - 1], 0));
          if ((st = launch_one(P, W, L, X, A, X_, C, k_lo * per_key, k_hi * per_key, counter, ls, sms))) return st;
          ++launches;
          a0 = a1;
        }
      } else {
        for (int li = 0; li < nl; ++li) {
          const LaunchHost& X = L.launches[li];
          cudaStream_t ls = (li == 0 || !conc) ? s : P->side[li - 1];
          unsigned* counter = P->d_counters + counter_idx++;
          if (X.item_off.back() == 0) continue;
          if ((st = launch_one(P, W, L, X, A, X_, C, 0, X.item_off.back(), counter, ls, sms))) return st;
          ++launches;
        }
      }
      if (conc) {
        for (int i = 1; i < std::max(nl, 2); ++i) {
          CUDA_TRY(cudaEventRecord(P->join[i - 1], P->side[i - 1]));
          CUDA_TRY(cudaStreamWaitEvent(s, P->join[i - 1], 0));
        }
      }
      if (P->timing) {
        CUDA_TRY(cudaEventRecord(P->events[2 * level_idx + 1], s));
        P->launch_level.push_back(L.k);
        P->launch_flops.push_back(L.flops);
      }
      ++level_idx;
      trace_mark(pipe, "wave" + std::to_string(wi) + " level" + std::to_string(L.k) + " done", s);
      if (pipe && L.k == 0) {
        // this wave's C blocks are final: download them (runs of consecutive ranks)
        CUDA_TRY(cudaEventRecord(P->wave_ev[wi], s));
        CUDA_TRY(cudaStreamWaitEvent(P->copy_out, P->wave_ev[wi], 0));
        CUDA_TRY(cudaStreamWaitEvent(P->copy_out2, P->wave_ev[wi], 0));
        int which = 0;  // alternate two DMA streams so per-copy setup overlaps
        std::vector<int> ranks(L.child_call.begin(), L.child_call.end());
        std::sort(ranks.begin(), ranks.end());
        size_t i = 0;
        while (i < ranks.size()) {
          size_t j = i + 1;
          while (j < ranks.size() && ranks[j] == ranks[j - 1] + 1) ++j;
          const size_t off = (size_t)ranks[i] * blk_c;
          CUDA_TRY(cudaMemcpyAsync(pipe->c_host + off, C + off, (j - i) * blk_c * sizeof(double),
                                   cudaMemcpyDeviceToHost, (which ^= 1) ? P->copy_out : P->copy_out2));
          i = j;
        }
        trace_mark(pipe, "wave" + std::to_string(wi) + " C downloaded", P->copy_out);
        // submit what is queued so far (the driver otherwise batches it until a sync)
        cudaStreamQuery(s);
        cudaStreamQuery(P->copy_out);
        cudaStreamQuery(P->copy_out2);
      }
    }
  }
  P->last_launches = launches;
  return BCSS_OK;
}

bool is_pinned(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

}  // namespace

extern "C" {

int bcss_sttsm_run(bcss_plan* P, const double* A, const double* X_, double* C, void* stream) {
  if (!P) return fail(BCSS_ERR_STATE, "null plan");
  if (!A || !X_ || !C) return fail(BCSS_ERR_PARAMETER, "null buffer");
  return run_impl(P, A, X_, C, static_cast<cudaStream_t>(stream), nullptr);
}

int bcss_plan_set_stop_level(bcss_plan* P, int stop_level) {
  if (!P) return fail(BCSS_ERR_STATE, "null plan");
  if (stop_level < 0 || stop_level >= P->m) return fail(BCSS_ERR_RANGE, "stop level %d outside 0..%d", stop_level, P->m - 1);
  P->stop_level = stop_level;
  invalidate(P);
  return BCSS_OK;
}

int bcss_plan_set_start_calls(bcss_plan* P, int level, const int32_t* suffixes, int n_calls) {
  if (!P) return fail(BCSS_ERR_STATE, "null plan");
  if (level == P->m || level == 0) {  // back to a full run from A
    P->start_level = 0;
    P->start_suffixes.clear();
    invalidate(P);
    return BCSS_OK;
  }
  if (level < 1 || level >= P->m) return fail(BCSS_ERR_RANGE, "start level %d outside 1..%d", level, P->m - 1);
  if (n_calls < 0 || (n_calls > 0 && !suffixes)) return fail(BCSS_ERR_PARAMETER, "bad call list");
  const int sl = P->m - level;
  for (int c = 0; c < n_calls; ++c)
    for (int q = 0; q < sl; ++q) {
      const int32_t v = suffixes[c * sl + q];
      if (v < 0 || v >= P->pbar) return fail(BCSS_ERR_RANGE, "suffix entry %d outside 0..%lld", v, (long long)P->pbar - 1);
      if (q > 0 && v < suffixes[c * sl + q - 1]) return fail(BCSS_ERR_SHAPE, "suffix is not nondecreasing");
    }
  P->start_level = level;
  P->start_suffixes.assign(suffixes, suffixes + (size_t)n_calls * sl);
  invalidate(P);
  return BCSS_OK;
}

int bcss_plan_level_calls(bcss_plan* P, int k, int32_t* out, int64_t n_max, int64_t* out_n) {
  if (!P || !out_n) return fail(BCSS_ERR_STATE, "null argument");
  int st = build_plan(*P);
  if (st) return st;
  const int sl = P->m - k;
  int64_t cnt = 0;
  for (auto& W : P->waves)
    for (auto& L : W.levels)
      if (L.k == k) {
        for (int64_t c = 0; c < L.n_calls; ++c, ++cnt)
          if (out && cnt < n_max)
            for (int q = 0; q < sl; ++q) out[cnt * sl + q] = L.suffixes[(size_t)(c * sl + q)];
      }
  *out_n = cnt;
  if (out && cnt > n_max) return fail(BCSS_ERR_RANGE, "output array too small");
  return BCSS_OK;
}

int bcss_plan_io_elems(bcss_plan* P, int64_t* in_elems, int64_t* out_elems) {
  if (!P) return fail(BCSS_ERR_STATE, "null plan");
  int st = build_plan(*P);
  if (st) return st;
  if (in_elems) {
    if (P->start_level > 0)
      *in_elems = (int64_t)(P->start_suffixes.size() / (P->m - P->start_level)) * keys_at(*P, P->start_level) *
                  blk_at(*P, P->start_level);
    else
      *in_elems = bcss::simplex_count(P->nbar, P->m) * ipow(P->bA, P->m);
  }
  if (out_elems) {
    if (P->stop_level > 0) {
      int64_t calls = 0;
      for (auto& W : P->waves)
        for (auto& L : W.levels)
          if (L.k == P->stop_level) calls += L.n_calls;
      *out_elems = calls * keys_at(*P, P->stop_level) * blk_at(*P, P->stop_level);
    } else {
      *out_elems = bcss::simplex_count(P->pbar, P->m) * ipow(P->bC, P->m);
    }
  }
  return BCSS_OK;
}

int bcss_plan_set_pipeline(bcss_plan* P, int waves) {
  if (!P) return fail(BCSS_ERR_STATE, "null plan");
  if (waves < 0) return fail(BCSS_ERR_PARAMETER, "negative wave count");
  P->pipeline_waves = waves;
  invalidate(P);
  return BCSS_OK;
}

int bcss_sttsm_run_host(bcss_plan* P, const double* A, const double* X, double* C) {
  if (!P) return fail(BCSS_ERR_STATE, "null plan");
  if (!A || !X || !C) return fail(BCSS_ERR_PARAMETER, "null buffer");
  const size_t blk_a = (size_t)ipow(P->bA, P->m);
  const size_t a_bytes = (size_t)bcss::simplex_count(P->nbar, P->m) * blk_a * sizeof(double);
  const size_t x_bytes = (size_t)(P->p * P->n) * sizeof(double);
  const size_t c_bytes = (size_t)bcss::simplex_count(P->pbar, P->m) * ipow(P->bC, P->m) * sizeof(double);
  auto grow = [&](double*& ptr, size_t& cap, size_t need) -> int {
    if (cap >= need) return BCSS_OK;
    if (ptr) cudaFree(ptr);
    ptr = nullptr; cap = 0;
    CUDA_TRY(cudaMalloc(&ptr, need));
    cap = need;
    return BCSS_OK;
  };
  int st;
  if ((st = grow(P->hA, P->hA_bytes, a_bytes))) return st;
  if ((st = grow(P->hX, P->hX_bytes, x_bytes))) return st;
  if ((st = grow(P->hC, P->hC_bytes, c_bytes))) return st;
  if (!P->host_stream) CUDA_TRY(cudaStreamCreateWithFlags(&P->host_stream, cudaStreamNonBlocking));
  const bool pipelined = P->pipeline_waves > 0 && !P->units_set && !P->keep_temps && P->start_level == 0 &&
                         P->stop_level == 0 && is_pinned(A) &&
                         is_pinned(X) && is_pinned(C);
  if (!pipelined) {
    CUDA_TRY(cudaMemcpyAsync(P->hA, A, a_bytes, cudaMemcpyHostToDevice, P->host_stream));
    CUDA_TRY(cudaMemcpyAsync(P->hX, X, x_bytes, cudaMemcpyHostToDevice, P->host_stream));
    if (P->units_set) CUDA_TRY(cudaMemsetAsync(P->hC, 0, c_bytes, P->host_stream));
    if ((st = run_impl(P, P->hA, P->hX, P->hC, P->host_stream, nullptr))) return st;
    CUDA_TRY(cudaMemcpyAsync(C, P->hC, c_bytes, cudaMemcpyDeviceToHost, P->host_stream));
    CUDA_TRY(cudaStreamSynchronize(P->host_stream));
    return BCSS_OK;
  }
  const auto h0 = std::chrono::steady_clock::now();
  if ((st = build_plan(*P))) return st;
  if (!P->copy_in) CUDA_TRY(cudaStreamCreateWithFlags(&P->copy_in, cudaStreamNonBlocking));
  if (!P->copy_out) CUDA_TRY(cudaStreamCreateWithFlags(&P->copy_out, cudaStreamNonBlocking));
  if (!P->copy_out2) CUDA_TRY(cudaStreamCreateWithFlags(&P->copy_out2, cudaStreamNonBlocking));
  if (!P->out2_done) CUDA_TRY(cudaEventCreateWithFlags(&P->out2_done, cudaEventDisableTiming));
  auto need_events = [&](std::vector<cudaEvent_t>& v, size_t n) -> int {
    while (v.size() < n) {
      cudaEvent_t ev;
      CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      v.push_back(ev);
    }
    return BCSS_OK;
  };
  if ((st = need_events(P->chunk_ev, (size_t)P->nbar))) return st;
  if ((st = need_events(P->wave_ev, P->waves.size()))) return st;
  // everything below is ordered after work already queued on the host stream
  CUDA_TRY(cudaEventRecord(P->chunk_ev[0], P->host_stream));
  CUDA_TRY(cudaStreamWaitEvent(P->copy_in, P->chunk_ev[0], 0));
  CUDA_TRY(cudaStreamWaitEvent(P->copy_out, P->chunk_ev[0], 0));
  CUDA_TRY(cudaStreamWaitEvent(P->copy_out2, P->chunk_ev[0], 0));
  Pipe pipe;
  pipe.c_host = C;
  std::vector<std::pair<std::string, cudaEvent_t>> trace;
  const char* tr = getenv("BCSS_TRACE");
  if (tr && atoi(tr) == 1) pipe.trace = &trace;
  trace_mark(&pipe, "upload start", P->copy_in);
  CUDA_TRY(cudaMemcpyAsync(P->hX, X, x_bytes, cudaMemcpyHostToDevice, P->copy_in));
  for (int64_t a = 0; a < P->nbar; ++a) {
    const size_t r0 = (size_t)first_rank_with(a, P->m, P->nbar), r1 = (size_t)first_rank_with(a + 1, P->m, P->nbar);
    CUDA_TRY(cudaMemcpyAsync(P->hA + r0 * blk_a, A + r0 * blk_a, (r1 - r0) * blk_a * sizeof(double),
                             cudaMemcpyHostToDevice, P->copy_in));
    CUDA_TRY(cudaEventRecord(P->chunk_ev[a], P->copy_in));
    trace_mark(&pipe, "A chunk " + std::to_string(a) + " landed", P->copy_in);
  }
  cudaStreamQuery(P->copy_in);  // kick the driver to submit queued work now
  if ((st = run_impl(P, P->hA, P->hX, P->hC, P->host_stream, &pipe))) return st;
  if (pipe.trace) {
    fprintf(stderr, "[bcss trace] host enqueue took %.3f ms\n",
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count());
    // host-side polling timeline (first time each event is seen complete)
    std::vector<double> seen(trace.size(), -1.0);
    const auto t0 = std::chrono::steady_clock::now();
    size_t left = trace.size();
    while (left) {
      const double now = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      for (size_t i = 0; i < trace.size(); ++i)
        if (seen[i] < 0 && cudaEventQuery(trace[i].second) == cudaSuccess) { seen[i] = now; --left; }
    }
    fprintf(stderr, "[bcss trace] run_host pipeline timeline (host-polled ms, relative to upload start):\n");
    for (size_t i = 0; i < trace.size(); ++i) {
      fprintf(stderr, "  %-28s %8.3f\n", trace[i].first.c_str(), seen[i] - seen[0]);
      cudaEventDestroy(trace[i].second);
    }
  }
  const auto h1 = std::chrono::steady_clock::now();
  CUDA_TRY(cudaStreamSynchronize(P->copy_out));
  const auto h2 = std::chrono::steady_clock::now();
  CUDA_TRY(cudaStreamSynchronize(P->copy_out2));
  CUDA_TRY(cudaStreamSynchronize(P->host_stream));
  const auto h3 = std::chrono::steady_clock::now();
  if (tr && atoi(tr) == 2)
    fprintf(stderr, "[bcss trace] enqueue %.3f ms, copy_out sync at %.3f ms, all synced at %.3f ms\n",
            std::chrono::duration<double, std::milli>(h1 - h0).count(),
            std::chrono::duration<double, std::milli>(h2 - h0).count(),
            std::chrono::duration<double, std::milli>(h3 - h0).count());
  return BCSS_OK;
}

int bcss_plan_temp(bcss_plan* P, int k, const int32_t* suffix, const double** out_ptr, int64_t* out_elems) {
  if (!P || !suffix || !out_ptr || !out_elems) return fail(BCSS_ERR_STATE, "null argument");
  if (!P->keep_temps || !P->built || !P->d_ws) return fail(BCSS_ERR_STATE, "temporaries were not kept");
  if (k < 1 || k >= P->m) return fail(BCSS_ERR_RANGE, "level %d outside 1..%d", k, P->m - 1);
  const int sl = P->m - k;
  int64_t base_calls = 0;
  for (auto& W : P->waves) {
    const LevelHost& L = W.levels[P->m - 1 - k];
    for (int64_t c = 0; c < L.n_calls; ++c) {
      if (std::equal(suffix, suffix + sl, &L.suffixes[(size_t)(c * sl)])) {
        const int64_t elems = L.keys_out * L.blk_out;
        *out_ptr = region_for(*P, W, k) + (base_calls + c) * elems;
        *out_elems = elems;
        if (P->waves.size() != 1) return fail(BCSS_ERR_STATE, "temporaries span several waves");
        return BCSS_OK;
      }
    }
  }
  return fail(BCSS_ERR_RANGE, "no call with that suffix at level %d", k);
}

int bcss_plan_temp_copy(bcss_plan* P, int k, const int32_t* suffix, double* host_out, int64_t elems) {
  if (!host_out) return fail(BCSS_ERR_PARAMETER, "null output");
  const double* ptr = nullptr;
  int64_t have = 0;
  int st = bcss_plan_temp(P, k, suffix, &ptr, &have);
  if (st) return st;
  if (have != elems) return fail(BCSS_ERR_SHAPE, "temporary has %lld elements, buffer %lld", (long long)have, (long long)elems);
  CUDA_TRY(cudaDeviceSynchronize());
  CUDA_TRY(cudaMemcpy(host_out, ptr, (size_t)elems * sizeof(double), cudaMemcpyDeviceToHost));
  return BCSS_OK;
}

int bcss_plan_last_launches(bcss_plan* P, int64_t* out) {
  if (!P || !out) return fail(BCSS_ERR_STATE, "null argument");
  *out = P->last_launches;
  return BCSS_OK;
}

int bcss_plan_c_block_ranks(bcss_plan* P, int64_t* out_ranks, int64_t n_max, int64_t* out_n) {
  if (!P || !out_n) return fail(BCSS_ERR_STATE, "null argument");
  int st = build_plan(*P);
  if (st) return st;
  int64_t cnt = 0;
  for (auto& W : P->waves)
    for (auto& L : W.levels)
      if (L.k == 0)
        for (int r : L.child_call) {
          if (out_ranks && cnt < n_max) out_ranks[cnt] = r;
          ++cnt;
        }
  *out_n = cnt;
  if (out_ranks && cnt > n_max) return fail(BCSS_ERR_RANGE, "output array too small (%lld > %lld)", (long long)cnt, (long long)n_max);
  return BCSS_OK;
}

int bcss_plan_set_timing(bcss_plan* P, int on) {
  if (!P) return fail(BCSS_ERR_STATE, "null plan");
  P->timing = on != 0;
  return BCSS_OK;
}

int bcss_plan_launch_times(bcss_plan* P, int32_t* out_level, uint64_t* out_flops, float* out_ms, int64_t n_max,
                           int64_t* out_n) {
  if (!P || !out_n) return fail(BCSS_ERR_STATE, "null argument");
  if (!P->timing) return fail(BCSS_ERR_STATE, "timing is off");
  const int64_t n = (int64_t)P->launch_level.size();
  *out_n = n;
  if (n > n_max) return fail(BCSS_ERR_RANGE, "output arrays too small");
  CUDA_TRY(cudaStreamSynchronize(P->timed_stream));
  for (int64_t i = 0; i < n; ++i) {
    float ms = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&ms, P->events[2 * i], P->events[2 * i + 1]));
    if (out_level) out_level[i] = P->launch_level[i];
    if (out_flops) out_flops[i] = P->launch_flops[i];
    if (out_ms) out_ms[i] = ms;
  }
  return BCSS_OK;
}

int bcss_probe_fp64_peak(double* out_tflops) {
  if (!out_tflops) return fail(BCSS_ERR_PARAMETER, "null output");
  int dev, sms;
  CUDA_TRY(cudaGetDevice(&dev));
  CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  double* sink;
  CUDA_TRY(cudaMalloc(&sink, 1024 * sizeof(double)));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4000, threads = 256, grid = 2 * sms;
  dmma_peak_kernel<<<grid, threads>>>(sink, 16);
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0);
    dmma_peak_kernel<<<grid, threads>>>(sink, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = std::min(best, ms);
  }
  cudaError_t e = cudaGetLastError();
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  if (e != cudaSuccess) return fail(BCSS_ERR_CUDA, "peak probe failed: %s", cudaGetErrorString(e));
  const double flops = 2.0 * 256.0 * 16.0 * iters * (threads / 32) * (double)grid;
  *out_tflops = flops / (best * 1e-3) / 1e12;
  return BCSS_OK;
}

}  // extern "C"
