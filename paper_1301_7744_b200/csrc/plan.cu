// Plan construction: neighbour tables, waves, levels, per-shape launches and
// workspace layout; device tables and workspace (declared in plan.hpp).
// Replaces the reference's depth-first `descend` (change_of_basis.py:269-283)
// by breadth-first levels over waves of top-level units.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <stdexcept>

#include "plan.hpp"
#include "shape_costs.hpp"

namespace bcss_host {

thread_local std::string g_last_error;

// ---- kernel configurations ----------------------------------------------------

// The fast tile shapes' BM (bcss::BCSS_FAST_SHAPES order).
int shape_bm(int shape) { return bcss::kFast32[shape].BM; }

const KernelCfg& kernel_cfg(int cfg) {
  if (cfg == CFG_GENERIC) return bcss::kGeneric;
  if (cfg == CFG_GENERIC_PERM) return bcss::kGenericPerm;
  const KernelCfg* const fast[bcss::N_BA] = {bcss::kFast4, bcss::kFast8, bcss::kFast16, bcss::kFast32, bcss::kFast64};
  const KernelCfg* const gen[bcss::N_BA] = {bcss::kGen4, bcss::kGen8, bcss::kGen16, bcss::kGen32, bcss::kGen64};
  const int np0 = 1 + bcss::N_BA * N_SHAPES + bcss::N_BA * N_GEN;  // non-power-of-two b_a
  if (cfg >= np0 && cfg < np0 + bcss::N_NP * N_SHAPES) {
    const KernelCfg* const np[bcss::N_NP] = {bcss::kNP4, bcss::kNP12, bcss::kNP20, bcss::kNP24, bcss::kNP28};
    return np[(cfg - np0) % bcss::N_NP][(cfg - np0) / bcss::N_NP];
  }
  const int npp0 = np0 + bcss::N_NP * N_SHAPES;  // ... padded up to a multiple of the row group
  if (cfg >= npp0 && cfg < npp0 + bcss::N_NPP * N_SHAPES) {
    const KernelCfg* const npp[bcss::N_NPP] = {bcss::kNPP4,  bcss::kNPP8,  bcss::kNPP12, bcss::kNPP16,
                                               bcss::kNPP20, bcss::kNPP24, bcss::kNPP28};
    return npp[(cfg - npp0) % bcss::N_NPP][(cfg - npp0) / bcss::N_NPP];
  }
  const int ba = (cfg - 1) % bcss::N_BA;
  if (cfg > bcss::N_BA * N_SHAPES)  // general-redirection variants
    return gen[ba][(cfg - 1 - bcss::N_BA * N_SHAPES) / bcss::N_BA];
  return fast[ba][(cfg - 1) / bcss::N_BA];
}
// Non-power-of-two b_a (even >= 6, odd >= 15) on the fast kernels (POW2 =
// false): np_row_group returns the index of the row group RG and the block
// width b_a' the contraction index runs over - b_a itself when RG divides it
// (unpadded kernels, index into bcss::kNpRg), else b_a padded up to a multiple
// of RG (rows e >= b_a zero-filled; index into bcss::kNppRg).  -1: a power of
// two, or a b_a the generic kernel serves better.
// relative rate of the POW2 = false kernels by row group (measured full-size
// shapes, profiles/r02/padded_row_groups.txt and np_shapes.txt: RG 20 / 24 run
// at 28-31 TF, 28 at 26, 16 at ~24, 12 at 18-19, 8 at ~20, 4 at ~13)
static double np_rate(int64_t rg) {
  switch (rg) {
    case 4: return 0.45;
    case 8: return 0.70;
    case 12: return 0.65;
    case 16: return 0.82;
    case 28: return 0.80;  // (its [col][e] ring does not fit: level 0 gathers 8 bytes at a time)
    default: return 1.0;
  }
}
int np_row_group(int64_t bA, int m, int64_t* padded) {
  (void)m;  // (problems with fewer than 64 top-level columns per key never get here: fast_cfg)
  if (bA < 6 || is_pow2(bA)) return -1;
  // odd b_a moves 8 bytes per copy: below 15 the generic kernel is faster
  // (measured, m = 3: b_a = 13: 12.2 vs 12.9 TF, 7: 5.4 vs 11.9, 5: 2.0 vs 10.0)
  if ((bA & 1) && bA < 15) return -1;
  // candidates: a row group that divides b_a (unpadded kernels, index into
  // kNpRg), or b_a padded up to a multiple of a row group (index into
  // kNppRg); the least wasted DMMA work per unit rate wins, ties to the
  // larger row group (so 36 runs as 40 = 2 x 20 rather than 3 x 12, 44 as
  // 48 = 2 x 24 rather than 11 x 4)
  int best = -1;
  double best_score = 0;
  int64_t best_pad = 0, best_rg = 0;
  auto consider = [&](int j, int64_t rg, int64_t pad, double bonus) {
    const double score = (double)pad / (double)bA / np_rate(rg) * bonus;
    if (best < 0 || score < best_score - 1e-9 || (score < best_score + 1e-9 && rg > best_rg)) {
      best = j;
      best_score = score;
      best_pad = pad;
      best_rg = rg;
    }
  };
  for (int j = 0; j < bcss::N_NP; ++j)
    if (bA % bcss::kNpRg[j] == 0) consider(j, bcss::kNpRg[j], bA, 0.95);  // (near ties go to the unpadded kernels)
  for (int j = 0; j < bcss::N_NPP; ++j) {
    const int64_t rg = bcss::kNppRg[j];
    if (bA % rg != 0) consider(j, rg, (bA + rg - 1) / rg * rg, 1.0);
  }
  if (padded) *padded = best_pad;
  return best;
}
// contraction rows per block on the fast kernels: b_a, or its padded width
int64_t padded_ba(int64_t bA, int m) {
  int64_t pad = bA;
  if (fast_cfg(bA, m, 0) < 0 || np_row_group(bA, m, &pad) < 0) return bA;
  return pad;
}
// general-redirection configuration mirroring fast shape `shape` (one of BCSS_GEN_OF), else -1
int gen_cfg(int64_t bA, int m, int shape) {
  if (!is_pow2(bA)) return -1;  // general redirection: power-of-two b_a only
  const int f = fast_cfg(bA, m, 0);
  if (f < 0) return -1;
  for (int g = 0; g < N_GEN; ++g)
    if (bcss::BCSS_GEN_OF[g] == shape) return 1 + bcss::N_BA * N_SHAPES + g * bcss::N_BA + (f - 1);
  return -1;
}
// fast configuration of tile shape `shape` for power-of-two b_a in {4, 8, 16, 32, 64}, else -1
int fast_cfg(int64_t bA, int m, int shape) {
  if (getenv("BCSS_FORCE_GENERIC")) return -1;  // (experiments)
  // Few GEMM columns per key at the top level (b_a^(m-1) < 64, and every
  // m = 2 problem): the fast kernels' key-major tiles of 128..512 columns
  // are mostly empty, the generic kernel's flat (key, column) tiles are not
  // (measured: m=3 b=4 3.8 vs 9.0 TF, m=2 b=32 4.0 vs 9.6, m=2 b=64 8.1 vs
  // 13.5; at 64 columns with m >= 3 the fast kernels win: m=3 b=8 15.6 vs
  // 13.2, m=4 b=4 9.6 vs 7.1).  BCSS_FORCE_FAST keeps the fast kernels (tests).
  if ((m == 2 || std::pow((double)bA, m - 1) < 64.0) && !getenv("BCSS_FORCE_FAST")) return -1;
  int i;
  switch (bA) {
    case 4: i = 0; break;
    case 8: i = 1; break;
    case 16: i = 2; break;
    case 32: i = 3; break;
    case 64: i = 4; break;
    default: {
      int64_t pad = bA;
      const int j = np_row_group(bA, m, &pad);
      if (j < 0) return -1;
      const int np0 = 1 + bcss::N_BA * N_SHAPES + bcss::N_BA * N_GEN;
      if (pad == bA) return np0 + shape * bcss::N_NP + j;               // j indexes kNpRg
      return np0 + bcss::N_NP * N_SHAPES + shape * bcss::N_NPP + j;     // j indexes kNppRg
    }
  }
  return 1 + shape * bcss::N_BA + i;
}

// Tile-shape policy.  A parent's rows are cut into tiles of the fast shapes;
// a tile with fewer valid rows than its height skips the empty 8-row
// fragments, so its cost is the measured full-tile time scaled by
// kFragFrac (shape_costs.hpp).  The split minimizes the summed tile cost
// (knapsack over row counts).  BCSS_FORCE_SHAPE=i forces one shape.
struct ShapePolicy {
  int force = -1;
  ShapePolicy() {
    if (const char* f = getenv("BCSS_FORCE_SHAPE")) force = atoi(f);
  }
  static int table(int64_t bA) { return !is_pow2(bA) ? 4 : bA <= 4 ? 0 : bA == 8 ? 1 : bA == 16 ? 2 : 3; }
  // time (arbitrary units) of one tile of shape s holding v valid rows
  static double tile_cost(int bi, int s, int v) {
    const int bm = shape_bm(s);
    const int nf = (std::min(v, bm) + 7) / 8;
    return bm / bcss::kTileTflops[bi][s] * bcss::kFragFrac[bi][s][nf - 1];
  }
  // Row decomposition of a parent with `rows` rows into contiguous pieces,
  // each one tile shape: the full tiles of a shape form one piece, every
  // partial tile is a piece of its own.
  std::vector<std::pair<int, int>> split(int rows, int64_t bA, unsigned allowed = ~0u) const {
    if (force >= 0 && force < N_SHAPES && ((allowed >> force) & 1)) return {{force, rows}};
    const int bi = table(bA);
    std::vector<double> cost(rows + 1, 1e300);
    std::vector<int2> choice(rows + 1, int2{-1, 0});  // {shape, rows of the last tile}
    cost[0] = 0;
    for (int r = 1; r <= rows; ++r)
      for (int sidx = 0; sidx < bcss::N_POLICY_SHAPES; ++sidx) {
        if (!((allowed >> sidx) & 1)) continue;
        const int bm = shape_bm(sidx);
        const int vmax = std::min(bm, r);
        for (int nf = 1; nf <= (vmax + 7) / 8; ++nf) {  // last tile: nf valid fragments
          const int v = std::min(8 * nf, vmax);
          const double c = cost[r - v] + tile_cost(bi, sidx, v);
          if (c < cost[r] - 1e-12) { cost[r] = c; choice[r] = int2{sidx, v}; }
        }
      }
    std::map<int, int> full_rows;            // shape -> rows in full tiles
    std::vector<std::pair<int, int>> out;
    for (int r = rows; r > 0;) {
      const int2 c = choice[r];
      if (c.y == shape_bm(c.x)) full_rows[c.x] += c.y;
      else out.push_back({c.x, c.y});
      r -= c.y;
    }
    std::vector<std::pair<int, int>> pieces;
    for (auto it = full_rows.rbegin(); it != full_rows.rend(); ++it) pieces.push_back({it->first, it->second});
    pieces.insert(pieces.end(), out.begin(), out.end());
    return pieces;
  }
};

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

void build_wave_levels(bcss_plan& P, WaveHost& W, bool cascade_wave) {
  // The fast kernel needs power-of-two blocks and the insertion form of the
  // redirection; with reuse=False the levels below the top read dense block
  // tables with the identity mapping (contracted position k), which is that
  // form too - only the top level (unsorted keys into A) needs the generic kernel.
  // (any b_c: rows are (jb, c) pairs addressed by division, the tail modes
  // pass through the column index whole; the mirrored C order alone needs a
  // power-of-two b_c)
  const bool fast_shape = fast_cfg(P.bA, P.m, 0) >= 0;
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
    int n_w0_wholes = 0;  // cascade top level: leading parents of first-wave units
    if (k == P.m - 1 && P.start_level == 0) {
      const std::vector<int>& tu = W.top_units;
      for (size_t i = 0; i < tu.size(); ++i) {
        L.suffixes.push_back(tu[i]);
        L.child_call.push_back((int)i);
      }
      // contiguous runs of units; with the cascade, runs never mix first-wave
      // and later units, and the first wave's runs come first
      const bool split_w0 = cascade_wave && P.top_first;
      auto in_w0 = [&](int u) { return std::find(W.units.begin(), W.units.end(), u) != W.units.end(); };
      // X row block of unit u: u itself, or its position in the gathered X_top
      auto pos = [&](int u) {
        if (P.gather_rows.empty() || P.gather_level != k) return u;
        return (int)(std::lower_bound(P.gather_rows.begin(), P.gather_rows.end(), u) - P.gather_rows.begin());
      };
      std::vector<int4> later;
      size_t s = 0;
      while (s < tu.size()) {
        size_t e = s + 1;
        while (e < tu.size() && pos(tu[e]) == pos(tu[e - 1]) + 1 && (!split_w0 || in_w0(tu[e]) == in_w0(tu[s]))) ++e;
        const int4 par = int4{0, (int)(pos(tu[s]) * P.bC), (int)((e - s) * P.bC), (int)s};
        if (split_w0 && !in_w0(tu[s])) later.push_back(par);
        else parents.push_back(par);
        s = e;
      }
      n_w0_wholes = (int)parents.size();  // without top_first every top row belongs to the first wave
      parents.insert(parents.end(), later.begin(), later.end());
      L.n_calls = (int64_t)tu.size();
      // the lower levels of this wave start from its own units
      prev_call.assign(W.top_call.begin(), W.top_call.end());
    } else {
      int64_t running = 0;
      std::vector<int64_t> full(P.m);
      // start plan restricted to some children of its (single) start call:
      // one parent over the gathered X rows of those children
      const bool subset = k == k_first && P.start_level > 0 && !P.start_children.empty();
      for (int64_t c = 0; c < prev_calls; ++c) {
        const int32_t* sp = &prev_suffix[(size_t)(c * (sl - 1))];
        const int J = sp[0];
        std::vector<int> kids;
        if (subset) kids = P.start_children;
        else for (int jb = 0; jb <= J; ++jb) kids.push_back(jb);
        parents.push_back(int4{prev_call[(size_t)c], 0, (int)(kids.size() * P.bC), (int)running});
        for (int jb : kids) {
          L.suffixes.push_back(jb);
          for (int q = 0; q < sl - 1; ++q) L.suffixes.push_back(sp[q]);
          if (k == 0) {
            full[0] = jb;
            for (int q = 0; q < sl - 1; ++q) full[q + 1] = sp[q];
            if (P.mirror) {  // block of the original C: sorted = reversed mirrored tuple
              std::vector<int64_t> orig(P.m);
              for (int d = 0; d < P.m; ++d) orig[d] = P.pbar - 1 - full[P.m - 1 - d];
              L.child_call.push_back((int)bcss::hypertriangle_rank(orig.data(), P.m, P.pbar));
            } else {
              L.child_call.push_back((int)bcss::hypertriangle_rank(full.data(), P.m, P.pbar));
            }
          } else {
            L.child_call.push_back((int)running);
          }
          ++running;
        }
      }
      L.n_calls = running;
    }
    // b_a >= 32 levels of few rounds (e.g. config 2, and every level of a
    // multi-GPU shard) run entirely on 32x256 tiles with 16 consumer warps:
    // measured faster than the calibrated mix there (config 2: 5.09 -> 5.07
    // ms; its 8-GPU shards 0.80 -> 0.75 ms) - the finest row granularity
    // packs the last rounds best; large levels (config 5) keep the mix
    constexpr int kSmallLevelShape = 5;  // ws32x256c16 (kernel_table.cuh)
    int level_shape = -1;
    if (fast_shape && P.bA >= 32 && P.reuse && policy.force < 0 && !getenv("BCSS_NO_SMALL_LEVEL_SHAPE")) {
      const int bm = shape_bm(kSmallLevelShape), bn = bcss::kFast32[kSmallLevelShape].BN;
      double items = 0;
      for (const int4& w : parents) items += (double)((w.z + bm - 1) / bm);
      items *= (double)L.keys_out * (double)((L.rest + bn - 1) / bn);
      if (items < 148.0 * 128) level_shape = kSmallLevelShape;
    }
    // group parents into launches by tile configuration
    std::map<int, LaunchHost> by_cfg;
    for (size_t wi = 0; wi < parents.size(); ++wi) {
      const int4& whole = parents[wi];
      // a parent's rows may be split into pieces of different tile shapes; a
      // piece is a parent with a later row0 (its child index follows from
      // child_off + (jb - row0/b_c) in the epilogue)
      std::vector<std::pair<int, int>> pieces;
      const bool fast = fast_shape && (P.reuse || k < P.m - 1);
      // reuse=False top level: unsorted keys, general redirection permutations
      const bool gen = fast_shape && !fast && is_pow2(P.bA) && !getenv("BCSS_NO_GEN_TOP");
      unsigned gen_mask = 0;
      for (int g = 0; g < bcss::N_GEN; ++g) gen_mask |= 1u << bcss::BCSS_GEN_OF[g];
      if (fast && level_shape >= 0) pieces = {{level_shape, whole.z}};
      else if (fast) pieces = policy.split(whole.z, P.bA);
      else if (gen) pieces = policy.split(whole.z, P.bA, gen_mask);
      else pieces = {{-1, whole.z}};
      int r0 = 0;
      for (const auto& pc : pieces) {
        // generic kernel: the insertion-form addressing unless the level
        // redirects through general permutations (reuse=False top level)
        const int cfg = fast ? fast_cfg(P.bA, P.m, pc.first) : gen ? gen_cfg(P.bA, P.m, pc.first)
                        : (P.reuse || k < P.m - 1) ? CFG_GENERIC : CFG_GENERIC_PERM;
        int4 par = whole;
        par.y = whole.y + r0;
        par.z = pc.second;
        par.w = whole.w + r0 / (int)P.bC;
        r0 += pc.second;
        LaunchHost& X = by_cfg[cfg];
        const KernelCfg& C = kernel_cfg(cfg);
        // the generic kernel tiles the flat (key, column) space of a parent
        const bool flat = is_generic(cfg);
        if (X.parents.empty()) {
          X.cfg = cfg;
          const int64_t ncols = flat ? L.keys_out * L.rest : L.rest;
          if ((ncols + C.BN - 1) / C.BN > INT32_MAX) throw std::overflow_error("column tiles exceed int32");
          X.n_tiles = (int)((ncols + C.BN - 1) / C.BN);
          X.item_off.push_back(0);
        }
        X.parents.push_back(par);
        if ((int)wi < n_w0_wholes) X.n_w0 = (int)X.parents.size();
        X.item_off.push_back(X.item_off.back() +
                             (flat ? 1LL : (long long)L.keys_out) * X.n_tiles * ((par.z + C.BM - 1) / C.BM));
        X.flops += (uint64_t)2 * par.z * P.n * L.keys_out * L.rest;
        if (fast && pc.first >= 0 && pc.first < bcss::N_POLICY_SHAPES)  // modelled time per column (SM shares, run.cu)
          for (int r = 0; r < par.z; r += C.BM)
            X.cost += ShapePolicy::tile_cost(ShapePolicy::table(P.bA), pc.first, std::min(C.BM, par.z - r));
      }
    }
    const bool grouped = cascade_wave && k >= 1;
    for (auto& kv : by_cfg) {
      // flat work list: parent-major, then key, n-tile, m-tile (adjacent CTAs
      // share the B tile of one (key, n-tile)); cascade levels first split the
      // keys into first-index groups
      LaunchHost& X = kv.second;
      const int BM = kernel_cfg(X.cfg).BM;
      X.items.reserve((size_t)X.item_off.back());
      const int ng = grouped ? (int)P.group_a.size() - 1 : 1;
      for (int g = 0; g < ng; ++g) {
        const int64_t k_lo = grouped ? first_rank_with(P.group_a[g], k, P.nbar) : 0;
        const int64_t k_hi = grouped ? first_rank_with(P.group_a[g + 1], k, P.nbar) : L.keys_out;
        if (grouped) X.group_items.push_back((long long)X.items.size());
        for (size_t pi = 0; pi < X.parents.size(); ++pi) {
          if (grouped && (int)pi == X.n_w0) X.group_w0.push_back((long long)X.items.size());
          const int mtiles = (X.parents[pi].z + BM - 1) / BM;
          if (is_generic(X.cfg)) {  // flat (key, column) tiles (never in key-grouped cascade levels)
            if (grouped) throw std::logic_error("generic kernel in a cascade level");
            for (int nt = 0; nt < X.n_tiles; ++nt)
              for (int mt = 0; mt < mtiles; ++mt) X.items.push_back(int4{(int)pi, 0, nt, mt});
            continue;
          }
          // Tail slices: the GEMM columns' high part is the tail index (b_c
          // modes), which is also the slowest dimension of every T(k+1) block,
          // so a range of n-tiles reads one contiguous slice of each block.  A
          // parent whose T(k+1) exceeds the slice budget is walked slice by
          // slice (all keys per slice), so the k+1 reads of a block by
          // different keys meet in L2 instead of going back to HBM.
          int slices = 1;
          if (!grouped && k < P.m - 1 && P.slice_bytes > 0) {
            const double in_bytes = (double)L.keys_in * (double)L.blk_in * sizeof(double);
            slices = (int)std::min<double>((double)X.n_tiles, std::ceil(in_bytes / (double)P.slice_bytes));
            slices = std::max(slices, 1);
          }
          for (int sg = 0; sg < slices; ++sg) {
            const int nt_lo = (int)((int64_t)X.n_tiles * sg / slices), nt_hi = (int)((int64_t)X.n_tiles * (sg + 1) / slices);
            for (int64_t key = k_lo; key < k_hi; ++key)
              for (int nt = nt_lo; nt < nt_hi; ++nt)
                for (int mt = 0; mt < mtiles; ++mt) X.items.push_back(int4{(int)pi, (int)key, nt, mt});
          }
        }
        if (grouped && X.n_w0 >= (int)X.parents.size()) X.group_w0.push_back((long long)X.items.size());
      }
      if (grouped) X.group_items.push_back((long long)X.items.size());
      L.flops += kv.second.flops;
      L.launches.push_back(std::move(kv.second));
    }
    // Tail trim of a single-shape small level: when the launch's last round
    // would hold only r <= SMs/2 tiles (config 2 level 0: 3264 = 22 x 148 + 8),
    // those r tiles run as 2r half-width tiles (32x128) in a second launch, so
    // the level ends half a tile earlier.  Not for chunk-gated / grouped levels
    // (their item ranges follow keys) - and only when every tile is full.
    if (level_shape >= 0 && !grouped && L.launches.size() == 1 && (k < P.m - 1 || P.pipeline_waves <= 1) &&
        P.bC % 32 == 0 && L.rest % 256 == 0 && is_pow2(P.bA) && !getenv("BCSS_NO_TAIL_TRIM")) {
      static const int sms = [] {
        int dev = 0, v = 0;
        if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
          cudaGetLastError();
          return 148;
        }
        return v > 0 ? v : 148;
      }();
      LaunchHost& X = L.launches[0];
      const long long total = (long long)X.items.size(), r = total % sms;
      constexpr int kHalfShape = 10;  // ws32x128c16s5
      if (total > sms && r > 0 && r <= sms / 2) {
        LaunchHost T;
        T.cfg = fast_cfg(P.bA, P.m, kHalfShape);
        T.n_tiles = (int)(L.rest / kernel_cfg(T.cfg).BN);
        T.parents = X.parents;
        for (long long i = total - r; i < total; ++i) {
          const int4 it = X.items[(size_t)i];
          T.items.push_back(int4{it.x, it.y, 2 * it.z, it.w});
          T.items.push_back(int4{it.x, it.y, 2 * it.z + 1, it.w});
        }
        X.items.resize((size_t)(total - r));
        const uint64_t per = X.flops / (uint64_t)total;  // every tile is full: equal flops
        T.flops = per * (uint64_t)r;
        X.flops -= T.flops;
        X.item_off.assign({0, (long long)X.items.size()});
        T.item_off.assign({0, (long long)T.items.size()});
        L.launches.push_back(std::move(T));
      }
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
    if (getenv("BCSS_PLAN_DUMP")) {  // diagnostics: one line per launch
      for (const auto& X : L.launches) {
        std::map<int, int> rows_hist;
        for (const int4& par : X.parents) rows_hist[par.z] += 1;
        fprintf(stderr, "[bcss plan] level %d %-18s parents %zu items %lld gflop %.2f rows:", L.k,
                kernel_cfg(X.cfg).name, X.parents.size(), (long long)X.item_off.back(), X.flops / 1e9);
        for (auto& kv : rows_hist) fprintf(stderr, " %dx%d", kv.first, kv.second);
        if (!is_generic(X.cfg) && !is_pow2(P.bA)) {  // non-power-of-two b_a: its row group and padded width
          int64_t pad = P.bA;
          const int j = np_row_group(P.bA, P.m, &pad);
          if (j >= 0) fprintf(stderr, " (row group %d, b_a' %lld)", pad == P.bA ? bcss::kNpRg[j] : bcss::kNppRg[j], (long long)pad);
        }
        fprintf(stderr, "\n");
      }
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
    // contraction rows per block on the fast kernels (fixed with the plan's
    // kernel choice: the runs must not re-derive it from the environment)
    P.bAp = padded_ba(P.bA, P.m);
    // mirrored C order for pipelined full runs on the fast kernels
    P.mirror = P.pipeline_waves > 1 && !P.keep_temps && !P.units_set && P.start_level == 0 &&
               P.stop_level == 0 && P.reuse && is_pow2(P.bC) && fast_cfg(P.bA, P.m, 0) >= 0 &&
               !getenv("BCSS_NO_MIRROR");
    const bool cascade_ok = P.mirror && !getenv("BCSS_NO_CASCADE") && !P.cascade_nofit;
    P.cascade = false;  // decided by the pipeline model below
    P.group_a.clear();
    if (P.pipeline_waves > 1) {  // first-index groups of keys (A chunk boundaries of the gated top level)
      const int64_t nb = P.nbar;
      const int groups = (int)std::min<int64_t>(8, nb);
      P.group_a.push_back(0);
      for (int g = 0; g < groups; ++g)
        P.group_a.push_back(g == groups - 1 ? nb : std::max(P.group_a.back() + 1, (nb * (g + 1)) / groups));
    }
    if (!P.units_set)
      for (int u = 0; u < P.pbar; ++u) units.push_back(u);
    std::sort(units.begin(), units.end());
    units.erase(std::unique(units.begin(), units.end()), units.end());
    // shard plans with scattered units: the top level reads gathered X rows;
    // start plans with a child subset: their first level does
    P.gather_rows.clear();
    P.gather_level = -1;
    if (P.units_set && !P.mirror && P.start_level == 0 && units.size() > 1 &&
        units.back() - units.front() + 1 != (int)units.size() && !getenv("BCSS_NO_TOP_GATHER")) {
      P.gather_rows = units;
      P.gather_level = P.m - 1;
    }
    if (P.start_level > 0 && !P.start_children.empty()) {
      const int sl = P.m - P.start_level;
      if (P.start_suffixes.size() != (size_t)sl)
        return fail(BCSS_ERR_STATE, "start children need exactly one start call");
      for (int jb : P.start_children)
        if (jb > P.start_suffixes[0])
          return fail(BCSS_ERR_RANGE, "start child %d > first suffix index %d", jb, (int)P.start_suffixes[0]);
      P.gather_rows = P.start_children;
      P.gather_level = P.start_level - 1;
    }
    // pipeline groups: run_host computes T(m-1) of every unit first (it
    // overlaps the upload of A), then the groups' lower levels one after the
    // other while the previous group's C blocks download.  Contiguous groups
    // (in unit order, largest or smallest unit first) are chosen by a DP
    // over a two-resource model (device compute, then D2H of the group's C
    // blocks as runs of consecutive ranks) minimizing the last download's end.
    std::vector<std::vector<int>> groups;
    if (P.pipeline_waves > 1 && !P.keep_temps && units.size() > 1) {
      // flop/s, B/s, B/s, s per D2H copy, s per wave, s per gated sub-launch group (ramp + tail)
      const double rate_c = 33e12, rate_d = 55e9, rate_h = 55e9, t_copy = 3e-6, t_wave = 20e-6, t_sub = 25e-6;
      const int U = (int)units.size();
      const int W = std::min(P.pipeline_waves, U);
      const double blk_bytes = (double)ipow(P.bC, P.m) * sizeof(double);
      const int G = (int)P.group_a.size() - 1;
      // A chunk a (blocks of first index a) lands at t_land[a] (seconds from the upload start)
      std::vector<double> t_land(P.nbar);
      {
        double acc = 0;
        for (int64_t a = 0; a < P.nbar; ++a) {
          acc += (double)bcss::simplex_count(P.nbar - a, P.m - 1) * (double)ipow(P.bA, P.m) * sizeof(double);
          t_land[a] = acc / rate_h;
        }
      }
      const double t_up = t_land[P.nbar - 1];
      // flops of level k, key group g, for the given units (top level: all units)
      auto group_flops = [&](const std::vector<int>& us, int k, int g) {
        const double keys = (double)(first_rank_with(P.group_a[g + 1], k, P.nbar) - first_rank_with(P.group_a[g], k, P.nbar));
        return (double)calls_for(P, us, k) * 2.0 * P.bC * P.n * keys * (double)(ipow(P.bA, k) * ipow(P.bC, P.m - 1 - k));
      };
      // Compute of the first wave (units `us`) relative to the end of the upload:
      // list-schedule the gated groups (top level of all units; with the
      // cascade also the first wave's levels m-2..1) on one device at rate_c,
      // higher levels first; then the remaining levels.
      // cascade: later units' top-level rows of groups >= defer run after the first wave's level 0
      int defer = G;
      while (defer > 0 && t_land[P.group_a[defer] - 1] >= 0.85 * t_up) --defer;
      if (const char* e = getenv("BCSS_DEFER_GROUP")) defer = std::max(0, std::min(G, atoi(e)));
      auto level_flops = [&](const std::vector<int>& us, int k) {
        return (double)calls_for(P, us, k) * 2.0 * P.bC * P.n * keys_at(P, k) *
               (double)(ipow(P.bA, k) * ipow(P.bC, P.m - 1 - k));
      };
      // {end of the first wave's compute, time later waves may start}, both
      // relative to the end of the upload.  One device at rate_c list-schedules
      // the gated jobs (earliest start; ties to the first wave's chain).
      auto first_wave = [&](const std::vector<int>& us, bool cascade) -> std::pair<double, double> {
        std::vector<int> others;
        for (int u : units)
          if (std::find(us.begin(), us.end(), u) == us.end()) others.push_back(u);
        // chain jobs (k, g): cascade - the first wave's rows of levels m-1..1;
        // non-cascade - the top level of all units.  bg jobs: cascade only.
        const int kmin = cascade ? 1 : P.m - 1;
        const std::vector<int>& top_rows = cascade ? us : units;
        std::vector<std::vector<double>> done(P.m + 1, std::vector<double>(G, 0.0));
        std::vector<std::vector<bool>> fin(P.m, std::vector<bool>(G, false));
        std::vector<bool> bg_fin(G, !cascade);
        for (int g = defer; g < G; ++g) bg_fin[g] = true;  // deferred: after level 0
        double now = 0;
        for (;;) {
          int bk = -1, bgi = -1;
          double best = 1e300;
          for (int k = P.m - 1; k >= kmin; --k)
            for (int g = 0; g < G; ++g) {
              if (fin[k][g] || (g > 0 && !fin[k][g - 1])) continue;
              if (k < P.m - 1 && !fin[k + 1][g]) break;
              const double ready = std::max(k == P.m - 1 ? t_land[P.group_a[g + 1] - 1] : done[k + 1][g],
                                            g > 0 ? done[k][g - 1] : 0.0);
              const double key = std::max(ready, now);
              if (key < best - 1e-12) { best = key; bk = k; bgi = g; }
              break;
            }
          int bb = -1;
          for (int g = 0; g < G; ++g)
            if (!bg_fin[g]) {
              if (fin[P.m - 1][g]) {
                const double key = std::max(done[P.m - 1][g], now);
                if (key < best - 1e-12) { best = key; bk = -1; bb = g; }
              }
              break;
            }
          if (bk < 0 && bb < 0) break;
          if (bk >= 0) {
            now = best + group_flops(bk == P.m - 1 ? top_rows : us, bk, bgi) / rate_c + t_sub;
            done[bk][bgi] = now;
            fin[bk][bgi] = true;
          } else {
            now = best + group_flops(others, P.m - 1, bb) / rate_c + t_sub;
            bg_fin[bb] = true;
          }
        }
        double rest = 0;  // the first wave's levels below the gated ones (incl. level 0)
        for (int k = kmin - 1; k >= 0; --k) rest += level_flops(us, k);
        const double t1 = std::max(now, t_up) + rest / rate_c;
        double deferred = 0;
        if (cascade)
          for (int g = defer; g < G; ++g) deferred += group_flops(others, P.m - 1, g) + t_sub * rate_c;
        return {t1 - t_up + t_wave, t1 + deferred / rate_c - t_up + t_wave};
      };
      double mode_best[2] = {1e300, 1e300};
      std::vector<std::vector<int>> mode_groups[2];
      for (int mode = 0; mode < (cascade_ok ? 2 : 1); ++mode)
        for (int dir = 0; dir < 2; ++dir) {
          std::vector<int> order(units.begin(), units.end());
          if (dir == 0) std::reverse(order.begin(), order.end());  // largest unit first
          std::vector<double> fl(U + 1, 0.0), by(U + 1, 0.0);
          const double top = 2.0 * P.bC * P.n * keys_at(P, P.m - 1) * (double)ipow(P.bA, P.m - 1);
          for (int i = 0; i < U; ++i) {
            const int u = order[i];
            fl[i + 1] = fl[i] + unit_cost(P, u) - top;
            by[i + 1] = by[i] + (double)bcss::simplex_count(u + 1, P.m - 1) * blk_bytes;
          }
          // copies of a group of units (in value range [lo, hi]): one run per
          // sorted prefix of length m-1 whose last index is <= hi (mirrored: one)
          auto d2h = [&](int i, int j) {
            int hi = order[i];
            for (int q = i; q < j; ++q) hi = std::max(hi, order[q]);
            const double copies = P.mirror ? 1.0 : (double)bcss::simplex_count(hi + 1, P.m - 1);
            return (by[j] - by[i]) / rate_d + copies * t_copy;
          };
          for (int i1 = 1; i1 <= U; ++i1) {
            const std::pair<double, double> fw = first_wave(std::vector<int>(order.begin(), order.begin() + i1), mode == 1);
            const double tc1 = fw.first, tlater = std::max(fw.first, fw.second);
            if (getenv("BCSS_PLAN_DUMP") && atoi(getenv("BCSS_PLAN_DUMP")) > 2)
              fprintf(stderr, "[bcss plan]   mode %d dir %d first group %d units: compute %.3f ms after upload, d2h %.3f ms\n",
                      mode, dir, i1, tc1 * 1e3, d2h(0, i1) * 1e3);
            // td[g][j]: earliest end of the g-th group's download covering order[0, j)
            std::vector<std::vector<double>> td(W + 1, std::vector<double>(U + 1, 1e300));
            std::vector<std::vector<int>> from(W + 1, std::vector<int>(U + 1, -1));
            td[1][i1] = tc1 + d2h(0, i1);
            from[1][i1] = 0;
            for (int g = 2; g <= W; ++g)
              for (int j = i1 + 1; j <= U; ++j)
                for (int i = i1; i < j; ++i) {
                  if (td[g - 1][i] >= 1e299) continue;
                  const double tc = tlater + (fl[j] - fl[i1]) / rate_c + (g - 1) * t_wave;  // groups 1..g computed
                  const double t = std::max(td[g - 1][i], tc) + d2h(i, j);
                  if (t < td[g][j]) { td[g][j] = t; from[g][j] = i; }
                }
            for (int g = 1; g <= W; ++g) {
              if (td[g][U] >= mode_best[mode] - 1e-9) continue;
              mode_best[mode] = td[g][U];
              mode_groups[mode].clear();
              for (int j = U, gg = g; gg > 0; j = from[gg][j], --gg)
                mode_groups[mode].insert(mode_groups[mode].begin(),
                                         std::vector<int>(order.begin() + from[gg][j], order.begin() + j));
            }
          }
        }
      if (getenv("BCSS_PLAN_DUMP") && atoi(getenv("BCSS_PLAN_DUMP")) > 1)
        fprintf(stderr, "[bcss plan] model best: level-synchronous %.3f ms, cascade %.3f ms (after the upload)\n",
                mode_best[0] * 1e3, mode_best[1] * 1e3);
      // the cascade's model is less certain (many small gated launches): it
      // must promise a 5 % gain
      P.cascade = cascade_ok && (mode_best[1] < 0.95 * mode_best[0] || getenv("BCSS_FORCE_CASCADE"));
      groups = mode_groups[P.cascade ? 1 : 0];
      const double best_t = mode_best[P.cascade ? 1 : 0];
      // later units' top-level rows of the key groups whose chunks land in the
      // last 15 % of the upload run after the first wave's level 0
      P.defer_group = defer;
      for (auto& g : groups) std::sort(g.begin(), g.end());
      if (getenv("BCSS_PLAN_DUMP")) {
        fprintf(stderr, "[bcss plan] pipeline groups (model: %.3f ms after the upload, cascade %d):", best_t * 1e3,
                (int)P.cascade);
        for (auto& g : groups) fprintf(stderr, " [%d..%d]", g.front(), g.back());
        fprintf(stderr, "\n");
      }
    } else {
      groups.push_back(units);
    }
    // waves: greedy groups of units whose live temporaries fit the limit.  A
    // pipelined plan keeps T(m-1) of every unit resident (top-first) next to
    // the wave's lower levels, so that is what must fit.
    auto al256 = [](size_t v) { return (v + 255) / 256 * 256; };
    const size_t top_all = al256(level_bytes(P, units)[P.m - 1]);
    auto lower_bytes = [&](const std::vector<int>& us) -> size_t {
      const auto b = level_bytes(P, us);
      size_t r[2] = {0, 0};
      for (int k = 1; k < P.m - 1; ++k) r[(P.m - 2 - k) % 2] = std::max(r[(P.m - 2 - k) % 2], al256(b[k]));
      return r[0] + r[1];
    };
    bool tf_fits = true;  // every single unit fits next to the resident T(m-1)
    if (P.ws_limit > 0)
      for (int u : units) tf_fits = tf_fits && top_all + lower_bytes({u}) <= P.ws_limit;
    const bool tf_want = P.pipeline_waves > 1 && !P.keep_temps && tf_fits;
    auto wave_bytes = [&](const std::vector<int>& us) -> size_t {
      return tf_want ? top_all + lower_bytes(us) : peak_for(P, us);
    };
    P.waves.clear();
    for (const auto& grp : groups) {
      std::vector<int> cur;
      for (int u : grp) {
        std::vector<int> trial = cur;
        trial.push_back(u);
        if (!cur.empty() && !P.keep_temps && P.ws_limit > 0 && wave_bytes(trial) > P.ws_limit) {
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
        if (wave_bytes(W.units) > P.ws_limit)
          return fail(BCSS_ERR_NOMEM, "one top-level unit needs %zu workspace bytes > limit %zu",
                      wave_bytes(W.units), P.ws_limit);
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
      build_wave_levels(P, W, false);
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
    P.top_first = tf_want && P.waves.size() > 1;
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
      const bool disjoint = P.cascade && &W == &P.waves[0];  // cascade: levels overlap in time
      if (P.keep_temps || (disjoint && !P.top_first)) {
        for (int k = 1; k < P.m; ++k) { W.level_off[k] = end; end += al(b[k]); }
      } else if (disjoint) {
        W.level_off[P.m - 1] = 0;
        end = top_bytes;
        for (int k = P.m - 2; k >= 1; --k) { W.level_off[k] = end; end += al(b[k]); }
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
    if (P.cascade && P.ws_limit > 0 && P.ws_bytes > P.ws_limit) {
      // the first wave's disjoint regions do not fit: run it level-synchronously
      P.cascade_nofit = true;
      return build_plan(P);
    }
    }  // full run
    // tables
    P.nbr_off.assign(P.m, 0);
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 255) / 256 * 256; return o; };
    for (int k = 0; k < P.m; ++k)  // neighbour tables: built on the device (build_nbr_device)
      P.nbr_off[k] = take((size_t)keys_at(P, k) * (size_t)P.nbar * sizeof(int2));
    P.flops = 0;
    P.c_blocks = 0;
    const bool partial = P.start_level > 0 || P.stop_level > 0;
    for (auto& W : P.waves) {
      if (!partial) build_wave_levels(P, W, P.cascade && &W == &P.waves[0]);
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
    P.off_gather_rows = take(P.gather_rows.size() * sizeof(int));
    P.tables_bytes = off;
    P.built = true;
    return BCSS_OK;
  } catch (const std::exception& e) {
    return fail(BCSS_ERR_PARAMETER, "plan construction failed: %s", e.what());
  }
}

// ---- neighbour tables, built on the device ----------------------------------------
// The largest plan table is the neighbour table of each level: keys(k) x n/b_a
// entries {rank of the stored block sorted(K u ib) in T(k+1), code word of the
// redirection}.  It is generated straight into the device table buffer (one
// warp per key, lanes over ib), so neither its host construction nor its
// upload grows with (n/b_a)^(k+1).  Same entries as build_nbr (tested bitwise).

__device__ __forceinline__ long long dev_binom(long long n, int r) {
  if (r < 0 || n < r) return 0;
  if (r > n - r) r = (int)(n - r);
  unsigned long long acc = 1;
  for (int i = 1; i <= r; ++i) acc = acc * (unsigned long long)(n - r + i) / (unsigned long long)i;
  return (long long)acc;
}

__device__ __forceinline__ long long dev_rank(const int* idx, int m, long long extent) {
  const long long N = extent + m - 1;
  long long r = 0, cprev = -1;
  for (int t = 0; t < m; ++t) {
    const long long c = (long long)idx[t] + t;
    r += dev_binom(N - cprev - 1, m - t) - dev_binom(N - c, m - t);
    cprev = c;
  }
  return r;
}

// mode 0: sorted keys (reuse, hypertriangle order); 1: product keys with the
// general canonicalize mapping (reuse=False top level); 2: product keys of a
// dense block table (reuse=False below the top: identity mapping)
__global__ void build_nbr_kernel(int2* __restrict__ out, int k, long long nkeys, int nbar, int mode) {
  const int lane = threadIdx.x & 31;
  const long long warp0 = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long kr = warp0; kr < nkeys; kr += nwarps) {
    int key[8];
    if (mode == 0) {  // unrank kr among the nondecreasing k-tuples
      long long rank = kr;
      int lo = 0;
      for (int t = 0; t < k; ++t) {
        const int rem = k - 1 - t;
        int v = lo;
        for (;; ++v) {
          const long long cnt = rem > 0 ? dev_binom((long long)(nbar - v) + rem - 1, rem) : 1;
          if (rank < cnt) break;
          rank -= cnt;
        }
        key[t] = v;
        lo = v;
      }
    } else {
      long long r = kr;
      for (int d = k - 1; d >= 0; --d) { key[d] = (int)(r % nbar); r /= nbar; }
    }
    for (int ib = lane; ib < nbar; ib += 32) {
      int rank, code;
      if (mode == 2) {
        rank = (int)(kr * nbar + ib);
        code = k;
        for (int d = 0; d <= k; ++d) code |= d << (4 + 3 * d);
      } else {
        int idx[9], canon[9], map[9];
        for (int d = 0; d < k; ++d) idx[d] = key[d];
        idx[k] = ib;
        for (int d = 0; d <= k; ++d) canon[d] = idx[d];
        for (int a = 1; a <= k; ++a)  // insertion sort (k + 1 <= 8 entries)
          for (int b = a; b > 0 && canon[b - 1] > canon[b]; --b) {
            const int tmp = canon[b]; canon[b] = canon[b - 1]; canon[b - 1] = tmp;
          }
        unsigned used = 0;  // canonicalize: first unused position of each value
        for (int d = 0; d <= k; ++d)
          for (int q = 0; q <= k; ++q)
            if (!((used >> q) & 1u) && canon[q] == idx[d]) { used |= 1u << q; map[d] = q; break; }
        rank = (int)dev_rank(canon, k + 1, nbar);
        code = map[k];
        for (int d = 0; d <= k; ++d) code |= map[d] << (4 + 3 * d);
      }
      out[kr * nbar + ib] = make_int2(rank, code);
    }
  }
}

int build_nbr_device(const bcss_plan& P, int k, int2* dst, cudaStream_t stream) {
  const long long nkeys = keys_at(P, k);
  const int mode = P.reuse ? 0 : (k + 1 == P.m ? 1 : 2);
  const long long blocks = std::min<long long>((nkeys + 7) / 8, 148LL * 16);
  build_nbr_kernel<<<(unsigned)std::max<long long>(1, blocks), 256, 0, stream>>>(dst, k, nkeys, (int)P.nbar, mode);
  CUDA_TRY(cudaGetLastError());
  return BCSS_OK;
}

// Upload the device tables once per plan.  The copy is stream-ordered on the
// run's stream and synchronized: a plain cudaMemcpy from pageable memory can
// return before its DMA lands, and kernels on a non-blocking stream would
// then race it.
int upload_tables(bcss_plan& P, cudaStream_t stream) {
  int dev;
  CUDA_TRY(cudaGetDevice(&dev));
  if (P.d_tables && P.device == dev) return BCSS_OK;
  if (P.d_tables || (P.d_ws && P.device >= 0 && P.device != dev))
    // tables, workspace and host-run buffers live on the device of the first
    // run; a plan is bound to it
    return fail(BCSS_ERR_STATE, "plan is bound to device %d but device %d is current", P.device, dev);
  std::vector<char> host(P.tables_bytes, 0);
  for (auto& W : P.waves)
    for (auto& L : W.levels) {
      for (auto& X : L.launches) {
        memcpy(&host[X.off_parents], X.parents.data(), X.parents.size() * sizeof(int4));
        memcpy(&host[X.off_items], X.items.data(), X.items.size() * sizeof(int4));
      }
      memcpy(&host[L.off_child], L.child_call.data(), L.child_call.size() * sizeof(int));
    }
  if (!P.gather_rows.empty())
    memcpy(&host[P.off_gather_rows], P.gather_rows.data(), P.gather_rows.size() * sizeof(int));
  CUDA_TRY(cudaMalloc(&P.d_tables, std::max<size_t>(P.tables_bytes, 256)));
  CUDA_TRY(cudaMemcpyAsync(P.d_tables, host.data(), P.tables_bytes, cudaMemcpyHostToDevice, stream));
  int st;
  for (int k = 0; k < P.m; ++k)  // neighbour tables: generated on the device over the zeroed slots
    if ((st = build_nbr_device(P, k, reinterpret_cast<int2*>(static_cast<char*>(P.d_tables) + P.nbr_off[k]), stream)))
      return st;
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
  // the neighbour-table code word packs each mode's stored position in 3 bits
  if (m > 8) return fail(BCSS_ERR_PARAMETER, "order %d > 8 is not supported (at most 8 modes)", m);
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

// The device tables hold block ranks, key indices, call indices and C block
// ranks as int32 (nbr {rank, code}, work items {parent, key, ..}, parents
// {in_call, row0, rows, child_off}, child_call): reject problems whose counts
// would not fit instead of truncating them.
int check_int32_limits(int m, int64_t n, int64_t p, int64_t b_a, int64_t b_c, bool reuse) {
  const int64_t nbar = n / b_a, pbar = p / b_c, lim = INT32_MAX;
  auto too_big = [&](const char* what, long double v) {
    return fail(BCSS_ERR_PARAMETER, "%s (%.4Lg) exceeds the int32 range of the device tables", what, v);
  };
  try {
    // blocks of A and C (ranks in the neighbour table / child_call)
    if (bcss::simplex_count(nbar, m) > lim) return too_big("number of canonical blocks of A", (long double)bcss::simplex_count(nbar, m));
    if (bcss::simplex_count(pbar, m) > lim) return too_big("number of canonical blocks of C", (long double)bcss::simplex_count(pbar, m));
    for (int k = 1; k < m; ++k) {
      // keys of T(k) (work-item key, neighbour rank into T(k+1))
      const long double keys = reuse ? (long double)bcss::simplex_count(nbar, k) : powl((long double)nbar, k);
      if (keys * nbar > lim) return too_big("neighbour-table entries of one level", keys * nbar);
      // calls of level k (call indices), and rows of one parent (child rows)
      if (bcss::simplex_count(pbar, m - k) > lim) return too_big("calls of one level", (long double)bcss::simplex_count(pbar, m - k));
    }
    if ((long double)pbar * b_c > lim) return too_big("rows of one parent", (long double)pbar * b_c);
  } catch (const std::exception& e) {
    return fail(BCSS_ERR_PARAMETER, "problem size overflows: %s", e.what());
  }
  return BCSS_OK;
}

void invalidate(bcss_plan* P) {
  P->built = false;
  P->cascade_nofit = false;
  if (P->d_tables) { cudaFree(P->d_tables); P->d_tables = nullptr; }
}


}  // namespace bcss_host
