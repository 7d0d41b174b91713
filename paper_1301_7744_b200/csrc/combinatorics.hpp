// Combinatorics of BCSS block indices (host side, header-only).
//
// Restates, in integer arithmetic, the reference's
//   simplex_count        /root/reference/pkg/src/blocksym/indexing.py:64-68
//   hypertriangle_iter   /root/reference/pkg/src/blocksym/indexing.py:57-61 (lex order)
//   canonicalize         /root/reference/pkg/src/blocksym/indexing.py:34-54
//   bcss_costs(...).flops /root/reference/pkg/src/blocksym/costs.py:83-112
// The packed payload order of A, C and of every temporary is the
// hypertriangle (lexicographic) order, so a block's rank is its slot.
#pragma once

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <vector>

namespace bcss {

// Binomial coefficient C(n, r) in 128-bit, throwing on int64 overflow.
inline int64_t binom(int64_t n, int64_t r) {
  if (r < 0 || n < 0 || r > n) return 0;
  r = std::min(r, n - r);
  __int128 acc = 1;
  for (int64_t i = 1; i <= r; ++i) {
    acc = acc * (n - r + i) / i;  // exact: product of i consecutive integers / i!
    if (acc > (__int128)INT64_MAX) throw std::overflow_error("binomial overflows int64");
  }
  return (int64_t)acc;
}

// Number of nondecreasing m-tuples over 0..extent-1 (indexing.py:64-68).
inline int64_t simplex_count(int64_t extent, int m) {
  if (extent < 1 || m < 1) return m == 0 ? 1 : 0;
  return binom(extent + m - 1, m);
}

// Lexicographic rank of a nondecreasing tuple among hypertriangle_iter(extent, m).
// With c_t = idx[t] + t (strictly increasing over N = extent + m - 1 values,
// c_{-1} = -1) the tuples before idx number
//   sum_t sum_{v = c_{t-1}+1}^{c_t - 1} C(N-1-v, m-1-t)
// and the hockey-stick identity collapses each inner sum:
//   sum_t [ C(N - c_{t-1} - 1, m - t) - C(N - c_t, m - t) ]     (O(m) binomials)
template <class I>
inline int64_t hypertriangle_rank(const I* idx, int m, int64_t extent) {
  const int64_t N = extent + m - 1;
  int64_t r = 0, cprev = -1;
  for (int t = 0; t < m; ++t) {
    const int64_t c = (int64_t)idx[t] + t;
    r += binom(N - cprev - 1, m - t) - binom(N - c, m - t);
    cprev = c;
  }
  return r;
}

inline void hypertriangle_unrank(int64_t rank, int m, int64_t extent, int64_t* idx) {
  int64_t lo = 0;
  for (int t = 0; t < m; ++t) {
    const int rem = m - 1 - t;
    int64_t v = lo;
    for (;; ++v) {
      const int64_t cnt = rem > 0 ? simplex_count(extent - v, rem) : 1;
      if (rank < cnt) break;
      rank -= cnt;
    }
    idx[t] = v;
    lo = v;
  }
}

// All nondecreasing m-tuples over 0..extent-1 in lex order (row-major, m per row).
inline std::vector<int32_t> hypertriangle_list(int64_t extent, int m) {
  std::vector<int32_t> out;
  if (m == 0) return out;
  std::vector<int32_t> cur(m, 0);
  for (;;) {
    out.insert(out.end(), cur.begin(), cur.end());
    int t = m - 1;
    while (t >= 0 && cur[t] == extent - 1) --t;
    if (t < 0) break;
    ++cur[t];
    for (int u = t + 1; u < m; ++u) cur[u] = cur[t];
  }
  return out;
}

// canonicalize(idx): sorted copy plus the lexicographically smallest mapping
// with canonical[mapping[d]] == idx[d] (first unused position of each value).
inline void canonical_mapping(const int32_t* idx, int m, int32_t* canonical, int32_t* mapping) {
  std::copy(idx, idx + m, canonical);
  std::sort(canonical, canonical + m);
  std::vector<char> used(m, 0);
  for (int d = 0; d < m; ++d) {
    for (int q = 0; q < m; ++q) {
      if (!used[q] && canonical[q] == idx[d]) { used[q] = 1; mapping[d] = q; break; }
    }
  }
}

// Exact blocked flop count (costs.py:83-112).  The (b_c/b_a)^d factors are kept
// exact by scaling every term to the common denominator b_a^(m-1).
inline uint64_t blocked_flops(int m, int64_t n, int64_t p, int64_t b_a, int64_t b_c, bool reuse) {
  const int64_t nbar = n / b_a, pbar = p / b_c;
  // flops = 2*nbar*b_c * sum_d C(pbar+d, d+1) * blocks(d) * b_c^d * b_a^(m-d)
  unsigned __int128 total = 0;
  for (int d = 0; d < m; ++d) {
    unsigned __int128 term = (unsigned __int128)binom(pbar + d, d + 1);
    int64_t blocks;
    if (reuse) {
      blocks = (m - d - 1 >= 1) ? simplex_count(nbar, m - d - 1) : 1;
    } else {
      blocks = 1;
      for (int q = 0; q < m - 1 - d; ++q) blocks *= nbar;
    }
    term *= (unsigned __int128)blocks;
    for (int q = 0; q < d; ++q) term *= (unsigned __int128)b_c;
    for (int q = 0; q < m - d; ++q) term *= (unsigned __int128)b_a;
    total += term;
  }
  total *= (unsigned __int128)(2 * nbar * b_c);
  if (total > (unsigned __int128)UINT64_MAX) throw std::overflow_error("flop count overflows uint64");
  return (uint64_t)total;
}

}  // namespace bcss
