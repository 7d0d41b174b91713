// Blocked symmetrization of a packed BCSS payload on the device: the
// counterpart of the reference's `symmetrize` (change_of_basis.py:287-295;
// diagonal blocks of C carry 1-ulp asymmetry).
//
// A canonical block whose key repeats an index (a run of equal entries in the
// sorted key) is symmetric in the modes of every run; averaging over the
// permutations of those modes makes the tensor the payload represents exactly
// symmetric.  Each element belongs to one orbit of the product of the runs'
// permutation groups; the thread of the orbit's representative (digits
// nondecreasing inside every run) sums the orbit's distinct elements and
// writes their mean back to all of them, so the update is in place and every
// orbit ends with one value (exact symmetry, not just to rounding).
// HBM-bound byte work: each affected element is read once and written once.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "plan.hpp"

namespace {

constexpr int kMaxM = 8;

// next lexicographic arrangement of v[lo..hi) (std::next_permutation)
__device__ __forceinline__ bool next_perm(int* v, int lo, int hi) {
  if (hi - lo < 2) return false;
  int i = hi - 2;
  while (i >= lo && v[i] >= v[i + 1]) --i;
  if (i < lo) {  // last arrangement: wrap to the first (sorted) one
    for (int a = lo, b = hi - 1; a < b; ++a, --b) { const int t = v[a]; v[a] = v[b]; v[b] = t; }
    return false;
  }
  int j = hi - 1;
  while (v[j] <= v[i]) --j;
  { const int t = v[i]; v[i] = v[j]; v[j] = t; }
  for (int a = i + 1, b = hi - 1; a < b; ++a, --b) { const int t = v[a]; v[a] = v[b]; v[b] = t; }
  return true;
}

// blocks[i] = rank of a block with repeats, runs[i] = bit d (d >= 1) set when
// key[d] == key[d-1]
__global__ void symmetrize_kernel(double* __restrict__ payload, const int* __restrict__ blocks,
                                  const unsigned* __restrict__ runs, long long nblk, int m, int b,
                                  long long blk_elems) {
  const long long total = nblk * blk_elems;
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < total;
       g += (long long)gridDim.x * blockDim.x) {
    const long long bi = g / blk_elems;
    long long e = g - bi * blk_elems;
    const unsigned run = __ldg(runs + bi);
    int dig[kMaxM];
    for (int d = 0; d < m; ++d) { dig[d] = (int)(e % b); e /= b; }
    bool rep = true;  // digits nondecreasing inside every run of equal key entries
    for (int d = 1; d < m; ++d)
      if (((run >> d) & 1u) && dig[d] < dig[d - 1]) rep = false;
    if (!rep) continue;
    int lo[kMaxM], hi[kMaxM], nr = 0;
    for (int d = 0; d < m;) {
      int q = d + 1;
      while (q < m && ((run >> q) & 1u)) ++q;
      if (q - d > 1) { lo[nr] = d; hi[nr] = q; ++nr; }
      d = q;
    }
    double* blk = payload + (long long)__ldg(blocks + bi) * blk_elems;
    auto offset = [&](const int* v) {
      long long o = 0;
      for (int d = m - 1; d >= 0; --d) o = o * b + v[d];
      return o;
    };
    // odometer over the runs' distinct arrangements (starts and ends sorted)
    int v[kMaxM];
    for (int d = 0; d < m; ++d) v[d] = dig[d];
    double sum = 0.0;
    long long cnt = 0;
    for (;;) {
      sum += blk[offset(v)];
      ++cnt;
      int r = 0;
      while (r < nr && !next_perm(v, lo[r], hi[r])) ++r;
      if (r == nr) break;
    }
    const double mean = sum / (double)cnt;
    for (;;) {
      blk[offset(v)] = mean;
      int r = 0;
      while (r < nr && !next_perm(v, lo[r], hi[r])) ++r;
      if (r == nr) break;
    }
  }
}

}  // namespace

using namespace bcss_host;

extern "C" int bcss_symmetrize_blocks(double* payload, int m, int64_t dim, int64_t b, void* stream) {
  if (!payload) return fail(BCSS_ERR_PARAMETER, "null payload");
  if (m < 1 || m > kMaxM) return fail(BCSS_ERR_PARAMETER, "order %d outside 1..%d", m, kMaxM);
  if (b < 1 || dim % b) return fail(BCSS_ERR_BLOCK_DIVISIBILITY, "block dimension %lld does not divide %lld",
                                    (long long)b, (long long)dim);
  const int64_t grid = dim / b;
  std::vector<int> blocks;
  std::vector<unsigned> runs;
  try {
    const std::vector<int32_t> keys = bcss::hypertriangle_list(grid, m);
    const int64_t n = (int64_t)keys.size() / m;
    for (int64_t r = 0; r < n; ++r) {
      unsigned run = 0;
      for (int d = 1; d < m; ++d)
        if (keys[(size_t)(r * m + d)] == keys[(size_t)(r * m + d - 1)]) run |= 1u << d;
      if (run) { blocks.push_back((int)r); runs.push_back(run); }
    }
  } catch (const std::exception& e) {
    return fail(BCSS_ERR_PARAMETER, "%s", e.what());
  }
  if (blocks.empty()) return BCSS_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int* d_blocks = nullptr;
  unsigned* d_runs = nullptr;
  CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&d_blocks), blocks.size() * sizeof(int), s));
  CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&d_runs), runs.size() * sizeof(unsigned), s));
  CUDA_TRY(cudaMemcpyAsync(d_blocks, blocks.data(), blocks.size() * sizeof(int), cudaMemcpyHostToDevice, s));
  CUDA_TRY(cudaMemcpyAsync(d_runs, runs.data(), runs.size() * sizeof(unsigned), cudaMemcpyHostToDevice, s));
  long long be = 1;
  for (int d = 0; d < m; ++d) be *= b;
  const long long total = (long long)blocks.size() * be;
  const unsigned grid_sz = (unsigned)std::min<long long>((total + 255) / 256, 148LL * 32);
  symmetrize_kernel<<<grid_sz, 256, 0, s>>>(payload, d_blocks, d_runs, (long long)blocks.size(), m, (int)b, be);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaFreeAsync(d_blocks, s));
  CUDA_TRY(cudaFreeAsync(d_runs, s));
  // the host vectors were copied by pageable cudaMemcpyAsync, which returns
  // only after staging them, so they may go out of scope here
  return BCSS_OK;
}
