// Symmetric-aware upload of a packed BCSS payload (pipelined host runs).
//
// A canonical block whose key repeats an index is symmetric in the modes of
// every run of equal key entries (a BCSS tensor represents a symmetric tensor;
// the reference's compress(t, b, tol=0) stores exactly symmetric blocks,
// storage.py:177-216).  Only one element per orbit carries information, so the
// upload moves:
//   * blocks with distinct key entries: whole, by DMA (cudaMemcpyAsync of runs
//     of consecutive ranks, copy_in stream, one event per first-index chunk);
//   * blocks with repeats: only the 32-byte sectors that hold an orbit
//     representative (digits nondecreasing inside every run), read straight
//     from mapped pinned host memory by a persistent streaming kernel on a few
//     SMs (zero-copy: SM loads skip the sectors nobody asks for; one warp per
//     block, blocks taken in chunk order from a ticket counter, a per-chunk
//     counter bumped after each block);
//   * then, per chunk, a short fill kernel on a high-priority stream (it waits
//     for the chunk's counter with a stream wait-value operation) writes every
//     other element of the chunk's repeated-key blocks from its representative
//     in HBM and records the chunk's fill event.
// The compute streams wait for the chunk's DMA event and fill event.  For
// config 5 (m=4, n=512, b=32) 72 % of A's bytes cross PCIe.
//
// The streaming kernel of call i+1 is launched right behind call i's (so it
// takes the SMs call i's kernel frees) and spins, on the device, until the
// previous call on its device buffer set has finished computing (a flag the
// compute stream writes with cuStreamWriteValue32); the compute launches of a
// symmetric-upload run leave those SMs free.  Counters, tickets and flags are
// cumulative across calls, so nothing is reset between them.
//
// Results are bitwise those of the full upload when the repeated-key blocks
// are exactly symmetric (compress(..., tol=0), bcss_symmetrize_blocks); for
// blocks symmetric to rounding (the reference's random_bcss: about 1 ulp)
// every orbit contributes its representative's value.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <string>
#include <vector>

#include "plan.hpp"

namespace {

// Element e of a block (32-bit: blocks of < 2^31 doubles) has digits
// d_j = (e >> j*lb) & (b-1), mode 0 least significant.  `run` bit j (j >= 1)
// says modes j-1 and j are a run of equal key entries.
template <int M>
__device__ __forceinline__ void digits(unsigned e, int lb, int (&d)[M]) {
  const unsigned mask = (1u << lb) - 1u;
#pragma unroll
  for (int j = 0; j < M; ++j) d[j] = (int)((e >> (j * lb)) & mask);
}

// the 32-byte sector (4 doubles along mode 0) of this element is uploaded: it
// holds an orbit representative (nondecreasing digits inside every run)
template <int M>
__device__ __forceinline__ bool fetched(const int (&d)[M], unsigned run) {
  bool ok = !((run >> 1) & 1u) || (d[0] >> 2) <= (d[1] >> 2);
#pragma unroll
  for (int j = 2; j < M; ++j) ok = ok && (!((run >> j) & 1u) || d[j - 1] <= d[j]);
  return ok;
}

// representative of element d: digits sorted inside every run
template <int M>
__device__ __forceinline__ unsigned rep_of(int (&d)[M], unsigned run, int passes, int lb) {
  for (int pass = 0; pass < passes; ++pass)
#pragma unroll
    for (int j = 1; j < M; ++j)
      if (((run >> j) & 1u) && d[j - 1] > d[j]) { const int x = d[j]; d[j] = d[j - 1]; d[j - 1] = x; }
  unsigned r = 0;
#pragma unroll
  for (int j = M - 1; j >= 0; --j) r = (r << lb) | (unsigned)d[j];
  return r;
}

__device__ __forceinline__ int bubble_passes(unsigned run, int m) {
  int passes = 0;  // longest run of equal key entries - 1
  for (int d = 1, len = 0; d < m; ++d) {
    len = ((run >> d) & 1u) ? len + 1 : 0;
    passes = len > passes ? len : passes;
  }
  return passes;
}

struct UploadArgs {
  const double* src;          // device-mapped pointer of the pinned host payload
  double* dst;                // device payload
  const int* rank;            // per repeated-key block (chunk order)
  const unsigned* run;        // bit d (d >= 1): key[d] == key[d-1]
  const int* chunk;           // first key index of each repeated-key block
  unsigned* ctr;              // per-chunk uploaded blocks (cumulative)
  unsigned long long* work;   // ticket counter (cumulative)
  unsigned long long base;    // tickets issued before this upload
  const unsigned* set_free;   // computes finished on this device buffer set
  unsigned set_target;        // ... needed before dst may be overwritten
  long long n_diag;           // blocks on the zero-copy list
  long long blk;              // b^m
  int lb;                     // log2 b (b >= 4)
};

// Streaming half: one warp per repeated-key block, only the representatives'
// sectors, U1 16-byte zero-copy loads in flight per lane.
#ifndef BCSS_SYM_THREADS
#define BCSS_SYM_THREADS 512
#endif
constexpr int kSymThreads = BCSS_SYM_THREADS;
template <int M>
__global__ void __launch_bounds__(kSymThreads, 1) sym_upload_kernel(const UploadArgs a) {
#ifndef BCSS_SYM_U1
#define BCSS_SYM_U1 12
#endif
  constexpr int U1 = BCSS_SYM_U1;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    // the previous call on this buffer set must have stopped reading dst;
    // a broken pipeline must not hang the GPU: give up after ~60 s
    long long spins = 0;
    while (true) {
      unsigned v;
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.set_free) : "memory");
      if ((int)(v - a.set_target) >= 0) break;
      __nanosleep(2000);
      if (++spins > 30000000LL) __trap();
    }
  }
  __syncthreads();
  const unsigned blk = (unsigned)a.blk;
  const unsigned pairs = blk >> 1;
  for (;;) {
    unsigned long long tk = 0;
    if (lane == 0) tk = atomicAdd(a.work, 1ull);
    const long long t = (long long)(__shfl_sync(0xffffffffu, tk, 0) - a.base);
    if (t >= a.n_diag) break;
    const unsigned run = __ldg(a.run + t);
    const long long off = (long long)__ldg(a.rank + t) * a.blk;
    const double2* src = reinterpret_cast<const double2*>(a.src + off);
    double2* dst = reinterpret_cast<double2*>(a.dst + off);
    if (run == 0) {  // a distinct-key block: all of it, no predicates
      for (unsigned p0 = lane; p0 < pairs; p0 += 32 * U1) {
        double2 v[U1];
#pragma unroll
        for (int u = 0; u < U1; ++u)
          if (p0 + 32 * u < pairs) v[u] = src[p0 + 32 * u];
#pragma unroll
        for (int u = 0; u < U1; ++u)
          if (p0 + 32 * u < pairs) dst[p0 + 32 * u] = v[u];
      }
    } else
    for (unsigned p0 = lane; p0 < pairs; p0 += 32 * U1) {  // a pair shares a sector
      double2 v[U1];
      bool need[U1];
#pragma unroll
      for (int u = 0; u < U1; ++u) {
        const unsigned p = p0 + 32 * u;
        int d[M];
        digits<M>(p << 1, a.lb, d);
        need[u] = p < pairs && fetched<M>(d, run);
        if (need[u]) v[u] = src[p];
      }
#pragma unroll
      for (int u = 0; u < U1; ++u)
        if (need[u]) dst[p0 + 32 * u] = v[u];
    }
    __syncwarp();
    if (lane == 0) {
      __threadfence();  // the block's stores before its chunk counter
      atomicAdd(a.ctr + __ldg(a.chunk + t), 1u);
    }
  }
}

// Fill half, one launch per chunk: blockIdx.y = repeated-key block of the
// chunk, threads over its elements; every element left out gets its
// representative's value (uploaded, same block: no element is both read and
// written).  HBM/L2-bound, U loads in flight per thread.
template <int M>
__global__ void __launch_bounds__(256) sym_fill_kernel(double* __restrict__ dst, const int* __restrict__ rank,
                                                      const unsigned* __restrict__ runs, long long blk, int lb) {
  constexpr int U = 8;
  const unsigned run = __ldg(runs + blockIdx.y);
  const int passes = bubble_passes(run, M);
  double* base = dst + (long long)__ldg(rank + blockIdx.y) * blk;
  const unsigned n = (unsigned)blk;
  for (unsigned e0 = blockIdx.x * blockDim.x * U + threadIdx.x; e0 < n; e0 += gridDim.x * blockDim.x * U) {
    unsigned r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const unsigned e = e0 + u * blockDim.x;
      int d[M];
      digits<M>(e, lb, d);
      r[u] = (e < n && !fetched<M>(d, run)) ? rep_of<M>(d, run, passes, lb) : 0xffffffffu;
    }
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (r[u] != 0xffffffffu) v[u] = base[r[u]];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (r[u] != 0xffffffffu) base[e0 + u * blockDim.x] = v[u];
  }
}

using UploadFn = void (*)(const UploadArgs&, int, cudaStream_t);
template <int M>
void upload_m(const UploadArgs& a, int ctas, cudaStream_t s) {
  sym_upload_kernel<M><<<ctas, kSymThreads, 0, s>>>(a);
}
using FillFn = void (*)(double*, const int*, const unsigned*, long long, int, dim3, cudaStream_t);
template <int M>
void fill_m(double* dst, const int* rank, const unsigned* runs, long long blk, int lb, dim3 grid, cudaStream_t s) {
  sym_fill_kernel<M><<<grid, 256, 0, s>>>(dst, rank, runs, blk, lb);
}

using WaitFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using WriteFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
template <class F>
F driver_fn(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return reinterpret_cast<F>(p);
}
WaitFn wait_value_fn() {
  static WaitFn fn = driver_fn<WaitFn>("cuStreamWaitValue32");
  return fn;
}
WriteFn write_value_fn() {
  static WriteFn fn = driver_fn<WriteFn>("cuStreamWriteValue32");
  return fn;
}

int64_t binom(int64_t n, int64_t k) {
  if (k < 0 || n < k) return 0;
  int64_t r = 1;
  for (int64_t i = 1; i <= k; ++i) r = r * (n - k + i) / i;
  return r;
}

// doubles uploaded for one block with the given run bits (sector granular)
int64_t fetched_elems(unsigned run, int m, int64_t b) {
  int64_t total = 1;
  for (int d = 0; d < m;) {
    int q = d + 1;
    while (q < m && ((run >> q) & 1u)) ++q;
    const int r = q - d;  // run of r equal key entries: modes d..q-1
    if (d > 0 || r == 1) {
      total *= binom(b + r - 1, r);  // nondecreasing r-tuples
    } else {
      // first run, mode 0 by sectors: rows (d1 <= ... <= d_{r-1}) carry the
      // sectors of mode 0 up to d1's
      int64_t s = 0;
      for (int64_t d1 = 0; d1 < b; ++d1)
        s += binom(b - d1 + r - 3, r - 2) * std::min<int64_t>(b, (d1 / 4 + 1) * 4);
      total *= s;
    }
    d = q;
  }
  return total;
}

}  // namespace

namespace bcss_host {

bool sym_eligible(const bcss_plan& P) {
  return P.sym_upload && P.m >= 2 && P.m <= 8 && is_pow2(P.bA) && P.bA >= 4 && ipow(P.bA, P.m) < (int64_t(1) << 31);
}

bool sym_supported() { return wait_value_fn() != nullptr && write_value_fn() != nullptr; }

int sym_prepare(bcss_plan& P) {
  if (P.sym_built) return BCSS_OK;
  const int m = P.m;
  const int64_t nb = P.nbar;
  const int64_t blk = ipow(P.bA, m);
  std::vector<int32_t> keys;
  try {
    keys = bcss::hypertriangle_list(nb, m);
  } catch (const std::exception& e) {
    return fail(BCSS_ERR_PARAMETER, "%s", e.what());
  }
  const int64_t n = (int64_t)keys.size() / m;
  std::vector<unsigned> run_of((size_t)n, 0);
  std::vector<std::vector<std::pair<int64_t, int64_t>>> runs((size_t)nb);
  int64_t n_runs = 0, distinct = 0;
  for (int64_t r = 0; r < n; ++r) {
    const int32_t* k = &keys[(size_t)(r * m)];
    unsigned run = 0;
    for (int d = 1; d < m; ++d)
      if (k[d] == k[d - 1]) run |= 1u << d;
    run_of[(size_t)r] = run;
    if (!run) {
      auto& rs = runs[(size_t)k[0]];
      if (!rs.empty() && rs.back().second == r) rs.back().second = r + 1;
      else { rs.emplace_back(r, r + 1); ++n_runs; }
      ++distinct;
    }
  }
  // distinct-key blocks go by DMA: while the previous call computes, zero-copy
  // reads from the SMs get ~23 GB/s (51 alone) but the copy engines keep
  // ~49 GB/s, even in the short runs of small blocks (config 4 streamed:
  // 26.3 ms with DMA, 28.3 ms with every block on the zero-copy kernel).
  // BCSS_SYM_DMA=0 puts them on the kernel (whole blocks, nothing to fill).
  (void)n_runs;
  (void)distinct;
  P.sym_dma = true;
  if (const char* e = getenv("BCSS_SYM_DMA")) P.sym_dma = atoi(e) != 0;
  P.sym_runs.assign((size_t)nb, {});
  if (P.sym_dma) P.sym_runs = runs;
  P.sym_nzc.assign((size_t)nb, 0);
  P.sym_nfill.assign((size_t)nb, 0);
  P.sym_h_rank.clear(); P.sym_h_chunk.clear(); P.sym_h_run.clear();
  P.sym_h_frank.clear(); P.sym_h_frun.clear();
  P.sym_fetch_elems = 0;
  for (int64_t r = 0; r < n; ++r) {  // packed order is chunk order
    const int a = keys[(size_t)(r * m)];
    const unsigned run = run_of[(size_t)r];
    if (run || !P.sym_dma) {
      P.sym_h_rank.push_back((int)r);
      P.sym_h_chunk.push_back(a);
      P.sym_h_run.push_back(run);
      ++P.sym_nzc[(size_t)a];
    }
    if (run) {
      P.sym_h_frank.push_back((int)r);
      P.sym_h_frun.push_back(run);
      ++P.sym_nfill[(size_t)a];
    }
    P.sym_fetch_elems += run ? fetched_elems(run, m, P.bA) : blk;
  }
  P.sym_n_zc = (int64_t)P.sym_h_rank.size();
  P.sym_built = true;
  return BCSS_OK;
}

// device tables and counters of the symmetric upload (on first use):
// [0,64) ticket counter, [64,128) per-set "computes done" flags, then the
// per-chunk counters and the tables
int sym_device(bcss_plan& P) {
  if (P.d_sym) return BCSS_OK;
  const int64_t nb = P.nbar;
  const size_t nd = P.sym_h_rank.size(), nf = P.sym_h_frank.size();
  const size_t head = 128 + (size_t)nb * sizeof(unsigned);
  const size_t bytes = head + nd * (2 * sizeof(int) + sizeof(unsigned)) + nf * (sizeof(int) + sizeof(unsigned));
  CUDA_TRY(cudaMalloc(&P.d_sym, bytes));
  char* base = static_cast<char*>(P.d_sym);
  P.d_sym_work = reinterpret_cast<unsigned long long*>(base);
  P.d_sym_free = reinterpret_cast<unsigned*>(base + 64);
  P.d_sym_ctr = reinterpret_cast<unsigned*>(base + 128);
  int* d_rank = reinterpret_cast<int*>(base + head);
  int* d_chunk = d_rank + nd;
  unsigned* d_run = reinterpret_cast<unsigned*>(d_chunk + nd);
  int* d_frank = reinterpret_cast<int*>(d_run + nd);
  unsigned* d_frun = reinterpret_cast<unsigned*>(d_frank + nf);
  CUDA_TRY(cudaMemset(base, 0, head));
  if (nf) {
    CUDA_TRY(cudaMemcpy(d_frank, P.sym_h_frank.data(), nf * sizeof(int), cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(d_frun, P.sym_h_frun.data(), nf * sizeof(unsigned), cudaMemcpyHostToDevice));
  }
  P.d_sym_frank = d_frank;
  P.d_sym_frun = d_frun;
  if (nd) {
    CUDA_TRY(cudaMemcpy(d_rank, P.sym_h_rank.data(), nd * sizeof(int), cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(d_chunk, P.sym_h_chunk.data(), nd * sizeof(int), cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(d_run, P.sym_h_run.data(), nd * sizeof(unsigned), cudaMemcpyHostToDevice));
  }
  P.d_sym_rank = d_rank;
  P.d_sym_chunk = d_chunk;
  P.d_sym_run = d_run;
  P.sym_uploads = 0;
  P.sym_ticket_base = 0;
  P.sym_set_issued[0] = P.sym_set_issued[1] = 0;
  P.sym_set_released[0] = P.sym_set_released[1] = 0;
  return BCSS_OK;
}

// SMs (one CTA each) for the streaming kernel, measured on config 5
// (tools/sym_upload_timing.py): streamed calls 4 / 5 / 6 / 8 / 10 / 12 CTAs ->
// 516 / 510 / 507 / 495 / 493 / 507 ms per call, synchronous calls 6 / 8 / 10
// -> 639 / 645 / 657 ms.  BCSS_SYM_CTAS overrides both.
int sym_upload_ctas(bool async) {
  static int env = [] {
    const char* e = getenv("BCSS_SYM_CTAS");
    return e ? std::max(1, atoi(e)) : 0;
  }();
  return env ? env : (async ? 8 : 6);
}

// Issue one symmetric upload of A (pinned host `A`, device `dA`, buffer set
// `set`): the DMA half on copy_in (chunk events), the streaming kernel on
// P->sym_stream, the per-chunk fills on P->fill_stream (fill events).
int sym_upload_issue(bcss_plan* P, const double* A, double* dA, int set, bool async, bool green,
                     cudaStream_t copy_in, cudaStream_t up_stream, Pipe& pipe) {
  const size_t blk = (size_t)ipow(P->bA, P->m);
  int st = sym_device(*P);
  if (st) return st;
  const double* srcd = nullptr;
  if (P->sym_n_zc) CUDA_TRY(cudaHostGetDevicePointer((void**)&srcd, const_cast<double*>(A), 0));
  // one call's upload at a time on PCIe: this call's DMA starts when the
  // previous call's zero-copy half has landed (otherwise it takes the link
  // from that kernel and the previous call's last chunks arrive late)
  if (!P->sym_prev_done) CUDA_TRY(cudaEventCreateWithFlags(&P->sym_prev_done, cudaEventDisableTiming));
  else CUDA_TRY(cudaStreamWaitEvent(copy_in, P->sym_prev_done, 0));
  for (int64_t a = 0; a < P->nbar; ++a) {
    for (const auto& r : P->sym_runs[(size_t)a])
      CUDA_TRY(cudaMemcpyAsync(dA + (size_t)r.first * blk, A + (size_t)r.first * blk,
                               (size_t)(r.second - r.first) * blk * sizeof(double), cudaMemcpyHostToDevice, copy_in));
    CUDA_TRY(cudaEventRecord(P->chunk_ev[(size_t)a], copy_in));
  }
  pipe.fill_ev = nullptr;
  if (P->sym_n_zc == 0) return BCSS_OK;
  // keep the cumulative chunk counters inside 32 bits (rare reset)
  int64_t maxd = 0;
  for (int64_t v : P->sym_nzc) maxd = std::max(maxd, v);
  if ((uint64_t)maxd * (P->sym_uploads + 2) >= (1ull << 31)) {
    CUDA_TRY(cudaDeviceSynchronize());
    CUDA_TRY(cudaMemset(P->d_sym_ctr, 0, (size_t)P->nbar * sizeof(unsigned)));
    P->sym_uploads = 0;
  }
  const uint64_t u = P->sym_uploads++;
  UploadArgs ua;
  ua.src = srcd;
  ua.dst = dA;
  ua.rank = P->d_sym_rank;
  ua.run = P->d_sym_run;
  ua.chunk = P->d_sym_chunk;
  ua.ctr = P->d_sym_ctr;
  ua.work = P->d_sym_work;
  ua.base = P->sym_ticket_base;
  ua.set_free = P->d_sym_free + set;
  ua.set_target = P->sym_set_issued[set];  // computes on this set enqueued before this call
  ua.n_diag = P->sym_n_zc;
  ua.blk = (long long)blk;
  ua.lb = ilog2(P->bA);
  static const UploadFn ups[9] = {nullptr, nullptr, upload_m<2>, upload_m<3>, upload_m<4>,
                                  upload_m<5>, upload_m<6>, upload_m<7>, upload_m<8>};
  static const FillFn fills[9] = {nullptr, nullptr, fill_m<2>, fill_m<3>, fill_m<4>,
                                  fill_m<5>, fill_m<6>, fill_m<7>, fill_m<8>};
  // the upload kernel's SMs: its green partition, or SMs the compute grids leave
  // free (then streamed calls issue one compute launch at a time)
  const int ctas = green ? P->g_up_sms : sym_upload_ctas(async);
  pipe.reserve_sms = ctas;
  pipe.serial = async && !green;
  ups[P->m](ua, ctas, up_stream);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaEventRecord(P->sym_prev_done, up_stream));
  // every warp takes tickets until one is past the list: n_diag + warps in all
  P->sym_ticket_base += (uint64_t)P->sym_n_zc + (uint64_t)ctas * (kSymThreads / 32);
  // fills, chunk by chunk, as the chunk's repeated-key blocks land
  while (P->fill_ev.size() < (size_t)P->nbar) {
    cudaEvent_t ev;
    CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    P->fill_ev.push_back(ev);
  }
  WaitFn wait = wait_value_fn();
  int64_t first = 0;
  const unsigned per_blk_ctas = (unsigned)std::max<int64_t>(1, std::min<int64_t>(16, (int64_t)blk / (256 * 8 * 4)));
  for (int64_t a = 0; a < P->nbar; ++a) {
    const int64_t nz = P->sym_nzc[(size_t)a], nf = P->sym_nfill[(size_t)a];
    if (nz) {  // the chunk's zero-copy blocks landed
      const unsigned target = (unsigned)((u + 1) * (uint64_t)nz);
      const CUresult r = wait(reinterpret_cast<CUstream>(P->fill_stream),
                              reinterpret_cast<CUdeviceptr>(P->d_sym_ctr + a), target, CU_STREAM_WAIT_VALUE_GEQ);
      if (r != CUDA_SUCCESS) return fail(BCSS_ERR_CUDA, "cuStreamWaitValue32 failed (%d)", (int)r);
    }
    if (nf) {  // fill its repeated-key blocks
      fills[P->m](dA, P->d_sym_frank + first, P->d_sym_frun + first, (long long)blk, ilog2(P->bA),
                  dim3(per_blk_ctas, (unsigned)nf), P->fill_stream);
      CUDA_TRY(cudaGetLastError());
      first += nf;
    }
    CUDA_TRY(cudaEventRecord(P->fill_ev[(size_t)a], P->fill_stream));
    if (a % 4 == 3) trace_mark(&pipe, "A chunk " + std::to_string(a) + " filled", P->fill_stream);
  }
  pipe.fill_ev = P->fill_ev.data();
  return BCSS_OK;
}

// Everything that reads buffer set `set` in this call is enqueued on `s` up
// to here: release the next symmetric upload into that set.  Called once per
// symmetric-upload call (also on its error paths, so no upload kernel waits
// for a call that never comes).
int sym_release_set(bcss_plan* P, int set, cudaStream_t s) {
  if (!P->d_sym_free) return BCSS_OK;
  // the counts advance only with the write that makes them true, so a failed
  // write leaves the next upload's target at what the flag will hold
  const CUresult r = write_value_fn()(reinterpret_cast<CUstream>(s),
                                      reinterpret_cast<CUdeviceptr>(P->d_sym_free + set),
                                      (cuuint32_t)(P->sym_set_released[set] + 1), 0);
  if (r != CUDA_SUCCESS) return fail(BCSS_ERR_CUDA, "cuStreamWriteValue32 failed (%d)", (int)r);
  ++P->sym_set_released[set];
  ++P->sym_set_issued[set];
  return BCSS_OK;
}

// ---- SM partition (green contexts) ---------------------------------------------
// A streamed call's upload kernel must stay resident while the previous call
// computes.  Green contexts split the SMs: the upload kernel's stream lives in
// a small partition, every compute stream of a symmetric-upload run in the
// complementary one, so concurrent launches and the cascade can no longer take
// the upload's SMs (measured: tools/green_probe.cu, disjoint SM sets, runtime
// launches into green-context streams on primary-context memory).  Driver
// entry points are looked up at run time.  Opt-in (BCSS_SYM_GREEN=1); by
// default streamed symmetric runs issue one compute launch at a time instead.
namespace {
using GetResFn = CUresult (*)(CUdevice, CUdevResource*, CUdevResourceType);
using SplitFn = CUresult (*)(CUdevResource*, unsigned*, const CUdevResource*, CUdevResource*, unsigned, unsigned);
using DescFn = CUresult (*)(CUdevResourceDesc*, CUdevResource*, unsigned);
using GreenCreateFn = CUresult (*)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned);
using GreenStreamFn = CUresult (*)(CUstream*, CUgreenCtx, unsigned, int);
using GreenDestroyFn = CUresult (*)(CUgreenCtx);
using DeviceGetFn = CUresult (*)(CUdevice*, int);
}  // namespace

int sym_green(bcss_plan* P) {
  if (P->green_state != 0) return P->green_state > 0 ? BCSS_OK : BCSS_ERR_STATE;
  P->green_state = -1;
  // opt-in: on config 5 the partition measured slightly slower than leaving the
  // upload's SMs free by grid size (streamed 500 vs 490 ms, one call 651 vs 639
  // ms), on config 4 slightly faster (26.3 vs 27.1 ms streamed)
  const char* e = getenv("BCSS_SYM_GREEN");
  if (!e || !atoi(e)) return BCSS_ERR_STATE;
  auto dget = driver_fn<DeviceGetFn>("cuDeviceGet");
  auto getres = driver_fn<GetResFn>("cuDeviceGetDevResource");
  auto split = driver_fn<SplitFn>("cuDevSmResourceSplitByCount");
  auto gdesc = driver_fn<DescFn>("cuDevResourceGenerateDesc");
  auto gcreate = driver_fn<GreenCreateFn>("cuGreenCtxCreate");
  auto gstream = driver_fn<GreenStreamFn>("cuGreenCtxStreamCreate");
  if (!dget || !getres || !split || !gdesc || !gcreate || !gstream) return BCSS_ERR_STATE;
  int ord = 0;
  if (cudaGetDevice(&ord) != cudaSuccess) return BCSS_ERR_STATE;
  CUdevice dev;
  CUdevResource all, grp[1], rem;
  unsigned nb = 1;
  CUdevResourceDesc d_up, d_comp;
  if (dget(&dev, ord) || getres(dev, &all, CU_DEV_RESOURCE_TYPE_SM) ||
      split(grp, &nb, &all, &rem, 0, (unsigned)sym_upload_ctas(true)) || nb != 1 || rem.sm.smCount == 0 ||
      gdesc(&d_up, grp, 1) || gdesc(&d_comp, &rem, 1)) {
    cudaGetLastError();
    return BCSS_ERR_STATE;
  }
  auto gdestroy = driver_fn<GreenDestroyFn>("cuGreenCtxDestroy");
  CUgreenCtx g_up = nullptr, g_comp = nullptr;
  CUstream up = nullptr, host = nullptr;
  auto undo = [&]() {  // a partial setup leaves nothing behind
    if (up) cudaStreamDestroy(reinterpret_cast<cudaStream_t>(up));
    if (host) cudaStreamDestroy(reinterpret_cast<cudaStream_t>(host));
    if (gdestroy && g_up) gdestroy(g_up);
    if (gdestroy && g_comp) gdestroy(g_comp);
    cudaGetLastError();
    return BCSS_ERR_STATE;
  };
  if (gcreate(&g_up, d_up, dev, CU_GREEN_CTX_DEFAULT_STREAM) ||
      gcreate(&g_comp, d_comp, dev, CU_GREEN_CTX_DEFAULT_STREAM))
    return undo();
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  if (gstream(&up, g_up, CU_STREAM_NON_BLOCKING, hi) || gstream(&host, g_comp, CU_STREAM_NON_BLOCKING, 0))
    return undo();
  P->g_up = g_up;
  P->g_comp = g_comp;
  P->g_sym_stream = reinterpret_cast<cudaStream_t>(up);
  P->g_host_stream = reinterpret_cast<cudaStream_t>(host);
  P->g_up_sms = (int)grp[0].sm.smCount;
  P->green_state = 1;
  return BCSS_OK;
}

// a stream in the compute partition (green runs' side and level streams)
int green_compute_stream(bcss_plan* P, int priority, cudaStream_t* out) {
  auto gstream = driver_fn<GreenStreamFn>("cuGreenCtxStreamCreate");
  CUstream s = nullptr;
  if (!gstream || !P->g_comp || gstream(&s, static_cast<CUgreenCtx>(P->g_comp), CU_STREAM_NON_BLOCKING, priority))
    return fail(BCSS_ERR_CUDA, "cuGreenCtxStreamCreate failed");
  *out = reinterpret_cast<cudaStream_t>(s);
  return BCSS_OK;
}

void green_destroy(bcss_plan* P) {
  auto gdestroy = driver_fn<GreenDestroyFn>("cuGreenCtxDestroy");
  for (cudaStream_t q : P->g_side) cudaStreamDestroy(q);
  for (cudaStream_t q : P->g_lvl_stream) cudaStreamDestroy(q);
  if (P->g_sym_stream) cudaStreamDestroy(P->g_sym_stream);
  if (P->g_host_stream) cudaStreamDestroy(P->g_host_stream);
  if (gdestroy) {
    if (P->g_up) gdestroy(static_cast<CUgreenCtx>(P->g_up));
    if (P->g_comp) gdestroy(static_cast<CUgreenCtx>(P->g_comp));
  }
  cudaGetLastError();
}

// stream s waits until A chunks 0..a are resident (DMA events + fill events)
int wait_chunks(bcss_plan* P, const Pipe* pipe, const cudaEvent_t* chunk_ev, cudaStream_t s, int64_t a) {
  (void)P;
  CUDA_TRY(cudaStreamWaitEvent(s, chunk_ev[a], 0));
  if (pipe && pipe->fill_ev) CUDA_TRY(cudaStreamWaitEvent(s, pipe->fill_ev[a], 0));
  return BCSS_OK;
}

}  // namespace bcss_host
