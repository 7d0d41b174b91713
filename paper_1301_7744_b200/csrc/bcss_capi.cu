// C ABI of the B200-native BCSS sttsm (declared in include/bcss_sttsm.h).
// Entry points validate arguments, drive the plan (plan.cu) and the runs
// (run.cu), and map failures to status codes + bcss_last_error(); nothing
// throws across the ABI.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <new>
#include <thread>
#include <vector>

#include "plan.hpp"

using namespace bcss_host;

namespace {

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
  if ((st = check_int32_limits(m, n, p, b_a, b_c, reuse != 0))) return st;
  bcss_plan* P = new (std::nothrow) bcss_plan();
  if (!P) return fail(BCSS_ERR_NOMEM, "out of host memory");
  P->m = m; P->n = n; P->p = p; P->bA = b_a; P->bC = b_c;
  P->nbar = n / b_a; P->pbar = p / b_c; P->reuse = reuse != 0;
  if (const char* e = getenv("BCSS_SERIAL_LAUNCH")) P->concurrent = atoi(e) == 0;
  if (const char* e = getenv("BCSS_SLICE_MB")) P->slice_bytes = (size_t)std::max(0.0, atof(e) * 1048576.0);
  if (const char* e = getenv("BCSS_SHARE")) P->share_frac = std::min(1.0, std::max(0.0, atof(e)));
  *out_plan = P;
  return BCSS_OK;
}

int bcss_plan_destroy(bcss_plan* P) {
  if (!P) return BCSS_OK;
  // nothing of this plan may still run when its buffers go (a streamed
  // symmetric upload's kernel and fills live on their own streams)
  for (cudaStream_t q : {P->copy_in, P->copy_out, P->copy_out2, P->host_stream, P->sym_stream, P->fill_stream,
                         P->g_host_stream, P->g_sym_stream})
    if (q) cudaStreamSynchronize(q);
  for (cudaStream_t q : P->g_side) cudaStreamSynchronize(q);
  for (cudaStream_t q : P->g_lvl_stream) cudaStreamSynchronize(q);
  cudaGetLastError();
  if (P->d_tables) cudaFree(P->d_tables);
  if (P->d_ws && P->own_ws) cudaFree(P->d_ws);
  if (P->hA) cudaFree(P->hA);
  if (P->hX) cudaFree(P->hX);
  if (P->dXm) cudaFree(P->dXm);
  if (P->dXp) cudaFree(P->dXp);
  if (P->dXt) cudaFree(P->dXt);
  if (P->dXtp) cudaFree(P->dXtp);
  if (P->hA1) cudaFree(P->hA1);
  if (P->hX1) cudaFree(P->hX1);
  if (P->hC1) cudaFree(P->hC1);
  for (int q = 0; q < 2; ++q) {
    if (P->set_compute_done[q]) cudaEventDestroy(P->set_compute_done[q]);
    if (P->set_d2h_done[q]) cudaEventDestroy(P->set_d2h_done[q]);
  }
  if (P->pinA) cudaFreeHost(P->pinA);
  if (P->pinX) cudaFreeHost(P->pinX);
  if (P->pinC) cudaFreeHost(P->pinC);
  if (P->d_call_out) cudaFree(P->d_call_out);
  if (P->hC) cudaFree(P->hC);
  if (P->host_stream) cudaStreamDestroy(P->host_stream);
  for (auto ev : P->events) cudaEventDestroy(ev);
  for (auto ev : P->join) cudaEventDestroy(ev);
  for (auto ss : P->side) cudaStreamDestroy(ss);
  if (P->fork) cudaEventDestroy(P->fork);
  for (auto ev : P->chunk_ev) cudaEventDestroy(ev);
  for (auto ev : P->wave_ev) cudaEventDestroy(ev);
  for (auto ev : P->grp_ev) cudaEventDestroy(ev);
  for (auto ss : P->lvl_stream) cudaStreamDestroy(ss);
  if (P->cascade_start) cudaEventDestroy(P->cascade_start);
  for (auto ev : P->bg_ev)
    if (ev) cudaEventDestroy(ev);
  if (P->copy_in) cudaStreamDestroy(P->copy_in);
  if (P->copy_out) cudaStreamDestroy(P->copy_out);
  if (P->copy_out2) cudaStreamDestroy(P->copy_out2);
  if (P->out2_done) cudaEventDestroy(P->out2_done);
  if (P->d_sym) cudaFree(P->d_sym);
  if (P->sym_stream) cudaStreamDestroy(P->sym_stream);
  if (P->fill_stream) cudaStreamDestroy(P->fill_stream);
  if (P->sym_prev_done) cudaEventDestroy(P->sym_prev_done);
  bcss_host::green_destroy(P);
  for (auto ev : P->fill_ev) cudaEventDestroy(ev);
  delete P;
  return BCSS_OK;
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

int bcss_plan_kernel_mix(bcss_plan* P, int64_t* fast_launches, int64_t* generic_launches) {
  if (!P) return fail(BCSS_ERR_STATE, "null plan");
  int st = build_plan(*P);
  if (st) return st;
  int64_t f = 0, g = 0;
  for (auto& W : P->waves)
    for (auto& L : W.levels)
      for (auto& X : L.launches)
        if (X.item_off.back() > 0) (is_generic(X.cfg) ? g : f) += 1;
  if (fast_launches) *fast_launches = f;
  if (generic_launches) *generic_launches = g;
  return BCSS_OK;
}

int bcss_plan_neighbour_table(bcss_plan* P, int k, int from_device, int32_t* out, int64_t n_max, int64_t* out_n) {
  if (!P || !out_n) return fail(BCSS_ERR_STATE, "null argument");
  if (k < 0 || k >= P->m) return fail(BCSS_ERR_RANGE, "level %d outside 0..%d", k, P->m - 1);
  int st = build_plan(*P);
  if (st) return st;
  const int64_t n = keys_at(*P, k) * P->nbar;
  *out_n = 2 * n;
  if (!out) return BCSS_OK;
  if (2 * n > n_max) return fail(BCSS_ERR_RANGE, "output array too small");
  if (from_device) {
    if ((st = upload_tables(*P, nullptr))) return st;
    CUDA_TRY(cudaMemcpy(out, static_cast<char*>(P->d_tables) + P->nbr_off[k], (size_t)n * sizeof(int2),
                        cudaMemcpyDeviceToHost));
  } else {
    std::vector<int2> h;
    try { build_nbr(*P, k, h); } catch (const std::exception& e) { return fail(BCSS_ERR_PARAMETER, "%s", e.what()); }
    memcpy(out, h.data(), (size_t)n * sizeof(int2));
  }
  return BCSS_OK;
}

int bcss_sttsm_run(bcss_plan* P, const double* A, const double* X_, double* C, void* stream) {
  if (!P) return fail(BCSS_ERR_STATE, "null plan");
  if (!A || !X_ || !C) return fail(BCSS_ERR_PARAMETER, "null buffer");
  return run_impl(P, A, X_, C, static_cast<cudaStream_t>(stream), nullptr);
}

int bcss_sttsm_run_gated(bcss_plan* P, const double* A, const double* X_, double* C, void* stream,
                         const void* const* chunk_events, int n_events) {
  if (!P) return fail(BCSS_ERR_STATE, "null plan");
  if (!A || !X_ || !C) return fail(BCSS_ERR_PARAMETER, "null buffer");
  if (n_events != (int)P->nbar || !chunk_events)
    return fail(BCSS_ERR_SHAPE, "%d chunk events for %lld first-index chunks of A", n_events, (long long)P->nbar);
  for (int a = 0; a < n_events; ++a)
    if (!chunk_events[a]) return fail(BCSS_ERR_PARAMETER, "null event for chunk %d", a);
  if (P->start_level > 0)  // nothing reads A: a plain run
    return run_impl(P, A, X_, C, static_cast<cudaStream_t>(stream), nullptr);
  std::vector<cudaEvent_t> evs((size_t)n_events);
  for (int a = 0; a < n_events; ++a) evs[(size_t)a] = static_cast<cudaEvent_t>(const_cast<void*>(chunk_events[a]));
  Pipe pipe;  // no per-wave downloads; the caller reads C after the run
  pipe.chunk_ev = evs.data();
  return run_impl(P, A, X_, C, static_cast<cudaStream_t>(stream), &pipe);
}

int bcss_plan_set_stop_level(bcss_plan* P, int stop_level) {
  if (!P) return fail(BCSS_ERR_STATE, "null plan");
  if (stop_level < 0 || stop_level >= P->m) return fail(BCSS_ERR_RANGE, "stop level %d outside 0..%d", stop_level, P->m - 1);
  P->stop_level = stop_level;
  invalidate(P);
  return BCSS_OK;
}

int bcss_plan_set_call_outputs(bcss_plan* P, const void* const* ptrs, int64_t n) {
  if (!P) return fail(BCSS_ERR_STATE, "null plan");
  if (n == 0) {
    P->call_out.clear();
    P->call_out_dirty = true;
    return BCSS_OK;
  }
  if (!ptrs || n < 0) return fail(BCSS_ERR_PARAMETER, "bad pointer table");
  if (P->stop_level <= 0) return fail(BCSS_ERR_STATE, "call outputs need a stop level > 0");
  int st = build_plan(*P);
  if (st) return st;
  int64_t calls = 0;
  for (auto& W : P->waves)
    for (auto& L : W.levels)
      if (L.k == P->stop_level) calls += L.n_calls;
  if (n != calls) return fail(BCSS_ERR_SHAPE, "%lld pointers for %lld stop-level calls", (long long)n, (long long)calls);
  P->call_out.assign(reinterpret_cast<const double* const*>(ptrs), reinterpret_cast<const double* const*>(ptrs) + n);
  P->call_out_dirty = true;
  return BCSS_OK;
}

int bcss_device_alloc(size_t bytes, void** out_ptr) {
  if (!out_ptr) return fail(BCSS_ERR_PARAMETER, "null output");
  *out_ptr = nullptr;
  cudaError_t e = cudaMalloc(out_ptr, std::max<size_t>(bytes, 256));
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(BCSS_ERR_NOMEM, "cudaMalloc of %zu bytes failed: %s", bytes, cudaGetErrorString(e));
  }
  return BCSS_OK;
}

int bcss_device_free(void* ptr) {
  CUDA_TRY(cudaFree(ptr));
  return BCSS_OK;
}

int bcss_ipc_get_handle(const void* dev_ptr, void* out_handle64) {
  if (!dev_ptr || !out_handle64) return fail(BCSS_ERR_PARAMETER, "null argument");
  cudaIpcMemHandle_t h;
  CUDA_TRY(cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr)));
  static_assert(sizeof(h) == 64, "IPC handle size");
  memcpy(out_handle64, &h, sizeof(h));
  return BCSS_OK;
}

int bcss_ipc_open_handle(const void* handle64, void** out_ptr) {
  if (!handle64 || !out_ptr) return fail(BCSS_ERR_PARAMETER, "null argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, sizeof(h));
  CUDA_TRY(cudaIpcOpenMemHandle(out_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return BCSS_OK;
}

int bcss_copy_async(void* dst, const void* src, size_t bytes, void* stream) {
  if ((!dst || !src) && bytes) return fail(BCSS_ERR_PARAMETER, "null buffer");
  CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, static_cast<cudaStream_t>(stream)));
  return BCSS_OK;
}

int bcss_ipc_close_handle(void* ptr) {
  CUDA_TRY(cudaIpcCloseMemHandle(ptr));
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

int bcss_plan_set_start_children(bcss_plan* P, const int32_t* jbs, int n) {
  if (!P) return fail(BCSS_ERR_STATE, "null plan");
  if (n < 0 || (n > 0 && !jbs)) return fail(BCSS_ERR_PARAMETER, "bad child list");
  for (int i = 0; i < n; ++i) {
    if (jbs[i] < 0 || jbs[i] >= P->pbar) return fail(BCSS_ERR_RANGE, "child %d outside 0..%lld", jbs[i], (long long)P->pbar - 1);
    if (i > 0 && jbs[i] <= jbs[i - 1]) return fail(BCSS_ERR_SHAPE, "children must be strictly increasing");
  }
  P->start_children.assign(jbs, jbs + n);
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

int bcss_plan_set_symmetric_upload(bcss_plan* P, int on) {
  if (!P) return fail(BCSS_ERR_STATE, "null plan");
  P->sym_upload = on != 0;
  return BCSS_OK;
}

int bcss_plan_last_upload_bytes(bcss_plan* P, int64_t* out_bytes) {
  if (!P || !out_bytes) return fail(BCSS_ERR_STATE, "null argument");
  *out_bytes = P->last_upload_bytes;
  return BCSS_OK;
}

int bcss_plan_upload_bytes(bcss_plan* P, int64_t* out_bytes) {
  if (!P || !out_bytes) return fail(BCSS_ERR_STATE, "null argument");
  int64_t in_elems = 0, out_elems = 0;
  int st = bcss_plan_io_elems(P, &in_elems, &out_elems);
  if (st) return st;
  *out_bytes = in_elems * (int64_t)sizeof(double);
  if (bcss_host::sym_eligible(*P) && P->pipeline_waves > 0 && !P->units_set && !P->keep_temps &&
      P->start_level == 0 && P->stop_level == 0) {
    if ((st = bcss_host::sym_prepare(*P))) return st;
    *out_bytes = P->sym_fetch_elems * (int64_t)sizeof(double);
  }
  return BCSS_OK;
}

namespace {
// memcpy with the host's cores (pageable <-> pinned staging)
void par_copy(void* dst, const void* src, size_t bytes) {
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const size_t min_chunk = size_t(8) << 20;
  const unsigned t = (unsigned)std::min<size_t>(std::min(hw, 32u), std::max<size_t>(1, bytes / min_chunk));
  if (t <= 1) {
    memcpy(dst, src, bytes);
    return;
  }
  const size_t per = (bytes / t + 63) / 64 * 64;
  std::vector<std::thread> th;
  for (unsigned i = 0; i < t; ++i) {
    const size_t lo = std::min(bytes, i * per), hi = std::min(bytes, lo + per);
    if (hi > lo)
      th.emplace_back([=] { memcpy(static_cast<char*>(dst) + lo, static_cast<const char*>(src) + lo, hi - lo); });
  }
  for (auto& x : th) x.join();
}
}  // namespace

static int run_host_pinned(bcss_plan* P, const double* A, const double* X, double* C, bool async);

int bcss_sttsm_run_host(bcss_plan* P, const double* A, const double* X, double* C) {
  if (!P) return fail(BCSS_ERR_STATE, "null plan");
  if (!A || !X || !C) return fail(BCSS_ERR_PARAMETER, "null buffer");
  const bool can_pipe = P->pipeline_waves > 0 && !P->units_set && !P->keep_temps && P->start_level == 0 &&
                        P->stop_level == 0;
  const bool pa = is_pinned(A), px = is_pinned(X), pc = is_pinned(C);
  if (can_pipe && !(pa && px && pc)) {
    // pageable buffers: stage only those through plan-owned pinned memory
    // with all host cores (the DMA engines then run at PCIe speed and the
    // pipeline applies); pinned or registered buffers (bcss_host_register)
    // are used in place
    const size_t a_b = (size_t)bcss::simplex_count(P->nbar, P->m) * (size_t)ipow(P->bA, P->m) * sizeof(double);
    const size_t x_b = (size_t)(P->p * P->n) * sizeof(double);
    const size_t c_b = (size_t)bcss::simplex_count(P->pbar, P->m) * (size_t)ipow(P->bC, P->m) * sizeof(double);
    auto grow_pinned = [&](double*& ptr, size_t& cap, size_t need) -> int {
      if (cap >= need) return BCSS_OK;
      if (ptr) cudaFreeHost(ptr);
      ptr = nullptr;
      cap = 0;
      CUDA_TRY(cudaMallocHost(&ptr, std::max<size_t>(need, 64)));
      cap = need;
      return BCSS_OK;
    };
    int st;
    if (!pa && (st = grow_pinned(P->pinA, P->pinA_bytes, a_b))) return st;
    if (!px && (st = grow_pinned(P->pinX, P->pinX_bytes, x_b))) return st;
    if (!pc && (st = grow_pinned(P->pinC, P->pinC_bytes, c_b))) return st;
    // (measured: staging the whole buffers around the pipelined run beats
    // chunk-gated staging overlapped with the DMA on this host's 16 cores)
    if (!pa) par_copy(P->pinA, A, a_b);
    if (!px) memcpy(P->pinX, X, x_b);
    if ((st = run_host_pinned(P, pa ? A : P->pinA, px ? X : P->pinX, pc ? C : P->pinC, false))) return st;
    if (!pc) par_copy(C, P->pinC, c_b);
    return BCSS_OK;
  }
  return run_host_pinned(P, A, X, C, false);
}

int bcss_host_register(void* ptr, size_t bytes) {
  if (!ptr || !bytes) return fail(BCSS_ERR_PARAMETER, "null or empty host range");
  if (is_pinned(ptr)) return BCSS_OK;
  const cudaError_t e = cudaHostRegister(ptr, bytes, cudaHostRegisterPortable | cudaHostRegisterMapped);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(BCSS_ERR_CUDA, "cudaHostRegister of %zu bytes failed: %s", bytes, cudaGetErrorString(e));
  }
  return BCSS_OK;
}

int bcss_host_unregister(void* ptr) {
  if (!ptr) return fail(BCSS_ERR_PARAMETER, "null host pointer");
  const cudaError_t e = cudaHostUnregister(ptr);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(BCSS_ERR_CUDA, "cudaHostUnregister failed: %s", cudaGetErrorString(e));
  }
  return BCSS_OK;
}

int bcss_host_alloc(size_t bytes, void** out_ptr) {
  if (!out_ptr) return fail(BCSS_ERR_PARAMETER, "null output");
  *out_ptr = nullptr;
  const cudaError_t e = cudaMallocHost(out_ptr, std::max<size_t>(bytes, 64));
  if (e != cudaSuccess) {
    cudaGetLastError();
    *out_ptr = nullptr;
    return fail(BCSS_ERR_NOMEM, "cudaMallocHost of %zu bytes failed: %s", bytes, cudaGetErrorString(e));
  }
  return BCSS_OK;
}

int bcss_host_free(void* ptr) {
  if (ptr) CUDA_TRY(cudaFreeHost(ptr));
  return BCSS_OK;
}

int bcss_host_is_pinned(const void* ptr, int* out) {
  if (!out) return fail(BCSS_ERR_PARAMETER, "null output");
  *out = ptr && is_pinned(ptr) ? 1 : 0;
  return BCSS_OK;
}

int bcss_sttsm_run_host_async(bcss_plan* P, const double* A, const double* X, double* C) {
  if (!P) return fail(BCSS_ERR_STATE, "null plan");
  if (!A || !X || !C) return fail(BCSS_ERR_PARAMETER, "null buffer");
  const bool can_pipe = P->pipeline_waves > 0 && !P->units_set && !P->keep_temps && P->start_level == 0 &&
                        P->stop_level == 0;
  if (!can_pipe || !is_pinned(A) || !is_pinned(X) || !is_pinned(C))
    return fail(BCSS_ERR_STATE, "asynchronous host runs need a pipelined full plan and pinned buffers");
  return run_host_pinned(P, A, X, C, true);
}

int bcss_plan_wait(bcss_plan* P) {
  if (!P) return fail(BCSS_ERR_STATE, "null plan");
  for (cudaStream_t q : {P->copy_in, P->copy_out, P->copy_out2, P->host_stream, P->sym_stream, P->fill_stream,
                         P->g_host_stream, P->g_sym_stream})
    if (q) CUDA_TRY(cudaStreamSynchronize(q));
  if (!P->atrace.empty()) {  // BCSS_TRACE=3: device timeline of the streamed calls
    fprintf(stderr, "[bcss trace] streamed host runs (device ms since the first mark):\n");
    for (auto& t : P->atrace) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, P->atrace.front().second, t.second);
      fprintf(stderr, "  %-34s %9.3f\n", t.first.c_str(), ms);
    }
    for (auto& t : P->atrace) cudaEventDestroy(t.second);
    P->atrace.clear();
  }
  return BCSS_OK;
}

namespace {
// BCSS_TRACE=3: timing event on `s`, printed by bcss_plan_wait
void amark(bcss_plan* P, const std::string& name, cudaStream_t s) {
  static const bool on = [] { const char* t = getenv("BCSS_TRACE"); return t && atoi(t) == 3; }();
  if (!on) return;
  cudaEvent_t ev;
  if (cudaEventCreate(&ev) != cudaSuccess || cudaEventRecord(ev, s) != cudaSuccess) return;
  P->atrace.emplace_back("call " + std::to_string(P->host_calls) + " " + name, ev);
}
}  // namespace

static int run_host_pinned(bcss_plan* P, const double* A, const double* X, double* C, bool async) {
  const size_t blk_a = (size_t)ipow(P->bA, P->m);
  // input / output sizes of this plan: A and C for a full run, the
  // start-level temporaries in / stop-level temporaries out for partial plans
  int64_t in_elems = 0, out_elems = 0;
  int st = bcss_plan_io_elems(P, &in_elems, &out_elems);
  if (st) return st;
  const size_t a_bytes = (size_t)in_elems * sizeof(double);
  const size_t x_bytes = (size_t)(P->p * P->n) * sizeof(double);
  const size_t c_bytes = (size_t)out_elems * sizeof(double);
  auto grow = [&](double*& ptr, size_t& cap, size_t need) -> int {
    if (cap >= need) return BCSS_OK;
    if (ptr) cudaFree(ptr);
    ptr = nullptr; cap = 0;
    const cudaError_t e = cudaMalloc(&ptr, need);
    if (e != cudaSuccess) {
      cudaGetLastError();
      ptr = nullptr;
      return fail(BCSS_ERR_NOMEM, "cudaMalloc of %zu host-run bytes failed: %s", need, cudaGetErrorString(e));
    }
    cap = need;
    return BCSS_OK;
  };
  if ((st = grow(P->hA, P->hA_bytes, a_bytes))) return st;
  if ((st = grow(P->hX, P->hX_bytes, x_bytes))) return st;
  if ((st = grow(P->hC, P->hC_bytes, c_bytes))) return st;
  if (!P->host_stream) CUDA_TRY(cudaStreamCreateWithFlags(&P->host_stream, cudaStreamNonBlocking));
  const bool pipelined = P->pipeline_waves > 0 && !P->units_set && !P->keep_temps && P->start_level == 0 &&
                         P->stop_level == 0 && is_pinned(A) &&
                         is_pinned(X) && is_pinned(C);
  P->last_upload_bytes = (int64_t)a_bytes;
  if (!pipelined) {
    CUDA_TRY(cudaMemcpyAsync(P->hA, A, a_bytes, cudaMemcpyHostToDevice, P->host_stream));
    CUDA_TRY(cudaMemcpyAsync(P->hX, X, x_bytes, cudaMemcpyHostToDevice, P->host_stream));
    if ((st = run_impl(P, P->hA, P->hX, P->hC, P->host_stream, nullptr))) return st;
    if ((P->units_set || P->start_level > 0) && P->stop_level == 0) {
      // a shard: only this plan's C blocks come back (runs of consecutive
      // ranks); the caller's other blocks are left as they are
      std::vector<int> ranks;
      for (auto& W : P->waves)
        for (auto& L : W.levels)
          if (L.k == 0) ranks.insert(ranks.end(), L.child_call.begin(), L.child_call.end());
      std::sort(ranks.begin(), ranks.end());
      const size_t blk_c = (size_t)ipow(P->bC, P->m);
      for (size_t i = 0; i < ranks.size();) {
        size_t j = i + 1;
        while (j < ranks.size() && ranks[j] == ranks[j - 1] + 1) ++j;
        const size_t off = (size_t)ranks[i] * blk_c;
        CUDA_TRY(cudaMemcpyAsync(C + off, P->hC + off, (j - i) * blk_c * sizeof(double), cudaMemcpyDeviceToHost,
                                 P->host_stream));
        i = j;
      }
    } else {
      CUDA_TRY(cudaMemcpyAsync(C, P->hC, c_bytes, cudaMemcpyDeviceToHost, P->host_stream));
    }
    CUDA_TRY(cudaStreamSynchronize(P->host_stream));
    return BCSS_OK;
  }
  const auto h0 = std::chrono::steady_clock::now();
  if ((st = build_plan(*P))) return st;
  // alternate device buffer sets between consecutive asynchronous calls (a
  // synchronous call has finished with its set when it returns: set 0)
  const int set = async ? (int)(P->host_calls++ & 1) : 0;
  double* dA = P->hA;
  double* dX = P->hX;
  double* dC = P->hC;
  if (set == 1) {
    if ((st = grow(P->hA1, P->hA1_bytes, a_bytes))) return st;
    if ((st = grow(P->hX1, P->hX1_bytes, x_bytes))) return st;
    if ((st = grow(P->hC1, P->hC1_bytes, c_bytes))) return st;
    dA = P->hA1;
    dX = P->hX1;
    dC = P->hC1;
  }
  for (int q = 0; q < 2; ++q) {
    if (!P->set_compute_done[q]) CUDA_TRY(cudaEventCreateWithFlags(&P->set_compute_done[q], cudaEventDisableTiming));
    if (!P->set_d2h_done[q]) CUDA_TRY(cudaEventCreateWithFlags(&P->set_d2h_done[q], cudaEventDisableTiming));
  }
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
  // symmetric upload: distinct-key blocks by DMA, repeated-key blocks by the
  // zero-copy streaming kernel + per-chunk fills (sym_upload.cu); with an SM
  // partition (green contexts) its kernel and the compute never share SMs
  bool sym = bcss_host::sym_eligible(*P) && bcss_host::sym_supported();
  if (sym) {
    cudaPointerAttributes at;
    sym = cudaPointerGetAttributes(&at, A) == cudaSuccess && at.devicePointer != nullptr;
    cudaGetLastError();
  }
  if (sym && (st = bcss_host::sym_prepare(*P))) return st;
  const bool green = sym && P->sym_n_zc > 0 && bcss_host::sym_green(P) == BCSS_OK;
  cudaGetLastError();
  cudaStream_t hs = green ? P->g_host_stream : P->host_stream;  // the compute's main stream
  // this set's device buffers: the upload waits until the set's previous call
  // stopped reading A / X, the kernels until its C was downloaded
  CUDA_TRY(cudaStreamWaitEvent(P->copy_in, P->set_compute_done[set], 0));
  CUDA_TRY(cudaStreamWaitEvent(hs, P->set_d2h_done[set], 0));
  Pipe pipe;
  pipe.c_host = C;
  std::vector<std::pair<std::string, cudaEvent_t>> trace;
  const char* tr = getenv("BCSS_TRACE");
  if (tr && atoi(tr) == 1) pipe.trace = &trace;
  trace_mark(&pipe, "upload start", P->copy_in);
  amark(P, "upload start (copy_in)", P->copy_in);
  CUDA_TRY(cudaMemcpyAsync(dX, X, x_bytes, cudaMemcpyHostToDevice, P->copy_in));
  if (sym) {
    int lo = 0, hi = 0;
    CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    if (!P->sym_stream) CUDA_TRY(cudaStreamCreateWithPriority(&P->sym_stream, cudaStreamNonBlocking, hi));
    if (!P->fill_stream) CUDA_TRY(cudaStreamCreateWithPriority(&P->fill_stream, cudaStreamNonBlocking, hi));
    cudaStream_t us = green ? P->g_sym_stream : P->sym_stream;
    // the kernel waits on the device for the set's previous symmetric run; a
    // previous full-upload run on this set is waited for here
    if (!P->sym_set_last[set]) CUDA_TRY(cudaStreamWaitEvent(us, P->set_compute_done[set], 0));
    // A streamed call that finds the pipeline empty (both sets' earlier
    // computes finished: the first call of a burst) has no previous call whose
    // compute its upload kernel must squeeze beside, so it runs like a
    // synchronous call - cascade and concurrent launches while A uploads -
    // instead of one compute launch at a time (first call of a config-5 burst:
    // 939 -> ~640 ms; the following calls are unchanged).
    bool idle = true;
    for (int q = 0; q < 2; ++q)
      if (cudaEventQuery(P->set_compute_done[q]) != cudaSuccess) idle = false;
    cudaGetLastError();
    if (getenv("BCSS_SYM_NO_IDLE_START")) idle = false;  // (A/B switch)
    if ((st = bcss_host::sym_upload_issue(P, A, dA, set, async && !idle, green, P->copy_in, us, pipe))) return st;
    P->last_upload_bytes = P->sym_fetch_elems * (int64_t)sizeof(double);
    trace_mark(&pipe, "A DMA half landed", P->copy_in);
    amark(P, "DMA half landed", P->copy_in);
    amark(P, "zero-copy half landed", us);
    amark(P, "fills done", P->fill_stream);
    trace_mark(&pipe, "A zero-copy half landed", us);
    trace_mark(&pipe, "A repeated-key blocks filled", P->fill_stream);
    cudaStreamQuery(us);
    cudaStreamQuery(P->fill_stream);
  } else {
    for (int64_t a = 0; a < P->nbar; ++a) {
      const size_t r0 = (size_t)first_rank_with(a, P->m, P->nbar), r1 = (size_t)first_rank_with(a + 1, P->m, P->nbar);
      CUDA_TRY(cudaMemcpyAsync(dA + r0 * blk_a, A + r0 * blk_a, (r1 - r0) * blk_a * sizeof(double),
                               cudaMemcpyHostToDevice, P->copy_in));
      CUDA_TRY(cudaEventRecord(P->chunk_ev[a], P->copy_in));
      trace_mark(&pipe, "A chunk " + std::to_string(a) + " landed", P->copy_in);
    }
  }
  cudaStreamQuery(P->copy_in);  // kick the driver to submit queued work now
  amark(P, "compute enqueued from here", hs);
  if (green) {  // side and level streams of the compute partition
    std::swap(P->side, P->g_side);
    std::swap(P->lvl_stream, P->g_lvl_stream);
    P->green_active = true;
  }
  st = run_impl(P, dA, dX, dC, hs, &pipe);
  if (green) {
    std::swap(P->side, P->g_side);
    std::swap(P->lvl_stream, P->g_lvl_stream);
    P->green_active = false;
  }
  if (sym && P->d_sym_free) {
    // release the next symmetric upload into this set once this call's
    // kernels are done (also after a failed enqueue: nothing may wait forever)
    const int st2 = bcss_host::sym_release_set(P, set, hs);
    if (!st) st = st2;
  }
  P->sym_set_last[set] = sym;
  if (st) return st;
  CUDA_TRY(cudaEventRecord(P->set_compute_done[set], hs));
  amark(P, "compute done", hs);
  CUDA_TRY(cudaEventRecord(P->out2_done, P->copy_out2));
  CUDA_TRY(cudaStreamWaitEvent(P->copy_out, P->out2_done, 0));
  CUDA_TRY(cudaEventRecord(P->set_d2h_done[set], P->copy_out));
  amark(P, "C downloaded", P->copy_out);
  if (async) {
    cudaStreamQuery(hs);  // submit
    return BCSS_OK;
  }
  if (pipe.trace) {
    fprintf(stderr, "[bcss trace] host enqueue took %.3f ms\n",
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count());
    // host-side polling timeline (first time each event is seen complete)
    std::vector<double> seen(trace.size(), -1.0);
    const auto t0 = h0;  // times relative to the start of this call
    size_t left = trace.size();
    while (left) {
      const double now = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      for (size_t i = 0; i < trace.size(); ++i)
        if (seen[i] < 0 && cudaEventQuery(trace[i].second) == cudaSuccess) { seen[i] = now; --left; }
    }
    fprintf(stderr, "[bcss trace] run_host pipeline timeline (host-polled ms since the call began):\n");
    for (size_t i = 0; i < trace.size(); ++i) {
      fprintf(stderr, "  %-28s %8.3f\n", trace[i].first.c_str(), seen[i]);
      cudaEventDestroy(trace[i].second);
    }
  }
  const auto h1 = std::chrono::steady_clock::now();
  CUDA_TRY(cudaStreamSynchronize(P->copy_out));
  const auto h2 = std::chrono::steady_clock::now();
  CUDA_TRY(cudaStreamSynchronize(P->copy_out2));
  CUDA_TRY(cudaStreamSynchronize(hs));
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
