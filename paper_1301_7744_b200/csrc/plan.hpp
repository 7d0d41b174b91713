// Host-side plan of the BCSS sttsm C ABI: structures and helpers shared by
// plan.cu (construction), run.cu (launch orchestration) and bcss_capi.cu.
#pragma once

#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <string>
#include <utility>
#include <vector>

#include "../../include/bcss_sttsm.h"
#include "combinatorics.hpp"
#include "kernel_table.cuh"

namespace bcss_host {

extern thread_local std::string g_last_error;

inline int fail(int code, const char* fmt, ...) {
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

inline bool is_pow2(int64_t v) { return v > 0 && (v & (v - 1)) == 0; }
inline int ilog2(int64_t v) { int r = 0; while ((int64_t(1) << r) < v) ++r; return r; }
inline int64_t ipow(int64_t b, int e) { int64_t r = 1; while (e-- > 0) r *= b; return r; }

using bcss::KernelCfg;
using bcss::N_SHAPES;
using bcss::N_GEN;
constexpr int N_CFGS = 2 + bcss::N_BA * N_SHAPES + bcss::N_BA * N_GEN + (bcss::N_NP + bcss::N_NPP) * N_SHAPES;
enum { CFG_GENERIC = 0, CFG_GENERIC_PERM = N_CFGS - 1 };
inline bool is_generic(int cfg) { return cfg == CFG_GENERIC || cfg == CFG_GENERIC_PERM; }
const KernelCfg& kernel_cfg(int cfg);
int fast_cfg(int64_t bA, int m, int shape);
int np_row_group(int64_t bA, int m, int64_t* padded);
int64_t padded_ba(int64_t bA, int m);
int gen_cfg(int64_t bA, int m, int shape);

// ---- plan ----------------------------------------------------------------------
// One kernel launch: the parents of a level that share a tile configuration.
struct LaunchHost {
  int cfg = 0;
  int n_tiles = 0;
  uint64_t flops = 0;
  double cost = 0;                 // modelled time (ShapePolicy::tile_cost units per column), 0 = unknown
  std::vector<int4> parents;       // {in_call, row0, rows, child_off}
  std::vector<long long> item_off; // prefix sums of work items, size parents+1
  std::vector<int4> items;         // per work item {parent, key, n-tile, m-tile}
  // cascade levels: items are ordered by key group (first key index in
  // [group_a[g], group_a[g+1])) first; group g is items [group_items[g], group_items[g+1])
  std::vector<long long> group_items;
  // cascade top level: the first n_w0 parents hold the first wave's unit rows;
  // within group g, items [group_items[g], group_w0[g]) are theirs
  int n_w0 = 0;
  std::vector<long long> group_w0;
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

}  // namespace bcss_host

using bcss_host::LaunchHost;
using bcss_host::LevelHost;
using bcss_host::WaveHost;

struct bcss_plan {
  int m = 0;
  int64_t n = 0, p = 0, bA = 0, bC = 0, nbar = 0, pbar = 0;
  int64_t bAp = 0;                  // b_a, or its padded width on the fast kernels (set by build_plan)
  bool reuse = true;
  std::vector<int> units;
  bool units_set = false;
  size_t ws_limit = 0;
  bool keep_temps = false;

  bool built = false;
  std::vector<WaveHost> waves;
  std::vector<size_t> nbr_off;         // per k, into the table buffer (neighbour tables built on device)
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
  // second device buffer set of pipelined host runs: consecutive calls
  // alternate sets so call i+1 uploads while call i computes / downloads
  double *hA1 = nullptr, *hX1 = nullptr, *hC1 = nullptr;
  size_t hA1_bytes = 0, hX1_bytes = 0, hC1_bytes = 0;
  cudaEvent_t set_compute_done[2] = {nullptr, nullptr};  // kernels of the set's last call finished
  cudaEvent_t set_d2h_done[2] = {nullptr, nullptr};      // downloads of the set's last call finished
  uint64_t host_calls = 0;
  double *pinA = nullptr, *pinX = nullptr, *pinC = nullptr;  // pinned staging for pageable host buffers
  size_t pinA_bytes = 0, pinX_bytes = 0, pinC_bytes = 0;
  cudaStream_t host_stream = nullptr;
  int64_t last_launches = 0;
  bool timing = false;
  bool concurrent = true;           // concurrent launches per level (BCSS_SERIAL_LAUNCH=1 disables)
  size_t slice_bytes = 0;           // > 0: parents whose T(k+1) is larger are walked in tail slices of about this size (plan.cu); BCSS_SLICE_MB
  double share_frac = 0;            // > 0: a level's tile shapes run side by side on SM shares (run.cu); BCSS_SHARE
  int pipeline_waves = 0;           // run_host: overlap H2D / compute / D2H over this many waves
  bool top_first = false;           // first wave computes T(m-1) for all units
  // Mirrored C-block order (pipelined plans): the plan contracts X' (row blocks
  // reversed, jb -> p̄-1-jb), so its top-level unit u is the SMALLEST index
  // p̄-1-u of the C blocks below it, whose ranks are then one contiguous range
  // (one D2H per wave).  Level 0 writes each block through the inverse map
  // (block rank of the reversed mirrored tuple, element digits reversed).
  std::vector<const double*> call_out;  // stop level: per-call destinations (bcss_plan_set_call_outputs)
  const double** d_call_out = nullptr;   // device copy
  size_t d_call_out_cap = 0;
  bool call_out_dirty = false;
  bool mirror = false;
  // Cascade (pipelined host runs): the first wave's levels m-1..1 run as key
  // groups of equal first index; group g of level k needs only A chunks /
  // T(k+1) groups <= g, so the levels below the top proceed while A is still
  // uploading.  The first wave's temporaries then get disjoint regions.
  bool cascade = false;
  bool cascade_nofit = false;       // the disjoint first-wave regions exceeded the workspace limit
  std::vector<int64_t> group_a;     // first-index boundaries of the key groups
  int defer_group = 0;              // cascade: top-level rows of later waves in groups >= this run after wave 0
  double* dXp = nullptr;            // X with every b_a column block zero-padded to b_a' columns (device, p x n')
  size_t dXp_bytes = 0;
  double* dXm = nullptr;            // X' (device, p x n)
  size_t dXm_bytes = 0;
  // Gathered X rows for one level (gather_level): row block i of X_g is row
  // block gather_rows[i] of X.  Shard plans whose units are not one contiguous
  // range (e.g. LPT pairs {j, p̄-1-j}) run their top level as ONE parent of
  // |units|·b_C rows (taller tiles, each A tile read once per rank) instead of
  // one short parent per run of units; start plans restricted to a subset of
  // the first level's children (start_children) contract only those rows.
  // Empty: every level reads X itself.
  std::vector<int> start_children;  // first computed level of a start plan: these jb only
  std::vector<int> gather_rows;
  int gather_level = -1;
  size_t off_gather_rows = 0;       // into the device table buffer
  double* dXt = nullptr;            // X_g (device, |gather_rows|·b_C x n)
  double* dXtp = nullptr;           // X_g with padded column blocks (see dXp)
  size_t dXtp_bytes = 0;
  size_t dXt_bytes = 0;
  int start_level = 0;              // 0 = from A; else compute below caller-provided T(start_level)
  std::vector<int32_t> start_suffixes;  // their calls (m - start_level entries each)
  int stop_level = 0;               // last level computed; its T goes to the caller's output buffer
  cudaStream_t copy_in = nullptr, copy_out = nullptr, copy_out2 = nullptr;
  cudaEvent_t out2_done = nullptr;
  std::vector<cudaEvent_t> chunk_ev;  // A chunk (first block index a) landed
  std::vector<cudaEvent_t> wave_ev;   // a wave's C blocks are final
  std::vector<cudaStream_t> lvl_stream;  // cascade: one stream per level
  std::vector<cudaEvent_t> grp_ev;       // cascade: [k * groups + g] = groups 0..g of level k done
  cudaEvent_t cascade_start = nullptr;
  cudaEvent_t bg_ev[2] = {nullptr, nullptr};  // cascade: non-deferred top rows of later waves done
  std::vector<cudaStream_t> side;   // concurrent launches of one level
  std::vector<cudaEvent_t> join;
  cudaEvent_t fork = nullptr;
  std::vector<cudaEvent_t> events;  // 2 per timed level
  std::vector<int> launch_level;
  std::vector<uint64_t> launch_flops;
  cudaStream_t timed_stream = nullptr;
  // symmetric-aware upload of pipelined host runs (sym_upload.cu): distinct-key
  // blocks by DMA, repeated-key blocks by a zero-copy kernel that reads only
  // the sectors holding orbit representatives and fills the rest in HBM
  bool sym_upload = false;
  bool sym_built = false;
  std::vector<std::vector<std::pair<int64_t, int64_t>>> sym_runs;  // per chunk: DMA rank runs [r0, r1)
  bool sym_dma = true;              // distinct-key blocks by DMA (long runs) or by the zero-copy kernel
  std::vector<int64_t> sym_nzc, sym_nfill;  // per chunk: zero-copy blocks, repeated-key blocks to fill
  int64_t sym_n_zc = 0;
  std::vector<int> sym_h_rank, sym_h_chunk;  // the zero-copy kernel's blocks in chunk order: rank, chunk
  std::vector<unsigned> sym_h_run;           // and run bits (bit d: key[d] == key[d-1]; 0: distinct key)
  std::vector<int> sym_h_frank;              // repeated-key blocks (the fills), chunk order
  std::vector<unsigned> sym_h_frun;
  int64_t sym_fetch_elems = 0;
  int64_t last_upload_bytes = -1;   // bytes of A the last host run moved (-1: none yet)      // doubles one symmetric upload moves over PCIe
  void* d_sym = nullptr;            // device tables + counters
  unsigned long long* d_sym_work = nullptr;
  unsigned* d_sym_ctr = nullptr;
  unsigned* d_sym_free = nullptr;   // per device buffer set: calls whose compute is enqueued (stream-written)
  uint64_t sym_set_issued[2] = {0, 0}, sym_set_released[2] = {0, 0};
  bool sym_set_last[2] = {false, false};  // the set's last host run used the symmetric upload
  cudaStream_t fill_stream = nullptr;
  cudaEvent_t sym_prev_done = nullptr;  // the last symmetric upload's zero-copy half landed
  // SM partition for symmetric-upload runs (green contexts, sym_upload.cu)
  int green_state = 0;              // 0 untried, 1 ready, -1 unavailable
  void* g_up = nullptr;             // CUgreenCtx: the upload kernel's SMs
  void* g_comp = nullptr;           // CUgreenCtx: the rest (compute)
  int g_up_sms = 0;
  cudaStream_t g_sym_stream = nullptr, g_host_stream = nullptr;
  std::vector<cudaStream_t> g_side, g_lvl_stream;  // swapped into side / lvl_stream during green runs
  bool green_active = false;
  std::vector<std::pair<std::string, cudaEvent_t>> atrace;  // BCSS_TRACE=3 marks
  std::vector<cudaEvent_t> fill_ev;  // per chunk: its repeated-key blocks are complete
  const int* d_sym_rank = nullptr;
  const int* d_sym_chunk = nullptr;
  const unsigned* d_sym_run = nullptr;
  const int* d_sym_frank = nullptr;
  const unsigned* d_sym_frun = nullptr;
  uint64_t sym_uploads = 0, sym_ticket_base = 0;
  cudaStream_t sym_stream = nullptr;
};


namespace bcss_host {

int64_t keys_at(const bcss_plan& P, int k);
int64_t blk_at(const bcss_plan& P, int k);
int build_plan(bcss_plan& P);
void build_nbr(bcss_plan& P, int k, std::vector<int2>& out);  // host reference of the device builder
int upload_tables(bcss_plan& P, cudaStream_t stream);
int ensure_workspace(bcss_plan& P);
double* region_for(bcss_plan& P, const WaveHost& W, int k);
int validate_problem(int m, int64_t n, int64_t p, int64_t b_a, int64_t b_c);
int check_int32_limits(int m, int64_t n, int64_t p, int64_t b_a, int64_t b_c, bool reuse);
void invalidate(bcss_plan* P);
int64_t first_rank_with(int64_t a, int m, int64_t extent);
bool is_pinned(const void* p);

// Host-transfer pipeline of run_host: A arrives in chunks (blocks whose first
// index is a, a contiguous range of the packed payload), wave 0's top level
// is split by key ranges that need only the chunks already landed, and each
// wave's C blocks are downloaded while later waves compute.
struct Pipe {
  double* c_host = nullptr;         // per-wave C downloads go here (null: no downloads)
  // A chunk a (blocks with first index a) is resident once chunk_ev[a] fired;
  // null = the plan's own upload events (run_host)
  const cudaEvent_t* chunk_ev = nullptr;
  // symmetric upload: chunk a is also complete once fill_ev[a] fired
  const cudaEvent_t* fill_ev = nullptr;
  int reserve_sms = 0;              // SMs held by the upload kernel (compute grids leave them)
  bool serial = false;              // one compute launch at a time (streamed symmetric uploads)
  // BCSS_TRACE=1: completion events (name, event) polled after the run
  std::vector<std::pair<std::string, cudaEvent_t>>* trace = nullptr;
};
void trace_mark(const Pipe* pipe, const std::string& name, cudaStream_t s);
int run_impl(bcss_plan* P, const double* A, const double* X_, double* C, cudaStream_t s, const Pipe* pipe);
bool sym_eligible(const bcss_plan& P);
bool sym_supported();  // the driver exposes stream wait-value operations
int sym_prepare(bcss_plan& P);
int sym_device(bcss_plan& P);
int sym_upload_ctas(bool async);
int sym_upload_issue(bcss_plan* P, const double* A, double* dA, int set, bool async, bool green,
                     cudaStream_t copy_in, cudaStream_t up_stream, Pipe& pipe);
int sym_green(bcss_plan* P);
int green_compute_stream(bcss_plan* P, int priority, cudaStream_t* out);
void green_destroy(bcss_plan* P);
int sym_release_set(bcss_plan* P, int set, cudaStream_t s);
int wait_chunks(bcss_plan* P, const Pipe* pipe, const cudaEvent_t* chunk_ev, cudaStream_t s, int64_t a);

}  // namespace bcss_host
