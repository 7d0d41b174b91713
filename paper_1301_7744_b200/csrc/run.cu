// Run orchestration: per-level launches (concurrent per tile shape), the
// host-transfer pipeline of bcss_sttsm_run_host, trace marks (plan.hpp).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "plan.hpp"

namespace bcss_host {

// Host-transfer pipeline of run_host: A arrives in chunks (blocks whose first
// index is a, a contiguous range of the packed payload), wave 0's top level
// is split by key ranges that need only the chunks already landed, and each
// wave's C blocks are downloaded while later waves compute.

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
               const double* X_, double* C, long long item_lo, long long item_hi,
               cudaStream_t ls, int sms) {
  const long long total = item_hi - item_lo;
  if (total <= 0) return BCSS_OK;
  const KernelCfg& K = kernel_cfg(X.cfg);
  char* tbl = static_cast<char*>(P->d_tables);
  bcss::LevelArgs a;
  memset(&a, 0, sizeof(a));
  // fast kernels on a b_a that no row group divides contract over blocks
  // padded to b_a' rows: they read the zero-padded copy of X (p x n')
  const int64_t bAp = is_generic(X.cfg) ? P->bA : P->bAp;
  const bool padded = bAp != P->bA;
  const bool gathered = L.k == P->gather_level && !P->gather_rows.empty();
  a.X = gathered ? (padded ? P->dXtp : P->dXt) : (padded ? P->dXp : X_);
  const bool from_input = (P->start_level == 0 && L.k == P->m - 1) || (P->start_level > 0 && L.k == P->start_level - 1);
  a.Tin = from_input ? A : region_for(*P, W, L.k + 1);
  a.Tout = (L.k == P->stop_level) ? C : region_for(*P, W, L.k);
  a.parents = reinterpret_cast<const int4*>(tbl + X.off_parents);
  a.items = reinterpret_cast<const int4*>(tbl + X.off_items) + item_lo;
  a.child_call = reinterpret_cast<const int*>(tbl + L.off_child);
  a.nbr = reinterpret_cast<const int2*>(tbl + P->nbr_off[L.k]);
  a.total_items = total;
  a.keys_in = L.keys_in; a.keys_out = L.keys_out;
  a.blk_in = L.blk_in; a.blk_out = L.blk_out;
  a.n_parents = (int)X.parents.size();
  a.n = (int)(P->nbar * bAp); a.ldx = a.n; a.p_rows = (int)P->p;
  a.nbar = (int)P->nbar; a.bA = (int)P->bA; a.bC = (int)P->bC;
  a.bAp = (int)bAp;
  a.lbA = is_pow2(P->bA) ? ilog2(P->bA) : -1;
  a.k = L.k;
  a.rest = (int)L.rest; a.bAk = (int)L.bAk;
  a.n_tiles = X.n_tiles;
  a.call_out = (P->stop_level > 0 && L.k == P->stop_level && !P->call_out.empty()) ? P->d_call_out : nullptr;
  a.row_mul = L.bAk;
  a.mirror_digits = 0;
  a.lbc = is_pow2(P->bC) ? ilog2(P->bC) : 0;
  if (P->mirror && L.k == 0) {
    a.row_mul = ipow(P->bC, P->m - 1);
    a.mirror_digits = (int)P->m - 1;
  }
  for (int i = 0; i < 10; ++i) a.pw[i] = (long long)std::min<double>(std::pow((double)P->bA, i), 9.0e18);
  int occ = 1;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, K.fn, K.NT, K.smem));
  const long long grid = std::min<long long>(total, (long long)sms * std::max(occ, 1));
  K.fn<<<(unsigned)grid, K.NT, K.smem, ls>>>(a);
  CUDA_TRY(cudaGetLastError());
  return BCSS_OK;
}

// X' for mirrored plans: row block jb of X' is row block p̄-1-jb of X
__global__ void reverse_row_blocks(const double* __restrict__ src, double* __restrict__ dst, long long p, long long n,
                                   long long bc) {
  const long long total = p * n;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / n, c = i - r * n;
    const long long pbar = p / bc, jb = r / bc;
    dst[i] = src[((pbar - 1 - jb) * bc + (r - jb * bc)) * n + c];
  }
}

// X with every b_a column block padded to b_a' columns of zeros behind it
// (fast kernels on a b_a that no row group divides): dst is rows x nbar*b_a'
__global__ void pad_column_blocks(const double* __restrict__ src, double* __restrict__ dst, long long rows,
                                  long long nbar, long long ba, long long bap) {
  const long long np = nbar * bap, total = rows * np;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / np, c = i - r * np;
    const long long ib = c / bap, e = c - ib * bap;
    dst[i] = e < ba ? src[r * nbar * ba + ib * ba + e] : 0.0;
  }
}

int pad_x(bcss_plan* P, const double* src, long long rows, double** buf, size_t* cap, cudaStream_t s) {
  const int64_t bAp = P->bAp;
  const size_t xb = (size_t)(rows * P->nbar * bAp) * sizeof(double);
  if (*cap < xb) {
    if (*buf) cudaFree(*buf);
    *buf = nullptr;
    *cap = 0;
    CUDA_TRY(cudaMalloc(buf, xb));
    *cap = xb;
  }
  pad_column_blocks<<<296, 256, 0, s>>>(src, *buf, rows, P->nbar, P->bA, bAp);
  CUDA_TRY(cudaGetLastError());
  return BCSS_OK;
}

// gathered X rows (plan.hpp gather_rows): row block i of dst is row block rows[i] of src
__global__ void gather_row_blocks(const double* __restrict__ src, double* __restrict__ dst,
                                  const int* __restrict__ rows, long long nblk, long long n, long long bc) {
  const long long per = bc * n;  // doubles per row block (contiguous in both)
  const long long total = nblk * per;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long b = i / per;
    dst[i] = src[(long long)__ldg(rows + b) * per + (i - b * per)];
  }
}

int ensure_side(bcss_plan* P, int n) {
  while ((int)P->side.size() < n) {
    cudaStream_t ss;
    if (P->green_active) {  // a green symmetric-upload run: the compute partition
      const int st = green_compute_stream(P, 0, &ss);
      if (st) return st;
    } else {
      CUDA_TRY(cudaStreamCreateWithFlags(&ss, cudaStreamNonBlocking));
    }
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
  const cudaEvent_t* chunk_ev = pipe && pipe->chunk_ev ? pipe->chunk_ev : P->chunk_ev.data();
  // Without a caller workspace or an explicit limit, fit the temporaries into
  // the free HBM by splitting the units into more waves.
  if (!P->d_ws && P->ws_limit == 0 && !P->keep_temps && P->start_level == 0 && P->stop_level == 0) {
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess && P->ws_bytes > free_b / 10 * 9) {
      P->ws_limit = free_b / 20 * 17;
      invalidate(P);
      if ((st = build_plan(*P))) return st;
    }
  }
  if ((st = upload_tables(*P, s))) return st;
  if (P->call_out_dirty) {  // per-call destinations of the stop level
    if (!P->call_out.empty()) {
      const size_t nb = P->call_out.size() * sizeof(double*);
      if (P->d_call_out_cap < nb) {
        if (P->d_call_out) cudaFree(P->d_call_out);
        P->d_call_out = nullptr;
        P->d_call_out_cap = 0;
        CUDA_TRY(cudaMalloc(&P->d_call_out, nb));
        P->d_call_out_cap = nb;
      }
      CUDA_TRY(cudaMemcpyAsync(P->d_call_out, P->call_out.data(), nb, cudaMemcpyHostToDevice, s));
      CUDA_TRY(cudaStreamSynchronize(s));
    }
    P->call_out_dirty = false;
  }
  if (P->mirror) {  // the kernels contract X' (row blocks reversed)
    const size_t xb = (size_t)(P->p * P->n) * sizeof(double);
    if (P->dXm_bytes < xb) {
      if (P->dXm) cudaFree(P->dXm);
      P->dXm = nullptr;
      P->dXm_bytes = 0;
      CUDA_TRY(cudaMalloc(&P->dXm, xb));
      P->dXm_bytes = xb;
    }
    // pipelined host run: X is uploaded on copy_in ahead of A chunk 0
    if (pipe) CUDA_TRY(cudaStreamWaitEvent(s, chunk_ev[0], 0));
    reverse_row_blocks<<<296, 256, 0, s>>>(X_, P->dXm, P->p, P->n, P->bC);
    CUDA_TRY(cudaGetLastError());
    X_ = P->dXm;
  }
  const bool pad = P->bAp != P->bA;  // (generic launches, if any, keep reading the plain X)
  if (pad) {
    if (pipe && !P->mirror) CUDA_TRY(cudaStreamWaitEvent(s, chunk_ev[0], 0));  // X was uploaded ahead of A chunk 0
    if ((st = pad_x(P, X_, P->p, &P->dXp, &P->dXp_bytes, s))) return st;
  }
  if (!P->gather_rows.empty()) {  // gathered X rows of one level (shard / child-subset plans)
    const size_t xb = P->gather_rows.size() * (size_t)(P->bC * P->n) * sizeof(double);
    if (P->dXt_bytes < xb) {
      if (P->dXt) cudaFree(P->dXt);
      P->dXt = nullptr;
      P->dXt_bytes = 0;
      CUDA_TRY(cudaMalloc(&P->dXt, xb));
      P->dXt_bytes = xb;
    }
    if (pipe) CUDA_TRY(cudaStreamWaitEvent(s, chunk_ev[0], 0));  // X was uploaded ahead of A chunk 0
    const int* rows = reinterpret_cast<const int*>(static_cast<char*>(P->d_tables) + P->off_gather_rows);
    gather_row_blocks<<<296, 256, 0, s>>>(X_, P->dXt, rows, (long long)P->gather_rows.size(), P->n, P->bC);
    CUDA_TRY(cudaGetLastError());
    if (pad && (st = pad_x(P, P->dXt, (long long)P->gather_rows.size() * P->bC, &P->dXtp, &P->dXtp_bytes, s))) return st;
  }
  if ((st = ensure_workspace(*P)) == BCSS_ERR_NOMEM && !P->d_ws && !P->keep_temps && P->start_level == 0 &&
      P->stop_level == 0 && P->ws_bytes > 0) {
    // the allocation failed although the plan looked like it fit (other
    // allocations, fragmentation): split into more waves and retry once
    cudaGetLastError();
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess) {
      P->ws_limit = std::min(P->ws_bytes / 2, free_b / 20 * 17);
      invalidate(P);
      if ((st = build_plan(*P))) return st;
      if ((st = upload_tables(*P, s))) return st;
      st = ensure_workspace(*P);
    }
  }
  if (st) return st;
  int dev, sms;
  CUDA_TRY(cudaGetDevice(&dev));
  CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  // a symmetric upload's kernel holds pipe->reserve_sms SMs for the whole
  // call: persistent grids that counted on them would wait a tile's worth
  if (pipe && pipe->reserve_sms) sms = std::max(1, sms - pipe->reserve_sms);
  int64_t launches = 0;
  if (P->timing) {
    P->launch_level.clear();
    P->launch_flops.clear();
    P->timed_stream = s;
  }
  // Launches of one level (one per tile shape) are independent: they run
  // concurrently on side streams, so one launch's tail overlaps the next
  // launch's CTAs instead of idling SMs.
  int level_idx = 0;
  const size_t blk_c = (size_t)ipow(P->bC, P->m);
  for (size_t wi = 0; wi < P->waves.size(); ++wi) {
    const WaveHost& W = P->waves[wi];
    // a streamed symmetric upload's kernel must become resident on the SMs
    // the compute grids leave free while the previous call computes: those
    // runs issue one compute launch at a time (concurrent launches would fill
    // the free SMs, and the next call's upload kernel would wait for them)
    const bool serial = pipe && pipe->serial;
    const bool cascade = pipe && P->cascade && wi == 0 && !serial;
    if (cascade) {
      // Levels m-1..1 of the first wave as key-group sub-launches, one stream
      // per level: group g of the top level waits for A chunks 0..a_{g+1}-1,
      // group g of level k for groups 0..g of level k+1 (a key of first index a
      // only reads blocks whose first index is <= a), so the lower levels run
      // while A is still uploading.
      const int G = (int)P->group_a.size() - 1;
      if ((int)P->lvl_stream.size() < 2 * P->m) {
        // two streams per level (groups alternate); higher levels get higher
        // priority so the gated top level keeps pace with the upload and the
        // levels below fill the idle SMs
        int lo = 0, hi = 0;
        CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        while ((int)P->lvl_stream.size() < 2 * P->m) {
          const int k = (int)P->lvl_stream.size() / 2;
          // (the greatest priority stays free for the symmetric upload's streams)
          const int top = hi < lo ? hi + 1 : hi;
          const int prio = std::max(top, lo - (k * (lo - top) + P->m - 2) / std::max(1, P->m - 1));
          cudaStream_t ss;
          if (P->green_active) {
            if ((st = green_compute_stream(P, prio, &ss))) return st;
          } else {
            CUDA_TRY(cudaStreamCreateWithPriority(&ss, cudaStreamNonBlocking, prio));
          }
          P->lvl_stream.push_back(ss);
        }
      }
      while (P->grp_ev.size() < (size_t)(P->m * G)) {
        cudaEvent_t ev;
        CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        P->grp_ev.push_back(ev);
      }
      if (!P->cascade_start) CUDA_TRY(cudaEventCreateWithFlags(&P->cascade_start, cudaEventDisableTiming));
      for (int q = 0; q < 2; ++q)
        if (!P->bg_ev[q]) CUDA_TRY(cudaEventCreateWithFlags(&P->bg_ev[q], cudaEventDisableTiming));
      CUDA_TRY(cudaEventRecord(P->cascade_start, s));  // tables and X' are ready
      for (const LevelHost& L : W.levels) {
        if (L.k == 0) continue;
        for (int q = 0; q < 2; ++q) CUDA_TRY(cudaStreamWaitEvent(P->lvl_stream[2 * L.k + q], P->cascade_start, 0));
        for (int g = 0; g < G; ++g) {
          cudaStream_t ls = P->lvl_stream[2 * L.k + (g & 1)];
          if (L.k == P->m - 1) {
            if ((st = wait_chunks(P, pipe, chunk_ev, ls, P->group_a[g + 1] - 1))) return st;
          } else {  // groups <= g of level k+1: g on one stream, g-1 (and earlier) on the other
            CUDA_TRY(cudaStreamWaitEvent(ls, P->grp_ev[(L.k + 1) * G + g], 0));
            if (g > 0) CUDA_TRY(cudaStreamWaitEvent(ls, P->grp_ev[(L.k + 1) * G + g - 1], 0));
          }
          // top level: the first wave's unit rows first (its lower levels only
          // read those), the other units' rows after the group's event; their
          // late groups (>= defer_group) wait until the first wave's level 0
          const bool top = L.k == P->m - 1;
          for (size_t li = 0; li < L.launches.size(); ++li) {
            const LaunchHost& X = L.launches[li];
            const long long lo = X.group_items[g], hi = top ? X.group_w0[g] : X.group_items[g + 1];
            if (hi <= lo) continue;
            if ((st = launch_one(P, W, L, X, A, X_, C, lo, hi, ls, sms))) return st;
            ++launches;
          }
          if (g > 0) CUDA_TRY(cudaStreamWaitEvent(ls, P->grp_ev[L.k * G + g - 1], 0));  // groups <= g done
          CUDA_TRY(cudaEventRecord(P->grp_ev[L.k * G + g], ls));
          if (top && g < P->defer_group) {
            for (size_t li = 0; li < L.launches.size(); ++li) {
              const LaunchHost& X = L.launches[li];
              const long long lo = X.group_w0[g], hi = X.group_items[g + 1];
              if (hi <= lo) continue;
              if ((st = launch_one(P, W, L, X, A, X_, C, lo, hi, ls, sms))) return st;
              ++launches;
            }
          }
        }
        if (L.k == P->m - 1)  // the non-deferred rows of later units: done when both streams are
          for (int q = 0; q < 2; ++q) CUDA_TRY(cudaEventRecord(P->bg_ev[q], P->lvl_stream[2 * L.k + q]));
        trace_mark(pipe, "wave0 level" + std::to_string(L.k) + " done", P->lvl_stream[2 * L.k + ((G - 1) & 1)]);
      }
      CUDA_TRY(cudaStreamWaitEvent(s, P->grp_ev[1 * G + G - 1], 0));
    }
    for (const LevelHost& L : W.levels) {
      if (cascade && L.k >= 1) continue;
      const int nl = (int)L.launches.size();
      // chunk-gated top level of the first wave (pipelined host run)
      const bool gate = pipe && wi == 0 && L.k == P->m - 1;
      // every launch of the top level holds one piece of the single top parent;
      // key ranges follow A's chunks only for sorted keys (reuse=True): a
      // product key K reads blocks whose first index is min(K), not K[0]
      bool gate_split = gate && P->reuse;
      for (const LaunchHost& X : L.launches)
        gate_split = gate_split && X.parents.size() == 1 && !is_generic(X.cfg);  // key-major items only
      if (gate && !gate_split && (st = wait_chunks(P, pipe, chunk_ev, s, P->nbar - 1))) return st;
      const bool conc = !serial && ((P->concurrent && nl > 1) || gate_split);
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
        // keys with first index <= a need only A chunks 0..a: ~8 key groups per
        // launch (tile shape), issued group-major so every shape's early keys
        // run first; sub-launches alternate between two streams, each waiting
        // for its group's last chunk
        const int64_t nb = P->nbar;
        const int groups = (int)std::min<int64_t>(8, nb);
        int64_t a0 = 0;
        int sub = 0;
        for (int g = 0; g < groups; ++g) {
          int64_t a1 = (g == groups - 1) ? nb : std::max(a0 + 1, (nb * (g + 1)) / groups);
          const int64_t k_lo = first_rank_with(a0, P->m - 1, nb), k_hi = first_rank_with(a1, P->m - 1, nb);
          for (int li = 0; li < nl; ++li) {
            const LaunchHost& X = L.launches[li];
            const int64_t per_key = X.item_off.back() / L.keys_out;
            if (per_key == 0 || k_hi <= k_lo) continue;
            cudaStream_t ls = (serial || sub++ % 2 == 0) ? s : P->side[0];
            if ((st = wait_chunks(P, pipe, chunk_ev, ls, a1 - 1))) return st;
            if ((st = launch_one(P, W, L, X, A, X_, C, k_lo * per_key, k_hi * per_key, ls, sms)))
              return st;
            ++launches;
          }
          a0 = a1;
        }
      } else {
        // SM shares: the tile shapes of one level run side by side for the
        // whole level, each on a share of the SMs proportional to its modelled
        // time, so the memory-bound small-row shapes (8/16-row parents) draw
        // on HBM while the tall shapes keep the DMMA pipes busy, instead of
        // one after the other.  The first share_frac of every launch's items
        // runs on its share; the rest follows on the same stream as a
        // full-width grid of short CTAs that fills SMs as the shares finish.
        std::vector<int> share(nl, 0);
        bool shared = conc && nl > 1 && P->share_frac > 0;
        if (shared) {
          double total = 0;
          int live = 0;
          for (const LaunchHost& X : L.launches) {
            if (X.item_off.back() == 0) continue;
            if (X.cost <= 0 || is_generic(X.cfg)) shared = false;
            total += X.cost;
            ++live;
          }
          shared = shared && live > 1 && live <= sms && total > 0;
          if (shared) {
            // largest-remainder apportionment with at least one SM per launch
            std::vector<std::pair<double, int>> rem;
            int used = 0;
            for (int li = 0; li < nl; ++li) {
              const LaunchHost& X = L.launches[li];
              if (X.item_off.back() == 0) continue;
              const double q = X.cost / total * sms;
              share[li] = std::max(1, (int)q);
              used += share[li];
              rem.push_back({q - (int)q, li});
            }
            std::sort(rem.begin(), rem.end(), [](auto& x, auto& y) { return x.first > y.first; });
            for (size_t i = 0; used < sms && !rem.empty(); i = (i + 1) % rem.size()) { ++share[rem[i].second]; ++used; }
            for (size_t i = 0; used > sms; i = (i + 1) % rem.size())
              if (share[rem[rem.size() - 1 - i].second] > 1) { --share[rem[rem.size() - 1 - i].second]; --used; }
          }
        }
        for (int li = 0; li < nl; ++li) {
          const LaunchHost& X = L.launches[li];
          cudaStream_t ls = (li == 0 || !conc) ? s : P->side[li - 1];
          const long long total = X.item_off.back();
          if (total == 0) continue;
          if (shared) {
            long long head = (long long)((double)total * P->share_frac);
            head -= head % share[li];  // whole rounds of the share
            if (head > 0) {
              if ((st = launch_one(P, W, L, X, A, X_, C, 0, head, ls, share[li]))) return st;
              ++launches;
            }
            if (head < total) {
              if ((st = launch_one(P, W, L, X, A, X_, C, head, total, ls, sms))) return st;
              ++launches;
            }
            continue;
          }
          if ((st = launch_one(P, W, L, X, A, X_, C, 0, total, ls, sms))) return st;
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
      if (pipe && L.k == 0 && pipe->c_host) {
        // this wave's C blocks are final: download them (runs of consecutive ranks)
        while (P->wave_ev.size() <= wi) {  // the plan may have been rebuilt with more waves
          cudaEvent_t ev;
          CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
          P->wave_ev.push_back(ev);
        }
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
      }
      if (pipe && L.k == 0) {
        if (cascade) {
          // deferred top-level rows of the later waves, then every later wave
          // may read T(m-1)
          const LevelHost& T = W.levels.front();
          const int G = (int)P->group_a.size() - 1;
          for (int g = P->defer_group; g < G; ++g)
            for (size_t li = 0; li < T.launches.size(); ++li) {
              const LaunchHost& X = T.launches[li];
              const long long lo = X.group_w0[g], hi = X.group_items[g + 1];
              if (hi <= lo) continue;
              if ((st = launch_one(P, W, T, X, A, X_, C, lo, hi, s, sms))) return st;
              ++launches;
            }
          for (int q = 0; q < 2; ++q) CUDA_TRY(cudaStreamWaitEvent(s, P->bg_ev[q], 0));
        }
        // submit what is queued so far (the driver otherwise batches it until a sync)
        cudaStreamQuery(s);
        if (P->copy_out) cudaStreamQuery(P->copy_out);
        if (P->copy_out2) cudaStreamQuery(P->copy_out2);
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

}  // namespace bcss_host
