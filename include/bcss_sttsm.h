/*
 * bcss_sttsm.h — C ABI of the B200-native BCSS change of basis ("sttsm").
 *
 * Computes C = [A; X, ..., X] = A x_0 X x_1 X ... x_{m-1} X for a symmetric
 * order-m tensor A (dimension n) held in Blocked Compact Symmetric Storage,
 * with the algorithm-by-blocks that reuses partially-symmetric temporaries.
 * This is the drop-in for the reference hot path
 *   blocksym.sttsm_bcss(a, x, b_c, counter, reuse, temp_hook)
 *   (/root/reference/pkg/src/blocksym/change_of_basis.py:239-284).
 *
 * Buffer contract (identical to the reference's .bcss payload,
 * /root/reference/pkg/src/blocksym/io.py:50-55):
 *   A_packed : simplex_count(n/b_a, m) canonical blocks in hypertriangle
 *              (lexicographic, nondecreasing-index) order, each b_a^m doubles
 *              in dimensional (Fortran) order.
 *   X        : p x n doubles, row-major (numpy C-order; the reference slices
 *              x[jb*b_c:(jb+1)*b_c, ib*b_a:(ib+1)*b_a], change_of_basis.py:229).
 *   C_packed : simplex_count(p/b_c, m) blocks of b_c^m doubles, same order.
 *
 * No torch or CUDA types appear in the signatures: streams are passed as
 * void* (a cudaStream_t), device buffers as plain pointers.  Functions return
 * BCSS_OK (0) or a status code; bcss_last_error() holds the message of the
 * last failure on the calling thread.  Nothing throws across the ABI.
 */
#ifndef BCSS_STTSM_H
#define BCSS_STTSM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes.  The Python host layer maps them onto the reference's
 * exception types (/root/reference/pkg/src/blocksym/errors.py:4-25). */
enum bcss_status {
  BCSS_OK = 0,
  BCSS_ERR_PARAMETER = 1,          /* ParameterError (e.g. m < 2, change_of_basis.py:56-57) */
  BCSS_ERR_SHAPE = 2,              /* ShapeError (dims / X shape, change_of_basis.py:58-62) */
  BCSS_ERR_BLOCK_DIVISIBILITY = 3, /* BlockDivisibilityError (change_of_basis.py:264-265) */
  BCSS_ERR_RANGE = 4,              /* RangeError (index outside the grid, storage.py:131-133) */
  BCSS_ERR_CUDA = 5,               /* CUDA runtime failure (device, launch, memory) */
  BCSS_ERR_NOMEM = 6,              /* workspace does not fit */
  BCSS_ERR_STATE = 7               /* API misuse (null plan, missing workspace, ...) */
};

typedef struct bcss_plan bcss_plan; /* opaque */

/* Message of the last failure on this thread ("" if none). */
const char* bcss_last_error(void);
/* ABI version of this library (major*100 + minor). */
int bcss_abi_version(void);

/* ---- combinatorics and cost model (host only, no GPU needed) ------------- */

/* C(extent+m-1, m): number of nondecreasing m-tuples over 0..extent-1.
 * Replaces simplex_count (indexing.py:64-68). Returns -1 on bad arguments. */
int64_t bcss_simplex_count(int64_t extent, int m);

/* Lexicographic rank of the nondecreasing tuple idx[0..m-1] among
 * hypertriangle_iter(extent, m) (indexing.py:57-61); this is the block's
 * position in a packed payload. */
int bcss_hypertriangle_rank(const int64_t* idx, int m, int64_t extent, int64_t* out_rank);

/* Inverse of bcss_hypertriangle_rank: the rank-th nondecreasing tuple. */
int bcss_hypertriangle_unrank(int64_t rank, int m, int64_t extent, int64_t* out_idx);

/* Exact flop count of the blocked algorithm, bcss_costs(...).flops
 * (costs.py:83-112): 2*nbar*b_c*b_a^m * sum_d C(pbar+d,d+1)*blocks(d)*(b_c/b_a)^d.
 * reuse=0 selects the plain algorithm-by-blocks count. */
int bcss_blocked_flops(int m, int64_t n, int64_t p, int64_t b_a, int64_t b_c, int reuse,
                       uint64_t* out_flops);

/* ---- plans ---------------------------------------------------------------- */

/* Validate the problem (change_of_basis.py:54-63, 259-266) and build the
 * level/work-list plan.  reuse=1 is the reference default (canonical blocks of
 * every temporary only); reuse=0 materializes every temporary block
 * (_DenseBlockTable, change_of_basis.py:157-167). */
int bcss_plan_create(int m, int64_t n, int64_t p, int64_t b_a, int64_t b_c, int reuse,
                     bcss_plan** out_plan);
int bcss_plan_destroy(bcss_plan* plan);

/* Restrict the plan to a subset of the top-level output block rows
 * ("units": values of jb_{m-1}, the outermost loop of descend,
 * change_of_basis.py:269-283).  Only the C blocks whose largest block index
 * lies in the subset are written.  Used to shard C across GPUs. */
int bcss_plan_set_units(bcss_plan* plan, const int32_t* units, int n_units);

/* Upper bound on workspace bytes; the plan processes the units in waves so
 * that live temporaries fit.  0 = no limit. */
int bcss_plan_set_workspace_limit(bcss_plan* plan, size_t bytes);

/* Keep every temporary of every level resident (for temp_hook replays). */
int bcss_plan_set_keep_temps(bcss_plan* plan, int keep);

/* Device workspace the plan needs (temporaries + tables) for its settings. */
int bcss_plan_workspace_bytes(bcss_plan* plan, size_t* out_bytes);

/* Caller-provided device workspace (>= bcss_plan_workspace_bytes).  Without
 * it the plan allocates its own with cudaMalloc on first run. */
int bcss_plan_set_workspace(bcss_plan* plan, void* dev_ptr, size_t bytes);

/* Plan statistics: waves, kernel launches per run, exact flops of the
 * assigned units, and number of C blocks written. */
int bcss_plan_stats(bcss_plan* plan, int64_t* waves, int64_t* launches, uint64_t* flops,
                    int64_t* c_blocks);

/* Launches per run on the warp-specialized DMMA kernels (b_a in {4, 8, 16,
 * 32, 64}, any b_c) and on the generic kernel (other b_a, e.g. 1, 2, 3). */
int bcss_plan_kernel_mix(bcss_plan* plan, int64_t* fast_launches, int64_t* generic_launches);

/* Level k's neighbour table as int32 pairs {rank of the stored block of
 * T(k+1) holding the logical block (K, ib), redirection code word}, keys x
 * n/b_a entries (2 * that many int32): from_device = 1 copies the table the
 * device builder generated (the plan's tables are built on the device: the
 * BCSS block index and redirection enumeration, canonicalize of
 * indexing.py:34-54, rank of indexing.py:57-68), 0 builds the same table
 * on the host (reference for tests).  out = NULL returns the size only. */
int bcss_plan_neighbour_table(bcss_plan* plan, int k, int from_device, int32_t* out, int64_t n_max,
                              int64_t* out_n);

/* ---- execution ------------------------------------------------------------ */

/* Device-resident run: A_packed, X, C_packed are device pointers; the work is
 * enqueued on `stream` (cudaStream_t, NULL = legacy default) and returns
 * without synchronizing. */
int bcss_sttsm_run(bcss_plan* plan, const double* A_packed, const double* X, double* C_packed,
                   void* stream);

/* Device-resident run whose input A is still arriving: chunk_events[a]
 * (cudaEvent_t, one per first block index a = 0..n/b_a-1) fires once the
 * blocks of A whose first index is a (one contiguous range of the packed
 * payload) are resident.  The top level's key groups wait only for the
 * chunks they read (a key of first index a reads chunks 0..a), so the
 * compute overlaps the rest of the transfer - e.g. the per-chunk NCCL
 * broadcasts of the multi-GPU host path, where every rank uploads only its
 * share of A over its own PCIe link.  Results are bit-identical to
 * bcss_sttsm_run.  Plans that start below A (start calls) ignore the events. */
int bcss_sttsm_run_gated(bcss_plan* plan, const double* A_packed, const double* X, double* C_packed,
                         void* stream, const void* const* chunk_events, int n_events);

/* Host-buffer run (the reference's call shape): copies A and X to the device,
 * runs, copies C back and synchronizes.  The host buffers are sized by
 * bcss_plan_io_elems: A / C for a full plan, the start-level temporaries in
 * and the stop-level temporaries out for partial plans.  Pinned host memory gives full
 * PCIe bandwidth; pageable memory works too.  With a pipeline set (below) and
 * pinned buffers, the A upload, the compute and the C download overlap.  A
 * plan restricted to some units (bcss_plan_set_units) or to start calls writes
 * only its own C blocks into C_packed and leaves the others untouched.  A
 * pipelined plan given pageable buffers stages those (only) through plan-owned
 * pinned memory (all host cores) and then runs the pipeline. */
int bcss_sttsm_run_host(bcss_plan* plan, const double* A_packed, const double* X,
                        double* C_packed);
/* Streaming form of the pipelined host run (pinned buffers, pipeline set):
 * enqueues upload, compute and download and returns.  Consecutive calls
 * alternate two device buffer sets, so call i+1's upload overlaps call i's
 * compute and download (PCIe is full duplex).  The caller keeps A, X, C alive
 * and unmodified until bcss_plan_wait; C is complete after it. */
int bcss_sttsm_run_host_async(bcss_plan* plan, const double* A_packed, const double* X,
                              double* C_packed);
int bcss_plan_wait(bcss_plan* plan);

/* Page-lock a caller-owned host range in place (cudaHostRegister), so host
 * runs read / write it by DMA at PCIe speed instead of staging it through
 * plan-owned pinned memory.  The drop-in registers a BcssTensor's packed
 * payload once and unregisters it when the tensor is released; the reference
 * has no counterpart (its arrays never leave the host).  Already-pinned
 * ranges are accepted as they are. */
int bcss_host_register(void* ptr, size_t bytes);
int bcss_host_unregister(void* ptr);
/* Pinned host allocations (cudaMallocHost) for results the drop-in returns. */
int bcss_host_alloc(size_t bytes, void** out_ptr);
int bcss_host_free(void* ptr);
/* *out = 1 if ptr is pinned (cudaHostAlloc / registered) host memory. */
int bcss_host_is_pinned(const void* ptr, int* out);

/* Overlap host transfers with compute in bcss_sttsm_run_host: A is uploaded
 * in chunks (blocks with first index a) that gate the top-level work (and, when
 * the plan's model predicts a gain, the first wave's lower levels: key groups of
 * equal first index), and the top-level units are split into at most `waves`
 * groups whose C blocks download while later groups compute.  Such a plan
 * contracts the C modes in mirrored order (X with reversed row blocks) so every
 * group's C blocks form one contiguous range: its results equal the plain
 * plan's to rounding (~1e-16 relative), not bit for bit, and are identical
 * between bcss_sttsm_run and bcss_sttsm_run_host.  0 = off. */
int bcss_plan_set_pipeline(bcss_plan* plan, int waves);

/* Symmetric-aware upload for pipelined host runs (no reference counterpart:
 * it exploits the symmetry a BCSS tensor represents, storage.py:177-216).
 * Blocks whose key repeats an index carry each orbit of their repeated modes'
 * permutations once; with `on`, bcss_sttsm_run_host[_async] moves only the
 * 32-byte sectors holding orbit representatives of those blocks (read by a
 * zero-copy kernel from the mapped pinned A; the other elements are filled from
 * the representatives in HBM) and the distinct-key blocks by DMA.  Results are
 * bit-identical to the full upload when the repeated-key blocks are exactly
 * symmetric (the reference's compress(..., tol=0), bcss_symmetrize_blocks);
 * otherwise every orbit contributes its representative's value.  Needs
 * power-of-two b_a >= 4 and a pinned, device-mapped A; other runs upload all of
 * A.  bcss_plan_upload_bytes: bytes of A one host run moves over PCIe. */
int bcss_plan_set_symmetric_upload(bcss_plan* plan, int on);
int bcss_plan_upload_bytes(bcss_plan* plan, int64_t* out_bytes);
/* bytes of A the plan's last host run moved (-1 before the first) */
int bcss_plan_last_upload_bytes(bcss_plan* plan, int64_t* out_bytes);

/* Partial runs, the exchange points of the multi-GPU schedule:
 * stop_level > 0 computes levels m-1 .. stop_level only and writes T(stop_level)
 * (calls in bcss_plan_level_calls order, each keys x block doubles) to the
 * run's output buffer instead of C;
 * start calls make the plan compute below the given calls of level `level`
 * (m-level suffix entries each), reading their T(level) from the run's input
 * buffer (in the given call order) instead of A.  level = m restores a full run. */
int bcss_plan_set_stop_level(bcss_plan* plan, int stop_level);
/* Fused exchange for a stop-level plan: the kernel computing T(stop_level)
 * writes call i (bcss_plan_level_calls order, keys x block doubles) straight
 * to ptrs[i] - e.g. a slot of another GPU's receive buffer opened with
 * bcss_ipc_open_handle (NVLink peer stores) - instead of the output buffer;
 * a NULL entry keeps the default slot.  n must equal the number of stop-level
 * calls; n = 0 clears the table.  Replaces the owner -> assignee send/recv of
 * the multi-GPU schedule S5. */
int bcss_plan_set_call_outputs(bcss_plan* plan, const void* const* ptrs, int64_t n);
/* Device memory for exchange buffers and its CUDA IPC handle (64 bytes), so
 * the other ranks' kernels can address it. */
int bcss_device_alloc(size_t bytes, void** out_ptr);
int bcss_device_free(void* ptr);
int bcss_ipc_get_handle(const void* dev_ptr, void* out_handle64);
int bcss_ipc_open_handle(const void* handle64, void** out_ptr);
int bcss_ipc_close_handle(void* ptr);
/* Stream-ordered copy between any two device addresses of this process,
 * including peer buffers opened with bcss_ipc_open_handle (NVLink DMA): the
 * T(m-1) hand-over from an owner GPU to its helper in the S5 schedule. */
int bcss_copy_async(void* dst, const void* src, size_t bytes, void* stream);
int bcss_plan_set_start_calls(bcss_plan* plan, int level, const int32_t* suffixes, int n_calls);
/* With exactly one start call (J, ...): its first computed level produces only
 * the children (jb, J, ...) for jb in `jbs` (strictly increasing, each <= J)
 * instead of all jb <= J - a slice of the owner's level work handed to a
 * helper GPU that received the start temporary.  Bit-identical to the same
 * calls of the full plan.  n = 0 clears. */
int bcss_plan_set_start_children(bcss_plan* plan, const int32_t* jbs, int n);
/* Suffixes (m-k entries each) of the plan's level-k calls, in buffer order. */
int bcss_plan_level_calls(bcss_plan* plan, int k, int32_t* out, int64_t n_max, int64_t* out_n);
/* Element counts of the run's input (A or start temporaries) and output
 * (C or stop-level temporaries) buffers. */
int bcss_plan_io_elems(bcss_plan* plan, int64_t* in_elems, int64_t* out_elems);

/* Device pointer and element count of the temporary T(k) produced for the
 * call whose suffix is (jb_k, ..., jb_{m-1}) (nondecreasing, m-k entries),
 * valid after a run with keep_temps=1.  Blocks are canonical keys in
 * hypertriangle order (reuse=1) or all keys in product order (reuse=0), each
 * b_a^k * b_c^(m-k) doubles in the reference's block layout
 * (a_0..a_{k-1}, c_k..c_{m-1}), Fortran order (change_of_basis.py:231-235). */
int bcss_plan_temp(bcss_plan* plan, int k, const int32_t* suffix, const double** out_ptr,
                   int64_t* out_elems);

/* Copy that temporary to host memory (elems must equal the temporary's size);
 * synchronizes the device. */
int bcss_plan_temp_copy(bcss_plan* plan, int k, const int32_t* suffix, double* host_out,
                        int64_t elems);

/* Number of user kernels the last run launched. */
int bcss_plan_last_launches(bcss_plan* plan, int64_t* out_launches);

/* Packed-payload ranks of the C blocks this plan writes (its units), in the
 * order they are produced; n_max bounds the output array.  Used to gather a
 * sharded C. */
int bcss_plan_c_block_ranks(bcss_plan* plan, int64_t* out_ranks, int64_t n_max, int64_t* out_n);

/* Per-launch timing: with timing on, every launch of the next runs is
 * bracketed by CUDA events on the run's stream; bcss_plan_launch_times
 * returns, for the last run, each launch's level k, exact flops and
 * device milliseconds (synchronizes the stream). */
int bcss_plan_set_timing(bcss_plan* plan, int on);
int bcss_plan_launch_times(bcss_plan* plan, int32_t* out_level, uint64_t* out_flops,
                           float* out_ms, int64_t n_max, int64_t* out_n);

/* Blocked symmetrization of a packed BCSS payload in device memory (order m,
 * dimension dim, block dimension b), in place on `stream`: every canonical
 * block whose key repeats an index is averaged over the permutations of the
 * modes of each run of equal indices, so the represented tensor becomes
 * exactly symmetric - the blocked counterpart of the reference's
 * symmetrize (change_of_basis.py:287-295). */
int bcss_symmetrize_blocks(double* payload, int m, int64_t dim, int64_t b, void* stream);

/* Diagnostic: FP64 tensor-core (DMMA) peak of the current device, measured
 * with a register-resident mma.sync m8n8k4 f64 loop over all SMs (TFLOP/s).
 * Used as the roofline denominator; no reference counterpart. */
int bcss_probe_fp64_peak(double* out_tflops);

#ifdef __cplusplus
}
#endif

#endif /* BCSS_STTSM_H */
