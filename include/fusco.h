/*
 * fusco.h — C ABI of the B200-native Fusco MoE token shuffle (libfusco.so).
 *
 * One handle per (process, GPU) = one expert-parallel rank.  Every call is
 * asynchronous on the caller's CUDA stream, allocates nothing, and returns
 * 0 on success or a negative FS_E* code (message via fs_last_error()).
 * No C++ exceptions and no torch types cross this boundary: plain pointers
 * (device pointers unless stated) and sizes only.
 *
 * Reference interfaces each entry point replaces (paths relative to the
 * reference package root pkg/src/shuffleforge/):
 *
 *   fs_layout    planner.py:138-159  _activation_layouts  (row order (expert,
 *                source, token) and the inverse map row_of[t,k])
 *                planner.py:178-196  dispatch_loads       (per-rank dedup bytes)
 *                routing.py:86-98    derive_token_node    (first_mask)
 *                planner.py:485-497  build_plan_pair      (the on-device plan)
 *   fs_dispatch  engine.py:266-276   apply_node_level + apply_expert_level
 *                (dispatch direction) and their pipelined/threaded form
 *                engine.py:799-851  _wallclock_dispatch
 *   fs_combine   engine.py:266-276   apply_expert_level + apply_node_level
 *                (combine direction) fused with engine.py:313-338
 *                _reduce_one / reduce_outputs (k-ascending weighted sum)
 *                and engine.py:967-1049 _wallclock_combine
 *   fs_sym_* / fs_ipc_*  the simulated link substrate (RingBuffer/TokenBucket,
 *                engine.py:637-680) becomes NVLink P2P over symmetric,
 *                IPC-mapped device regions.
 *
 * SPEC.md names these ops build_plan / execute_dispatch / execute_combine
 * (SPEC.md:260,396,405).
 */
#ifndef FUSCO_H_
#define FUSCO_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FS_ABI_VERSION 2
#define FS_MAX_RANKS 32

/* return codes */
#define FS_OK 0
#define FS_EINVAL (-1)    /* bad argument (ValueError in the Python layer) */
#define FS_ECUDA (-2)     /* a CUDA runtime call failed */
#define FS_ETIMEOUT (-3)  /* a peer flag wait exceeded the timeout */
#define FS_ERANGE (-4)    /* routing data out of range (expert id, row cap) */

/* phase bits: production calls pass FS_PHASE_ALL.  Single-GPU emulation of
 * P ranks calls LOCAL for every rank, then REMOTE for every rank, so that no
 * kernel ever waits on a kernel that has not been launched yet. */
#define FS_PHASE_LOCAL 1  /* work that only publishes to peers            */
#define FS_PHASE_REMOTE 2 /* work that waits for what peers published     */
#define FS_PHASE_ALL 3

/* payload dtypes for the combine reduction */
#define FS_DTYPE_F32 0
#define FS_DTYPE_BF16 1

/* combine source buffer on the expert ranks */
#define FS_SRC_ACT 0     /* dispatch output itself (identity expert)      */
#define FS_SRC_ACT_OUT 1 /* the symmetric expert-output buffer           */

/* combine accumulation */
#define FS_ACC_F32 0 /* fp32 FMA, k ascending (production)                  */
#define FS_ACC_F64 1 /* f64 mul then add, k ascending: bit-exact with
                        engine.py:322-331 when weights are f64            */

/* layout statistics (int64 stats[FS_NSTATS]) */
#define FS_STAT_ROWS 0          /* activation rows this rank receives      */
#define FS_STAT_DEDUP_SEND 1    /* Σ_t |distinct remote ranks of t|        */
#define FS_STAT_NAIVE_SEND 2    /* #(t,k) owned by another rank            */
#define FS_STAT_LOCAL_ROWS 3    /* #(t,k) owned by this rank               */
#define FS_STAT_NODE_DEDUP 4    /* Σ_t |distinct remote nodes of t| = dispatch_loads/tb */
#define FS_NSTATS 8

/* trace slots (globaltimer ns, CTA 0 thread 0) when created with FUSCO_TRACE=1 */
#define FS_TRACE_LAYOUT_BEGIN 0
#define FS_TRACE_LAYOUT_HIST 1
#define FS_TRACE_LAYOUT_GRIDSYNC 2
#define FS_TRACE_LAYOUT_PUBLISH 3
#define FS_TRACE_LAYOUT_WAIT 4
#define FS_TRACE_LAYOUT_END 5
#define FS_TRACE_DISPATCH_SIGNAL 7 /* sender: the last completion block released (any CTA) */
#define FS_TRACE_DISPATCH_BEGIN 8
#define FS_TRACE_DISPATCH_PUSHED 9
#define FS_TRACE_DISPATCH_ARRIVED 10
#define FS_TRACE_DISPATCH_END 11
#define FS_TRACE_COMBINE_BEGIN 12
#define FS_TRACE_COMBINE_READY 13
#define FS_TRACE_COMBINE_END 14
#define FS_TRACE_LAYOUT_LAST 16   /* thread 0 of the last CTA to leave the kernel */
#define FS_TRACE_DISPATCH_LAST 17
#define FS_TRACE_COMBINE_LAST 18
#define FS_NTRACE 24                /* slots 20-22: exit counters behind the *_LAST stamps */

typedef struct fs_ctx* fs_handle_t;

int fs_abi_version(void);
const char* fs_last_error(void);

/* ---- symmetric memory: one region per rank, identical layout everywhere -- */

/* Bytes of one rank's symmetric region for this configuration (count
 * words, dispatch block words and duplicate lists, activation rows,
 * optional expert-output rows). */
int fs_region_bytes(int world, int num_experts, int topk, int token_bytes, int max_tokens,
                    long long max_rows, int with_act_out, size_t* bytes_out);

/* cudaMalloc + zero-fill on `device` (not the torch caching allocator, so
 * the region can be exported with CUDA IPC).  Every entry point takes or
 * remembers an explicit device ordinal: the library's CUDA runtime keeps its
 * own current-device state, independent of the caller's. */
int fs_sym_alloc(int device, size_t bytes, void** ptr_out);
int fs_sym_free(int device, void* ptr);
/* CUDA IPC export/import of a region (64-byte opaque handle, host memory). */
int fs_ipc_handle(int device, void* ptr, uint8_t* handle64_out);
int fs_ipc_open(int device, const uint8_t* handle64, void** ptr_out);
int fs_ipc_close(int device, void* ptr);
/* Map peer_device's memory into device's address space (one process driving
 * several GPUs, e.g. the phased multi-GPU emulation the NVLink counter
 * profile uses; production ranks map peers through CUDA IPC instead). */
int fs_enable_peer_access(int device, int peer_device);

/* ---- handle ------------------------------------------------------------- */

/* expert_owner[num_experts] (host): rank owning each expert (reference
 * ExpertPlacement.owner, topology.py:69-105).  node_of[world] (host, may be
 * NULL = identity): node of each rank, used only for first_mask / node-dedup
 * statistics (routing.py:86-98 with gpus_per_node > 1).
 * peer_regions[world] (host array of device pointers): every rank's
 * symmetric region mapped into this process (own one at [rank]).
 * grid_ctas: persistent grid of dispatch/combine; must be equal on all
 * ranks (0 = one CTA per SM times occupancy, computed identically).
 * timeout_ms: bound on every peer-flag wait (0 = 10000). */
int fs_create(int device, int rank, int world, int num_experts, int topk, int token_bytes,
              int max_tokens, long long max_rows, int with_act_out,
              const int32_t* expert_owner, const int32_t* node_of,
              void* const* peer_regions, int grid_ctas, int timeout_ms,
              fs_handle_t* out);
int fs_destroy(fs_handle_t h);

/* Local experts (ascending id) and device pointers into the own region. */
int fs_num_local_experts(fs_handle_t h, int* n_out);
int fs_grid_ctas(fs_handle_t h, int* n_out);
/* which: 0 = act, 1 = act_out (fixed addresses for the handle's lifetime) */
int fs_buffer_ptr(fs_handle_t h, int which, void** ptr_out);
long long fs_max_rows(fs_handle_t h);
/* Current epoch (incremented by every fs_layout with the LOCAL phase). */
unsigned int fs_epoch(fs_handle_t h);
/* Per-rank dispatch dedup on (0, default) or off (1: every (token, k) row
 * crosses the link) — the reference's "planner" ablation (engine.py:384-420,
 * build_direct_plans planner.py:563-659).  Takes effect from the next
 * fs_dispatch; set it identically on every rank. */
int fs_set_nodedup(fs_handle_t h, int on);
/* Load balancer on (1, default) or off (0) — the reference's "balancer"
 * ablation (balancer.py:73-90, engine.py:384-420).  On: push units,
 * fan-out units and combine items are claimed dynamically from per-epoch
 * counters, and each token's destination order is rotated so concurrent
 * warps of a rank spread their first stores over different peers.  Off:
 * static striding of the same work over the grid, no rotation.  Takes
 * effect from the next kernel; set it identically on every rank. */
int fs_set_balance(fs_handle_t h, int on);

/* ---- the hot path --------------------------------------------------------- */

/* Layout planner.  topk_idx[num_tokens, topk] (int32 if idx_bytes==4, int64
 * if 8).  Outputs (device): row_of[num_tokens, topk] int32 = row in the
 * owner's activation buffer; expert_counts[E_local]; expert_offsets
 * [E_local+1]; first_mask[num_tokens, topk] u8 (may be NULL);
 * rank_mask[num_tokens] u32 bitmask of destination ranks (may be NULL);
 * stats[FS_NSTATS] int64 (may be NULL).  All outputs are complete after the
 * REMOTE phase. */
int fs_layout(fs_handle_t h, const void* topk_idx, int idx_bytes, int num_tokens,
              int32_t* row_of, int32_t* expert_counts, int32_t* expert_offsets,
              uint8_t* first_mask, uint32_t* rank_mask, int64_t* stats,
              int phase, void* stream);

/* Dispatch: x[num_tokens, token_bytes] (any dtype, raw bytes) is written
 * straight into every owner's expert-major activation rows, one NVLink
 * crossing per (token, destination rank); duplicates on the same rank are
 * fanned out receiver-side.  Output: this rank's act buffer rows
 * [0, expert_offsets[E_local]).  x must be complete before fs_layout of the
 * same step is enqueued: the dispatch is launched as a programmatic
 * dependent of the planner and may start streaming x in while it runs. */
int fs_dispatch(fs_handle_t h, const void* x, const void* topk_idx, int idx_bytes,
                const int32_t* row_of, int num_tokens, int phase, void* stream);

/* fs_dispatch with the router weights topk_w[num_tokens, topk] (fp32 if
 * w_bytes==4, f64 if 8; the same array the combine gets).  With weights the
 * dispatch also describes, for each token with several experts on one remote
 * owner, that group to the owner, and a combine of this step with fp32
 * accumulation lets the owner pre-reduce the group (one fp32 partial per
 * (token, owner) pulled instead of its rows; see fs_combine).  topk_w NULL
 * is fs_dispatch.  Replaces the same reference calls as fs_dispatch. */
int fs_dispatch_w(fs_handle_t h, const void* x, const void* topk_idx, int idx_bytes,
                  const int32_t* row_of, const void* topk_w, int w_bytes, int num_tokens,
                  int phase, void* stream);

/* Combine: out[t] = Σ_{k ascending} w[t,k] · src_owner(t,k)[row_of[t,k]],
 * pulled from the peers' act / act_out rows.  topk_w is f32 (w_bytes 4) or
 * f64 (w_bytes 8); out has the payload dtype. */
int fs_combine(fs_handle_t h, const void* topk_idx, int idx_bytes,
               const int32_t* row_of, const void* topk_w, int w_bytes,
               int num_tokens, void* out, int dtype, int src, int acc,
               int phase, void* stream);

/* Synchronise the stream and return the device status word (FS_OK, or the
 * first FS_ETIMEOUT / FS_ERANGE a kernel recorded); clears it. */
int fs_check(fs_handle_t h, void* stream);

/* Copy the trace stamps (FS_NTRACE u64, 0 when never written) to host
 * memory; synchronises the stream.  FS_EINVAL unless created with
 * FUSCO_TRACE=1 in the environment. */
int fs_trace(fs_handle_t h, uint64_t* host_out, void* stream);

/* P2P/HBM copy-bandwidth probe: copies `bytes` from src to dst with the
 * same 16-byte warp copy loop the engine uses (used by bench.py to measure
 * the link/HBM peak in-run).  src == NULL: write-only fill of dst. */
int fs_probe_copy(int device, void* dst, const void* src, size_t bytes, int ctas, void* stream);

/* Row-scatter probe, the dispatch's HBM write pattern without its metadata:
 * warp w reads row src[r] (r = w, w + warps, ...; nrows_src rows) and writes
 * it to the `fanout` rows perm[r * fanout + j] of dst (device int32 array),
 * row_bytes each (multiple of 16).  src == NULL: write-only.  Used by
 * tools/hbm_probe.py to measure the ceiling of the P=1 dispatch's pattern. */
int fs_probe_scatter(int device, void* dst, const void* src, const int32_t* perm, int nrows_src, int fanout,
                     int row_bytes, int ctas, void* stream);

/* All-to-all copy probe: npairs (<= 32) concurrent copies srcs[j] -> dsts[j]
 * of `bytes` each (host arrays of device pointers, local or peer-mapped).
 * mode 0 = warp 16-byte loads/stores, 1 = TMA bulk copies through shared
 * memory.  Used by tools/p2p_probe.py to measure achievable NVLink push /
 * pull bandwidth with the engines' own data movers. */
int fs_probe_a2a(int device, void* const* dsts, const void* const* srcs, int npairs, size_t bytes,
                 int mode, int ctas, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* FUSCO_H_ */
