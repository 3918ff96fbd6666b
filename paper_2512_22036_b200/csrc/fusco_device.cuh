// fusco_device.cuh — device-side primitives for the NVLink shuffle kernels.
//
// Memory-ordering protocol over NVLink/NVSwitch (replaces the reference's
// ring-buffer + expected-byte counters, engine.py:637-694, 979-1031):
//   writer: payload stores (weak st.global to peer addresses) -> bar.sync
//           -> thread 0: fence.acq_rel.sys, then an acq_rel.gpu count on a
//              local counter; the last arrival issues st.release.sys on the
//              peer flag (signal_pushed below)
//   reader: one thread per flag spins ld.acquire.sys until the epoch value
//           -> bar.sync -> payload loads.
// Flags never reset: they carry the monotonically increasing epoch (or an
// epoch-scaled arrival count), so consecutive iterations need no barrier.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "../../include/fusco.h"

namespace fusco {

constexpr uint32_t kFull = 0xffffffffu;

// Offsets inside the 4 KiB signal block at the start of every region.
constexpr int kMoveThreads = 256;  // dispatch / combine warp-mover CTA size
constexpr size_t kSigBytes = 4096;
constexpr size_t kOffCountFlag = 0;    // u32[FS_MAX_RANKS]: reserved (the counts are epoch-tagged words)
constexpr size_t kOffReadyFlag = 256;  // u32[FS_MAX_RANKS]: expert outputs ready
constexpr size_t kOffModeFlag = 512;   // u32[FS_MAX_RANKS]: owner g pre-reduced this epoch (= epoch)

// Owner-side pre-reduction (combine, fp32 accumulate, P > 1): for a token
// with m >= 3 (bf16 rows; m >= 2 for fp32 rows) of its K experts on one
// remote owner, the owner sums w_k * y_k over those rows in fp32 (k
// ascending) and the source pulls that one fp32 partial instead of the m
// rows.  The source describes each such (token, owner) group during the
// dispatch: a record in the owner's region, slot [source][token].
constexpr int kGrpMaxK = 8;
struct GrpRec {
  uint32_t epoch;
  uint32_t kmask;  // the token's k's owned by this rank
  int32_t rows[kGrpMaxK];
  float w[kGrpMaxK];
  uint32_t pad[2];
};
static_assert(sizeof(GrpRec) == 80, "GrpRec layout");

// Completion blocks of the dispatch (P > 1): a source's tokens are cut into
// blocks of FsArgs::blk tokens; when every unit of block b has been pushed, the
// source releases one epoch-tagged word per destination rank carrying the
// number of duplicate rows it listed there for that block, and the
// destination fans those rows out while later blocks are still in flight.
// Tokens per completion block: max_tokens / 16 rounded up to a multiple of
// 128 (at least 128, at most 2048; FsArgs::blk, equal on every rank).  Every
// block completion costs a system-scope release per destination, so blocks
// stay few; 16 per source still lets the fan-out start after the first
// sixteenth of the push.
constexpr int kBlockTarget = 16;
__host__ __device__ inline int block_tokens(int max_tokens) {
#ifdef FUSCO_BLOCK_TOKENS
  return FUSCO_BLOCK_TOKENS;
#else
  const int per = (max_tokens + kBlockTarget - 1) / kBlockTarget;
  const int r = ((per + 127) / 128) * 128;
  return r < 128 ? 128 : (r > 2048 ? 2048 : r);
#endif
}
constexpr int kBlkStride = 32;  // u32 words per block counter (one 128-byte line each)

struct FsArgs {
  int rank, world, E, K, tb, T;
  int idx64;      // topk_idx element size 8 (else 4)
  int nodedup;    // 1: every (token, k) row crosses the link (the reference's "planner" ablation)
  int balance;    // 1 (default): dynamic work claiming + rotated destination order; 0: static striding
  // Iteration counter in device memory (per handle), so a captured CUDA graph
  // replays correctly: fs_layout's LOCAL phase uses *epoch + 1 and stores it;
  // every later phase/kernel of the iteration reads it.  parity = epoch & 1
  // selects the count-matrix copy and the per-epoch scratch (work counters,
  // block accounting).
  uint32_t* epoch_ptr;
  long long max_rows;
  const int32_t* owner;      // [E] expert -> rank
  const int32_t* node_of;    // [P] rank -> node (first_mask statistics)
  const int32_t* perm;       // [E] experts sorted by (owner, id)
  const int32_t* seg_begin;  // [P+1] segment of rank g in perm
  char* peer[FS_MAX_RANKS];  // every rank's region, mapped here
  size_t off_count, off_blkflag, off_dupq, off_act, off_actout;
  size_t count_stride, act_stride;  // bytes per parity copy
  int blk;                   // tokens per completion block (block_tokens(max_tokens))
  int nbmax;                 // completion blocks per source (ceil(max_tokens / blk))
  long long dupq_cap;        // duplicate-list entries per source in a region (max_tokens * (K - 1))
  int push_warps;            // warps per CTA that push first (the rest fan out from the start)
  int dbg_relaxed;           // timing experiments only: block counts without release ordering
  // owner-side pre-reduction (0 in every field when the handle has no partial buffers)
  size_t off_grp, off_part;  // region offsets: GrpRec[P][max_tokens], fp32 partials [P][max_tokens][2 * tb]
  int max_tokens;
  const void* disp_w;        // fs_dispatch_w: the router weights [T, K] (records are written when set)
  int disp_w64;
  int reduce;                // combine: pre-reduce as owner and pull partials as source (this epoch)
  int push_rounds;           // 1: completion counted per CTA round (FUSCO_PUSH_ROUNDS=1), 0: per unit (default)
  int fan_split;             // 1: fan-out units are row slices (small batches), 0: whole rows
  int fan_poll;              // 1: fan-out waits poll through a per-CTA shared-memory cache (FUSCO_FAN_POLL)
  int32_t* chunk_cnt;        // [chunks][E] scratch (per handle)
  int32_t* totals;           // [2][E] per-parity per-expert atomic totals (per handle)
  long long* stat_part;      // [2][8] per-parity atomic statistics accumulators
  int* status;               // [2]: first error code (FS_OK when clean), ErrSite of a timeout
  int* num_rows;             // rows of the own activation buffer this epoch
  unsigned long long timeout_ns;
  unsigned long long* trace;  // optional globaltimer stamps (FUSCO_TRACE=1), see FS_TRACE_*
  unsigned long long* work;   // [2][8][kWorkStride] per-parity dynamic work counters (zeroed one epoch ahead)
  // sender-side block accounting, per parity (zeroed one epoch ahead by the planner)
  uint32_t* blkdone;          // [2][nbmax][kBlkStride] units of block b pushed (word 0 of a line)
  uint32_t* dupcnt;           // [2][P][nbmax] duplicate rows listed at rank g for block b
  // receiver-side fan-out schedule (this epoch): published jobs in arrival order
  unsigned long long* fan_jcum;  // [P * nbmax] cumulative fan-out units after job k
  uint32_t* fan_jorder;          // [P * nbmax] job k = (source << 16) | block
};

// dynamic work counters (slot within work[parity][*])
constexpr int kWorkDispatch = 0;
constexpr int kWorkFanout = 1;    // fan-out unit claims (groups of kFanGroup units)
constexpr int kWorkCombine = 2;
constexpr int kWorkFanReady = 4;  // (published jobs << 40) | published fan-out units
constexpr int kWorkFanDone = 5;   // every job published (or the wait timed out)
constexpr int kWorkSlots = 8;
// one 128-byte line per counter: the words fan-out workers poll must not
// share a line with the counters pushers claim from
constexpr int kWorkStride = 16;
constexpr size_t kWorkWords = 2 * kWorkSlots * kWorkStride;  // [2 parities][8 slots][16]

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Phase timestamps written by CTA 0 / thread 0 when tracing is enabled.
__device__ __forceinline__ void trace_stamp(const FsArgs& a, int slot) {
  if (a.trace != nullptr && blockIdx.x == 0 && threadIdx.x == 0) a.trace[slot] = globaltimer();
}
// Tracing only: stamps `slot` when thread 0 of the last CTA of the launch
// leaves the kernel (any return path: a destructor), so the tail after CTA 0
// is visible.  Counter slot = slot + 4; same grid size every launch assumed.
struct TraceLast {
  const FsArgs& a;
  int slot;
  __device__ TraceLast(const FsArgs& args, int s) : a(args), slot(s) {}
  __device__ ~TraceLast() {
    if (a.trace != nullptr && threadIdx.x == 0) {
      const unsigned long long old = atomicAdd(a.trace + slot + 4, 1ull);
      if ((old + 1) % gridDim.x == 0) a.trace[slot] = globaltimer();
    }
  }
};

// Where a kernel gave up (status word 1, read back by fs_check with the code).
enum ErrSite : int {
  kSiteNone = 0,
  kSiteLayoutCounts = 1,     // planner: a peer's count words of this epoch
  kSiteDispTokens = 2,       // dispatch watcher: a source's token count word
  kSiteDispBlocks = 3,       // dispatch watcher: a source's block words
  kSiteDispWorker = 4,       // dispatch fan-out worker: the published schedule
  kSiteDispSchedule = 5,     // dispatch fan-out worker: inconsistent schedule
  kSiteCombineReady = 6,     // combine: a peer's "outputs ready" flag
  kSiteCombinePipe = 7,      // combine TMA engine: shared-memory stage pipeline
  kSiteDispatchPipe = 8,     // dispatch TMA engine: shared-memory slot pipeline
  kSiteRows = 9,             // a row index outside the activation buffer
};
__device__ __forceinline__ void record_error(int* status, int code, int site = kSiteNone) {
  if (atomicCAS(status, FS_OK, code) == FS_OK) status[1] = site;
}

__device__ __forceinline__ uint32_t ld_acquire_sys_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_sys_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ int ld_relaxed_sys_s32(const int32_t* p) {
  int v;
  asm volatile("ld.relaxed.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long atom_add_acq_rel_gpu_u64(unsigned long long* p,
                                                                        unsigned long long v) {
  unsigned long long old;
  asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(v) : "memory");
  return old;
}
__device__ __forceinline__ void red_release_sys_add_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Spin until *p >= target (wrap-safe for u32 epochs); false on timeout.
__device__ __forceinline__ bool wait_u32_geq(const uint32_t* p, uint32_t target, const FsArgs& a,
                                             int site = kSiteCombineReady) {
  const unsigned long long t0 = globaltimer();
  while ((int32_t)(ld_acquire_sys_u32(p) - target) < 0) {
    if (globaltimer() - t0 > a.timeout_ns) {
      record_error(a.status, FS_ETIMEOUT, site);
      return false;
    }
  }
  return true;
}
__device__ __forceinline__ bool wait_u64_geq(const unsigned long long* p, unsigned long long target,
                                             const FsArgs& a) {
  const unsigned long long t0 = globaltimer();
  while (ld_acquire_sys_u64(p) < target) {
    if (globaltimer() - t0 > a.timeout_ns) {
      record_error(a.status, FS_ETIMEOUT);
      return false;
    }
  }
  return true;
}

// ---- count all-gather, epoch-tagged words ("LL") ---------------------------
// Each word of the P x E count matrix carries (epoch << 32 | count): a reader
// polls the words themselves, so the publisher needs neither a release fence
// nor a separate flag (one NVLink traversal instead of data + fence + flag).
// Row s of the matrix has E + 1 words: the per-expert counts, then the
// source's token count (the receiver's dispatch derives its blocks from it).
__device__ __forceinline__ void publish_count(const FsArgs& a, int parity, uint32_t epoch, int e, int count) {
  const unsigned long long w = ((unsigned long long)epoch << 32) | (uint32_t)count;
  for (int g = 0; g < a.world; ++g) {
    unsigned long long* m =
        reinterpret_cast<unsigned long long*>(a.peer[g] + a.off_count + (size_t)parity * a.count_stride);
    st_relaxed_sys_u64(m + (size_t)a.rank * (a.E + 1) + e, w);
  }
}
// One epoch-tagged count word of source q (waits for this epoch's value).
__device__ __forceinline__ int read_count_word(const FsArgs& a, int parity, uint32_t epoch, int q, int e) {
  const unsigned long long* p = reinterpret_cast<const unsigned long long*>(
                                    a.peer[a.rank] + a.off_count + (size_t)parity * a.count_stride) +
                                (size_t)q * (a.E + 1) + e;
  unsigned long long w = ld_acquire_sys_u64(p);
  if ((uint32_t)(w >> 32) != epoch) {
    const unsigned long long t0 = globaltimer();
    do {
      if (globaltimer() - t0 > a.timeout_ns) {
        record_error(a.status, FS_ETIMEOUT, kSiteDispTokens);
        return 0;
      }
      w = ld_acquire_sys_u64(p);
    } while ((uint32_t)(w >> 32) != epoch);
  }
  return (int)(uint32_t)w;
}
// Σ_q cnt[q][e] and Σ_{q<rank} cnt[q][e] from this rank's matrix, waiting for
// every source's word of this epoch.
__device__ __forceinline__ void gather_counts(const FsArgs& a, int parity, uint32_t epoch, int e, int* tot,
                                              int* before) {
  const unsigned long long* m =
      reinterpret_cast<const unsigned long long*>(a.peer[a.rank] + a.off_count + (size_t)parity * a.count_stride);
  int t = 0, b = 0;
  for (int q = 0; q < a.world; ++q) {
    const unsigned long long* p = m + (size_t)q * (a.E + 1) + e;
    unsigned long long w = ld_acquire_sys_u64(p);
    if ((uint32_t)(w >> 32) != epoch) {
      const unsigned long long t0 = globaltimer();
      do {
        if (globaltimer() - t0 > a.timeout_ns) {
          record_error(a.status, FS_ETIMEOUT, kSiteLayoutCounts);
          break;
        }
        w = ld_acquire_sys_u64(p);
      } while ((uint32_t)(w >> 32) != epoch);
    }
    const int v = (int)(uint32_t)w;
    t += v;
    b += (q < a.rank) ? v : 0;
  }
  *tot = t;
  *before = b;
}

// ---- completion blocks (sender side) -----------------------------------
// A unit of block b is done: count it on the block's local counter with
// acq_rel at gpu scope (a release over the pusher's peer stores, which
// precede it in program order).  The arrival that completes the block has
// acquired every other unit's release; its st.release.sys of the block word
// on each destination, (epoch << 32) | number of duplicate-list entries, is
// cumulative over everything it acquired, so by the PTX memory model's
// causality order (release.gpu -> acquire.gpu -> release.sys ->
// acquire.sys) every one of the block's NVLink stores is visible to the
// receiver's ld.acquire.sys of the word.  One flag per (source, destination,
// block) instead of one per unit: a per-unit system fence waits for the deep
// NVLink store queue and was measured slower, and an extra
// fence.sc.sys before the flags cost 8-12% of the push (measured, round 2).
__device__ __forceinline__ uint32_t atom_add_acq_rel_gpu_u32(uint32_t* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ uint32_t ld_relaxed_gpu_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long* blkflag_ptr(const FsArgs& a, int g, int src, int b) {
  return reinterpret_cast<unsigned long long*>(a.peer[g] + a.off_blkflag) + (size_t)src * a.nbmax + b;
}
// Count n units of block b; returns the previous count (the caller that
// brings it to the block's total completes the block).
__device__ __forceinline__ uint32_t block_count(const FsArgs& a, uint32_t epoch, int b, uint32_t n) {
  uint32_t* ctr = a.blkdone + ((size_t)(epoch & 1u) * a.nbmax + b) * kBlkStride;
  // a.dbg_relaxed (FUSCO_DBG_BLK=1, timing experiments only): relaxed count, no ordering
  return a.dbg_relaxed ? atomicAdd(ctr, n) : atom_add_acq_rel_gpu_u32(ctr, n);
}
// Every unit of block b is counted (and acquired): release the block word on
// every destination with its duplicate-list length.
__device__ __forceinline__ void block_complete(const FsArgs& a, uint32_t epoch, int b) {
  const int par = (int)(epoch & 1u);
#ifdef FUSCO_BLKFENCE  // A/B only: an explicit fence.sc.sys before the release stores
  __threadfence_system();
#endif
  for (int g = 0; g < a.world; ++g) {
    if (g == a.rank) continue;
    const uint32_t nd = ld_relaxed_gpu_u32(a.dupcnt + ((size_t)par * a.world + g) * a.nbmax + b);
    st_release_sys_u64(blkflag_ptr(a, g, a.rank, b), ((unsigned long long)epoch << 32) | nd);
  }
  if (a.trace != nullptr && b == (a.T - 1) / a.blk) a.trace[FS_TRACE_DISPATCH_SIGNAL] = globaltimer();
}
__device__ __forceinline__ void block_units_done(const FsArgs& a, uint32_t epoch, int b, uint32_t n,
                                                 uint32_t total) {
  if (block_count(a, epoch, b, n) + n == total) block_complete(a, epoch, b);
}
// Duplicate-list entry of (dup row, primary row) on rank g for block b.
__device__ __forceinline__ void list_duplicate(const FsArgs& a, uint32_t epoch, int g, int b, int row, int prim) {
  uint32_t* cnt = a.dupcnt + ((size_t)(epoch & 1u) * a.world + g) * a.nbmax + b;
  const uint32_t slot = atomicAdd(cnt, 1u);
  int2* q = reinterpret_cast<int2*>(a.peer[g] + a.off_dupq) + (size_t)a.rank * a.dupq_cap +
            (size_t)b * a.blk * (a.K - 1) + slot;
  *q = make_int2(row, prim);
}

// ---- 16-byte / 4-byte vector moves ----------------------------------------
// Read-only inputs (x, peers' finished act/act_out): non-coherent path, no L1
// allocation (streaming).  Data written by peers inside the same kernel
// (fan-out sources): .cg (L2, coherent).  Stores: plain weak st.global; the
// release fence publishes them.
__device__ __forceinline__ int4 ld_nc(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ int ld_nc(const int* p) {
  int r;
  asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ int4 ld_cg(const int4* p) {
  int4 r;
  asm volatile("ld.global.cg.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ int ld_cg(const int* p) {
  int r;
  asm volatile("ld.global.cg.s32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ void st_na(int4* p, const int4& v) {
  asm volatile("st.global.L1::no_allocate.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ void st_na(int* p, const int& v) {
  asm volatile("st.global.L1::no_allocate.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <typename V>
__device__ __forceinline__ uint32_t word(const V& v, int j) {
  return reinterpret_cast<const uint32_t*>(&v)[j];
}
template <typename V>
__device__ __forceinline__ void set_word(V& v, int j, uint32_t x) {
  reinterpret_cast<uint32_t*>(&v)[j] = x;
}

__device__ __forceinline__ int warp_incl_scan(int v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int n = __shfl_up_sync(kFull, v, o);
    if (lane >= o) v += n;
  }
  return v;
}

// One lane claims the next work unit for the warp (dynamic load balancing:
// warps that drew light units simply claim more).
__device__ __forceinline__ long long claim_warp(unsigned long long* ctr) {
  unsigned long long v = 0;
  if ((threadIdx.x & 31) == 0) v = atomicAdd(ctr, 1ull);
  return (long long)__shfl_sync(0xffffffffu, v, 0);
}
__device__ __forceinline__ unsigned long long* work_ctr(const FsArgs& a, uint32_t epoch, int slot) {
  return a.work + ((size_t)(epoch & 1u) * kWorkSlots + slot) * kWorkStride;
}

__device__ __forceinline__ uint32_t load_epoch(const FsArgs& a) {
  return *reinterpret_cast<volatile const uint32_t*>(a.epoch_ptr);
}

__device__ __forceinline__ long long load_idx(const void* idx, size_t pos, int idx64) {
  return idx64 ? reinterpret_cast<const long long*>(idx)[pos]
               : (long long)reinterpret_cast<const int32_t*>(idx)[pos];
}

// ---- mbarrier + bulk-copy (TMA) primitives --------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// The engines' pipeline waits: bounded like every flag wait, so a lost
// transaction surfaces as FS_ETIMEOUT through fs_check instead of a hang.
__device__ __forceinline__ void mbar_wait_bounded(uint64_t* bar, uint32_t parity, const FsArgs& a, int site) {
  if (mbar_try_wait(bar, parity)) return;
  const unsigned long long t0 = globaltimer();
  while (!mbar_try_wait(bar, parity)) {
    if (globaltimer() - t0 > a.timeout_ns) {
      record_error(a.status, FS_ETIMEOUT, site);
      return;
    }
  }
}
// global -> shared (this CTA), completion counted on an mbarrier
__device__ __forceinline__ void bulk_load(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// shared -> global (local HBM or a peer's HBM over NVLink), bulk-group tracked
__device__ __forceinline__ void bulk_store(void* gdst, const void* smem_src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
               "r"(smem_u32(smem_src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// ---- programmatic dependent launch (PDL) ----------------------------------
// The planner lets the next kernel on the stream start launching right away;
// the dependent kernel does independent prologue work and then waits for the
// planner's completion (and memory visibility) with griddepcontrol.wait.  Both
// are no-ops for kernels launched without the PDL attribute.
__device__ __forceinline__ void griddep_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// ---- thread-block cluster / distributed shared memory ----------------------
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Load a u32 from the same shared-memory offset in CTA `rank` of the cluster.
__device__ __forceinline__ uint32_t ld_dsmem_u32(const void* local_smem, uint32_t rank) {
  uint32_t remote, v;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(local_smem)), "r"(rank));
  asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(remote) : "memory");
  return v;
}

}  // namespace fusco
