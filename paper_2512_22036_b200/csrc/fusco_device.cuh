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
constexpr size_t kOffArrive = 512;     // u32[FS_MAX_RANKS]: source s finished pushing here (epoch)
constexpr size_t kOffDone = 1024;      // u64: reserved

struct FsArgs {
  int rank, world, E, K, tb, T;
  int idx64;      // topk_idx element size 8 (else 4)
  int nodedup;    // 1: every (token, k) row crosses the link (the reference's "planner" ablation)
  // Iteration counter in device memory (per handle), so a captured CUDA graph
  // replays correctly: fs_layout's LOCAL phase uses *epoch + 1 and stores it;
  // every later phase/kernel of the iteration reads it.  parity = epoch & 1
  // selects the act / count / fan_src copy.
  uint32_t* epoch_ptr;
  long long max_rows;
  const int32_t* owner;      // [E] expert -> rank
  const int32_t* node_of;    // [P] rank -> node (first_mask statistics)
  const int32_t* perm;       // [E] experts sorted by (owner, id)
  const int32_t* seg_begin;  // [P+1] segment of rank g in perm
  char* peer[FS_MAX_RANKS];  // every rank's region, mapped here
  size_t off_count, off_fansrc, off_act, off_actout;
  size_t count_stride, fansrc_stride, act_stride;  // bytes per parity copy
  int32_t* chunk_cnt;        // [chunks][E] scratch (per handle)
  int32_t* totals;           // [2][E] per-parity per-expert atomic totals (per handle)
  long long* stat_part;      // [2][8] per-parity atomic statistics accumulators
  int* status;               // first error code, FS_OK when clean
  int* num_rows;             // rows of the own activation buffer this epoch
  unsigned long long timeout_ns;
  unsigned long long* trace;  // optional globaltimer stamps (FUSCO_TRACE=1), see FS_TRACE_*
  unsigned long long* work;   // [2][8] per-parity dynamic work counters (zeroed one epoch ahead)
  int2* fan_list;             // [max_rows] receiver fan-out list (row, primary row), P > 1
};

// dynamic work counters (slot within work[parity][*])
constexpr int kWorkDispatch = 0;
constexpr int kWorkFanout = 1;
constexpr int kWorkCombine = 2;
constexpr int kWorkDone = 3;  // dispatch CTAs of this epoch done pushing (target gridDim.x)

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

__device__ __forceinline__ void record_error(int* status, int code) {
  atomicCAS(status, FS_OK, code);
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
__device__ __forceinline__ bool wait_u32_geq(const uint32_t* p, uint32_t target, const FsArgs& a) {
  const unsigned long long t0 = globaltimer();
  while ((int32_t)(ld_acquire_sys_u32(p) - target) < 0) {
    if (globaltimer() - t0 > a.timeout_ns) {
      record_error(a.status, FS_ETIMEOUT);
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
__device__ __forceinline__ void publish_count(const FsArgs& a, int parity, uint32_t epoch, int e, int count) {
  const unsigned long long w = ((unsigned long long)epoch << 32) | (uint32_t)count;
  for (int g = 0; g < a.world; ++g) {
    unsigned long long* m =
        reinterpret_cast<unsigned long long*>(a.peer[g] + a.off_count + (size_t)parity * a.count_stride);
    st_relaxed_sys_u64(m + (size_t)a.rank * a.E + e, w);
  }
}
// Σ_q cnt[q][e] and Σ_{q<rank} cnt[q][e] from this rank's matrix, waiting for
// every source's word of this epoch.
__device__ __forceinline__ void gather_counts(const FsArgs& a, int parity, uint32_t epoch, int e, int* tot,
                                              int* before) {
  const unsigned long long* m =
      reinterpret_cast<const unsigned long long*>(a.peer[a.rank] + a.off_count + (size_t)parity * a.count_stride);
  int t = 0, b = 0;
  for (int q = 0; q < a.world; ++q) {
    const unsigned long long* p = m + (size_t)q * a.E + e;
    unsigned long long w = ld_acquire_sys_u64(p);
    if ((uint32_t)(w >> 32) != epoch) {
      const unsigned long long t0 = globaltimer();
      do {
        if (globaltimer() - t0 > a.timeout_ns) {
          record_error(a.status, FS_ETIMEOUT);
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

// End of a rank's push phase: every CTA makes its peer stores visible at
// system scope (bar.sync, then one fence.acq_rel.sys by thread 0) and counts
// itself done on a local counter; the last CTA of the epoch then releases
// one flag per peer (value = epoch).  One NVLink signal per (source,
// destination) instead of one per CTA.
__device__ __forceinline__ void signal_pushed(const FsArgs& a, uint32_t epoch) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    // per-parity counter, zeroed by the planner for the next epoch, so the
    // grid may differ between launches
    unsigned long long* done = a.work + (size_t)(epoch & 1u) * 8 + kWorkDone;
    const unsigned long long prev = atom_add_acq_rel_gpu_u64(done, 1ull);
    if (prev + 1 == (unsigned long long)gridDim.x) {
      if (a.trace != nullptr) a.trace[7] = globaltimer();  // the last CTA's signal
      for (int g = 0; g < a.world; ++g)
        st_release_sys_u32(reinterpret_cast<uint32_t*>(a.peer[g] + kOffArrive) + a.rank, epoch);
    }
  }
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
  return a.work + (size_t)(epoch & 1u) * 8 + slot;
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
