// dispatch.cuh — the push dispatch and the receiver fan-out (fs_dispatch)
#pragma once
#include <cooperative_groups.h>

#include "fusco_device.cuh"

namespace fusco {
namespace cg = cooperative_groups;

// ===========================================================================
// Dispatch
//
// Work unit = (token, slice of SLICE = 32 lanes x U vector words).  Lane k<K
// of the warp holds (owner g_k, row r_k) of the token's k-th expert.  Per
// destination rank only the first k crosses NVLink (the per-rank dedup of
// routing.py:94-97 / planner.py:231 with one GPU per "node"); for the own
// rank every k is written directly from registers.  The sender records, for
// each destination row, the row holding its bytes (fan_src): itself, or the
// primary row of the same token on that rank.  After every source's CTAs
// have signalled arrival, the receiver copies primary -> duplicate rows in
// its own HBM.  The activation buffer is single: a rank's next dispatch
// cannot start before every peer published its next-epoch counts, i.e.
// finished pulling this epoch's rows in combine (fusco.cu region_layout).
// ===========================================================================
template <typename V>
struct MoveCfg {
  static constexpr int U = sizeof(V) == 16 ? 8 : 16;  // words per lane per unit (4 KB / 2 KB)
  static constexpr int kSliceWords = 32 * U;
};

// Lane k < K of a warp holds (expert, row) of token i's k-th choice: two
// independent global loads, issued one work item ahead of use; the owner is
// looked up later in a shared-memory copy of the expert table.
struct KMeta {
  int e, r;
};
__device__ __forceinline__ KMeta load_meta(const FsArgs& a, const void* idx, const int32_t* row_of, int i,
                                           int lane) {
  KMeta m{0, -1};
  if (lane < a.K) {
    const long long e = load_idx(idx, (size_t)i * a.K + lane, a.idx64);
    m.e = (e < 0 || e >= a.E) ? 0 : (int)e;
    m.r = row_of[(size_t)i * a.K + lane];
  }
  return m;
}
constexpr int kMaxExperts = 1024;  // shared-memory expert table bound (checked by fs_create)

__device__ __forceinline__ void load_owner_table(const FsArgs& a, int32_t* owner_sm) {
  for (int e = threadIdx.x; e < a.E; e += blockDim.x) owner_sm[e] = a.owner[e];
  __syncthreads();
}

template <typename V>
__device__ __forceinline__ void warp_copy_row_cg(V* __restrict__ dst, const V* __restrict__ src, int nv,
                                                 int lane) {
  constexpr int U = MoveCfg<V>::U;
  for (int w0 = 0; w0 < nv; w0 += 32 * U) {
    V v[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int w = w0 + j * 32 + lane;
      if (w < nv) v[j] = ld_cg(src + w);
    }
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int w = w0 + j * 32 + lane;
      if (w < nv) st_na(dst + w, v[j]);
    }
  }
}

// Receiver-side fan-out: rows whose fan_src points at another row (a
// duplicate destination of a token that crossed NVLink once) are copied from
// that primary row.  Two steps over the whole (cooperative) grid: every warp
// scans 32 rows per load (most rows are primaries) and appends the
// duplicates to a list with one atomic per warp; after a grid barrier the
// (row, slice) copy units of the list are strided over every warp.  Balanced
// whatever the duplicates' distribution over the rows (sources, experts).
template <typename V>
__device__ __forceinline__ void fan_out_rows(const FsArgs& a, size_t act_off, size_t fan_off, int nv,
                                             uint32_t epoch) {
  constexpr int U = MoveCfg<V>::U;
  constexpr int SW = 32 * U;
  const int lane = threadIdx.x & 31;
  const long long gw = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = (gridDim.x * (long long)blockDim.x) >> 5;
  // the planner records FS_ERANGE (and fs_check raises) when the rows exceed
  // the buffer; never walk past it meanwhile
  const long long rows_all = *reinterpret_cast<volatile int*>(a.num_rows);
  const int rows = (int)(rows_all < a.max_rows ? rows_all : a.max_rows);
  const int S = (nv + SW - 1) / SW;
  const int32_t* fs = reinterpret_cast<const int32_t*>(a.peer[a.rank] + fan_off);
  V* act = reinterpret_cast<V*>(a.peer[a.rank] + act_off);
  unsigned long long* cnt = work_ctr(a, epoch, kWorkFanout);
  const uint32_t lt = (1u << lane) - 1u;
  for (long long b = gw * 32; b < rows; b += nw * 32) {
    const int r = (int)b + lane;
    const int f = r < rows ? ld_cg(fs + r) : r;
    const bool dup = r < rows && f != r && f >= 0 && f < rows;
    const uint32_t m = __ballot_sync(kFull, dup);
    if (m) {
      unsigned long long base = 0;
      if (lane == 0) base = atomicAdd(cnt, (unsigned long long)__popc(m));
      base = __shfl_sync(kFull, base, 0);
      if (dup) a.fan_list[base + __popc(m & lt)] = make_int2(r, f);
    }
  }
  cg::this_grid().sync();
  const uint32_t units = (uint32_t)*reinterpret_cast<volatile unsigned long long*>(cnt) * (uint32_t)S;
  for (uint32_t u = (uint32_t)gw; u < units; u += (uint32_t)nw) {
    const uint32_t ri = u / (uint32_t)S;
    const int2 rf = __ldcg(a.fan_list + ri);
    const int w0 = (int)(u - ri * (uint32_t)S) * SW, rem = nv - w0;
    const V* src = act + (size_t)rf.y * nv + w0;
    V* dst = act + (size_t)rf.x * nv + w0;
    V v[U];
#pragma unroll
    for (int j = 0; j < U; ++j)
      if (j * 32 + lane < rem) v[j] = ld_cg(src + j * 32 + lane);
#pragma unroll
    for (int j = 0; j < U; ++j)
      if (j * 32 + lane < rem) st_na(dst + j * 32 + lane, v[j]);
  }
}

template <typename V>
__global__ void __launch_bounds__(kMoveThreads)
    dispatch_kernel(FsArgs a, const V* __restrict__ x, const void* __restrict__ idx,
                    const int32_t* __restrict__ row_of, int phase) {
  TraceLast trace_last_(a, FS_TRACE_DISPATCH_LAST);
  constexpr int U = MoveCfg<V>::U;
  constexpr int SW = MoveCfg<V>::kSliceWords;
  const int K = a.K, T = a.T, P = a.world, s = a.rank;
  const int nv = a.tb / (int)sizeof(V);
  const int S = (nv + SW - 1) / SW;
  const int lane = threadIdx.x & 31;
  const int gw = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int nw = (int)((gridDim.x * blockDim.x) >> 5);
  __shared__ int32_t owner_sm[kMaxExperts];
  if (phase & FS_PHASE_LOCAL) load_owner_table(a, owner_sm);  // static table: before the PDL wait
  griddep_wait();  // row_of / the epoch come from the planner
  const uint32_t epoch = load_epoch(a);
  const int parity = (int)(epoch & 1u);
  const size_t act_off = a.off_act;
  const size_t fan_off = a.off_fansrc + (size_t)parity * a.fansrc_stride;
  trace_stamp(a, FS_TRACE_DISPATCH_BEGIN);

  if (phase & FS_PHASE_LOCAL) {
    const long long units = (long long)T * S;
    const uint32_t uS = (uint32_t)S;
    unsigned long long* ctr = work_ctr(a, epoch, kWorkDispatch);
    long long u = claim_warp(ctr);
    KMeta nxt = u < units ? load_meta(a, idx, row_of, (int)((uint32_t)u / uS), lane) : KMeta{0, -1};
    while (u < units) {
      const int i = (int)((uint32_t)u / uS);
      const int sl = (int)((uint32_t)u - (uint32_t)i * uS);
      const KMeta cur = nxt;
      const long long un = claim_warp(ctr);  // next unit: claimed and prefetched during this one
      if (un < units) nxt = load_meta(a, idx, row_of, (int)((uint32_t)un / uS), lane);
      // payload loads first: they do not depend on the destinations
      const int w0 = sl * SW;
      const V* src = x + (size_t)i * nv + w0;
      const int rem = nv - w0;
      V v[U];
#pragma unroll
      for (int j = 0; j < U; ++j) {
        const int w = j * 32 + lane;
        if (w < rem) v[j] = ld_nc(src + w);
      }
      int g = -1 - lane, r = -1;  // lanes >= K get unique negative keys
      if (lane < K) {
        g = owner_sm[cur.e];
        r = (cur.r < 0 || cur.r >= a.max_rows) ? -1 : cur.r;
      }
      const uint32_t same = __match_any_sync(kFull, g);
      const int first_lane = __ffs(same) - 1;
      const int r_first = __shfl_sync(kFull, r, first_lane);
      const bool direct = lane < K && r >= 0 && (a.nodedup || first_lane == lane || g == s);
      const uint32_t dmask = __ballot_sync(kFull, direct);
      if (sl == 0 && lane < K && r >= 0) {
        int32_t* fs = reinterpret_cast<int32_t*>(a.peer[g] + fan_off);
        fs[r] = direct ? r : r_first;
      }
      // Rotate the destination order by token so concurrent warps of this
      // rank spread their first stores over different peers.
      uint32_t m = dmask;
      const int rot = (i + s) % K;
      m = (m >> rot) | (rot ? (m << (32 - rot)) : 0u);
      while (m) {
        const int d0 = __ffs(m) - 1;
        m &= m - 1;
        const int d = (d0 + rot) & 31;
        const int gd = __shfl_sync(kFull, g, d);
        const int rd = __shfl_sync(kFull, r, d);
        V* dst = reinterpret_cast<V*>(a.peer[gd] + act_off) + (size_t)rd * nv + w0;
#pragma unroll
        for (int j = 0; j < U; ++j) {
          const int w = j * 32 + lane;
          if (w < rem) st_na(dst + w, v[j]);
        }
      }
      u = un;
    }
    if (P > 1) signal_pushed(a, epoch);
  }
  griddep_launch_dependents();  // the combine may start its prologue

  trace_stamp(a, FS_TRACE_DISPATCH_PUSHED);
  if ((phase & FS_PHASE_REMOTE) && P > 1) {
    if (threadIdx.x < P)
      wait_u32_geq(reinterpret_cast<const uint32_t*>(a.peer[s] + kOffArrive) + threadIdx.x, epoch, a);
    __syncthreads();
    trace_stamp(a, FS_TRACE_DISPATCH_ARRIVED);
    fan_out_rows<V>(a, act_off, fan_off, nv, epoch);
  }
  trace_stamp(a, FS_TRACE_DISPATCH_END);
}

// ===========================================================================
// Dispatch, TMA engine
//
// Same protocol and outputs as dispatch_kernel, different data mover: per
// CTA a ring of NS shared-memory row slots.  Warp 0 (one elected thread)
// streams whole token rows global->shared with cp.async.bulk, completion on
// a per-slot mbarrier (expect_tx).  Warp 1 resolves the token's destinations
// (same per-rank dedup as above) and one lane issues one cp.async.bulk
// shared->global store per destination row — local HBM or a peer's HBM over
// NVLink — committing one bulk group per token; a slot is handed back to the
// producer once its group has finished reading shared memory
// (wait_group.read with a lag).  The registers never hold payload: bytes in
// flight per SM are NS rows, independent of occupancy.
// ===========================================================================
constexpr int kTmaThreads = 128;
constexpr int kTmaMaxSlots = 32;

__host__ __device__ inline int tma_slot_bytes(int tb) { return (tb + 127) & ~127; }

template <int LAG>
__global__ void __launch_bounds__(kTmaThreads)
    dispatch_tma_kernel(FsArgs a, const char* __restrict__ x, const void* __restrict__ idx,
                        const int32_t* __restrict__ row_of, int phase, int nslots) {
  TraceLast trace_last_(a, FS_TRACE_DISPATCH_LAST);
  extern __shared__ __align__(128) char tsm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(tsm);
  uint64_t* empty = full + kTmaMaxSlots;
  char* ring = tsm + 2 * kTmaMaxSlots * sizeof(uint64_t);
  const int K = a.K, T = a.T, P = a.world, s = a.rank, tb = a.tb;
  const int slot_bytes = tma_slot_bytes(tb);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ int32_t owner_tma[kMaxExperts];
  // Prologue independent of the planner (launched with PDL behind it): barrier
  // init, expert table, and the first ring-full of token rows streaming in.
  if ((phase & FS_PHASE_LOCAL) && threadIdx.x == 0) {
    for (int q = 0; q < nslots; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], 1);
    }
    mbar_fence_init();
  }
  if (phase & FS_PHASE_LOCAL) load_owner_table(a, owner_tma);
  if ((phase & FS_PHASE_LOCAL) && threadIdx.x == 0) {
    int n = 0;
    for (int i = blockIdx.x; i < T && n < nslots; i += gridDim.x, ++n) {
      mbar_arrive_expect_tx(&full[n], (uint32_t)tb);
      bulk_load(ring + (size_t)n * slot_bytes, x + (size_t)i * tb, (uint32_t)tb, &full[n]);
    }
  }
  griddep_wait();  // row_of / the epoch come from the planner
  const uint32_t epoch = load_epoch(a);
  const int parity = (int)(epoch & 1u);
  const size_t act_off = a.off_act;
  const size_t fan_off = a.off_fansrc + (size_t)parity * a.fansrc_stride;
  trace_stamp(a, FS_TRACE_DISPATCH_BEGIN);

  if (phase & FS_PHASE_LOCAL) {
    if (warp == 0) {
      if (lane == 0) {  // producer (the first nslots rows were issued in the prologue)
        int n = 0;
        for (int i = blockIdx.x; i < T; i += gridDim.x, ++n) {
          if (n < nslots) continue;
          const int q = n % nslots;
          mbar_wait(&empty[q], ((n / nslots) & 1) ^ 1);
          mbar_arrive_expect_tx(&full[q], (uint32_t)tb);
          bulk_load(ring + (size_t)q * slot_bytes, x + (size_t)i * tb, (uint32_t)tb, &full[q]);
        }
      }
    } else if (warp == 1) {  // destinations + bulk stores
      int n = 0;
      KMeta nxt = (int)blockIdx.x < T ? load_meta(a, idx, row_of, blockIdx.x, lane) : KMeta{0, -1};
      for (int i = blockIdx.x; i < T; i += gridDim.x, ++n) {
        const int q = n % nslots;
        const KMeta cur = nxt;
        if (i + (int)gridDim.x < T) nxt = load_meta(a, idx, row_of, i + gridDim.x, lane);
        int g = -1 - lane, r = -1;
        if (lane < K) {
          g = owner_tma[cur.e];
          r = (cur.r < 0 || cur.r >= a.max_rows) ? -1 : cur.r;
        }
        const uint32_t same = __match_any_sync(kFull, g);
        const int first_lane = __ffs(same) - 1;
        const int r_first = __shfl_sync(kFull, r, first_lane);
        const bool direct = lane < K && r >= 0 && (a.nodedup || first_lane == lane || g == s);
        if (lane < K && r >= 0) {
          int32_t* fs = reinterpret_cast<int32_t*>(a.peer[g] + fan_off);
          fs[r] = direct ? r : r_first;
        }
        mbar_wait(&full[q], (n / nslots) & 1);
        // each destination lane issues its own bulk store (per-thread bulk
        // groups); every lane commits one group per token so the lag below
        // counts tokens on all lanes
        if (direct)
          bulk_store(a.peer[g] + act_off + (size_t)r * tb, ring + (size_t)q * slot_bytes, (uint32_t)tb);
        bulk_commit();
        bulk_wait_read<LAG>();
        __syncwarp();
        if (lane == 0 && n >= LAG) mbar_arrive(&empty[(n - LAG) % nslots]);
      }
      bulk_wait<0>();
      fence_proxy_async_global();
    }
    if (P > 1) signal_pushed(a, epoch);
  }
  griddep_launch_dependents();  // the combine may start its prologue

  trace_stamp(a, FS_TRACE_DISPATCH_PUSHED);
  if ((phase & FS_PHASE_REMOTE) && P > 1) {
    if (threadIdx.x < P)
      wait_u32_geq(reinterpret_cast<const uint32_t*>(a.peer[s] + kOffArrive) + threadIdx.x, epoch, a);
    __syncthreads();
    trace_stamp(a, FS_TRACE_DISPATCH_ARRIVED);
    fan_out_rows<int4>(a, act_off, fan_off, tb / 16, epoch);
  }
  trace_stamp(a, FS_TRACE_DISPATCH_END);
}

}  // namespace fusco
