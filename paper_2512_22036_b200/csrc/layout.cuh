// layout.cuh — the on-device layout planner (fs_layout)
#pragma once
#include <cooperative_groups.h>

#include "fusco_device.cuh"

namespace fusco {
namespace cg = cooperative_groups;

constexpr int kLayoutThreads = 256;  // one token per thread per chunk
constexpr int kLayoutWarps = kLayoutThreads / 32;

// Shared memory of the layout kernel (bytes):
//   owner table [E] + node table [32]
//   LOCAL : bits[8][E] + wbase[8][E]            (REMOTE aliases: tot/base/before/pre [4][E])
//   chunk : e_s[256*K] (expert ids of the chunk) + pos_s[256*K] (in-chunk positions)
__host__ __device__ inline size_t layout_smem_bytes(int E, int K) {
  const size_t tables = (3ull * E + 32 + 33) * sizeof(int32_t);  // owner, perm, node, seg, cnt
  const size_t a = 2ull * kLayoutWarps * E * sizeof(uint32_t);
  const size_t b = (5ull * E + 1) * sizeof(int32_t);
  const size_t chunk = 2ull * kLayoutThreads * K * sizeof(int32_t);
  return tables + (a > b ? a : b) + chunk;
}


// base_g(e) for every expert: exclusive scan of tot[] in (owner, expert)
// order (perm_s), restarted at each owner's segment — one block-wide scan
// over shared memory (no serial per-rank loop, no global loads).  ex_s gets
// E+1 entries.  Returns nothing; rows of rank s = ex_s[seg_s[s+1]] - ex_s[seg_s[s]].
template <int NT>
__device__ __forceinline__ void block_segmented_base(int E, const int32_t* tot, const int32_t* perm_s,
                                                     const int32_t* seg_s, const int32_t* owner_s,
                                                     int32_t* ex_s, int32_t* base, int* warp_tot) {
  constexpr int NW = NT / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (E <= 32) {  // one warp scans, one barrier
    if (warp == 0) {
      const int v = lane < E ? tot[perm_s[lane]] : 0;
      const int incl = warp_incl_scan(v, lane);
      if (lane < E) ex_s[lane] = incl - v;
      if (lane == E - 1) ex_s[E] = incl;
    }
    __syncthreads();
    if (tid < E) {
      const int e = perm_s[tid];
      base[e] = ex_s[tid] - ex_s[seg_s[owner_s[e]]];
    }
    return;
  }
  const int per = (E + NT - 1) / NT;  // consecutive elements per thread
  const int j0 = tid * per;
  int loc = 0;
  for (int q = 0; q < per; ++q) {
    const int j = j0 + q;
    if (j < E) loc += tot[perm_s[j]];
  }
  const int incl = warp_incl_scan(loc, lane);
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int v = lane < NW ? warp_tot[lane] : 0;
    const int wi = warp_incl_scan(v, lane);
    if (lane < NW) warp_tot[lane] = wi - v;  // exclusive warp offsets
  }
  __syncthreads();
  int run = warp_tot[warp] + incl - loc;
  for (int q = 0; q < per; ++q) {
    const int j = j0 + q;
    if (j < E) {
      ex_s[j] = run;
      run += tot[perm_s[j]];
    }
  }
  if (tid == NT - 1) ex_s[E] = run;  // the last thread's running sum is the grand total
  __syncthreads();
  for (int j = tid; j < E; j += NT) {
    const int e = perm_s[j];
    base[e] = ex_s[j] - ex_s[seg_s[owner_s[e]]];
  }
}

// pre[e] += Σ chunk_cnt[j] over j < n with j % E == e (the counts of the
// chunks before this one).  When E divides the block size every thread owns
// one expert column, so its loads are independent and accumulate in a
// register (one L2 round trip per batch instead of one per element).
__device__ __forceinline__ void chunk_prefix(const int32_t* cnt, int n, int E, int32_t* pre) {
  const int tid = threadIdx.x;
  if (kLayoutThreads % E == 0) {
    int v[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int j = tid;
    for (; j + 7 * kLayoutThreads < n; j += 8 * kLayoutThreads) {
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] += ld_cg(cnt + j + q * kLayoutThreads);
    }
    for (; j < n; j += kLayoutThreads) v[0] += ld_cg(cnt + j);
    const int acc = v[0] + v[1] + v[2] + v[3] + v[4] + v[5] + v[6] + v[7];
    if (acc) atomicAdd(&pre[tid % E], acc);
  } else {
    for (int j = tid; j < n; j += kLayoutThreads) {
      const int v = ld_cg(cnt + j);
      if (v) atomicAdd(&pre[j % E], v);
    }
  }
}

// The next epoch's dispatch block counters (sender side, P > 1): zeroed one
// epoch ahead, like the work counters.
__device__ __forceinline__ void zero_next_blocks(const FsArgs& a, int parity, int tid, int nthreads) {
  if (a.world == 1) return;
  const int nb = a.nbmax;
  uint32_t* done = a.blkdone + (size_t)(parity ^ 1) * nb * kBlkStride;
  uint32_t* dup = a.dupcnt + (size_t)(parity ^ 1) * a.world * nb;
  for (int j = tid; j < nb; j += nthreads) done[(size_t)j * kBlkStride] = 0u;
  for (int j = tid; j < a.world * nb; j += nthreads) dup[j] = 0u;
}

// ===========================================================================
// Layout planner
//
// Row order on rank g (Appendix A of SURVEY.md, planner.py:147-151):
//   rows sorted by (expert asc, source rank asc, local token index asc)
//   row_of[i,k] = base_g(e) + Σ_{s'<s} cnt[s'][e] + chunk_off[c][e]
//                 + (position of token i among chunk c's tokens routed to e)
// The in-chunk position is computed without atomics on positions: each warp
// ORs a lane bit into a per-(warp, expert) word; a token's rank among the
// earlier tokens of its warp is popc(word & lanemask_lt), plus the sum of the
// popcounts of the earlier warps.  Deterministic, hence bit-exact.  Per-expert
// totals are accumulated with commutative atomics (exact integers), so one
// CTA can publish them right after the single grid barrier.
//
// Global scratch per handle: chunk_cnt[chunks][E] (chunk counts), and
// totals[2][E] (per-parity atomic accumulators; this epoch zeroes the other
// parity for the next one).
// ===========================================================================
__global__ void __launch_bounds__(kLayoutThreads)
    layout_kernel(FsArgs a, const void* __restrict__ idx, int32_t* __restrict__ row_of,
                  uint8_t* __restrict__ first_mask, uint32_t* __restrict__ rank_mask,
                  long long* __restrict__ stats, int32_t* __restrict__ expert_counts,
                  int32_t* __restrict__ expert_offsets, int phase) {
  TraceLast trace_last_(a, FS_TRACE_LAYOUT_LAST);
  extern __shared__ __align__(16) uint32_t sm[];
  __shared__ long long red[kLayoutWarps][4];
  __shared__ int rows_total;
  cg::grid_group grid = cg::this_grid();
  const int E = a.E, K = a.K, T = a.T, P = a.world, s = a.rank;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nchunks = (T + kLayoutThreads - 1) / kLayoutThreads;
  const uint32_t lt_mask = (1u << lane) - 1u;
  const uint32_t epoch = load_epoch(a) + ((phase & FS_PHASE_LOCAL) ? 1u : 0u);
  const int parity = (int)(epoch & 1u);
  trace_stamp(a, FS_TRACE_LAYOUT_BEGIN);
  // the dispatch may start its row prefetch now (measured: triggering after the
  // histogram instead, to spare the planner's loads the contention, is slower)
  griddep_launch_dependents();

  __shared__ int warp_tot[kLayoutWarps];
  int32_t* owner_s = reinterpret_cast<int32_t*>(sm);
  int32_t* node_s = owner_s + E;
  int32_t* perm_s = node_s + 32;
  int32_t* seg_s = perm_s + E;        // [33]
  int32_t* cnt_s = seg_s + 33;        // [E] this CTA's last chunk counts
  uint32_t* work = reinterpret_cast<uint32_t*>(cnt_s + E);
  const size_t work_words = (size_t)(2 * kLayoutWarps * E > 5 * E + 1 ? 2 * kLayoutWarps * E : 5 * E + 1);
  // a single CTA owning the only chunk needs no grid barrier and already holds the totals
  const bool single = gridDim.x == 1 && nchunks <= 1;
  int32_t* e_s = reinterpret_cast<int32_t*>(work + work_words);
  int32_t* pos_s = e_s + kLayoutThreads * K;
  int32_t* totals = a.totals + (size_t)parity * E;
  long long* stat_acc = a.stat_part + parity * 8;  // [2][8] per-parity atomic accumulators
  // positions survive the grid barrier in shared memory when every CTA owns
  // exactly one chunk and both phases run in this launch (production)
  const bool keep_pos = (phase == FS_PHASE_ALL) && nchunks <= (int)gridDim.x;

  // stage the expert table and this CTA's first chunk of indices together
  // (one memory round trip instead of two)
  for (int e = tid; e < E; e += kLayoutThreads) {
    owner_s[e] = a.owner[e];
    perm_s[e] = a.perm[e];
    cnt_s[e] = 0;  // a rank without tokens publishes zero counts
  }
  if (tid < P) node_s[tid] = a.node_of[tid];
  if (tid <= P) seg_s[tid] = a.seg_begin[tid];
  auto stage_chunk = [&](int c) {
    const int t0 = c * kLayoutThreads;
    const int nel = min(kLayoutThreads, T - t0) * K;
    const size_t base_el = (size_t)t0 * K;
    // 8 independent loads in flight per thread before any is consumed
    for (int j0 = tid; j0 < nel; j0 += 8 * kLayoutThreads) {
      long long v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int j = j0 + q * kLayoutThreads;
        v[q] = j < nel ? load_idx(idx, base_el + j, a.idx64) : 0;
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int j = j0 + q * kLayoutThreads;
        if (j < nel) {
          long long e = v[q];
          if (e < 0 || e >= E) {
            record_error(a.status, FS_ERANGE);
            e = 0;
          }
          e_s[j] = (int32_t)e;
        }
      }
    }
  };
  if ((phase & FS_PHASE_LOCAL) && (int)blockIdx.x < nchunks) stage_chunk(blockIdx.x);

  if (phase & FS_PHASE_LOCAL) {
    uint32_t* bits = work;                       // [8][E]
    uint32_t* wbase = work + kLayoutWarps * E;   // [8][E]
    long long st_dedup = 0, st_naive = 0, st_local = 0, st_node = 0;
    for (int c = blockIdx.x; c < nchunks; c += gridDim.x) {
      const int t0 = c * kLayoutThreads;
      const int ntok = min(kLayoutThreads, T - t0);
      const int nel = ntok * K;
      const size_t base_el = (size_t)t0 * K;
      if (c != (int)blockIdx.x) {
        __syncthreads();
        stage_chunk(c);
      }
      for (int j = tid; j < kLayoutWarps * E; j += kLayoutThreads) bits[j] = 0u;
      __syncthreads();
      trace_stamp(a, 6);
      const int my_node = node_s[s];
      if (tid < ntok) {
        uint32_t seen_node = 0u, seen_rank = 0u;
        // groups of 8 experts: all smem lookups of a group issue before the
        // first is consumed (short dependent chains instead of K long ones)
        for (int k0 = 0; k0 < K; k0 += 8) {
          int ev[8], gv[8], nv[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) ev[q] = (k0 + q < K) ? e_s[tid * K + k0 + q] : 0;
#pragma unroll
          for (int q = 0; q < 8; ++q) gv[q] = owner_s[ev[q]];
#pragma unroll
          for (int q = 0; q < 8; ++q) nv[q] = node_s[gv[q]];
          uint32_t old[8];
#pragma unroll
          for (int q = 0; q < 8; ++q)
            old[q] = (k0 + q < K) ? atomicOr(&bits[warp * E + ev[q]], 1u << lane) : 0u;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            if (k0 + q < K) {
              const int g = gv[q], n = nv[q];
              const bool first = !((seen_node >> n) & 1u);
              seen_node |= 1u << n;
              seen_rank |= 1u << g;
              pos_s[tid * K + k0 + q] = first ? 1 : 0;  // first_mask staged here until positions overwrite it
              st_naive += (g != s);
              st_local += (g == s);
              st_node += (first && n != my_node);
              if (old[q] & (1u << lane)) record_error(a.status, FS_EINVAL);  // duplicate expert in a row
            }
          }
        }
        if (rank_mask) rank_mask[t0 + tid] = seen_rank;
        st_dedup += __popc(seen_rank & ~(1u << s));
      }
      __syncthreads();
      if (first_mask)
        for (int j = tid; j < nel; j += kLayoutThreads) first_mask[base_el + j] = (uint8_t)pos_s[j];
      for (int e = tid; e < E; e += kLayoutThreads) {
        uint32_t run = 0;
#pragma unroll
        for (int w = 0; w < kLayoutWarps; ++w) {
          wbase[w * E + e] = run;
          run += __popc(bits[w * E + e]);
        }
        a.chunk_cnt[(size_t)c * E + e] = (int32_t)run;
        cnt_s[e] = (int32_t)run;
        if (run) atomicAdd(&totals[e], (int)run);
      }
      __syncthreads();
      if (tid < ntok) {
        for (int k0 = 0; k0 < K; k0 += 8) {
          int ev[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) ev[q] = (k0 + q < K) ? e_s[tid * K + k0 + q] : 0;
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (k0 + q < K)
              pos_s[tid * K + k0 + q] =
                  (int32_t)(wbase[warp * E + ev[q]] + __popc(bits[warp * E + ev[q]] & lt_mask));
        }
      }
      __syncthreads();
      if (!keep_pos)
        for (int j = tid; j < nel; j += kLayoutThreads) row_of[base_el + j] = pos_s[j];
    }
    // statistics: block reduce, then one commutative atomic per counter (a
    // single rank's are constants: every row is local, nothing is sent)
    if (P > 1) {
      long long v[4] = {st_dedup, st_naive, st_local, st_node};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[j] += __shfl_xor_sync(kFull, v[j], o);
        if (lane == 0) red[warp][j] = v[j];
      }
      __syncthreads();
      if (tid < 4) {
        long long acc = 0;
        for (int w = 0; w < kLayoutWarps; ++w) acc += red[w][tid];
        if (acc) atomicAdd(reinterpret_cast<unsigned long long*>(stat_acc + tid), (unsigned long long)acc);
      }
    }
    trace_stamp(a, FS_TRACE_LAYOUT_HIST);
    if (single) __syncthreads();
    else grid.sync();
    trace_stamp(a, FS_TRACE_LAYOUT_GRIDSYNC);

    // One CTA publishes this rank's per-expert totals into every peer's count
    // matrix row [s] (the P x E count all-gather, 16 KB of epoch-tagged words
    // at P=8, E=256).  A single rank needs no publication.
    if (blockIdx.x == 0) {
      int32_t* next_totals = a.totals + (size_t)(parity ^ 1) * E;
      long long* next_stats = a.stat_part + (parity ^ 1) * 8;
      if (P > 1)
        for (int e = tid; e <= E; e += kLayoutThreads)
          publish_count(a, parity, epoch, e, e == E ? T : (single ? cnt_s[e] : ld_cg(totals + e)));
      for (int e = tid; e < E; e += kLayoutThreads) next_totals[e] = 0;
      zero_next_blocks(a, parity, tid, kLayoutThreads);
      if (stats && tid >= 5 && tid < FS_NSTATS) stats[tid] = 0;
      if (tid < 8) {
        next_stats[tid] = 0;
        a.work[((size_t)(parity ^ 1) * kWorkSlots + tid) * kWorkStride] = 0ull;  // the next epoch's work counters
      }
      // every CTA read the old epoch before the grid barrier: safe to bump
      if (tid == 0) *a.epoch_ptr = epoch;
      trace_stamp(a, FS_TRACE_LAYOUT_PUBLISH);
    }
  }

  if (phase & FS_PHASE_REMOTE) {
    int32_t* tot = reinterpret_cast<int32_t*>(work);
    int32_t* base = tot + E;
    int32_t* before = base + E;
    int32_t* pre = before + E;
    // this CTA's chunk offsets Σ_{c'<c} cnt[c'][e] — issued before the peer
    // wait so their latency overlaps it (only the CTA's first chunk here).
    // All threads sweep the contiguous [c][E] prefix (coalesced, independent
    // loads) and fold into shared memory.
    const int c_first = blockIdx.x;
    const bool from_smem = single && (phase & FS_PHASE_LOCAL);
    const bool one_e = E <= kLayoutThreads;  // one expert column per thread
    int tv = 0;  // P == 1: this thread's expert total, loaded alongside the chunk prefix
    if (P == 1 && one_e && tid < E) tv = from_smem ? cnt_s[tid] : ld_cg(totals + tid);
    for (int e = tid; e < E; e += kLayoutThreads) pre[e] = 0;
    __syncthreads();
    if (c_first < nchunks) chunk_prefix(a.chunk_cnt, c_first * E, E, pre);
    if (P > 1) {
      for (int e = tid; e < E; e += kLayoutThreads) gather_counts(a, parity, epoch, e, tot + e, before + e);
      trace_stamp(a, FS_TRACE_LAYOUT_WAIT);
    } else if (one_e) {
      if (tid < E) {
        tot[tid] = tv;
        before[tid] = 0;
      }
    } else {
      for (int e = tid; e < E; e += kLayoutThreads) {
        tot[e] = from_smem ? cnt_s[e] : ld_cg(totals + e);
        before[e] = 0;
      }
    }
    __syncthreads();
    trace_stamp(a, 15);
    // base_g(e): exclusive scan of totals over rank g's experts
    int32_t* ex_s = pre + E;  // [E+1]
    block_segmented_base<kLayoutThreads>(E, tot, perm_s, seg_s, owner_s, ex_s, base, warp_tot);
    if (tid == 0) rows_total = ex_s[seg_s[s + 1]] - ex_s[seg_s[s]];
    __syncthreads();
    trace_stamp(a, 19);
    for (int c = blockIdx.x; c < nchunks; c += gridDim.x) {
      if (c != c_first) {  // later chunks of this CTA (T > grid * 256)
        __syncthreads();
        for (int e = tid; e < E; e += kLayoutThreads) pre[e] = 0;
        __syncthreads();
        chunk_prefix(a.chunk_cnt, c * E, E, pre);
        __syncthreads();
      }
      for (int e = tid; e < E; e += kLayoutThreads) pre[e] += base[e] + before[e];
      __syncthreads();
      trace_stamp(a, 23);
      const int t0 = c * kLayoutThreads;
      const int nel = min(kLayoutThreads, T - t0) * K;
      const size_t base_el = (size_t)t0 * K;
      for (int j = tid; j < nel; j += kLayoutThreads) {  // coalesced, element-wise
        int e = keep_pos ? e_s[j] : (int)load_idx(idx, base_el + j, a.idx64);
        if (e < 0 || e >= E) e = 0;
        const long long r = (long long)(keep_pos ? pos_s[j] : row_of[base_el + j]) + pre[e];
        if (r >= a.max_rows) record_error(a.status, FS_ERANGE);
        row_of[base_el + j] = (int32_t)r;
      }
    }
    if (blockIdx.x == 0) {
      const int jb = seg_s[s], je = seg_s[s + 1];
      for (int j = jb + tid; j < je; j += kLayoutThreads) {
        const int e = perm_s[j];
        if (expert_counts) expert_counts[j - jb] = tot[e];
        if (expert_offsets) expert_offsets[j - jb] = base[e];
      }
      // the statistics sums (complete since the grid barrier) are read back
      // last: the round trip stays off the count publication's path
      if (stats && tid < 4) {
        const int slot[4] = {FS_STAT_DEDUP_SEND, FS_STAT_NAIVE_SEND, FS_STAT_LOCAL_ROWS, FS_STAT_NODE_DEDUP};
        stats[slot[tid]] = P > 1 ? *reinterpret_cast<volatile long long*>(a.stat_part + parity * 8 + tid)
                                 : (tid == 2 ? (long long)T * K : 0ll);
      }
      if (tid == 0) {
        if (expert_offsets) expert_offsets[je - jb] = rows_total;
        *a.num_rows = rows_total;
        if (stats) stats[FS_STAT_ROWS] = rows_total;
        trace_stamp(a, FS_TRACE_LAYOUT_END);
        if (rows_total > a.max_rows) record_error(a.status, FS_ERANGE);
      }
    }
  }
}

// ===========================================================================
// Layout planner, cluster engine (production, one launch for both phases)
//
// For E <= 256, K <= 8, T <= 8 x 1024: ONE thread-block cluster of CS <= 8
// CTAs x 1024 threads, one token per thread.  Each CTA builds its chunk's
// per-expert counts and in-chunk positions exactly as layout_kernel does
// (warp bitmasks, 32 warps), then the chunk offsets and per-expert totals come
// from the other CTAs' shared memory over DSMEM after one cluster barrier —
// no global atomics, no cooperative grid barrier.  Cluster rank 0 publishes
// the totals to the peers (P > 1).
// ===========================================================================
constexpr int kClusterThreads = 1024;
constexpr int kClusterWarps = kClusterThreads / 32;
constexpr int kClusterMaxCtas = 8;
constexpr int kClusterMaxE = 256;
constexpr int kClusterMaxK = 8;

__host__ __device__ inline size_t layout_cluster_smem_bytes(int E, int K) {
  // owner[E] node[32] bits[32][E] wbase[32][E] e_s[1024K] pos_s[1024K] cnt[E] tot/base/before/pre[4E]
  return sizeof(int32_t) * (2ull * E + 32 + 33 + 2ull * kClusterWarps * E + 2ull * kClusterThreads * K + 6ull * E + 1);
}

__global__ void __launch_bounds__(kClusterThreads, 1)
    layout_cluster_kernel(FsArgs a, const void* __restrict__ idx, int32_t* __restrict__ row_of,
                          uint8_t* __restrict__ first_mask, uint32_t* __restrict__ rank_mask,
                          long long* __restrict__ stats, int32_t* __restrict__ expert_counts,
                          int32_t* __restrict__ expert_offsets) {
  extern __shared__ __align__(16) uint32_t sm[];
  __shared__ long long red[kClusterWarps][4];
  __shared__ long long cta_stats[4];
  __shared__ int rows_total;
  const int E = a.E, K = a.K, T = a.T, P = a.world, s = a.rank;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t crank = cluster_ctarank();
  const int CS = (int)gridDim.x;
  const uint32_t lt_mask = (1u << lane) - 1u;
  const uint32_t epoch = load_epoch(a) + 1u;
  const int parity = (int)(epoch & 1u);
  trace_stamp(a, FS_TRACE_LAYOUT_BEGIN);
  griddep_launch_dependents();

  __shared__ int warp_tot[kClusterWarps];
  int32_t* owner_s = reinterpret_cast<int32_t*>(sm);
  int32_t* node_s = owner_s + E;
  int32_t* perm_s = node_s + 32;
  int32_t* seg_s = perm_s + E;  // [33]
  uint32_t* bits = reinterpret_cast<uint32_t*>(seg_s + 33);     // [32][E]
  uint32_t* wbase = bits + kClusterWarps * E;                   // [32][E]
  int32_t* e_s = reinterpret_cast<int32_t*>(wbase + kClusterWarps * E);
  int32_t* pos_s = e_s + kClusterThreads * K;
  int32_t* cnt = pos_s + kClusterThreads * K;                   // this CTA's per-expert counts
  int32_t* tot = cnt + E;
  int32_t* base = tot + E;
  int32_t* before = base + E;
  int32_t* pre = before + E;
  int32_t* ex_s = pre + E;  // [E+1]

  const int t0 = (int)crank * kClusterThreads;
  const int ntok = max(0, min(kClusterThreads, T - t0));
  const int nel = ntok * K;
  const size_t base_el = (size_t)t0 * K;
  // one round trip: expert table, node table and this CTA's indices together
  for (int e = tid; e < E; e += kClusterThreads) {
    owner_s[e] = a.owner[e];
    perm_s[e] = a.perm[e];
  }
  if (tid < P) node_s[tid] = a.node_of[tid];
  if (tid <= P) seg_s[tid] = a.seg_begin[tid];
  for (int j = tid; j < nel; j += kClusterThreads) {
    long long e = load_idx(idx, base_el + j, a.idx64);
    if (e < 0 || e >= E) {
      record_error(a.status, FS_ERANGE);
      e = 0;
    }
    e_s[j] = (int32_t)e;
  }
  for (int j = tid; j < kClusterWarps * E; j += kClusterThreads) bits[j] = 0u;
  if (tid < 4) cta_stats[tid] = 0;
  __syncthreads();

  long long st_dedup = 0, st_naive = 0, st_local = 0, st_node = 0;
  if (tid < ntok) {
    const int my_node = node_s[s];
    uint32_t seen_node = 0u, seen_rank = 0u;
    for (int k = 0; k < K; ++k) {
      const int e = e_s[tid * K + k];
      const int g = owner_s[e];
      const int n = node_s[g];
      const bool first = !((seen_node >> n) & 1u);
      seen_node |= 1u << n;
      seen_rank |= 1u << g;
      pos_s[tid * K + k] = first ? 1 : 0;
      st_naive += (g != s);
      st_local += (g == s);
      st_node += (first && n != my_node);
      const uint32_t old = atomicOr(&bits[warp * E + e], 1u << lane);
      if (old & (1u << lane)) record_error(a.status, FS_EINVAL);
    }
    if (rank_mask) rank_mask[t0 + tid] = seen_rank;
    st_dedup += __popc(seen_rank & ~(1u << s));
  }
  {
    long long v[4] = {st_dedup, st_naive, st_local, st_node};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v[j] += __shfl_xor_sync(kFull, v[j], o);
      if (lane == 0) red[warp][j] = v[j];
    }
  }
  __syncthreads();
  if (first_mask)
    for (int j = tid; j < nel; j += kClusterThreads) first_mask[base_el + j] = (uint8_t)pos_s[j];
  if (tid < 4) {
    long long acc = 0;
    for (int w = 0; w < kClusterWarps; ++w) acc += red[w][tid];
    cta_stats[tid] = acc;
  }
  // per-expert warp prefixes: 8 warps x 32 lanes cover the experts, each lane
  // walks the 32 warps' words of its expert
  for (int e = tid; e < E; e += kClusterThreads) {
    uint32_t run = 0;
#pragma unroll 8
    for (int w = 0; w < kClusterWarps; ++w) {
      wbase[w * E + e] = run;
      run += __popc(bits[w * E + e]);
    }
    cnt[e] = (int32_t)run;
  }
  __syncthreads();
  if (tid < ntok)
    for (int k = 0; k < K; ++k) {
      const int e = e_s[tid * K + k];
      pos_s[tid * K + k] = (int32_t)(wbase[warp * E + e] + __popc(bits[warp * E + e] & lt_mask));
    }
  trace_stamp(a, FS_TRACE_LAYOUT_HIST);
  cluster_sync_all();  // every CTA's cnt[] and cta_stats[] are final
  trace_stamp(a, FS_TRACE_LAYOUT_GRIDSYNC);

  // chunk offset (earlier CTAs) and rank totals from the cluster's smem
  for (int e = tid; e < E; e += kClusterThreads) {
    int p_acc = 0, t_acc = 0;
    for (int r = 0; r < CS; ++r) {
      const int v = (r == (int)crank) ? cnt[e] : (int)ld_dsmem_u32(&cnt[e], (uint32_t)r);
      t_acc += v;
      p_acc += (r < (int)crank) ? v : 0;
    }
    pre[e] = p_acc;
    tot[e] = t_acc;
  }
  __syncthreads();
  if (crank == 0) {
    if (P > 1)
      for (int e = tid; e <= E; e += kClusterThreads) publish_count(a, parity, epoch, e, e == E ? T : tot[e]);
    zero_next_blocks(a, parity, tid, kClusterThreads);
    if (stats && tid < 4) {
      long long acc = 0;
      for (int r = 0; r < CS; ++r) {
        const uint32_t lo = (r == 0) ? (uint32_t)(cta_stats[tid] & 0xffffffffu)
                                     : ld_dsmem_u32(reinterpret_cast<const uint32_t*>(&cta_stats[tid]), r);
        const uint32_t hi = (r == 0) ? (uint32_t)((unsigned long long)cta_stats[tid] >> 32)
                                     : ld_dsmem_u32(reinterpret_cast<const uint32_t*>(&cta_stats[tid]) + 1, r);
        acc += (long long)(((unsigned long long)hi << 32) | lo);
      }
      const int slot[4] = {FS_STAT_DEDUP_SEND, FS_STAT_NAIVE_SEND, FS_STAT_LOCAL_ROWS, FS_STAT_NODE_DEDUP};
      stats[slot[tid]] = acc;
    }
    if (stats && tid >= 5 && tid < FS_NSTATS) stats[tid] = 0;
    // the next epoch's accumulators (the grid planner relies on them being
    // zeroed one epoch ahead, and either planner may run next)
    for (int e = tid; e < E; e += kClusterThreads) a.totals[(size_t)(parity ^ 1) * E + e] = 0;
    if (tid < 8) {
      a.stat_part[(parity ^ 1) * 8 + tid] = 0;
      a.work[((size_t)(parity ^ 1) * kWorkSlots + tid) * kWorkStride] = 0ull;
    }
    if (tid == 0) *a.epoch_ptr = epoch;  // every CTA read the old epoch before the cluster barrier
    trace_stamp(a, FS_TRACE_LAYOUT_PUBLISH);
  }

  if (P > 1) {
    // tot[] is overwritten with the all-source totals (the DSMEM values were
    // this rank's own, already published above)
    __syncthreads();
    for (int e = tid; e < E; e += kClusterThreads) gather_counts(a, parity, epoch, e, tot + e, before + e);
    trace_stamp(a, FS_TRACE_LAYOUT_WAIT);
  } else {
    for (int e = tid; e < E; e += kClusterThreads) before[e] = 0;
  }
  __syncthreads();
  block_segmented_base<kClusterThreads>(E, tot, perm_s, seg_s, owner_s, ex_s, base, warp_tot);
  if (tid == 0) rows_total = ex_s[seg_s[s + 1]] - ex_s[seg_s[s]];
  __syncthreads();
  for (int e = tid; e < E; e += kClusterThreads) pre[e] += base[e] + before[e];
  __syncthreads();
  for (int j = tid; j < nel; j += kClusterThreads) {
    const long long r = (long long)pos_s[j] + pre[e_s[j]];
    if (r >= a.max_rows) record_error(a.status, FS_ERANGE);
    row_of[base_el + j] = (int32_t)r;
  }
  if (crank == 0) {
    const int jb = seg_s[s], je = seg_s[s + 1];
    for (int j = jb + tid; j < je; j += kClusterThreads) {
      const int e = perm_s[j];
      if (expert_counts) expert_counts[j - jb] = tot[e];
      if (expert_offsets) expert_offsets[j - jb] = base[e];
    }
    if (tid == 0) {
      if (expert_offsets) expert_offsets[je - jb] = rows_total;
      *a.num_rows = rows_total;
      if (stats) stats[FS_STAT_ROWS] = rows_total;
      trace_stamp(a, FS_TRACE_LAYOUT_END);
      if (rows_total > a.max_rows) record_error(a.status, FS_ERANGE);
    }
  }
  cluster_sync_all();  // keep every CTA's shared memory alive until all DSMEM reads are done
}

}  // namespace fusco
