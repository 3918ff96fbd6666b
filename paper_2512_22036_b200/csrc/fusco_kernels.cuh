// fusco_kernels.cuh — the three hot-path kernels of the shuffle.
//
//   layout_kernel    on-device planner: per-(rank, expert) counts, offsets,
//                    row_of[t,k], first_mask, dedup statistics
//                    (reference planner.py:126-196, routing.py:86-98)
//   dispatch_kernel  push: token rows -> owners' expert-major rows over NVLink,
//                    one crossing per (token, rank), receiver-side fan-out
//                    (reference engine.py:266-276 dispatch, 799-851)
//   combine_kernel   pull + k-ascending weighted reduction back to token order
//                    (reference engine.py:266-276 combine, 313-338, 967-1049)
//
// All three are persistent cooperative launches; their cross-rank waits are
// split into an explicit REMOTE phase so that P ranks can be emulated on one
// GPU by launching LOCAL for every rank, then REMOTE for every rank.
#pragma once
#include <cooperative_groups.h>

#include "fusco_device.cuh"

namespace fusco {
namespace cg = cooperative_groups;

constexpr int kLayoutThreads = 256;  // one token per thread per chunk
constexpr int kLayoutWarps = kLayoutThreads / 32;
constexpr int kMoveThreads = 256;    // dispatch / combine CTA size

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
        for (int e = tid; e < E; e += kLayoutThreads)
          publish_count(a, parity, epoch, e, single ? cnt_s[e] : ld_cg(totals + e));
      for (int e = tid; e < E; e += kLayoutThreads) next_totals[e] = 0;
      if (stats && tid >= 5 && tid < FS_NSTATS) stats[tid] = 0;
      if (tid < 8) {
        next_stats[tid] = 0;
        a.work[(size_t)(parity ^ 1) * 8 + tid] = 0ull;  // the next epoch's work counters
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
      for (int e = tid; e < E; e += kClusterThreads) publish_count(a, parity, epoch, e, tot[e]);
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
    if (tid < 8) a.work[(size_t)(parity ^ 1) * 8 + tid] = 0ull;
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
// its own HBM.  The activation buffer is double-buffered by epoch parity so
// that a fast rank's next dispatch cannot overwrite rows a slow rank is
// still pulling in combine.
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
  const int rows = *reinterpret_cast<volatile int*>(a.num_rows);
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

// ===========================================================================
// Combine
//
// out[i] = Σ_{k=0..K-1} w[i,k] · src_{owner(e_ik)}[row_of[i,k]]  (k ascending)
// pulled straight from the owners' rows; no staging buffer, no second pass.
// ACC64 reproduces engine.py:322-331 bit for bit (f64 multiply, then f64 add,
// k ascending, one final rounding); otherwise fp32 FMA.
// ===========================================================================
template <typename V, bool BF16>
struct Elem {
  static constexpr int kWords = sizeof(V) / 4;
  static constexpr int kPerWord = BF16 ? 2 : 1;
  static constexpr int N = kWords * kPerWord;
  __device__ __forceinline__ static float get(const V& v, int j) {
    const uint32_t w = word(v, j / kPerWord);
    if constexpr (BF16) return __uint_as_float((j & 1) ? (w & 0xffff0000u) : (w << 16));
    else return __uint_as_float(w);
  }
};

template <typename Acc>
__device__ __forceinline__ Acc fma_acc(Acc w, float y, Acc acc);
template <>
__device__ __forceinline__ float fma_acc<float>(float w, float y, float acc) {
  return __fmaf_rn(w, y, acc);
}
template <>
__device__ __forceinline__ double fma_acc<double>(double w, float y, double acc) {
  return __dadd_rn(acc, __dmul_rn(w, (double)y));  // no contraction: matches numpy
}

__device__ __forceinline__ uint32_t pack_out(float lo, float hi) {
  // one cvt.rn.bf16x2.f32 (round-to-nearest-even, same as two __float2bfloat16_rn)
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ uint32_t pack_out(double lo, double hi) {
  const __nv_bfloat16 a = __double2bfloat16(lo), b = __double2bfloat16(hi);
  return (uint32_t)__bfloat16_as_ushort(a) | ((uint32_t)__bfloat16_as_ushort(b) << 16);
}
__device__ __forceinline__ uint32_t f32_bits(float v) { return __float_as_uint(v); }
__device__ __forceinline__ uint32_t f32_bits(double v) { return __float_as_uint(__double2float_rn(v)); }

template <typename V, bool BF16, bool ACC64, int U, int KG>
__global__ void __launch_bounds__(kMoveThreads, 2)
    combine_kernel(FsArgs a, const void* __restrict__ idx, const int32_t* __restrict__ row_of,
                   const void* __restrict__ topk_w, int w64, V* __restrict__ out, int src_sel,
                   int phase) {
  TraceLast trace_last_(a, FS_TRACE_COMBINE_LAST);
  using Acc = typename std::conditional<ACC64, double, float>::type;
  using EL = Elem<V, BF16>;
  // U vector words per lane per unit; KG experts' rows in flight together
  // (KG = min(K, 4) so no registers are reserved for loads that never issue)
  constexpr int SW = 32 * U;
  const int K = a.K, T = a.T, P = a.world, s = a.rank;
  const int nv = a.tb / (int)sizeof(V);
  const int S = (nv + SW - 1) / SW;
  const int lane = threadIdx.x & 31;
  const int gw = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int nw = (int)((gridDim.x * blockDim.x) >> 5);
  griddep_wait();  // rows / the epoch from the previous kernel (PDL launch)
  const uint32_t epoch = load_epoch(a);
  const size_t src_off =
      src_sel == FS_SRC_ACT_OUT ? a.off_actout : a.off_act;

  trace_stamp(a, FS_TRACE_COMBINE_BEGIN);
  // "expert outputs ready" handshake: this rank's act/act_out rows were
  // completed by earlier kernels on this stream; one release store per peer
  // publishes them, and the pull waits for every peer's.  A single rank has
  // nobody to wait for.
  if ((phase & FS_PHASE_LOCAL) && P > 1) {
    if (blockIdx.x == 0 && threadIdx.x < P)
      st_release_sys_u32(reinterpret_cast<uint32_t*>(a.peer[threadIdx.x] + kOffReadyFlag) + s, epoch);
  }
  if (phase & FS_PHASE_REMOTE) {
    if (P > 1) {
      if (threadIdx.x < P)
        wait_u32_geq(reinterpret_cast<const uint32_t*>(a.peer[s] + kOffReadyFlag) + threadIdx.x, epoch, a);
      __syncthreads();
    }
    trace_stamp(a, FS_TRACE_COMBINE_READY);
    __shared__ int32_t owner_sm[kMaxExperts];
    load_owner_table(a, owner_sm);
    const uint32_t units = (uint32_t)T * (uint32_t)S, uS = (uint32_t)S;  // 32-bit unit arithmetic
    auto load_w = [&](int i) -> Acc {
      if (lane >= K) return (Acc)0;
      const size_t pos = (size_t)i * K + lane;
      return w64 ? (Acc)reinterpret_cast<const double*>(topk_w)[pos]
                 : (Acc)reinterpret_cast<const float*>(topk_w)[pos];
    };
    uint32_t u = (uint32_t)gw;
    KMeta nxt = u < units ? load_meta(a, idx, row_of, (int)(u / uS), lane) : KMeta{0, 0};
    Acc nxt_w = u < units ? load_w((int)(u / uS)) : (Acc)0;
    for (; u < units; u += (uint32_t)nw) {
      const int i = (int)(u / uS);
      const int sl = (int)(u - (uint32_t)i * uS);
      const KMeta cur = nxt;
      const Acc wk = nxt_w;
      if (u + (uint32_t)nw < units) {
        const int inext = (int)((u + (uint32_t)nw) / uS);
        nxt = load_meta(a, idx, row_of, inext, lane);
        nxt_w = load_w(inext);
      }
      int g = 0, r = 0;
      if (lane < K) {
        g = owner_sm[cur.e];
        r = (cur.r < 0 || cur.r >= a.max_rows) ? 0 : cur.r;
      }
      const int w0 = sl * SW;
      const int rem = nv - w0;
      Acc acc[U][EL::N];
#pragma unroll
      for (int j = 0; j < U; ++j)
#pragma unroll
        for (int q = 0; q < EL::N; ++q) acc[j][q] = (Acc)0;
      for (int k0 = 0; k0 < K; k0 += KG) {
        V v[KG][U];
        Acc wg[KG];
#pragma unroll
        for (int kk = 0; kk < KG; ++kk) {
          const int k = k0 + kk;
          const int gk = __shfl_sync(kFull, g, k & 31);
          const int rk = __shfl_sync(kFull, r, k & 31);
          wg[kk] = __shfl_sync(kFull, wk, k & 31);
          if (k < K) {
            const V* src = reinterpret_cast<const V*>(a.peer[gk] + src_off) + (size_t)rk * nv + w0;
#pragma unroll
            for (int j = 0; j < U; ++j) {
              const int w = j * 32 + lane;
              if (w < rem) v[kk][j] = ld_nc(src + w);
            }
          }
        }
#pragma unroll
        for (int kk = 0; kk < KG; ++kk) {
          if (k0 + kk < K) {
#pragma unroll
            for (int j = 0; j < U; ++j) {
              if (j * 32 + lane < rem) {
#pragma unroll
                for (int q = 0; q < EL::N; ++q)
                  acc[j][q] = fma_acc<Acc>(wg[kk], EL::get(v[kk][j], q), acc[j][q]);
              }
            }
          }
        }
      }
      V* dst = out + (size_t)i * nv + w0;
#pragma unroll
      for (int j = 0; j < U; ++j) {
        const int w = j * 32 + lane;
        if (w < rem) {
          V o;
#pragma unroll
          for (int q = 0; q < EL::kWords; ++q) {
            if constexpr (BF16) set_word(o, q, pack_out(acc[j][2 * q], acc[j][2 * q + 1]));
            else set_word(o, q, f32_bits(acc[j][q]));
          }
          st_na(dst + w, o);
        }
      }
    }
  }
  trace_stamp(a, FS_TRACE_COMBINE_END);
}

// ===========================================================================
// Combine, software-pipelined warp engine for K <= 2 (Mixtral-like top-2)
//
// Same math and order as combine_kernel, but each warp keeps two units in
// flight: the row loads of unit n+1 are issued before unit n is reduced and
// stored, and the (expert, row) metadata is prefetched two units ahead, so a
// warp's memory parallelism doubles without more warps.
// ===========================================================================
template <bool BF16, bool ACC64>
__global__ void __launch_bounds__(kMoveThreads)
    combine_k2_kernel(FsArgs a, const void* __restrict__ idx, const int32_t* __restrict__ row_of,
                      const void* __restrict__ topk_w, int w64, int4* __restrict__ out, int src_sel, int phase) {
  TraceLast trace_last_(a, FS_TRACE_COMBINE_LAST);
  using Acc = typename std::conditional<ACC64, double, float>::type;
  using EL = Elem<int4, BF16>;
  constexpr int U = 4;
  constexpr int SW = 32 * U;
  const int K = a.K, T = a.T, P = a.world, s = a.rank;
  const int nv = a.tb / 16;
  const int S = (nv + SW - 1) / SW;
  const int lane = threadIdx.x & 31;
  // unit indices fit in 32 bits (fs_create bounds max_tokens x slices):
  // 32-bit division, and the token of a unit is computed once
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  __shared__ int32_t owner_sm[kMaxExperts];
  load_owner_table(a, owner_sm);  // prologue (static table) before the PDL wait
  griddep_wait();                 // dispatched rows / epoch from the previous kernel
  const uint32_t epoch = load_epoch(a);
  const size_t src_off =
      src_sel == FS_SRC_ACT_OUT ? a.off_actout : a.off_act;
  trace_stamp(a, FS_TRACE_COMBINE_BEGIN);
  if ((phase & FS_PHASE_LOCAL) && P > 1) {
    if (blockIdx.x == 0 && threadIdx.x < P)
      st_release_sys_u32(reinterpret_cast<uint32_t*>(a.peer[threadIdx.x] + kOffReadyFlag) + s, epoch);
  }
  if (!(phase & FS_PHASE_REMOTE)) return;
  if (P > 1) {
    if (threadIdx.x < P)
      wait_u32_geq(reinterpret_cast<const uint32_t*>(a.peer[s] + kOffReadyFlag) + threadIdx.x, epoch, a);
    __syncthreads();
  }
  trace_stamp(a, FS_TRACE_COMBINE_READY);
  const uint32_t units = (uint32_t)T * (uint32_t)S;

  struct Unit {
    uint32_t u;
    int i;
    const int4* src[2];
    Acc w[2];
    int w0, rem;
  };
  auto load_w = [&](int i) -> Acc {
    if (lane >= K) return (Acc)0;
    const size_t pos = (size_t)i * K + lane;
    return w64 ? (Acc)reinterpret_cast<const double*>(topk_w)[pos]
               : (Acc)reinterpret_cast<const float*>(topk_w)[pos];
  };
  // metadata (lanes 0..K-1) -> per-unit row pointers, broadcast to the warp
  auto resolve = [&](uint32_t uu, const KMeta& m, Acc wl) -> Unit {
    Unit x;
    x.u = uu;
    x.i = (int)(uu / (uint32_t)S);
    const int sl = (int)(uu - (uint32_t)x.i * (uint32_t)S);
    x.w0 = sl * SW;
    x.rem = nv - x.w0;
    int g = 0, r = 0;
    if (lane < K) {
      g = owner_sm[m.e];
      r = (m.r < 0 || m.r >= a.max_rows) ? 0 : m.r;
    }
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int gk = __shfl_sync(kFull, g, k);
      const int rk = __shfl_sync(kFull, r, k);
      x.w[k] = __shfl_sync(kFull, wl, k);
      x.src[k] = reinterpret_cast<const int4*>(a.peer[gk] + src_off) + (size_t)rk * nv + x.w0;
    }
    return x;
  };
  auto issue = [&](const Unit& x, int4 (&v)[2][U]) {
#pragma unroll
    for (int k = 0; k < 2; ++k)
#pragma unroll
      for (int j = 0; j < U; ++j) {
        const int w = j * 32 + lane;
        if (k < K && w < x.rem) v[k][j] = ld_nc(x.src[k] + w);
      }
  };
  auto finish = [&](const Unit& x, const int4 (&v)[2][U]) {
    int4* dst = out + (size_t)x.i * nv + x.w0;
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int w = j * 32 + lane;
      if (w < x.rem) {
        Acc acc[EL::N];
#pragma unroll
        for (int q = 0; q < EL::N; ++q) acc[q] = (Acc)0;
#pragma unroll
        for (int k = 0; k < 2; ++k)
          if (k < K)
#pragma unroll
            for (int q = 0; q < EL::N; ++q) acc[q] = fma_acc<Acc>(x.w[k], EL::get(v[k][j], q), acc[q]);
        int4 o;
#pragma unroll
        for (int q = 0; q < EL::kWords; ++q) {
          if constexpr (BF16) set_word(o, q, pack_out(acc[2 * q], acc[2 * q + 1]));
          else set_word(o, q, f32_bits(acc[q]));
        }
        st_na(dst + w, o);
      }
    }
  };

  const uint32_t u = gw;
  if (u >= units) return;
  KMeta m_next = load_meta(a, idx, row_of, (int)(u / (uint32_t)S), lane);
  Acc w_next = load_w((int)(u / (uint32_t)S));
  Unit cur = resolve(u, m_next, w_next);
  if (u + nw < units) {
    const int i1 = (int)((u + nw) / (uint32_t)S);
    m_next = load_meta(a, idx, row_of, i1, lane);
    w_next = load_w(i1);
  }
  int4 va[2][U], vb[2][U];
  issue(cur, va);
  for (;;) {
    // ---- cur in va; next goes to vb
    const uint32_t u1 = cur.u + nw;
    Unit nxt;
    if (u1 < units) {
      nxt = resolve(u1, m_next, w_next);
      if (u1 + nw < units) {
        const int in = (int)((u1 + nw) / (uint32_t)S);
        m_next = load_meta(a, idx, row_of, in, lane);
        w_next = load_w(in);
      }
      issue(nxt, vb);
    }
    finish(cur, va);
    if (u1 >= units) break;
    cur = nxt;
    // ---- cur in vb; next goes to va
    const uint32_t u2 = cur.u + nw;
    if (u2 < units) {
      nxt = resolve(u2, m_next, w_next);
      if (u2 + nw < units) {
        const int in = (int)((u2 + nw) / (uint32_t)S);
        m_next = load_meta(a, idx, row_of, in, lane);
        w_next = load_w(in);
      }
      issue(nxt, va);
    }
    finish(cur, vb);
    if (u2 >= units) break;
    cur = nxt;
  }
  trace_stamp(a, FS_TRACE_COMBINE_END);
}

// ===========================================================================
// Combine, TMA engine
//
// Work item = (token i, column slice j of SB bytes).  Warp 0 resolves the
// token's K (owner, row) pairs one item ahead and its lanes k<K each issue a
// cp.async.bulk of row slice (owner_k, row_k, j) — local HBM or a peer over
// NVLink — into stage q ([K][SB] bytes), all completing on full[q].
// kCombConsumers warps then reduce Σ_k w_k·row_k in k order straight out of
// shared memory (16 B per lane per step) and store the output slice; each
// consumer warp arrives on empty[q] when done.  Loads in flight per SM = NS
// stages of K·SB bytes, independent of register pressure.
// ===========================================================================
constexpr int kCombConsumers = 8;
constexpr int kCombThreads = 32 * (1 + kCombConsumers);
constexpr int kCombMaxStages = 16;
constexpr int kCombStageTarget = 24 * 1024;  // bytes of one stage (K row slices)

__host__ __device__ inline int comb_slice_bytes(int tb, int K, int stage_target = kCombStageTarget) {
  int sb = stage_target / K;
  sb = sb < 512 ? 512 : sb;
  if (sb >= tb) return tb;
  const int S = (tb + sb - 1) / sb;
  return (((tb + S - 1) / S) + 15) & ~15;
}

template <bool BF16, bool ACC64>
__global__ void __launch_bounds__(kCombThreads)
    combine_tma_kernel(FsArgs a, const void* __restrict__ idx, const int32_t* __restrict__ row_of,
                       const void* __restrict__ topk_w, int w64, char* __restrict__ out, int src_sel,
                       int phase, int nstages, int sb) {
  TraceLast trace_last_(a, FS_TRACE_COMBINE_LAST);
  using Acc = typename std::conditional<ACC64, double, float>::type;
  using EL = Elem<int4, BF16>;
  extern __shared__ __align__(128) char csm[];
  // per stage: the claimed item (-1 = no more work) and its K weights, written
  // by the producer before it arms the stage's full barrier
  __shared__ long long slot_item[kCombMaxStages];
  __shared__ Acc slot_w[kCombMaxStages][32];
  __shared__ int32_t owner_cmb[kMaxExperts];
  uint64_t* full = reinterpret_cast<uint64_t*>(csm);
  uint64_t* empty = full + kCombMaxStages;
  char* stages = csm + 2 * kCombMaxStages * sizeof(uint64_t);
  const int K = a.K, T = a.T, P = a.world, s = a.rank, tb = a.tb;
  const int S = (tb + sb - 1) / sb;
  const int stage_bytes = K * sb;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool remote = (phase & FS_PHASE_REMOTE) != 0;
  if (remote) {  // prologue independent of the previous kernel (PDL launch)
    for (int e = threadIdx.x; e < a.E; e += blockDim.x) owner_cmb[e] = a.owner[e];
    if (threadIdx.x == 0) {
      for (int q = 0; q < nstages; ++q) {
        mbar_init(&full[q], 1);
        mbar_init(&empty[q], kCombConsumers);
      }
      mbar_fence_init();
    }
  }
  griddep_wait();  // dispatched rows / the epoch
  const uint32_t epoch = load_epoch(a);
  const size_t src_off =
      src_sel == FS_SRC_ACT_OUT ? a.off_actout : a.off_act;
  trace_stamp(a, FS_TRACE_COMBINE_BEGIN);

  if ((phase & FS_PHASE_LOCAL) && P > 1) {
    if (blockIdx.x == 0 && threadIdx.x < P)
      st_release_sys_u32(reinterpret_cast<uint32_t*>(a.peer[threadIdx.x] + kOffReadyFlag) + s, epoch);
  }
  if (!remote) return;
  if (P > 1 && threadIdx.x < P)
    wait_u32_geq(reinterpret_cast<const uint32_t*>(a.peer[s] + kOffReadyFlag) + threadIdx.x, epoch, a);
  __syncthreads();
  // the rows the bulk copies (async proxy) read were published to generic-proxy acquires
  if (P > 1 && threadIdx.x < 32) fence_proxy_async_global();
  trace_stamp(a, FS_TRACE_COMBINE_READY);
  const long long items = (long long)T * S;

  if (warp == 0) {  // producer: claims items dynamically, one ahead (metadata + weights prefetched)
    unsigned long long* ctr = work_ctr(a, epoch, kWorkCombine);
    auto load_w = [&](long long uu) -> Acc {
      if (lane >= K) return (Acc)0;
      const size_t pos = (size_t)((uint32_t)uu / (uint32_t)S) * K + lane;
      return w64 ? (Acc)reinterpret_cast<const double*>(topk_w)[pos]
                 : (Acc)reinterpret_cast<const float*>(topk_w)[pos];
    };
    long long u = claim_warp(ctr);
    KMeta m = u < items ? load_meta(a, idx, row_of, (int)((uint32_t)u / (uint32_t)S), lane) : KMeta{0, 0};
    Acc wl = u < items ? load_w(u) : (Acc)0;
    int n = 0;
    for (;; ++n) {
      const int q = n % nstages;
      if (n >= nstages) mbar_wait(&empty[q], ((n / nstages) & 1) ^ 1);
      if (u >= items) {  // sentinel: consumers stop at this stage
        if (lane == 0) {
          slot_item[q] = -1;
          mbar_arrive(&full[q]);
        }
        break;
      }
      const long long un = claim_warp(ctr);  // claimed and prefetched while this item streams
      KMeta mn = KMeta{0, 0};
      Acc wn = (Acc)0;
      if (un < items) {
        mn = load_meta(a, idx, row_of, (int)((uint32_t)un / (uint32_t)S), lane);
        wn = load_w(un);
      }
      const int i = (int)((uint32_t)u / (uint32_t)S), j = (int)((uint32_t)u - (uint32_t)i * (uint32_t)S);
      (void)i;
      const int off = j * sb;
      const int len = min(sb, tb - off);
      int g = 0, r = 0;
      if (lane < K) {
        g = owner_cmb[m.e];
        r = (m.r < 0 || m.r >= a.max_rows) ? 0 : m.r;
        slot_w[q][lane] = wl;
      }
      if (lane == 0) slot_item[q] = u;
      __syncwarp();
      if (lane == 0) mbar_arrive_expect_tx(&full[q], (uint32_t)(K * len));
      __syncwarp();
      if (lane < K)
        bulk_load(stages + (size_t)q * stage_bytes + (size_t)lane * sb,
                  a.peer[g] + src_off + (size_t)r * tb + off, (uint32_t)len, &full[q]);
      u = un;
      m = mn;
      wl = wn;
    }
  } else {  // consumers
    const int ct = threadIdx.x - 32;  // 0 .. 32*kCombConsumers-1
    for (int n = 0;; ++n) {
      const int q = n % nstages;
      mbar_wait(&full[q], (n / nstages) & 1);
      const long long u = slot_item[q];
      if (u < 0) break;
      const int i = (int)((uint32_t)u / (uint32_t)S), j = (int)((uint32_t)u - (uint32_t)i * (uint32_t)S);
      const int off = j * sb;
      const int nv = min(sb, tb - off) / 16;
      const char* st = stages + (size_t)q * stage_bytes;
      for (int v = ct; v < nv; v += 32 * kCombConsumers) {
        Acc acc[EL::N];
#pragma unroll
        for (int e = 0; e < EL::N; ++e) acc[e] = (Acc)0;
        for (int k = 0; k < K; ++k) {
          const Acc wk = slot_w[q][k];
          const int4 x = *reinterpret_cast<const int4*>(st + (size_t)k * sb + (size_t)v * 16);
#pragma unroll
          for (int e = 0; e < EL::N; ++e) acc[e] = fma_acc<Acc>(wk, EL::get(x, e), acc[e]);
        }
        int4 o;
#pragma unroll
        for (int w = 0; w < EL::kWords; ++w) {
          if constexpr (BF16) set_word(o, w, pack_out(acc[2 * w], acc[2 * w + 1]));
          else set_word(o, w, f32_bits(acc[w]));
        }
        st_na(reinterpret_cast<int4*>(out + (size_t)i * tb + off) + v, o);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[q]);
    }
  }
  trace_stamp(a, FS_TRACE_COMBINE_END);
}

// ===========================================================================
// Copy-bandwidth probe (HBM or NVLink peer), same warp copy loop shape.
// ===========================================================================
__global__ void __launch_bounds__(kMoveThreads)
    probe_copy_kernel(int4* __restrict__ dst, const int4* __restrict__ src, size_t n16) {
  constexpr int U = 4;
  const size_t lane = threadIdx.x & 31;
  const size_t gw = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  const size_t nw = (gridDim.x * (size_t)blockDim.x) >> 5;
  for (size_t w0 = gw * 32 * U; w0 < n16; w0 += nw * 32 * U) {
    int4 v[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const size_t w = w0 + j * 32 + lane;
      if (w < n16) v[j] = ld_nc(src + w);
    }
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const size_t w = w0 + j * 32 + lane;
      if (w < n16) st_na(dst + w, v[j]);
    }
  }
}

// ===========================================================================
// All-to-all copy probe: pairs j = 0..n-1 copy src[j] -> dst[j] concurrently
// (chunks interleaved over CTAs so every pair progresses at once).  With
// src local / dst on peers it measures NVLink push bandwidth, with src on
// peers / dst local the pull bandwidth — with the engines' own movers
// (mode 0: warp 16 B loads/stores, mode 1: TMA bulk via a smem ring).
// ===========================================================================
struct ProbePairs {
  const char* src[FS_MAX_RANKS];
  char* dst[FS_MAX_RANKS];
};
constexpr int kProbeChunk = 16384;

__global__ void __launch_bounds__(kMoveThreads) probe_a2a_warp_kernel(ProbePairs pp, int npairs, size_t bytes) {
  const int lane = threadIdx.x & 31;
  const long long gw = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = (gridDim.x * (long long)blockDim.x) >> 5;
  const long long chunks = (long long)((bytes + kProbeChunk - 1) / kProbeChunk) * npairs;
  for (long long c = gw; c < chunks; c += nw) {
    const int j = (int)(c % npairs);
    const size_t off = (size_t)(c / npairs) * kProbeChunk;
    const int n16 = (int)(min((size_t)kProbeChunk, bytes - off) / 16);
    const int4* s = reinterpret_cast<const int4*>(pp.src[j] + off);
    int4* d = reinterpret_cast<int4*>(pp.dst[j] + off);
    for (int w0 = 0; w0 < n16; w0 += 32 * 8) {
      int4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (w0 + u * 32 + lane < n16) v[u] = ld_nc(s + w0 + u * 32 + lane);
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (w0 + u * 32 + lane < n16) st_na(d + w0 + u * 32 + lane, v[u]);
    }
  }
}

__global__ void __launch_bounds__(64) probe_a2a_tma_kernel(ProbePairs pp, int npairs, size_t bytes, int nslots) {
  extern __shared__ __align__(128) char psm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(psm);
  char* ring = psm + 32 * sizeof(uint64_t);
  if (threadIdx.x != 0) return;  // one thread drives loads and stores
  for (int q = 0; q < nslots; ++q) mbar_init(&full[q], 1);
  mbar_fence_init();
  const long long chunks = (long long)((bytes + kProbeChunk - 1) / kProbeChunk) * npairs;
  long long n = 0;
  // prologue: fill the ring
  long long c_load = blockIdx.x;
  for (int q = 0; q < nslots && c_load < chunks; ++q, c_load += gridDim.x) {
    const int j = (int)(c_load % npairs);
    const size_t off = (size_t)(c_load / npairs) * kProbeChunk;
    const uint32_t len = (uint32_t)min((size_t)kProbeChunk, bytes - off);
    mbar_arrive_expect_tx(&full[q], len);
    bulk_load(ring + (size_t)q * kProbeChunk, pp.src[j] + off, len, &full[q]);
  }
  for (long long c = blockIdx.x; c < chunks; c += gridDim.x, ++n) {
    const int q = (int)(n % nslots);
    mbar_wait(&full[q], (uint32_t)((n / nslots) & 1));
    const int j = (int)(c % npairs);
    const size_t off = (size_t)(c / npairs) * kProbeChunk;
    const uint32_t len = (uint32_t)min((size_t)kProbeChunk, bytes - off);
    bulk_store(pp.dst[j] + off, ring + (size_t)q * kProbeChunk, len);
    bulk_commit();
    bulk_wait_read<0>();
    if (c_load < chunks) {  // refill this slot
      const int j2 = (int)(c_load % npairs);
      const size_t off2 = (size_t)(c_load / npairs) * kProbeChunk;
      const uint32_t len2 = (uint32_t)min((size_t)kProbeChunk, bytes - off2);
      mbar_arrive_expect_tx(&full[q], len2);
      bulk_load(ring + (size_t)q * kProbeChunk, pp.src[j2] + off2, len2, &full[q]);
      c_load += gridDim.x;
    }
  }
  bulk_wait<0>();
}

}  // namespace fusco
