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
// rank every k is written directly from registers.  A token's further rows
// on an already-reached rank are listed (duplicate row, primary row) in that
// rank's duplicate list for the token's completion block; as each block of
// each source lands, the receiver copies primary -> duplicate rows in its
// own HBM (fan_watch / fan_work).  The activation buffer is single: a rank's next dispatch
// cannot start before every peer published its next-epoch counts, i.e.
// finished pulling this epoch's rows in combine (fusco.cu region_layout).
// ===========================================================================
#ifndef FUSCO_MOVE_U
#define FUSCO_MOVE_U 8  // 16-byte words per lane per dispatch unit (A/B builds)
#endif
template <typename V>
struct MoveCfg {
  static constexpr int U = sizeof(V) == 16 ? FUSCO_MOVE_U : 16;  // words per lane per unit (4 KB / 2 KB)
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

// ===========================================================================
// Receiver-side fan-out, block by block as the pushes land (P > 1)
//
// Jobs are (source q, block b).  One watcher warp (CTA 0's last warp) polls
// the block words of every pending job — lane l owns jobs l, l+32, ... in
// block-major order — and publishes each landed job with its duplicate
// count: jcum[k] (cumulative fan-out units after the k-th published job),
// jorder[k] = (q << 16) | b, then one release of (k << 40 | units) on the
// work word kWorkFanReady.  Every other warp with nothing left to push
// claims groups of kFanGroup units (one unit = one duplicate row) and
// copies primary -> duplicate rows in its own HBM once
// the published prefix covers them — so duplicates of early blocks are
// fanned out while later blocks are still crossing NVLink.  Replaces the
// reference's "forwarders fan out after all landings" (engine.py:845-847)
// and its expected-byte completion counters (engine.py:979-1031).
// ===========================================================================
constexpr int kFanGroup = 2;  // duplicate rows per fan-out claim

// Per-CTA cache of the published fan-out words (a.fan_poll).
struct FanPoll {
  unsigned long long seen, done;
  int lock;
};
__device__ __forceinline__ volatile FanPoll* fan_poll_sm() {
  __shared__ FanPoll fp;
  return &fp;
}
__device__ __forceinline__ void fan_poll_init() {
  if (threadIdx.x == 0) {
    volatile FanPoll* fp = fan_poll_sm();
    fp->seen = 0;
    fp->done = 0;
    fp->lock = 0;
  }
  __syncthreads();
}

__device__ __forceinline__ unsigned long long ld_acquire_gpu_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
constexpr unsigned long long kUnitMask = (1ull << 40) - 1;

// The watcher warp: publishes landed jobs until every one is in (or timeout).
// fs = fan-out units per duplicate row (1: whole rows; S: one unit per slice)
static __device__ void fan_watch(const FsArgs& a, uint32_t epoch, int fs) {
  const int P = a.world, s = a.rank, lane = threadIdx.x & 31;
  const int par = (int)(epoch & 1u);
  unsigned long long* ready = work_ctr(a, epoch, kWorkFanReady);
  unsigned long long* done = work_ctr(a, epoch, kWorkFanDone);
  // blocks per source from the sources' published token counts
  int nb = 0;
  if (lane < P && lane != s) {
    const int Tq = read_count_word(a, par, epoch, lane, a.E);
    nb = (Tq + a.blk - 1) / a.blk;
  }
  int nbm = nb;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) nbm = max(nbm, __shfl_xor_sync(kFull, nbm, o));
  const int Q = P - 1;
  const int J = nbm * Q;
  int j = lane;  // this lane's next pending job (block-major, sources rotated by the receiver)
  unsigned long long units = 0;
  uint32_t npub = 0;
  const unsigned long long t0 = globaltimer();
  bool timed_out = false;
  while (__any_sync(kFull, j < J)) {
    bool rdy = false;
    uint32_t nd = 0;
    int q = 0, b = 0;
    if (j < J) {
      b = j / Q;
      q = (s + 1 + j % Q) % P;
    }
    // lane q holds nb for source q: fetch the one this lane's job needs
    const int nb_q = __shfl_sync(kFull, nb, q & 31);
    if (j < J) {
      if (b >= nb_q) {
        rdy = true;  // the source has fewer blocks: nothing to wait for
      } else {
        const unsigned long long w = ld_acquire_sys_u64(blkflag_ptr(a, s, q, b));
        if ((uint32_t)(w >> 32) == epoch) {
          rdy = true;
          nd = (uint32_t)w;
        }
      }
    }
    const bool pub = rdy && nd > 0;
    const unsigned long long mine = pub ? (unsigned long long)nd * (unsigned)fs : 0ull;
    // inclusive warp scan of the newly published units
    unsigned long long inc = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long n = __shfl_up_sync(kFull, inc, o);
      if (lane >= o) inc += n;
    }
    const uint32_t pm = __ballot_sync(kFull, pub);
    if (pub) {
      const uint32_t k = npub + __popc(pm & ((1u << lane) - 1u));
      a.fan_jcum[k] = units + inc;
      a.fan_jorder[k] = ((uint32_t)q << 16) | (uint32_t)b;
    }
    units += __shfl_sync(kFull, inc, 31);
    npub += __popc(pm);
    if (rdy) j += 32;
    __syncwarp();
    if (pm && lane == 0) st_release_gpu_u64(ready, ((unsigned long long)npub << 40) | units);
    if (!pm) {
      if (globaltimer() - t0 > a.timeout_ns) {
        timed_out = true;
        break;
      }
      __nanosleep(64);
    }
  }
  if (timed_out && lane == 0) record_error(a.status, FS_ETIMEOUT, kSiteDispBlocks);
  if (a.trace != nullptr && lane == 0) a.trace[FS_TRACE_DISPATCH_ARRIVED] = globaltimer();
  __syncwarp();
  if (lane == 0) st_release_gpu_u64(done, 1ull);
}

// A fan-out worker warp: claims unit groups and copies duplicate rows.  A
// unit is a whole row (large batches: one schedule lookup per row) or, with
// a.fan_split (small batches: few rows, so a warp copying a 14 KB row slice
// after slice would serialise the phase), one slice of a row.
template <typename V>
__device__ __forceinline__ int fan_units_per_row(const FsArgs& a, int nv) {
  constexpr int SW = 32 * MoveCfg<V>::U;
  return a.fan_split ? (nv + SW - 1) / SW : 1;
}
template <typename V>
__device__ void fan_work(const FsArgs& a, uint32_t epoch, size_t act_off, int nv, int warps_per_cta) {
  constexpr int U = MoveCfg<V>::U;
  constexpr int SW = 32 * U;
  const int fs = fan_units_per_row<V>(a, nv);
  const int lane = threadIdx.x & 31;
  unsigned long long* ctr = work_ctr(a, epoch, kWorkFanout);
  const unsigned long long* ready = work_ctr(a, epoch, kWorkFanReady);
  const unsigned long long* done = work_ctr(a, epoch, kWorkFanDone);
  V* act = reinterpret_cast<V*>(a.peer[a.rank] + act_off);
  const int2* dq = reinterpret_cast<const int2*>(a.peer[a.rank] + a.off_dupq);
  const long long per_block = (long long)a.blk * (a.K - 1);
  unsigned long long seen = 0;  // last published word read by this warp
  uint32_t k = 0;               // job of the previous unit (units are claimed in increasing order)
  // balancer on: groups claimed dynamically; off: static striding over every warp
  const unsigned long long wid = (unsigned long long)blockIdx.x * warps_per_cta + (threadIdx.x >> 5);
  const unsigned long long nwk = (unsigned long long)gridDim.x * warps_per_cta;
  unsigned long long grp = wid;
  for (;; grp += nwk) {
    // small batches (a.fan_split: uniform 4 KB slice units, fewer than the
    // warps) stride statically: a claim atomic per group would serialise
    // ~1.5k claims on one address behind the block's arrival
    const unsigned long long g0 =
        ((a.balance && !a.fan_split) ? (unsigned long long)claim_warp(ctr) : grp) * kFanGroup;
    for (int gi = 0; gi < kFanGroup; ++gi) {
      const unsigned long long u = g0 + gi;
      // wait until the published prefix covers u (or every job is in)
      unsigned backoff = 64;
      unsigned long long tw = 0;
      while (u >= (seen & kUnitMask)) {
        // lane 0 polls (with backoff: thousands of warps may wait here).
        // a.fan_poll: one warp per CTA at a time reads the global words and
        // caches them in shared memory; the CTA's other waiting warps read
        // the cache (one L2 poller per CTA instead of one per warp)
        unsigned long long w = 0, d = 0;
        if (lane == 0) {
          if (a.fan_poll) {
            volatile FanPoll* fp = fan_poll_sm();
            w = fp->seen;
            d = fp->done;
            if (u >= (w & kUnitMask) && !d && atomicCAS(const_cast<int*>(&fp->lock), 0, 1) == 0) {
              d = ld_acquire_gpu_u64(done);
              w = ld_acquire_gpu_u64(ready);
              if (w > fp->seen) fp->seen = w;
              fp->done = d;
              __threadfence_block();
              atomicExch(const_cast<int*>(&fp->lock), 0);
            }
            __threadfence_block();
          } else {
            d = ld_acquire_gpu_u64(done);
            w = ld_acquire_gpu_u64(ready);
          }
        }
        w = __shfl_sync(kFull, w, 0);
        d = __shfl_sync(kFull, d, 0);
        seen = w;
        if (u < (seen & kUnitMask)) break;
        if (d) return;  // final prefix read after `done`: u is past the last unit
        // bounded like every wait (the watcher itself gives up after timeout_ns)
        if (tw == 0) {
          tw = globaltimer();
        } else if (globaltimer() - tw > 2 * a.timeout_ns) {
          if (lane == 0) record_error(a.status, FS_ETIMEOUT, kSiteDispWorker);
          return;
        }
        __nanosleep(backoff);
        backoff = backoff < 1024 ? backoff * 2 : 1024;
      }
      // job holding u: first k' >= k with jcum[k'] > u (lane-parallel window)
      const uint32_t npub = (uint32_t)(seen >> 40);
      while (k < npub) {
        const uint32_t kk = k + lane;
        const bool past = kk < npub && __ldcg(a.fan_jcum + kk) > u;
        const uint32_t m = __ballot_sync(kFull, past);
        if (m) {
          k += __ffs(m) - 1;
          break;
        }
        k += 32;
      }
      if (k >= npub) {  // cannot happen (jcum[npub-1] is the published total > u): fail loudly, never spin
        if (lane == 0) record_error(a.status, FS_ERANGE, kSiteDispSchedule);
        return;
      }
      const unsigned long long base = k ? __ldcg(a.fan_jcum + k - 1) : 0ull;
      const uint32_t jo = __ldcg(a.fan_jorder + k);
      const int q = (int)(jo >> 16), b = (int)(jo & 0xffffu);
      const int ju = (int)(u - base);
      const int entry = ju / fs, part = ju - entry * fs;  // the job's duplicate row, and its slice (fs > 1)
      const int2 rp = __ldcg(dq + (size_t)q * a.dupq_cap + (size_t)b * per_block + entry);
      if (rp.x < 0 || rp.x >= a.max_rows || rp.y < 0 || rp.y >= a.max_rows) {
        if (lane == 0) record_error(a.status, FS_ERANGE, kSiteRows);
        continue;
      }
      // the whole row slice by slice, or the unit's one slice
      const V* src = act + (size_t)rp.y * nv;
      V* dst = act + (size_t)rp.x * nv;
      const int wb = fs > 1 ? part * SW : 0, we = fs > 1 ? min(nv, wb + SW) : nv;
      for (int w0 = wb; w0 < we; w0 += SW) {
        const int rem = nv - w0;
        V v[U];
#pragma unroll
        for (int jj = 0; jj < U; ++jj)
          if (jj * 32 + lane < rem) v[jj] = ld_cg(src + w0 + jj * 32 + lane);
#pragma unroll
        for (int jj = 0; jj < U; ++jj)
          if (jj * 32 + lane < rem) st_na(dst + w0 + jj * 32 + lane, v[jj]);
      }
    }
  }
}

#ifndef FUSCO_DISP_MINB
#define FUSCO_DISP_MINB 3  // CTAs per SM the register budget is cut for
#endif
template <typename V>
__global__ void __launch_bounds__(kMoveThreads, FUSCO_DISP_MINB)
    dispatch_kernel(FsArgs a, const V* __restrict__ x, const void* __restrict__ idx,
                    const int32_t* __restrict__ row_of, int phase) {
  TraceLast trace_last_(a, FS_TRACE_DISPATCH_LAST);
  constexpr int U = MoveCfg<V>::U;
  constexpr int SW = MoveCfg<V>::kSliceWords;
  const int K = a.K, T = a.T, P = a.world, s = a.rank;
  const int nv = a.tb / (int)sizeof(V);
  const int S = (nv + SW - 1) / SW;
  const int lane = threadIdx.x & 31;
  const int wcta = threadIdx.x >> 5;
  constexpr int kWarps = kMoveThreads / 32;
  // roles: CTA 0's last warp watches the block words; warps below push_warps
  // push first; the others fan out from the start (LOCAL-only launches: all push)
  const bool remote = (phase & FS_PHASE_REMOTE) && P > 1;
  const bool watcher = remote && blockIdx.x == 0 && wcta == kWarps - 1;
  const bool pusher = (phase & FS_PHASE_LOCAL) && !watcher && (!remote || wcta < a.push_warps);
  __shared__ int32_t owner_sm[kMaxExperts];
  if (phase & FS_PHASE_REMOTE) fan_poll_init();
  if (phase & FS_PHASE_LOCAL) load_owner_table(a, owner_sm);  // static table: before the PDL wait
  const uint32_t uS = (uint32_t)S;
  const long long units = (long long)T * S;
  // pushing warps and this warp's static index among them
  const int npw = remote ? a.push_warps : kWarps;
  const bool wexcl = remote && a.push_warps == kWarps;  // CTA 0's last warp watches instead
  const long long pidx = (long long)blockIdx.x * npw + wcta - ((wexcl && blockIdx.x > 0) ? 1 : 0);
  const long long pnum = (long long)gridDim.x * npw - (wexcl ? 1 : 0);
  // Small batches (every pushing warp has at most one unit, e.g. decode):
  // static assignment, no claim atomic, and the unit's payload rows and
  // expert ids -- inputs, not planner outputs -- are loaded before the PDL
  // wait, so they stream in while the planner finishes.  Only row_of waits.
  const bool small = pusher && units <= pnum;
  V v[U];
  KMeta cur{0, -1};
  if (small && pidx < units) {
    const int i = (int)((uint32_t)pidx / uS), sl = (int)((uint32_t)pidx - (uint32_t)i * uS);
    const int w0 = sl * SW, rem = nv - w0;
#pragma unroll
    for (int j = 0; j < U; ++j)
      if (j * 32 + lane < rem) v[j] = ld_nc(x + (size_t)i * nv + w0 + j * 32 + lane);
    if (lane < K) {
      const long long e = load_idx(idx, (size_t)i * K + lane, a.idx64);
      cur.e = (e < 0 || e >= a.E) ? 0 : (int)e;
    }
  }
  griddep_wait();  // row_of / the epoch come from the planner
  const uint32_t epoch = load_epoch(a);
  const size_t act_off = a.off_act;
  trace_stamp(a, FS_TRACE_DISPATCH_BEGIN);

  // One unit (token i, slice sl) whose payload is in v and whose k-th expert
  // (and destination row) lane k holds in m: resolve destinations, list
  // duplicates, store.  Returns the unit's completion block.
  auto push_unit = [&](int i, int sl, const KMeta& m) -> int {
    const int w0 = sl * SW, rem = nv - w0;
    // destinations of the token (lane k < K: owner and row of its k-th expert)
    int g = -1 - lane, r = -1;  // lanes >= K get unique negative keys
    if (lane < K) {
      g = owner_sm[m.e];
      r = (m.r < 0 || m.r >= a.max_rows) ? -1 : m.r;
    }
    const uint32_t same = __match_any_sync(kFull, g);
    const int first_lane = __ffs(same) - 1;
    const int r_first = __shfl_sync(kFull, r, first_lane);
    const bool direct = lane < K && r >= 0 && (a.nodedup || first_lane == lane || g == s);
    const uint32_t dmask = __ballot_sync(kFull, direct);
    const int b = i / a.blk;
    // a further row of the token on an already-reached rank: listed for the
    // receiver's fan-out instead of crossing the link again
    if (P > 1 && sl == 0 && lane < K && r >= 0 && !direct && r_first >= 0)
      list_duplicate(a, epoch, g, b, r, r_first);
    // pre-reduction record for the owner of >= 2 of the token's rows (the
    // combine decides whether the group is large enough to pre-reduce); plain
    // stores, published with the unit's block like the rows themselves
    if (a.disp_w != nullptr && sl == 0 && lane < K && g != s && __popc(same) >= 2) {
      GrpRec* rec = reinterpret_cast<GrpRec*>(a.peer[g] + a.off_grp) + (size_t)s * a.max_tokens + i;
      const size_t wi = (size_t)i * K + lane;
      rec->rows[lane] = r;
      rec->w[lane] = a.disp_w64 ? (float)reinterpret_cast<const double*>(a.disp_w)[wi]
                                : reinterpret_cast<const float*>(a.disp_w)[wi];
      if (lane == first_lane) {
        rec->kmask = same;
        rec->epoch = epoch;
      }
    }
    // Rotate the destination order by token so concurrent warps of this
    // rank spread their first stores over different peers.
    const int rot = a.balance ? (i + s) % K : 0;
    uint32_t mm = (dmask >> rot) | (rot ? (dmask << (32 - rot)) : 0u);
    while (mm) {
      const int d0 = __ffs(mm) - 1;
      mm &= mm - 1;
      const int d = (d0 + rot) & 31;
      const int gd = __shfl_sync(kFull, g, d);
      const int rd = __shfl_sync(kFull, r, d);
      V* dst = reinterpret_cast<V*>(a.peer[gd] + act_off) + (size_t)rd * nv + w0;
#pragma unroll
      for (int j = 0; j < U; ++j)
        if (j * 32 + lane < rem) st_na(dst + j * 32 + lane, v[j]);
    }
    return b;
  };

  // pushing warps of this CTA (CTA 0's last warp watches at P > 1) and the
  // CTA's first static unit
  const int rcta = (wexcl && blockIdx.x == 0) ? kWarps - 1 : npw;
  const long long cta_first = pidx - wcta;
  // Completion accounting per CTA round (a.push_rounds, FUSCO_PUSH_ROUNDS=1):
  // the CTA's pushing warps each push one unit of a run of rcta consecutive
  // units, meet at a named barrier, and thread 0 counts the run into its (at
  // most two) blocks with one acq_rel atomic each -- the release that orders
  // the round's peer stores before the count (cumulative over the barrier).
  // Measured against the default per-unit count (the per-warp loop below):
  // 1-2 % slower at large batches (the barrier waits for the round's slowest
  // warp), equal at decode -- the per-unit release is not what bounds the push.
  // Thread 0 checks a round's counts one round later (pending arrays).
  int pb[2] = {-1, -1};
  uint32_t pc[2] = {0, 0}, pt[2] = {0, 0};
  auto count_run = [&](long long base, int n) {  // thread 0: count units [base, base + n)
    if (n <= 0) return;
    for (int q = 0; q < 2; ++q)
      if (pb[q] >= 0 && pc[q] == pt[q]) block_complete(a, epoch, pb[q]);
    pb[0] = pb[1] = -1;
    long long u0 = base;
    const long long u1 = base + n;
    for (int q = 0; q < 2 && u0 < u1; ++q) {
      const int b = (int)((uint32_t)u0 / uS) / a.blk;
      const long long bend = (long long)(b + 1) * a.blk * S;
      const uint32_t c = (uint32_t)((u1 < bend ? u1 : bend) - u0);
      pc[q] = block_count(a, epoch, b, c) + c;
      pt[q] = (uint32_t)(min(a.blk, T - b * a.blk) * S);
      pb[q] = b;
      u0 += c;
    }
  };
  auto finish_runs = [&]() {
    for (int q = 0; q < 2; ++q)
      if (pb[q] >= 0 && pc[q] == pt[q]) block_complete(a, epoch, pb[q]);
  };
  auto pusher_bar = [&]() { asm volatile("bar.sync 2, %0;" ::"r"(rcta * 32) : "memory"); };

  if (small) {
    // one round: this CTA's units [cta_first, cta_first + rcta)
    if (pidx < units) {
      const int i = (int)((uint32_t)pidx / uS), sl = (int)((uint32_t)pidx - (uint32_t)i * uS);
      if (lane < K) cur.r = row_of[(size_t)i * K + lane];
      const int b = push_unit(i, sl, cur);
      if (P > 1 && !a.push_rounds) {
        __syncwarp();
        if (lane == 0) block_units_done(a, epoch, b, 1u, (uint32_t)(min(a.blk, T - b * a.blk) * S));
      }
    }
    if (P > 1 && a.push_rounds) {
      pusher_bar();
      if (threadIdx.x == 0) {
        count_run(cta_first, (int)min((long long)rcta, units - cta_first));
        finish_runs();
      }
    }
  } else if (pusher && a.push_rounds) {
    __shared__ long long rbase[3];  // round bases, claimed two rounds ahead (triple buffer)
    unsigned long long* ctr = work_ctr(a, epoch, kWorkDispatch);
    const bool dyn = a.balance != 0;
    auto round_base = [&](long long r) -> long long {  // static striding: the CTA's r-th run
      return cta_first + r * pnum;
    };
    if (threadIdx.x == 0 && dyn) {
      rbase[0] = (long long)atomicAdd(ctr, (unsigned long long)rcta);
      rbase[1] = (long long)atomicAdd(ctr, (unsigned long long)rcta);
    }
    pusher_bar();
    long long base = dyn ? rbase[0] : round_base(0);
    long long nbase = dyn ? rbase[1] : round_base(1);
    KMeta nxt = base + wcta < units ? load_meta(a, idx, row_of, (int)((uint32_t)(base + wcta) / uS), lane)
                                    : KMeta{0, -1};
    for (long long r = 0; base < units; ++r) {
      unsigned long long claim = 0;
      if (threadIdx.x == 0 && dyn) claim = atomicAdd(ctr, (unsigned long long)rcta);  // round r + 2
      const long long u = base + wcta;
      cur = nxt;
      if (nbase + wcta < units) nxt = load_meta(a, idx, row_of, (int)((uint32_t)(nbase + wcta) / uS), lane);
      if (u < units) {
        const int i = (int)((uint32_t)u / uS), sl = (int)((uint32_t)u - (uint32_t)i * uS);
        const int w0 = sl * SW, rem = nv - w0;
#pragma unroll
        for (int j = 0; j < U; ++j)
          if (j * 32 + lane < rem) v[j] = ld_nc(x + (size_t)i * nv + w0 + j * 32 + lane);
        push_unit(i, sl, cur);
      }
      if (threadIdx.x == 0 && dyn) rbase[(r + 2) % 3] = (long long)claim;
      pusher_bar();  // the round's stores are issued; rbase[(r + 2) % 3] is visible
      if (P > 1 && threadIdx.x == 0) count_run(base, (int)min((long long)rcta, units - base));
      base = nbase;
      nbase = dyn ? rbase[(r + 2) % 3] : round_base(r + 2);
    }
    if (P > 1 && threadIdx.x == 0) finish_runs();
  } else if (pusher) {
    // Per-warp loop (default).  Work unit = (token, slice).  Per
    // iteration: claim the next unit and load its (expert, row) metadata
    // while this unit's payload streams in; resolve destinations; store;
    // count the unit into its completion block.  Lane 0 checks the count's
    // returned value one unit later.  Measured (tools/push_probe.py, Mixtral
    // EP=2): a loop that also deferred the claim and issued the payload loads
    // first was 10% slower, an immediate completion check 8%.
    unsigned long long* ctr = work_ctr(a, epoch, kWorkDispatch);
    // balancer on: units claimed dynamically (warps that drew light tokens
    // take more); off: static striding over the pushing warps
    const bool dyn = a.balance != 0;
    long long u = dyn ? claim_warp(ctr) : pidx;
    KMeta nxt = u < units ? load_meta(a, idx, row_of, (int)((uint32_t)u / uS), lane) : KMeta{0, -1};
    int pend_b = -1;  // lane 0: block of the previous unit, its count after the add, the block's total
    uint32_t pend_cnt = 0, pend_total = 0;
    while (u < units) {
      const int i = (int)((uint32_t)u / uS);
      const int sl = (int)((uint32_t)u - (uint32_t)i * uS);
      cur = nxt;
      const long long un = dyn ? claim_warp(ctr) : u + pnum;
      if (un < units) nxt = load_meta(a, idx, row_of, (int)((uint32_t)un / uS), lane);
      const int w0 = sl * SW, rem = nv - w0;
#pragma unroll
      for (int j = 0; j < U; ++j)
        if (j * 32 + lane < rem) v[j] = ld_nc(x + (size_t)i * nv + w0 + j * 32 + lane);
      const int b = push_unit(i, sl, cur);
      if (P > 1) {
        __syncwarp();
        if (lane == 0) {
          // the previous unit completed its block?  (the add returned long ago)
          if (pend_b >= 0 && pend_cnt == pend_total) block_complete(a, epoch, pend_b);
          pend_cnt = block_count(a, epoch, b, 1u) + 1u;
          pend_total = (uint32_t)(min(a.blk, T - b * a.blk) * S);
          pend_b = b;
        }
      }
      u = un;
    }
    if (P > 1 && lane == 0 && pend_b >= 0 && pend_cnt == pend_total) block_complete(a, epoch, pend_b);
  }
  griddep_launch_dependents();  // the combine may start its prologue
  trace_stamp(a, FS_TRACE_DISPATCH_PUSHED);
  if (remote) {
    if (watcher) fan_watch(a, epoch, fan_units_per_row<V>(a, nv));
    fan_work<V>(a, epoch, act_off, nv, kWarps);
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
                        const int32_t* __restrict__ row_of, int phase, int nslots, int whole, int ns, int sb) {
  TraceLast trace_last_(a, FS_TRACE_DISPATCH_LAST);
  extern __shared__ __align__(128) char tsm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(tsm);
  uint64_t* empty = full + kTmaMaxSlots;
  char* ring = tsm + 2 * kTmaMaxSlots * sizeof(uint64_t);
  const int K = a.K, T = a.T, P = a.world, s = a.rank, tb = a.tb;
  const int slot_bytes = tma_slot_bytes(tb);  // slots hold whole rows (host: tma_smem)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // Work units: tokens [0, whole) are whole rows, tokens [whole, T) are cut
  // into ns column slices of sb bytes (the last one shorter).  Default: all
  // whole rows (whole = T).  FUSCO_TMA_TAIL=1 sets whole = the full rounds of
  // the strided assignment so only the last, partial round is sliced over
  // the grid; FUSCO_TMA_SLICES=n slices every row.  Both measured no faster
  // (DESIGN.md §10): the engine is latency-bound per CTA.
  const int units = whole + (T - whole) * ns;
  struct Unit {
    int i;          // token
    uint32_t off;   // byte offset in the row
    uint32_t len;   // bytes
  };
  auto unit_of = [&](int u) -> Unit {
    if (u < whole) return Unit{u, 0u, (uint32_t)tb};
    const int r = u - whole;
    const int i = whole + r / ns, sl = r - (r / ns) * ns;
    return Unit{i, (uint32_t)(sl * sb), (uint32_t)min(sb, tb - sl * sb)};
  };
  // units of completion block b (P > 1 accounting)
  auto block_units = [&](int b) -> uint32_t {
    const int t0 = b * a.blk, t1 = min(T, t0 + a.blk);
    const int w = max(0, min(t1, whole) - t0);
    return (uint32_t)(w + (t1 - t0 - w) * ns);
  };
  __shared__ int32_t owner_tma[kMaxExperts];
  // Prologue independent of the planner (launched with PDL behind it): barrier
  // init, expert table, and the first ring-full of token slices streaming in.
  if ((phase & FS_PHASE_LOCAL) && threadIdx.x == 0) {
    for (int q = 0; q < nslots; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], 1);
    }
    mbar_fence_init();
  }
  if (phase & FS_PHASE_REMOTE) fan_poll_init();
  if (phase & FS_PHASE_LOCAL) load_owner_table(a, owner_tma);
  if ((phase & FS_PHASE_LOCAL) && threadIdx.x == 0) {
    int n = 0;
    for (int u = blockIdx.x; u < units && n < nslots; u += gridDim.x, ++n) {
      const Unit w = unit_of(u);
      mbar_arrive_expect_tx(&full[n], w.len);
      bulk_load(ring + (size_t)n * slot_bytes, x + (size_t)w.i * tb + w.off, w.len, &full[n]);
    }
  }
  griddep_wait();  // row_of / the epoch come from the planner
  const uint32_t epoch = load_epoch(a);
  const size_t act_off = a.off_act;
  trace_stamp(a, FS_TRACE_DISPATCH_BEGIN);
  const bool remote = (phase & FS_PHASE_REMOTE) && P > 1;

  if ((phase & FS_PHASE_LOCAL) && warp < 2) {
    if (warp == 0) {
      if (lane == 0) {  // producer (the first nslots units were issued in the prologue)
        int n = 0;
        for (int u = blockIdx.x; u < units; u += gridDim.x, ++n) {
          if (n < nslots) continue;
          const int q = n % nslots;
          const Unit w = unit_of(u);
          mbar_wait_bounded(&empty[q], ((n / nslots) & 1) ^ 1, a, kSiteDispatchPipe);
          mbar_arrive_expect_tx(&full[q], w.len);
          bulk_load(ring + (size_t)q * slot_bytes, x + (size_t)w.i * tb + w.off, w.len, &full[q]);
        }
      }
    } else if (warp == 1) {  // destinations + bulk stores
      int n = 0;
      KMeta nxt = (int)blockIdx.x < units ? load_meta(a, idx, row_of, unit_of(blockIdx.x).i, lane) : KMeta{0, -1};
      for (int u = blockIdx.x; u < units; u += gridDim.x, ++n) {
        const int q = n % nslots;
        const Unit w = unit_of(u);
        const int i = w.i;
        const KMeta cur = nxt;
        if (u + (int)gridDim.x < units) nxt = load_meta(a, idx, row_of, unit_of(u + gridDim.x).i, lane);
        int g = -1 - lane, r = -1;
        if (lane < K) {
          g = owner_tma[cur.e];
          r = (cur.r < 0 || cur.r >= a.max_rows) ? -1 : cur.r;
        }
        const uint32_t same = __match_any_sync(kFull, g);
        const int first_lane = __ffs(same) - 1;
        const int r_first = __shfl_sync(kFull, r, first_lane);
        const bool direct = lane < K && r >= 0 && (a.nodedup || first_lane == lane || g == s);
        if (P > 1 && w.off == 0 && lane < K && r >= 0 && !direct && r_first >= 0)
          list_duplicate(a, epoch, g, i / a.blk, r, r_first);
        mbar_wait_bounded(&full[q], (n / nslots) & 1, a, kSiteDispatchPipe);
        // each destination lane issues its own bulk store (per-thread bulk
        // groups); every lane commits one group per unit so the lag below
        // counts units on all lanes
        if (direct)
          bulk_store(a.peer[g] + act_off + (size_t)r * tb + w.off, ring + (size_t)q * slot_bytes, w.len);
        bulk_commit();
        bulk_wait_read<LAG>();
        __syncwarp();
        if (lane == 0 && n >= LAG) mbar_arrive(&empty[(n - LAG) % nslots]);
      }
      bulk_wait<0>();
      fence_proxy_async_global();
    }
    if (P > 1) {
      // every bulk store of this CTA is complete: count its units into their
      // blocks (units are strided over the grid, so the blocks complete when
      // the last CTA gets here)
      asm volatile("bar.sync 1, 64;" ::: "memory");  // warps 0-1 only: the others may be fanning out
      if (threadIdx.x == 0) {
        auto flush = [&](int b, uint32_t n) {
          block_units_done(a, epoch, b, n, block_units(b));
        };
        int b_cur = -1;
        uint32_t cnt = 0;
        for (int u = blockIdx.x; u < units; u += gridDim.x) {
          const int b = unit_of(u).i / a.blk;
          if (b != b_cur) {
            if (cnt) flush(b_cur, cnt);
            b_cur = b;
            cnt = 0;
          }
          ++cnt;
        }
        if (cnt) flush(b_cur, cnt);
      }
    }
  }
  griddep_launch_dependents();  // the combine may start its prologue

  trace_stamp(a, FS_TRACE_DISPATCH_PUSHED);
  if (remote) {  // watcher: CTA 0's warp 3; every warp fans out once it has no push work
    if (blockIdx.x == 0 && warp == 3) fan_watch(a, epoch, fan_units_per_row<int4>(a, tb / 16));
    fan_work<int4>(a, epoch, act_off, tb / 16, kTmaThreads / 32);
  }
  trace_stamp(a, FS_TRACE_DISPATCH_END);
}

}  // namespace fusco
