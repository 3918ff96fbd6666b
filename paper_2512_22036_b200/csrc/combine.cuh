// combine.cuh — the pull combine with the k-ordered weighted reduction (fs_combine)
#pragma once
#include <cooperative_groups.h>

#include "dispatch.cuh"

namespace fusco {
namespace cg = cooperative_groups;

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
// Owner-side pre-reduction (combine LOCAL phase, a.reduce): for every record a
// source wrote into this rank's region this epoch (dispatch_kernel) with at
// least mmin rows here, the partial Σ_{k in group, ascending} w_k · y[row_k]
// in fp32 goes to the partial slot [source][token] of this rank's region
// (2·tb bytes: fp32 of the hidden dim).  Every warp of the grid takes
// (source, token) slots in turn; lanes stride the 16-byte column chunks.
// ===========================================================================
template <bool BF16>
__device__ void owner_prereduce(const FsArgs& a, uint32_t epoch, size_t src_off, int mmin) {
  using EL = Elem<int4, BF16>;
  constexpr int kCh = 2;  // 16-byte column chunks per lane per item (loaded together below)
  const int P = a.world, s = a.rank, K = a.K, tb = a.tb, nv = tb / 16;
  const int lane = threadIdx.x & 31;
  const int par = (int)(epoch & 1u);
  const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  const char* src = a.peer[s] + src_off;
  const GrpRec* recs = reinterpret_cast<const GrpRec*>(a.peer[s] + a.off_grp);
  char* part = a.peer[s] + a.off_part;
  // Work items = (source q != s, token t < T_q, column part of 32 * kCh
  // chunks).  Measured: a warp per whole 14 KB row walks it chunk after
  // chunk, latency-bound (DeepSeek-V3 EP=2 step 460 vs 412 us); column parts
  // keep ~kCh x 4 loads per lane in flight.  T_q: the sources' token counts
  // this epoch (count words, complete since the planner), prefix over
  // sources in lane q, so no slot of the own rank or beyond T_q is visited.
  int tq = 0;
  if (lane < P && lane != s) tq = read_count_word(a, par, epoch, lane, a.E);
  int incl = tq;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int n = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += n;
  }
  const int t_total = __shfl_sync(kFull, incl, 31);
  const int parts = (nv + 32 * kCh - 1) / (32 * kCh);
  const int cols_per_part = 32 * kCh;  // 16-byte chunks of one item
  const long long items = (long long)t_total * parts;
  for (long long it = gw; it < items; it += nw) {
    const int gt = (int)(it / parts), pc = (int)(it - (long long)gt * parts);
    // source holding global token index gt: first lane whose inclusive prefix exceeds gt
    const uint32_t past = __ballot_sync(kFull, lane < P && incl > gt);
    const int q = __ffs(past) - 1;
    const int t = gt - (__shfl_sync(kFull, incl, q) - __shfl_sync(kFull, tq, q));
    const long long slot = (long long)q * a.max_tokens + t;
    const GrpRec* rec = recs + slot;
    // the whole record in one round trip: every lane the header, lane k < K
    // its row and weight (used only where the k-mask has the bit)
    const uint32_t e = __ldcg(&rec->epoch), km = __ldcg(&rec->kmask);
    int rk = 0;
    float wk = 0.f;
    if (lane < K) {
      rk = __ldcg(&rec->rows[lane]);
      wk = __ldcg(&rec->w[lane]);
    }
    if (e != epoch || __popc(km) < mmin) continue;
    if (lane < K && ((km >> lane) & 1u) && (rk < 0 || rk >= a.max_rows)) {
      record_error(a.status, FS_ERANGE, kSiteRows);
      rk = 0;
    }
    int rr[kGrpMaxK];
    float ww[kGrpMaxK];
#pragma unroll
    for (int k = 0; k < kGrpMaxK; ++k) {  // every lane takes part (before the column loop)
      rr[k] = __shfl_sync(kFull, rk, k);
      ww[k] = __shfl_sync(kFull, wk, k);
    }
    char* dst = part + (size_t)slot * 2 * tb;
    // the part's two chunks per lane: both chunks' loads of four rows in
    // flight together (a group rarely has more than four rows)
    const int va = pc * 32 * kCh + lane, vb = va + 32;
    const bool ha = va < nv, hb = vb < nv;
    float acc_a[EL::N], acc_b[EL::N];
#pragma unroll
    for (int e2 = 0; e2 < EL::N; ++e2) acc_a[e2] = acc_b[e2] = 0.f;
#pragma unroll
    for (int k0 = 0; k0 < kGrpMaxK; k0 += 4) {
      if (k0 > 0 && (km >> k0) == 0u) break;
      int4 xa[4], xb[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int k = k0 + j;
        xa[j] = xb[j] = make_int4(0, 0, 0, 0);
        if (k < K && ((km >> k) & 1u)) {
          const int4* row = reinterpret_cast<const int4*>(src + (size_t)rr[k] * tb);
          if (ha) xa[j] = ld_nc(row + va);
          if (hb) xb[j] = ld_nc(row + vb);
        }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int k = k0 + j;
        if (k < K && ((km >> k) & 1u)) {
#pragma unroll
          for (int e2 = 0; e2 < EL::N; ++e2) {
            acc_a[e2] = __fmaf_rn(ww[k], EL::get(xa[j], e2), acc_a[e2]);
            acc_b[e2] = __fmaf_rn(ww[k], EL::get(xb[j], e2), acc_b[e2]);
          }
        }
      }
    }
#pragma unroll
    for (int c = 0; c < kCh; ++c) {
      const int v = c ? vb : va;
      if (!(c ? hb : ha)) break;
      const float* acc = c ? acc_b : acc_a;
      int4* o = reinterpret_cast<int4*>(dst) + (size_t)v * (EL::N / 4);
#pragma unroll
      for (int h = 0; h < EL::N / 4; ++h)
        st_na(o + h, make_int4(__float_as_int(acc[4 * h]), __float_as_int(acc[4 * h + 1]),
                               __float_as_int(acc[4 * h + 2]), __float_as_int(acc[4 * h + 3])));
    }
  }
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
__global__ void __launch_bounds__(kCombThreads, 3)  // 3 CTAs/SM (the stage budget assumes it)
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
  __shared__ int8_t slot_kind[kCombMaxStages][32];  // per stage and lane: 0 row, 1/2 partial halves, 3 none
  __shared__ int8_t slot_k2[kCombMaxStages][32];    // lane holding the partial's second half (bf16)
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

  // owner-side pre-reduction (fp32 accumulate only; bf16 rows: groups of >= 3,
  // whose fp32 partial is smaller than the rows; fp32 rows: groups of >= 2)
  const bool red = !ACC64 && a.reduce && P > 1;
  const int mmin = BF16 ? 3 : 2;
  if ((phase & FS_PHASE_LOCAL) && P > 1) {
    if (red) {
      owner_prereduce<BF16>(a, epoch, src_off, mmin);
      cg::this_grid().sync();  // every partial written before the "ready" release below
    }
    if (blockIdx.x == 0 && threadIdx.x < P) {
      if (red) reinterpret_cast<volatile uint32_t*>(a.peer[threadIdx.x] + kOffModeFlag)[s] = epoch;
      st_release_sys_u32(reinterpret_cast<uint32_t*>(a.peer[threadIdx.x] + kOffReadyFlag) + s, epoch);
    }
  }
  if (!remote) return;
  __shared__ uint32_t red_mask;  // owners whose partials this CTA pulls (this epoch)
  if (threadIdx.x == 0) red_mask = 0u;
  __syncthreads();
  if (P > 1 && threadIdx.x < P) {
    wait_u32_geq(reinterpret_cast<const uint32_t*>(a.peer[s] + kOffReadyFlag) + threadIdx.x, epoch, a);
    // the owner's mode word precedes its ready release: read after the acquire
    if (red && threadIdx.x != s &&
        reinterpret_cast<volatile const uint32_t*>(a.peer[s] + kOffModeFlag)[threadIdx.x] == epoch)
      atomicOr(&red_mask, 1u << threadIdx.x);
  }
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
    // balancer on: items claimed dynamically; off: static striding over the CTAs
    // (static striding also when there are no more items than producers x 2:
    // decode batches, where every claim would be one more serialised atomic)
    const bool dyn = a.balance != 0 && items > 2LL * gridDim.x;
    long long u = dyn ? claim_warp(ctr) : (long long)blockIdx.x;
    KMeta m = u < items ? load_meta(a, idx, row_of, (int)((uint32_t)u / (uint32_t)S), lane) : KMeta{0, 0};
    Acc wl = u < items ? load_w(u) : (Acc)0;
    int n = 0;
    for (;; ++n) {
      const int q = n % nstages;
      if (n >= nstages) mbar_wait_bounded(&empty[q], ((n / nstages) & 1) ^ 1, a, kSiteCombinePipe);
      if (u >= items) {  // sentinel: consumers stop at this stage
        if (lane == 0) {
          slot_item[q] = -1;
          mbar_arrive(&full[q]);
        }
        break;
      }
      const long long un = dyn ? claim_warp(ctr) : u + gridDim.x;  // claimed and prefetched while this item streams
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
      // Source side of the pre-reduction: a group of >= mmin of the token's
      // rows on an owner that pre-reduced is one fp32 partial slice (2·len
      // bytes for bf16, loaded as two halves into the slots of the group's
      // first two lanes); its other lanes load nothing.  kind: 0 row,
      // 1 partial (first half), 2 partial second half, 3 skipped.
      int kind = 0, second = 0;
      if (red_mask) {
        const uint32_t same = __match_any_sync(kFull, lane < K ? g : -1 - lane);
        const bool grp = lane < K && ((red_mask >> g) & 1u) && __popc(same) >= mmin;
        const int first = __ffs(same) - 1;
        second = __ffs(same & ~(1u << first)) - 1;
        kind = !grp ? 0 : (lane == first ? 1 : ((BF16 && lane == second) ? 2 : 3));
      }
      if (lane < K) {
        slot_kind[q][lane] = (int8_t)kind;
        slot_k2[q][lane] = (int8_t)second;
      }
      if (lane == 0) slot_item[q] = u;
      const uint32_t nb = (lane < K && kind != 3) ? (uint32_t)len : 0u;
      const uint32_t tx = __reduce_add_sync(kFull, nb);
      __syncwarp();
      if (lane == 0) mbar_arrive_expect_tx(&full[q], tx);
      __syncwarp();
      if (lane < K) {
        char* dstage = stages + (size_t)q * stage_bytes + (size_t)lane * sb;
        if (kind == 0) {
          bulk_load(dstage, a.peer[g] + src_off + (size_t)r * tb + off, (uint32_t)len, &full[q]);
        } else if (kind != 3) {
          const int i = (int)((uint32_t)u / (uint32_t)S);
          const char* pp = a.peer[g] + a.off_part + ((size_t)s * a.max_tokens + i) * 2 * tb + (BF16 ? 2 * off : off);
          bulk_load(dstage, pp + (kind == 2 ? len : 0), (uint32_t)len, &full[q]);
        }
      }
      u = un;
      m = mn;
      wl = wn;
    }
  } else {  // consumers
    const int ct = threadIdx.x - 32;  // 0 .. 32*kCombConsumers-1
    for (int n = 0;; ++n) {
      const int q = n % nstages;
      mbar_wait_bounded(&full[q], (n / nstages) & 1, a, kSiteCombinePipe);
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
          const int kd = slot_kind[q][k];
          if (kd == 0) {
            const Acc wk = slot_w[q][k];
            const int4 x = *reinterpret_cast<const int4*>(st + (size_t)k * sb + (size_t)v * 16);
#pragma unroll
            for (int e = 0; e < EL::N; ++e) acc[e] = fma_acc<Acc>(wk, EL::get(x, e), acc[e]);
          } else if (kd == 1) {  // fp32 partial of the owner's group, already weighted
            const int len = nv * 16;
            const int k2 = slot_k2[q][k];
#pragma unroll
            for (int h = 0; h < EL::N / 4; ++h) {
              const int pb = v * EL::N * 4 + h * 16;  // byte offset in the slice's fp32 partial
              const char* src = pb < len ? st + (size_t)k * sb + pb : st + (size_t)k2 * sb + (pb - len);
              const int4 f = *reinterpret_cast<const int4*>(src);
              acc[4 * h] += (Acc)__int_as_float(f.x);
              acc[4 * h + 1] += (Acc)__int_as_float(f.y);
              acc[4 * h + 2] += (Acc)__int_as_float(f.z);
              acc[4 * h + 3] += (Acc)__int_as_float(f.w);
            }
          }
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

}  // namespace fusco
