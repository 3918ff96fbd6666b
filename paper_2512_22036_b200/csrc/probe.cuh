// probe.cuh — copy-bandwidth probes (fs_probe_copy, fs_probe_a2a)
#pragma once
#include <cooperative_groups.h>

#include "dispatch.cuh"

namespace fusco {
namespace cg = cooperative_groups;

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
      if (w < n16) v[j] = src ? ld_nc(src + w) : make_int4((int)w, j, 0, 0);
    }
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const size_t w = w0 + j * 32 + lane;
      if (w < n16) st_na(dst + w, v[j]);
    }
  }
}

// Row-scatter probe: the P=1 dispatch's pattern (read a row once, write it to
// `fanout` scattered rows) with the engine's 16-byte warp moves, no metadata.
__global__ void __launch_bounds__(kMoveThreads)
    probe_scatter_kernel(int4* __restrict__ dst, const int4* __restrict__ src, const int32_t* __restrict__ perm,
                         int nrows, int fanout, int nv) {
  constexpr int U = 8;
  const int lane = threadIdx.x & 31;
  const long long gw = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = (gridDim.x * (long long)blockDim.x) >> 5;
  for (long long r = gw; r < nrows; r += nw) {
    for (int w0 = 0; w0 < nv; w0 += 32 * U) {
      int4 v[U];
#pragma unroll
      for (int j = 0; j < U; ++j) {
        const int w = w0 + j * 32 + lane;
        if (w < nv) v[j] = src ? ld_nc(src + r * nv + w) : make_int4(w, j, 0, 0);
      }
      for (int f = 0; f < fanout; ++f) {
        int4* d = dst + (size_t)perm[r * fanout + f] * nv;
#pragma unroll
        for (int j = 0; j < U; ++j) {
          const int w = w0 + j * 32 + lane;
          if (w < nv) st_na(d + w, v[j]);
        }
      }
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
