// fusco.cu — libfusco.so: the extern "C" boundary (include/fusco.h) around
// the sm_100a shuffle kernels.  Host code here only validates, keeps the
// per-rank handle, and launches; it never touches payload bytes.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "fusco_kernels.cuh"

using namespace fusco;

namespace {

constexpr int kMaxCtasPerSm = 8;
constexpr int kFanSplitTokens = 512;  // batches up to this size fan out slice by slice
thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define FS_CUDA(call)                                                                   \
  do {                                                                                  \
    cudaError_t _e = (call);                                                            \
    if (_e != cudaSuccess)                                                              \
      return fail(FS_ECUDA, std::string(#call) + ": " + cudaGetErrorString(_e));        \
  } while (0)

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

struct RegionLayout {
  size_t off_count, count_stride, off_blkflag, off_dupq, off_act, act_stride, off_actout, total;
  int blk, nbmax;
  long long dupq_cap;
  size_t off_grp, off_part;  // owner-side pre-reduction (0: not configured)
};

int blocks_per_source(int max_tokens) {
  const int blk = block_tokens(max_tokens);
  return std::max(1, (max_tokens + blk - 1) / blk);
}

// Owner-side pre-reduction buffers are part of the region when P > 1 and
// 2 <= K <= 8, unless FUSCO_OWNER_REDUCE=0 (read identically by
// fs_region_bytes and fs_create, so every rank sizes its region the same).
bool owner_reduce_configured(int world, int K) {
  const char* e = getenv("FUSCO_OWNER_REDUCE");
  if (e && std::string(e) == "0") return false;
  return world > 1 && K >= 2 && K <= kGrpMaxK;
}

RegionLayout region_layout(int world, int E, int K, int tb, int max_tokens, long long max_rows, int with_act_out) {
  RegionLayout L;
  L.blk = block_tokens(max_tokens);
  L.nbmax = blocks_per_source(max_tokens);
  L.dupq_cap = (long long)std::max(max_tokens, 0) * (K - 1);
  L.off_count = kSigBytes;
  // epoch-tagged words: E per-expert counts + the source's token count
  L.count_stride = align256((size_t)world * (E + 1) * sizeof(uint64_t));
  L.off_blkflag = L.off_count + 2 * L.count_stride;
  // block words [source][block] and duplicate lists [source][max_tokens * (K-1)]
  L.off_dupq = L.off_blkflag + align256((size_t)world * L.nbmax * sizeof(uint64_t));
  L.off_act = L.off_dupq + align256((size_t)world * (size_t)L.dupq_cap * sizeof(int2));
  L.act_stride = align256((size_t)max_rows * (size_t)tb);
  // one activation buffer: a rank's next dispatch cannot start before every
  // rank has published the next epoch's counts, i.e. finished this combine
  L.off_actout = L.off_act + L.act_stride;
  L.total = L.off_actout + (with_act_out ? L.act_stride : 0);
  L.off_grp = L.off_part = 0;
  if (owner_reduce_configured(world, K)) {
    L.off_grp = align256(L.total);
    L.off_part = L.off_grp + align256((size_t)world * std::max(max_tokens, 0) * sizeof(GrpRec));
    L.total = L.off_part + (size_t)world * std::max(max_tokens, 0) * 2 * (size_t)tb;
  }
  return L;
}

}  // namespace

struct fs_ctx {
  int rank, world, E, K, tb, max_tokens, with_act_out;
  long long max_rows;
  int device;
  int nloc;
  int layout_grid_max;  // cooperative capacity of the layout kernel
  int move_grid;        // dispatch persistent grid (equal on all ranks)
  int dispatch_tma;     // 1: TMA bulk-copy dispatch engine (FUSCO_DISPATCH=tma)
  int tma_slots;        // smem ring slots per CTA of the TMA engine
  int tma_lag, tma_ctas;
  int tma_sb;           // slot payload bytes (a whole row)
  int tma_slices;       // FUSCO_TMA_SLICES: > 0 cuts every row into this many slices (A/B)
  int tma_tail;         // 1: slice the last partial round's rows (FUSCO_TMA_TAIL=1)
  size_t tma_smem;
  int pdl;              // 1: programmatic dependent launch planner -> dispatch (FUSCO_PDL=0 disables)
  int pdl_multi;        // 1: PDL for the cooperative P > 1 movers too (FUSCO_PDL_MULTI=0 disables)
  int nodedup;          // 1: no per-rank dedup on dispatch (FUSCO_NODEDUP=1; planner ablation)
  int balance;          // 1: dynamic claiming + rotation (default); 0: static striding (balancer ablation)
  int cluster_layout;   // 1: single-cluster DSMEM planner usable (E <= 256, K <= 8)
  size_t cluster_smem;
  int combine_tma;      // 1: TMA combine engine (FUSCO_COMBINE=tma)
  int comb_sb, comb_stages, comb_grid;
  size_t comb_smem;
  int sms;
  int combine_grid_cap; // 0 = occupancy-derived
  size_t layout_smem;
  uint32_t epoch;
  int disp_phases;  // dispatch phases already enqueued in this epoch (each runs once)
  int comb_phases;  // combine phases already enqueued in this epoch (repeats reset the claim counter)
  unsigned long long timeout_ns;
  RegionLayout L;
  std::vector<char*> peers;
  int32_t *owner_d, *node_of_d, *perm_d, *seg_d, *chunk_cnt_d, *totals_d;
  long long* stat_part_d;
  int* status_d;
  int* num_rows_d;
  uint32_t* epoch_d;  // device iteration counter (graph-replay safe)
  unsigned long long* work_d;  // [2][8][kWorkStride] dynamic work counters
  uint32_t *blkdone_d, *dupcnt_d;  // [2][nbmax], [2][P][nbmax] dispatch block accounting (P > 1)
  unsigned long long* jcum_d;      // [P * nbmax] receiver fan-out schedule
  uint32_t* jorder_d;              // [P * nbmax]
  int push_warps;                  // warps per dispatch CTA that push before fanning out
  int recs_written;                // this epoch's dispatch wrote pre-reduction records (fs_dispatch_w)
  int owner_reduce_off;            // no pre-reduction buffers (FUSCO_OWNER_REDUCE=0, or P = 1, K > 8)
  int owner_reduce_force;          // FUSCO_OWNER_REDUCE=1: pre-reduce at every P and batch size
  int push_rounds;                 // FUSCO_PUSH_ROUNDS=1: per-CTA-round completion counts (A/B; default per unit)
  int fan_split;                   // FUSCO_FAN_SPLIT: -1 auto (by batch size), 0 rows, 1 slices
  int fan_poll;                    // FUSCO_FAN_POLL: 1 = per-CTA cached fan-out polling
  int dbg_relaxed;                 // FUSCO_DBG_BLK=1: unordered block counts (timing experiments only)
  int disp_ctas_per_sm;            // P > 1 warp-mover grid cap (0 = occupancy)
  unsigned long long* trace_d;  // FS_NTRACE stamps when FUSCO_TRACE=1, else null
};

namespace {

FsArgs make_args(const fs_ctx* h, int T, int idx64) {
  FsArgs a;
  memset(&a, 0, sizeof(a));
  a.rank = h->rank;
  a.world = h->world;
  a.E = h->E;
  a.K = h->K;
  a.tb = h->tb;
  a.T = T;
  a.idx64 = idx64;
  a.nodedup = h->nodedup;
  a.balance = h->balance;
  a.epoch_ptr = h->epoch_d;
  a.max_rows = h->max_rows;
  a.owner = h->owner_d;
  a.node_of = h->node_of_d;
  a.perm = h->perm_d;
  a.seg_begin = h->seg_d;
  for (int g = 0; g < h->world; ++g) a.peer[g] = h->peers[g];
  a.off_count = h->L.off_count;
  a.off_blkflag = h->L.off_blkflag;
  a.off_dupq = h->L.off_dupq;
  a.off_act = h->L.off_act;
  a.off_actout = h->L.off_actout;
  a.count_stride = h->L.count_stride;
  a.act_stride = h->L.act_stride;
  a.blk = h->L.blk;
  a.off_grp = h->L.off_grp;
  a.off_part = h->L.off_part;
  a.max_tokens = h->max_tokens;
  a.nbmax = h->L.nbmax;
  a.dupq_cap = h->L.dupq_cap;
  a.push_warps = h->push_warps;
  a.dbg_relaxed = h->dbg_relaxed;
  a.fan_poll = h->fan_poll;
  a.push_rounds = h->push_rounds;
  a.blkdone = h->blkdone_d;
  a.dupcnt = h->dupcnt_d;
  a.fan_jcum = h->jcum_d;
  a.fan_jorder = h->jorder_d;
  a.chunk_cnt = h->chunk_cnt_d;
  a.totals = h->totals_d;
  a.stat_part = h->stat_part_d;
  a.status = h->status_d;
  a.num_rows = h->num_rows_d;
  a.timeout_ns = h->timeout_ns;
  a.trace = h->trace_d;
  a.work = h->work_d;
  return a;
}

int check_idx_bytes(int idx_bytes) {
  if (idx_bytes != 4 && idx_bytes != 8) return fail(FS_EINVAL, "idx_bytes must be 4 or 8");
  return FS_OK;
}

bool aligned(const void* p, size_t n) { return (reinterpret_cast<uintptr_t>(p) % n) == 0; }

template <typename Kern>
int occupancy(Kern kernel, int threads, size_t smem, int* out) {
  FS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, kernel, threads, smem));
  return FS_OK;
}

// Launch with optional cooperative (co-residency for cross-CTA waits) and
// programmatic-dependent-launch attributes (the kernel's prologue overlaps the
// previous kernel's tail; every kernel griddep_wait()s before reading its
// predecessor's outputs).
int launch_ex(const void* fn, int grid, int block, size_t smem, void* stream, void** args, bool coop, bool pdl) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[2];
  int n = 0;
  if (coop) {
    attr[n].id = cudaLaunchAttributeCooperative;
    attr[n].val.cooperative = 1;
    ++n;
  }
  if (pdl) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  FS_CUDA(cudaLaunchKernelExC(&cfg, fn, args));
  return FS_OK;
}

}  // namespace

extern "C" {

int fs_abi_version(void) { return FS_ABI_VERSION; }

const char* fs_last_error(void) { return g_err.c_str(); }

int fs_region_bytes(int world, int num_experts, int topk, int token_bytes, int max_tokens, long long max_rows,
                    int with_act_out, size_t* bytes_out) {
  if (!bytes_out || world < 1 || world > FS_MAX_RANKS || num_experts < 1 || topk < 1 || token_bytes <= 0 ||
      max_tokens < 0 || max_rows < 0)
    return fail(FS_EINVAL, "fs_region_bytes: bad arguments");
  *bytes_out = region_layout(world, num_experts, topk, token_bytes, max_tokens, max_rows, with_act_out).total;
  return FS_OK;
}

int fs_sym_alloc(int device, size_t bytes, void** ptr_out) {
  if (!ptr_out || bytes == 0) return fail(FS_EINVAL, "fs_sym_alloc: bad arguments");
  FS_CUDA(cudaSetDevice(device));
  void* p = nullptr;
  FS_CUDA(cudaMalloc(&p, bytes));
  FS_CUDA(cudaMemset(p, 0, bytes));
  FS_CUDA(cudaDeviceSynchronize());
  *ptr_out = p;
  return FS_OK;
}

int fs_sym_free(int device, void* ptr) {
  FS_CUDA(cudaSetDevice(device));
  if (ptr) FS_CUDA(cudaFree(ptr));
  return FS_OK;
}

int fs_ipc_handle(int device, void* ptr, uint8_t* handle64_out) {
  if (!ptr || !handle64_out) return fail(FS_EINVAL, "fs_ipc_handle: bad arguments");
  FS_CUDA(cudaSetDevice(device));
  cudaIpcMemHandle_t h;
  static_assert(sizeof(h) == 64, "CUDA IPC handle is 64 bytes");
  FS_CUDA(cudaIpcGetMemHandle(&h, ptr));
  memcpy(handle64_out, &h, 64);
  return FS_OK;
}

int fs_ipc_open(int device, const uint8_t* handle64, void** ptr_out) {
  if (!handle64 || !ptr_out) return fail(FS_EINVAL, "fs_ipc_open: bad arguments");
  FS_CUDA(cudaSetDevice(device));
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, 64);
  void* p = nullptr;
  FS_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  *ptr_out = p;
  return FS_OK;
}

int fs_enable_peer_access(int device, int peer_device) {
  if (device == peer_device) return FS_OK;
  FS_CUDA(cudaSetDevice(device));
  int can = 0;
  FS_CUDA(cudaDeviceCanAccessPeer(&can, device, peer_device));
  if (!can) return fail(FS_EINVAL, "fs_enable_peer_access: no peer access between these devices");
  cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return FS_OK;
  }
  FS_CUDA(e);
  return FS_OK;
}

int fs_ipc_close(int device, void* ptr) {
  FS_CUDA(cudaSetDevice(device));
  if (ptr) FS_CUDA(cudaIpcCloseMemHandle(ptr));
  return FS_OK;
}

int fs_create(int device, int rank, int world, int num_experts, int topk, int token_bytes, int max_tokens,
              long long max_rows, int with_act_out, const int32_t* expert_owner,
              const int32_t* node_of, void* const* peer_regions, int grid_ctas, int timeout_ms,
              fs_handle_t* out) {
  if (!out || !expert_owner || !peer_regions) return fail(FS_EINVAL, "fs_create: null argument");
  *out = nullptr;
  if (world < 1 || world > FS_MAX_RANKS) return fail(FS_EINVAL, "world must be in [1, 32]");
  if (rank < 0 || rank >= world) return fail(FS_EINVAL, "rank outside [0, world)");
  if (num_experts < 1 || num_experts > kMaxExperts) return fail(FS_EINVAL, "num_experts must be in [1, 1024]");
  if (topk < 1 || topk > 32 || topk > num_experts)
    return fail(FS_EINVAL, "topk must be in [1, min(32, num_experts)]");
  // (token, slice) work units are indexed in 32 bits (smallest slice: 512 B)
  if ((long long)max_tokens * (((long long)token_bytes + 511) / 512) >= (1ll << 31))
    return fail(FS_EINVAL, "max_tokens x token_bytes too large for 32-bit work-unit indices");
  if (token_bytes <= 0 || token_bytes % 4)
    return fail(FS_EINVAL, "token_bytes must be a positive multiple of 4");
  if (max_tokens < 0) return fail(FS_EINVAL, "max_tokens must be >= 0");
  // expert table and per-rank segments (experts sorted by (owner, id))
  std::vector<int32_t> owner(expert_owner, expert_owner + num_experts);
  std::vector<int32_t> nodes(world);
  for (int g = 0; g < world; ++g) nodes[g] = node_of ? node_of[g] : g;
  for (int e = 0; e < num_experts; ++e)
    if (owner[e] < 0 || owner[e] >= world) return fail(FS_EINVAL, "expert owner outside [0, world)");
  for (int g = 0; g < world; ++g)
    if (nodes[g] < 0 || nodes[g] >= world) return fail(FS_EINVAL, "node_of outside [0, world)");
  std::vector<int32_t> perm(num_experts), seg(world + 1, 0);
  for (int e = 0; e < num_experts; ++e) seg[owner[e] + 1]++;
  for (int g = 0; g < world; ++g) seg[g + 1] += seg[g];
  {
    std::vector<int32_t> fill(seg.begin(), seg.end() - 1);
    for (int e = 0; e < num_experts; ++e) perm[fill[owner[e]]++] = e;
  }
  int max_local = 0;
  for (int g = 0; g < world; ++g) max_local = std::max(max_local, seg[g + 1] - seg[g]);
  if (max_rows <= 0) max_rows = (long long)world * max_tokens * std::min(topk, std::max(1, max_local));
  if (max_rows < 1) max_rows = 1;
  if (max_rows > 0x7fffffffLL) return fail(FS_EINVAL, "max_rows exceeds int32 row indices");
  for (int g = 0; g < world; ++g)
    if (!peer_regions[g]) return fail(FS_EINVAL, "peer region pointer is null");

  FS_CUDA(cudaSetDevice(device));
  fs_ctx* h = new fs_ctx();
  h->device = device;
  h->rank = rank;
  h->world = world;
  h->E = num_experts;
  h->K = topk;
  h->tb = token_bytes;
  h->max_tokens = max_tokens;
  h->max_rows = max_rows;
  h->with_act_out = with_act_out ? 1 : 0;
  h->nloc = seg[rank + 1] - seg[rank];
  h->epoch = 0;
  h->timeout_ns = (unsigned long long)(timeout_ms > 0 ? timeout_ms : 10000) * 1000000ull;
  h->L = region_layout(world, num_experts, topk, token_bytes, max_tokens, max_rows, h->with_act_out);
  h->peers.assign((char* const*)peer_regions, (char* const*)peer_regions + world);
  h->layout_smem = layout_smem_bytes(num_experts, topk);
  auto cleanup = [&](int rc) {
    fs_destroy(h);
    return rc;
  };
  cudaError_t e;
  int sms = 0;
  e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device);
  if (e != cudaSuccess) return cleanup(fail(FS_ECUDA, cudaGetErrorString(e)));

  if (h->layout_smem > 48 * 1024) {
    e = cudaFuncSetAttribute(layout_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)h->layout_smem);
    if (e != cudaSuccess) return cleanup(fail(FS_ECUDA, cudaGetErrorString(e)));
  }
  if (grid_ctas <= 0) {  // experiment knob: cap the mover grids
    const char* gc = getenv("FUSCO_GRID_CTAS");
    if (gc) grid_ctas = atoi(gc);
  }
  int occ_l = 0;
  int rc = occupancy(layout_kernel, kLayoutThreads, h->layout_smem, &occ_l);
  if (rc) return cleanup(rc);
  if (occ_l < 1) return cleanup(fail(FS_EINVAL, "layout kernel cannot be resident (too many experts)"));
  const int max_chunks = std::max(1, (max_tokens + kLayoutThreads - 1) / kLayoutThreads);
  h->layout_grid_max = std::min(max_chunks, occ_l * sms);

  // Dispatch grid upper bound (occupancy x SMs); the warp mover sizes each
  // launch to its work (fs_dispatch), the TMA mover uses the bound.
  int occ_d = 0;
  if ((rc = occupancy(dispatch_kernel<int4>, kMoveThreads, 0, &occ_d))) return cleanup(rc);
  int o = 0;
  if ((rc = occupancy(dispatch_kernel<int>, kMoveThreads, 0, &o))) return cleanup(rc);
  occ_d = std::max(1, std::min(std::min(occ_d, o), kMaxCtasPerSm));
  h->move_grid = grid_ctas > 0 ? std::min(grid_ctas, occ_d * sms) : occ_d * sms;
  // TMA engine: ~100 KB of row slots per CTA, two CTAs per SM
  {
    // Engine selection (FUSCO_DISPATCH = tma | warp | auto, default auto).
    // Measured on B200: TMA wins the HBM-bound single-rank permutation, the
    // warp mover wins when pushes go over NVLink (profiles/).
    const char* mode = getenv("FUSCO_DISPATCH");
    const std::string dm = mode ? std::string(mode) : std::string("auto");
    const bool want_tma = dm == "tma" || (dm == "auto" && world == 1);
    h->dispatch_tma = (want_tma && token_bytes % 16 == 0) ? 1 : 0;
    const char* lag = getenv("FUSCO_TMA_LAG");
    h->tma_lag = (lag && atoi(lag) >= 4) ? 4 : 2;
    const char* ctas = getenv("FUSCO_TMA_CTAS");
    h->tma_ctas = ctas ? std::max(1, std::min(8, atoi(ctas))) : 3;
    // Work unit: whole rows (default).  Measured alternatives (A/B knobs):
    // FUSCO_TMA_TAIL=1 cuts only the last partial round of the strided
    // assignment into column slices (neutral: DeepSeek-V3 96.8 vs 97.2 us,
    // Mixtral 41.2 vs 40.2 -- the strided tail is not what bounds the
    // launch); FUSCO_TMA_SLICES=n cuts every row into n slices (slower: the
    // engine is latency-bound per CTA, 2 slices made the Mixtral P=1
    // dispatch 40% slower).
    {
      const char* sl = getenv("FUSCO_TMA_SLICES");
      h->tma_slices = (sl && atoi(sl) > 0) ? std::min(atoi(sl), std::max(1, token_bytes / 16)) : 0;
      const char* tl = getenv("FUSCO_TMA_TAIL");
      h->tma_tail = tl && std::string(tl) == "1";
      h->tma_sb = token_bytes;  // slots hold whole rows
    }
    const int slot = tma_slot_bytes(h->tma_sb);
    h->tma_slots = std::max(h->tma_lag + 2, std::min(kTmaMaxSlots, (int)((200 * 1024 / h->tma_ctas - 512) / slot)));
    h->tma_smem = 2 * kTmaMaxSlots * sizeof(uint64_t) + (size_t)h->tma_slots * slot;
    if (h->dispatch_tma) {
      if (h->tma_smem > 227 * 1024) return cleanup(fail(FS_EINVAL, "token too large for the TMA engine"));
      const void* tfn = h->tma_lag == 4 ? (const void*)dispatch_tma_kernel<4> : (const void*)dispatch_tma_kernel<2>;
      e = cudaFuncSetAttribute(tfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->tma_smem);
      if (e != cudaSuccess) return cleanup(fail(FS_ECUDA, cudaGetErrorString(e)));
      int occ_t = 0;
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_t, tfn, kTmaThreads, h->tma_smem);
      if (e != cudaSuccess) return cleanup(fail(FS_ECUDA, cudaGetErrorString(e)));
      occ_t = std::max(1, std::min(occ_t, h->tma_ctas));
      h->move_grid = grid_ctas > 0 ? std::min(grid_ctas, occ_t * sms) : occ_t * sms;
    }
  }
  h->sms = sms;
  {
    // dispatch warps per CTA that push before fanning out (P > 1; the others
    // fan out duplicates from the start): FUSCO_PUSH_WARPS, default all
    const char* pw = getenv("FUSCO_PUSH_WARPS");
    h->push_warps = pw ? std::max(1, std::min(kMoveThreads / 32, atoi(pw))) : kMoveThreads / 32;
    const char* db = getenv("FUSCO_DBG_BLK");
    h->dbg_relaxed = db && std::string(db) == "1";
    h->recs_written = 0;
    h->owner_reduce_off = !h->L.off_grp;
    {
      const char* orf = getenv("FUSCO_OWNER_REDUCE");
      h->owner_reduce_force = orf && std::string(orf) == "1";
    }
    const char* pr = getenv("FUSCO_PUSH_ROUNDS");
    h->push_rounds = pr && std::string(pr) == "1";
    const char* fsp = getenv("FUSCO_FAN_SPLIT");
    h->fan_split = fsp ? (atoi(fsp) ? 1 : 0) : -1;
    const char* fp = getenv("FUSCO_FAN_POLL");
    h->fan_poll = fp && std::string(fp) == "1";
    const char* dc = getenv("FUSCO_DISP_CTAS");  // P > 1 warp mover: CTAs per SM cap
    h->disp_ctas_per_sm = dc ? std::max(1, std::min(kMaxCtasPerSm, atoi(dc))) : 0;
    const char* nd = getenv("FUSCO_NODEDUP");
    h->nodedup = nd && std::string(nd) == "1";
    const char* bl = getenv("FUSCO_BALANCE");
    h->balance = !(bl && std::string(bl) == "0");
    const char* pd = getenv("FUSCO_PDL");
    h->pdl = !(pd && std::string(pd) == "0");
    const char* pm = getenv("FUSCO_PDL_MULTI");
    h->pdl_multi = h->pdl && !(pm && std::string(pm) == "0");
    const char* lm = getenv("FUSCO_LAYOUT");  // grid (default, measured faster) | cluster
    h->cluster_layout = (lm && std::string(lm) == "cluster") && num_experts <= kClusterMaxE && topk <= kClusterMaxK;
    h->cluster_smem = layout_cluster_smem_bytes(num_experts, topk);
    if (h->cluster_layout) {
      e = cudaFuncSetAttribute(layout_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->cluster_smem);
      if (e != cudaSuccess) h->cluster_layout = 0;  // fall back to the grid planner
      cudaGetLastError();
    }
  }
  // TMA combine: ~100 KB of [K][slice] stages per CTA, two CTAs per SM
  {
    // FUSCO_COMBINE = tma | warp | auto (default): warp pull for the local
    // (HBM) case, TMA stages for NVLink pulls (measured)
    const char* mode = getenv("FUSCO_COMBINE");
    const std::string cm = mode ? std::string(mode) : std::string("auto");
    const bool want_tma = cm == "tma" || (cm == "auto" && world > 1);
    h->combine_tma = (want_tma && token_bytes % 16 == 0) ? 1 : 0;
    const char* cst = getenv("FUSCO_COMB_STAGE");  // bytes per stage (K row slices), default 24 KiB
    const int stage_target = cst ? std::max(4096, std::min(96 * 1024, atoi(cst))) : kCombStageTarget;
    h->comb_sb = comb_slice_bytes(token_bytes, topk, stage_target);
    const int stage = topk * h->comb_sb;
    const char* cctas = getenv("FUSCO_TMA_CTAS");
    const int comb_ctas = cctas ? std::max(1, std::min(8, atoi(cctas))) : 3;
    h->comb_stages = std::max(2, std::min(kCombMaxStages, (200 * 1024 / comb_ctas) / stage));
    h->comb_smem = 2 * kCombMaxStages * sizeof(uint64_t) + (size_t)h->comb_stages * stage;
    h->comb_grid = 0;
    if (h->combine_tma) {
      if (h->comb_smem > 227 * 1024) return cleanup(fail(FS_EINVAL, "token too large for the TMA combine"));
      const void* fns[4] = {(const void*)combine_tma_kernel<false, false>, (const void*)combine_tma_kernel<false, true>,
                            (const void*)combine_tma_kernel<true, false>, (const void*)combine_tma_kernel<true, true>};
      int occ_c = 1 << 30;
      for (const void* f : fns) {
        e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->comb_smem);
        if (e != cudaSuccess) return cleanup(fail(FS_ECUDA, cudaGetErrorString(e)));
        int o2 = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, f, kCombThreads, h->comb_smem);
        if (e != cudaSuccess) return cleanup(fail(FS_ECUDA, cudaGetErrorString(e)));
        occ_c = std::min(occ_c, o2);
      }
      occ_c = std::max(1, std::min(occ_c, comb_ctas));
      h->comb_grid = grid_ctas > 0 ? std::min(grid_ctas, occ_c * sms) : occ_c * sms;
    }
  }
  h->combine_grid_cap = grid_ctas > 0 ? grid_ctas : 0;

  auto dalloc = [&](void** p, size_t n) -> cudaError_t { return cudaMalloc(p, std::max<size_t>(n, 16)); };
  if ((e = dalloc((void**)&h->owner_d, num_experts * 4)) != cudaSuccess ||
      (e = dalloc((void**)&h->node_of_d, world * 4)) != cudaSuccess ||
      (e = dalloc((void**)&h->perm_d, num_experts * 4)) != cudaSuccess ||
      (e = dalloc((void**)&h->seg_d, (world + 1) * 4)) != cudaSuccess ||
      (e = dalloc((void**)&h->chunk_cnt_d, (size_t)max_chunks * num_experts * 4)) != cudaSuccess ||
      (e = dalloc((void**)&h->totals_d, (size_t)2 * num_experts * 4)) != cudaSuccess ||
      (e = dalloc((void**)&h->stat_part_d, (size_t)2 * 8 * 8)) != cudaSuccess ||
      (e = dalloc((void**)&h->status_d, 8)) != cudaSuccess ||
      (e = dalloc((void**)&h->num_rows_d, 4)) != cudaSuccess ||
      (e = dalloc((void**)&h->epoch_d, 4)) != cudaSuccess ||
      (e = dalloc((void**)&h->work_d, kWorkWords * 8)) != cudaSuccess ||
      (e = dalloc((void**)&h->blkdone_d, (size_t)2 * h->L.nbmax * kBlkStride * 4)) != cudaSuccess ||
      (e = dalloc((void**)&h->dupcnt_d, (size_t)2 * world * h->L.nbmax * 4)) != cudaSuccess ||
      (e = dalloc((void**)&h->jcum_d, (size_t)world * h->L.nbmax * 8)) != cudaSuccess ||
      (e = dalloc((void**)&h->jorder_d, (size_t)world * h->L.nbmax * 4)) != cudaSuccess)
    return cleanup(fail(FS_ECUDA, std::string("fs_create alloc: ") + cudaGetErrorString(e)));
  if ((e = cudaMemcpy(h->owner_d, owner.data(), num_experts * 4, cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaMemcpy(h->node_of_d, nodes.data(), world * 4, cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaMemcpy(h->perm_d, perm.data(), num_experts * 4, cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaMemcpy(h->seg_d, seg.data(), (world + 1) * 4, cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaMemset(h->status_d, 0, 8)) != cudaSuccess ||
      (e = cudaMemset(h->num_rows_d, 0, 4)) != cudaSuccess ||
      (e = cudaMemset(h->epoch_d, 0, 4)) != cudaSuccess ||
      (e = cudaMemset(h->work_d, 0, kWorkWords * 8)) != cudaSuccess ||
      (e = cudaMemset(h->totals_d, 0, (size_t)2 * num_experts * 4)) != cudaSuccess ||
      (e = cudaMemset(h->stat_part_d, 0, (size_t)2 * 8 * 8)) != cudaSuccess ||
      (e = cudaMemset(h->blkdone_d, 0, (size_t)2 * h->L.nbmax * kBlkStride * 4)) != cudaSuccess ||
      (e = cudaMemset(h->dupcnt_d, 0, (size_t)2 * world * h->L.nbmax * 4)) != cudaSuccess ||
      (e = cudaDeviceSynchronize()) != cudaSuccess)
    return cleanup(fail(FS_ECUDA, std::string("fs_create init: ") + cudaGetErrorString(e)));
  {
    const char* tr = getenv("FUSCO_TRACE");
    if (tr && std::string(tr) == "1") {
      if ((e = cudaMalloc((void**)&h->trace_d, FS_NTRACE * 8)) != cudaSuccess ||
          (e = cudaMemset(h->trace_d, 0, FS_NTRACE * 8)) != cudaSuccess)
        return cleanup(fail(FS_ECUDA, cudaGetErrorString(e)));
    }
  }
  *out = h;
  return FS_OK;
}

int fs_destroy(fs_handle_t h) {
  if (!h) return FS_OK;
  cudaSetDevice(h->device);
  cudaFree(h->owner_d);
  cudaFree(h->node_of_d);
  cudaFree(h->perm_d);
  cudaFree(h->seg_d);
  cudaFree(h->chunk_cnt_d);
  cudaFree(h->totals_d);
  cudaFree(h->stat_part_d);
  cudaFree(h->status_d);
  cudaFree(h->num_rows_d);
  cudaFree(h->epoch_d);
  cudaFree(h->work_d);
  cudaFree(h->blkdone_d);
  cudaFree(h->dupcnt_d);
  cudaFree(h->jcum_d);
  cudaFree(h->jorder_d);
  if (h->trace_d) cudaFree(h->trace_d);
  delete h;
  return FS_OK;
}

int fs_num_local_experts(fs_handle_t h, int* n_out) {
  if (!h || !n_out) return fail(FS_EINVAL, "null argument");
  *n_out = h->nloc;
  return FS_OK;
}

int fs_grid_ctas(fs_handle_t h, int* n_out) {
  if (!h || !n_out) return fail(FS_EINVAL, "null argument");
  *n_out = h->move_grid;
  return FS_OK;
}

int fs_buffer_ptr(fs_handle_t h, int which, void** ptr_out) {
  if (!h || !ptr_out) return fail(FS_EINVAL, "null argument");
  char* base = h->peers[h->rank];
  if (which == 0) {
    *ptr_out = base + h->L.off_act;  // fixed address: safe to capture in a CUDA graph
  } else if (which == 1) {
    if (!h->with_act_out) return fail(FS_EINVAL, "handle was created without an act_out buffer");
    *ptr_out = base + h->L.off_actout;
  } else {
    return fail(FS_EINVAL, "which must be 0 (act) or 1 (act_out)");
  }
  return FS_OK;
}

long long fs_max_rows(fs_handle_t h) { return h ? h->max_rows : -1; }

unsigned int fs_epoch(fs_handle_t h) { return h ? h->epoch : 0u; }

int fs_set_nodedup(fs_handle_t h, int on) {
  if (!h) return fail(FS_EINVAL, "null handle");
  if (on != 0 && on != 1) return fail(FS_EINVAL, "on must be 0 or 1");
  h->nodedup = on;
  return FS_OK;
}

int fs_set_balance(fs_handle_t h, int on) {
  if (!h) return fail(FS_EINVAL, "null handle");
  if (on != 0 && on != 1) return fail(FS_EINVAL, "on must be 0 or 1");
  h->balance = on;
  return FS_OK;
}

int fs_layout(fs_handle_t h, const void* topk_idx, int idx_bytes, int num_tokens, int32_t* row_of,
              int32_t* expert_counts, int32_t* expert_offsets, uint8_t* first_mask,
              uint32_t* rank_mask, int64_t* stats, int phase, void* stream) {
  if (!h) return fail(FS_EINVAL, "null handle");
  FS_CUDA(cudaSetDevice(h->device));
  if (int rc = check_idx_bytes(idx_bytes)) return rc;
  if (num_tokens < 0 || num_tokens > h->max_tokens)
    return fail(FS_EINVAL, "num_tokens outside [0, max_tokens]");
  if ((phase & FS_PHASE_ALL) == 0 || (phase & ~FS_PHASE_ALL)) return fail(FS_EINVAL, "bad phase");
  if (num_tokens > 0 && (!topk_idx || !row_of)) return fail(FS_EINVAL, "null topk_idx / row_of");
  if (phase & FS_PHASE_LOCAL) {
    h->epoch++;
    h->disp_phases = h->comb_phases = 0;
  }
  FsArgs a = make_args(h, num_tokens, idx_bytes == 8);
  long long* st_ptr = reinterpret_cast<long long*>(stats);
  const int ncl = (num_tokens + kClusterThreads - 1) / kClusterThreads;
  if (phase == FS_PHASE_ALL && h->cluster_layout && ncl <= kClusterMaxCtas) {
    const int cs = std::max(1, ncl);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(kClusterThreads);
    cfg.dynamicSmemBytes = h->cluster_smem;
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    FS_CUDA(cudaLaunchKernelEx(&cfg, layout_cluster_kernel, a, topk_idx, row_of, first_mask, rank_mask, st_ptr,
                               expert_counts, expert_offsets));
    return FS_OK;
  }
  const int nchunks = (num_tokens + kLayoutThreads - 1) / kLayoutThreads;
  const int grid = std::max(1, std::min(nchunks, h->layout_grid_max));
  void* args[] = {&a, (void*)&topk_idx, &row_of, &first_mask, &rank_mask,
                  &st_ptr, &expert_counts, &expert_offsets, &phase};
  FS_CUDA(cudaLaunchCooperativeKernel((const void*)layout_kernel, dim3(grid), dim3(kLayoutThreads), args,
                                      h->layout_smem, (cudaStream_t)stream));
  return FS_OK;
}

int fs_dispatch(fs_handle_t h, const void* x, const void* topk_idx, int idx_bytes, const int32_t* row_of,
                int num_tokens, int phase, void* stream) {
  return fs_dispatch_w(h, x, topk_idx, idx_bytes, row_of, nullptr, 4, num_tokens, phase, stream);
}

int fs_dispatch_w(fs_handle_t h, const void* x, const void* topk_idx, int idx_bytes, const int32_t* row_of,
                  const void* topk_w, int w_bytes, int num_tokens, int phase, void* stream) {
  if (!h) return fail(FS_EINVAL, "null handle");
  if (topk_w && w_bytes != 4 && w_bytes != 8) return fail(FS_EINVAL, "w_bytes must be 4 or 8");
  FS_CUDA(cudaSetDevice(h->device));
  if (int rc = check_idx_bytes(idx_bytes)) return rc;
  if (num_tokens < 0 || num_tokens > h->max_tokens)
    return fail(FS_EINVAL, "num_tokens outside [0, max_tokens]");
  if ((phase & FS_PHASE_ALL) == 0 || (phase & ~FS_PHASE_ALL)) return fail(FS_EINVAL, "bad phase");
  if (num_tokens > 0 && (!x || !topk_idx || !row_of)) return fail(FS_EINVAL, "null input");
  if (h->epoch == 0) return fail(FS_EINVAL, "fs_dispatch before fs_layout");
  // the push claims / done counts / arrival flags are per epoch: a second
  // dispatch of the same phase needs a new plan (fs_layout) first
  if (h->disp_phases & phase) return fail(FS_EINVAL, "fs_dispatch already ran for this plan: call fs_layout first");
  h->disp_phases |= phase;
  FsArgs a = make_args(h, num_tokens, idx_bytes == 8);
  // owner-side pre-reduction records (warp engine, P > 1, weights given): the
  // combine of this epoch may then pull fp32 partials for them
  const bool vec16_x = (h->tb % 16 == 0) && aligned(x, 16);
  const bool recs = topk_w && h->L.off_grp && h->world > 1 && !(h->dispatch_tma && vec16_x);
  if (phase & FS_PHASE_LOCAL) h->recs_written = recs ? 1 : 0;
  if (recs) {
    a.disp_w = topk_w;
    a.disp_w64 = w_bytes == 8;
  }
  // receiver fan-out unit: a row slice at small batches (few duplicate rows:
  // spread them over every warp), a whole row otherwise (FUSCO_FAN_SPLIT=0|1 overrides)
  a.fan_split = h->fan_split >= 0 ? h->fan_split : (num_tokens <= kFanSplitTokens ? 1 : 0);
  const bool vec16 = (h->tb % 16 == 0) && aligned(x, 16);
  if (!aligned(x, 4)) return fail(FS_EINVAL, "x must be 4-byte aligned");
  if (h->dispatch_tma && vec16) {  // unaligned x falls back to the warp mover (same grid)
    int nslots = h->tma_slots, whole = num_tokens, ns = 1, sb = h->tb;
    {
      // rows of the full rounds stay whole; the last round's rows are sliced
      // so they spread over the grid (>= 2 KiB per slice)
      const int grid = h->move_grid;
      const int max_ns = std::max(1, h->tb / 2048);
      if (h->tma_slices > 0) {
        whole = 0;
        ns = h->tma_slices;
      } else if (h->tma_tail && num_tokens > 0) {
        whole = (num_tokens / grid) * grid;
        const int tail = num_tokens - whole;
        if (tail > 0) ns = std::min(max_ns, (grid + tail - 1) / tail);
      }
      sb = ((h->tb + ns - 1) / ns + 15) & ~15;
      ns = (h->tb + sb - 1) / sb;
      if (ns == 1) whole = num_tokens;
    }
    const void* tfn = h->tma_lag == 4 ? (const void*)dispatch_tma_kernel<4> : (const void*)dispatch_tma_kernel<2>;
    if (h->world == 1 && h->pdl) {
      // No cross-CTA or cross-rank waits at P=1: a plain launch with PDL behind
      // the planner, so row prefetch overlaps the planner's tail.
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(h->move_grid);
      cfg.blockDim = dim3(kTmaThreads);
      cfg.dynamicSmemBytes = h->tma_smem;
      cfg.stream = (cudaStream_t)stream;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      if (h->tma_lag == 4)
        FS_CUDA(cudaLaunchKernelEx(&cfg, dispatch_tma_kernel<4>, a, (const char*)x, topk_idx, row_of, phase, nslots, whole, ns, sb));
      else
        FS_CUDA(cudaLaunchKernelEx(&cfg, dispatch_tma_kernel<2>, a, (const char*)x, topk_idx, row_of, phase, nslots, whole, ns, sb));
      return FS_OK;
    }
    void* targs[] = {&a, (void*)&x, (void*)&topk_idx, (void*)&row_of, &phase, &nslots, &whole, &ns, &sb};
    return launch_ex(tfn, h->move_grid, kTmaThreads, h->tma_smem, stream, targs, true, h->pdl_multi);
  }
  void* args[] = {&a, (void*)&x, (void*)&topk_idx, (void*)&row_of, &phase};
  const void* fn = vec16 ? (const void*)dispatch_kernel<int4> : (const void*)dispatch_kernel<int>;
  // Grid sized to the work: every CTA joins the end-of-push count (one
  // acq_rel atomic each), so idle CTAs only add latency at decode sizes.
  // At least one CTA per SM (the receiver fan-out uses the same grid).
  const int U = vec16 ? MoveCfg<int4>::U : MoveCfg<int>::U, elem = vec16 ? 16 : 4;
  const long long slices = ((long long)h->tb / elem + 32 * U - 1) / (32 * U);
  const long long units = (long long)num_tokens * slices;
  const long long want = (units + kMoveThreads / 32 - 1) / (kMoveThreads / 32);
  int cap = h->move_grid;
  if (h->world > 1 && h->disp_ctas_per_sm > 0) cap = std::min(cap, h->disp_ctas_per_sm * h->sms);
  const int grid = (int)std::min<long long>(cap, std::max<long long>(want, h->sms));
  return launch_ex(fn, grid, kMoveThreads, 0, stream, args, true, h->pdl_multi);
}

int fs_combine(fs_handle_t h, const void* topk_idx, int idx_bytes, const int32_t* row_of, const void* topk_w,
               int w_bytes, int num_tokens, void* out, int dtype, int src, int acc, int phase,
               void* stream) {
  if (!h) return fail(FS_EINVAL, "null handle");
  FS_CUDA(cudaSetDevice(h->device));
  if (int rc = check_idx_bytes(idx_bytes)) return rc;
  if (w_bytes != 4 && w_bytes != 8) return fail(FS_EINVAL, "w_bytes must be 4 or 8");
  if (num_tokens < 0 || num_tokens > h->max_tokens)
    return fail(FS_EINVAL, "num_tokens outside [0, max_tokens]");
  if ((phase & FS_PHASE_ALL) == 0 || (phase & ~FS_PHASE_ALL)) return fail(FS_EINVAL, "bad phase");
  if (dtype != FS_DTYPE_F32 && dtype != FS_DTYPE_BF16) return fail(FS_EINVAL, "dtype must be f32 or bf16");
  if (src != FS_SRC_ACT && src != FS_SRC_ACT_OUT) return fail(FS_EINVAL, "src must be act or act_out");
  if (src == FS_SRC_ACT_OUT && !h->with_act_out)
    return fail(FS_EINVAL, "combine from act_out on a handle without act_out");
  if (acc != FS_ACC_F32 && acc != FS_ACC_F64) return fail(FS_EINVAL, "acc must be f32 or f64");
  if (num_tokens > 0 && (!topk_idx || !row_of || !topk_w || !out)) return fail(FS_EINVAL, "null input");
  if (h->epoch == 0) return fail(FS_EINVAL, "fs_combine before fs_layout");
  if (h->comb_phases & phase & FS_PHASE_REMOTE) {
    // a repeated combine of the same plan (e.g. another expert output):
    // re-arm the dynamic item counter (both parities: the other one is the
    // next epoch's, zeroed by its planner anyway), stream-ordered and graph-safe
    for (int q = 0; q < 2; ++q)
      FS_CUDA(cudaMemsetAsync(h->work_d + ((size_t)q * kWorkSlots + kWorkCombine) * kWorkStride, 0,
                              sizeof(unsigned long long), (cudaStream_t)stream));
  }
  h->comb_phases |= phase;
  FsArgs a = make_args(h, num_tokens, idx_bytes == 8);
  if (!aligned(out, 4)) return fail(FS_EINVAL, "out must be 4-byte aligned");
  const bool vec16 = (h->tb % 16 == 0) && aligned(out, 16);
  int w64 = w_bytes == 8;
  void* args[] = {&a, (void*)&topk_idx, (void*)&row_of, (void*)&topk_w, &w64, &out, &src, &phase};
  const void* fn;
  const bool bf = dtype == FS_DTYPE_BF16, f64 = acc == FS_ACC_F64;
  // owner-side pre-reduction: this epoch's dispatch wrote the records
  // (fs_dispatch_w), fp32 accumulation, the TMA engine (P > 1 default)
  // (groups need >= 3 bf16 rows / >= 2 fp32 rows: with fewer experts per token there is nothing to reduce)
  // Default (FUSCO_OWNER_REDUCE unset): more than kFanSplitTokens tokens and
  // P = 2, or P <= 4 with rows of >= 8 KB -- where it was measured faster:
  // EP=2 DeepSeek-V3 step 405 vs 508 us, Zipf 416 vs 547, Qwen3 158 vs 185;
  // EP=4 DeepSeek-V3 829 vs 850, Zipf 1008 vs 1077.  Slower: EP=4 Qwen3 (4 KB
  // rows) 297 vs 290, decode 72 vs 67 (the LOCAL-phase pass and grid barrier
  // outweigh the bytes saved), and at P >= 8 a token has ~1.5 rows per owner
  // (8 % fewer bytes).  FUSCO_OWNER_REDUCE=1 forces it on, =0 removes the
  // buffers.  Ranks may decide differently (ragged batches): a source pulls
  // an owner's partials only if that owner's mode word says it pre-reduced.
  const bool red_auto =
      num_tokens > kFanSplitTokens && (h->world == 2 || (h->world <= 4 && h->tb >= 8192));
  a.reduce = (h->combine_tma && vec16 && !f64 && h->world > 1 && h->recs_written && !h->owner_reduce_off &&
              h->K >= (bf ? 3 : 2) && (h->owner_reduce_force || red_auto)) ? 1 : 0;
  if (h->combine_tma && vec16) {
    fn = bf ? (f64 ? (const void*)combine_tma_kernel<true, true> : (const void*)combine_tma_kernel<true, false>)
            : (f64 ? (const void*)combine_tma_kernel<false, true> : (const void*)combine_tma_kernel<false, false>);
    int ns = h->comb_stages, sb = h->comb_sb;
    void* targs[] = {&a, (void*)&topk_idx, (void*)&row_of, (void*)&topk_w, &w64, &out, &src, &phase, &ns, &sb};
    return launch_ex(fn, h->comb_grid, kCombThreads, h->comb_smem, stream, targs, true, h->pdl_multi);
  }
  // rows in flight per unit: min(K, 4) (no registers reserved for loads that never issue)
  if (vec16 && h->K <= 2) {  // software-pipelined top-1/top-2 mover
    fn = bf ? (f64 ? (const void*)combine_k2_kernel<true, true> : (const void*)combine_k2_kernel<true, false>)
            : (f64 ? (const void*)combine_k2_kernel<false, true> : (const void*)combine_k2_kernel<false, false>);
    if (h->world == 1 && h->pdl) {  // no cross-CTA waits at P=1: PDL launch behind the dispatch
      int occ = 0;
      if (int rc = occupancy(fn, kMoveThreads, 0, &occ)) return rc;
      occ = std::max(1, std::min(occ, kMaxCtasPerSm));
      int grid = occ * h->sms;
      if (h->combine_grid_cap > 0) grid = std::min(grid, h->combine_grid_cap);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(grid);
      cfg.blockDim = dim3(kMoveThreads);
      cfg.stream = (cudaStream_t)stream;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      FS_CUDA(cudaLaunchKernelExC(&cfg, fn, args));
      return FS_OK;
    }
  } else if (vec16) {  // K > 2: four rows' 16-byte loads in flight per lane
    fn = bf ? (f64 ? (const void*)combine_kernel<int4, true, true, 4, 4> : (const void*)combine_kernel<int4, true, false, 4, 4>)
            : (f64 ? (const void*)combine_kernel<int4, false, true, 4, 4> : (const void*)combine_kernel<int4, false, false, 4, 4>);
  } else {
    fn = bf ? (f64 ? (const void*)combine_kernel<int, true, true, 8, 4> : (const void*)combine_kernel<int, true, false, 8, 4>)
            : (f64 ? (const void*)combine_kernel<int, false, true, 8, 4> : (const void*)combine_kernel<int, false, false, 8, 4>);
  }
  int occ = 0;
  if (int rc = occupancy(fn, kMoveThreads, 0, &occ)) return rc;
  occ = std::max(1, std::min(occ, kMaxCtasPerSm));
  int grid = occ * h->sms;
  if (h->combine_grid_cap > 0) grid = std::min(grid, h->combine_grid_cap);
  return launch_ex(fn, grid, kMoveThreads, 0, stream, args, true, h->pdl_multi);
}

int fs_check(fs_handle_t h, void* stream) {
  if (!h) return fail(FS_EINVAL, "null handle");
  FS_CUDA(cudaSetDevice(h->device));
  FS_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  int st[2] = {0, 0};
  FS_CUDA(cudaMemcpy(st, h->status_d, 8, cudaMemcpyDeviceToHost));
  FS_CUDA(cudaMemset(h->status_d, 0, 8));
  const int status = st[0];
  static const char* kSites[] = {"",
                                 " (planner: peer count words)",
                                 " (dispatch: a source's token count)",
                                 " (dispatch: a source's block words)",
                                 " (dispatch fan-out worker: published schedule)",
                                 " (dispatch fan-out worker: inconsistent schedule)",
                                 " (combine: a peer's outputs-ready flag)",
                                 " (combine: TMA stage pipeline)",
                                 " (dispatch: TMA slot pipeline)",
                                 " (row index outside the activation buffer)"};
  const std::string where = (st[1] > 0 && st[1] < (int)(sizeof(kSites) / sizeof(kSites[0]))) ? kSites[st[1]] : "";
  if (status == FS_ETIMEOUT) return fail(FS_ETIMEOUT, "a peer flag wait timed out" + where);
  if (status == FS_ERANGE) return fail(FS_ERANGE, "routing out of range (expert id or row capacity)" + where);
  if (status == FS_EINVAL) return fail(FS_EINVAL, "a token routes to the same expert twice");
  if (status != FS_OK) return fail(status, "device reported an error");
  return FS_OK;
}

int fs_trace(fs_handle_t h, uint64_t* host_out, void* stream) {
  if (!h || !host_out) return fail(FS_EINVAL, "null argument");
  if (!h->trace_d) return fail(FS_EINVAL, "handle created without FUSCO_TRACE=1");
  FS_CUDA(cudaSetDevice(h->device));
  FS_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  FS_CUDA(cudaMemcpy(host_out, h->trace_d, FS_NTRACE * 8, cudaMemcpyDeviceToHost));
  return FS_OK;
}

int fs_probe_a2a(int device, void* const* dsts, const void* const* srcs, int npairs, size_t bytes, int mode,
                 int ctas, void* stream) {
  if (!dsts || !srcs || npairs < 1 || npairs > FS_MAX_RANKS || bytes % 16 || ctas <= 0 || (mode != 0 && mode != 1))
    return fail(FS_EINVAL, "fs_probe_a2a: bad arguments");
  FS_CUDA(cudaSetDevice(device));
  ProbePairs pp;
  memset(&pp, 0, sizeof(pp));
  for (int j = 0; j < npairs; ++j) {
    if (!aligned(dsts[j], 16) || !aligned(srcs[j], 16)) return fail(FS_EINVAL, "fs_probe_a2a: 16-byte alignment");
    pp.dst[j] = (char*)dsts[j];
    pp.src[j] = (const char*)srcs[j];
  }
  if (mode == 0) {
    probe_a2a_warp_kernel<<<ctas, kMoveThreads, 0, (cudaStream_t)stream>>>(pp, npairs, bytes);
  } else {
    const int nslots = 6;
    const size_t smem = 32 * sizeof(uint64_t) + (size_t)nslots * kProbeChunk;
    FS_CUDA(cudaFuncSetAttribute(probe_a2a_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    probe_a2a_tma_kernel<<<ctas, 64, smem, (cudaStream_t)stream>>>(pp, npairs, bytes, nslots);
  }
  FS_CUDA(cudaGetLastError());
  return FS_OK;
}

int fs_probe_copy(int device, void* dst, const void* src, size_t bytes, int ctas, void* stream) {
  FS_CUDA(cudaSetDevice(device));
  // src == NULL: write-only fill (the write ceiling a write-heavy mover sees)
  if (!dst || bytes % 16 || !aligned(dst, 16) || (src && !aligned(src, 16)))
    return fail(FS_EINVAL, "fs_probe_copy: 16-byte aligned buffers and size required");
  if (ctas <= 0) return fail(FS_EINVAL, "fs_probe_copy: ctas must be > 0");
  probe_copy_kernel<<<ctas, kMoveThreads, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<int4*>(dst), reinterpret_cast<const int4*>(src), bytes / 16);
  FS_CUDA(cudaGetLastError());
  return FS_OK;
}

int fs_probe_scatter(int device, void* dst, const void* src, const int32_t* perm, int nrows_src, int fanout,
                     int row_bytes, int ctas, void* stream) {
  FS_CUDA(cudaSetDevice(device));
  if (!dst || !perm || row_bytes <= 0 || row_bytes % 16 || !aligned(dst, 16) || (src && !aligned(src, 16)) ||
      nrows_src < 0 || fanout <= 0 || ctas <= 0)
    return fail(FS_EINVAL, "fs_probe_scatter: bad arguments");
  probe_scatter_kernel<<<ctas, kMoveThreads, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<int4*>(dst), reinterpret_cast<const int4*>(src), perm, nrows_src, fanout, row_bytes / 16);
  FS_CUDA(cudaGetLastError());
  return FS_OK;
}

}  // extern "C"
