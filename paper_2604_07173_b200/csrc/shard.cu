// shard.cu -- the Sharded LoRA Server: LoRA Data Parallel over NVLink.
//
// P:288-291 (Sec. 4.1, Table 1 DP row): "evenly distribute LoRA adapters
// across the server GPUs ... activations from client GPUs must be routed
// accordingly ... the server GPUs perform a collective coordination step to
// determine which activations should be processed by which GPUs."  Skewed
// adapter popularity concentrates activations on a few server GPUs;
// the n_replicated hottest adapters are therefore stored on every rank
// and their rows never leave their rank.
//
// Push path (x and y registered with lora_shard_register).
// The paper moves activations and results with one-sided pushes in both
// directions (pull measured 2.63x slower) and overlaps receive,
// compute and send.  Here every transfer is fused into a compute
// kernel over NVLink peer mappings, so no row and no delta is staged:
//   1. bucket (1 CTA): rows this rank serves -> in-place id list; the rest
//      bucketed by owner into this rank's control area (ids + local row);
//      announce: the count row (+ a layout hash) is written into every peer's
//      mailbox, then a release flag carrying the apply's epoch
//   2. in-place plan + apply of the local rows (caller's stream), concurrently
//      on a second stream: recv-prep (waits for every peer's flag, pulls the
//      received rows' ids and origins from the sources' control areas) and
//      the owner-side plan, with the row count on the device
//   3. owner apply: the shrink kernels read each received x row from its
//      source's registered x buffer (dispatch fused into the shrink's loads),
//      the expand epilogues add each delta into the origin row of the source's
//      registered y with red.add (return fused into the epilogue; one writer
//      per element)
//   4. done: a release flag into every peer; wait: until every owner's flag
//      for this epoch has arrived (this rank's y is final)
// No host synchronisation, no allocation: the sharded step is captured in a
// CUDA graph.  The epoch lives in device memory, so graph replays advance it.
// Spin-waits give up after LORA_SHARD_TIMEOUT_MS (default 10 s): the sticky
// flag reports LORA_ERR_PEER instead of a hang.
//
// Unregistered buffers (NCCL control plane only): grouped ncclSend/ncclRecv of
// x rows + ids and of the deltas, one host sync for the count matrix.
// Deltas travel as fp32 when y is fp32 (sharded == unsharded bit for bit,
// DESIGN.md R18) and as bf16 when y is bf16 (one extra rounding of the
// delta: DESIGN.md R19), unless LORA_SHARD_FP32=1 (NCCL path).
// NCCL is loaded with dlopen("libnccl.so.2") (the copy torch already loaded),
// so the library itself has no link-time NCCL dependency.
#include <cuda.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "server.h"

using namespace lora;

namespace {

struct NcclApi {
  bool ok = false;
  std::string err;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api;
  tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    api.err = std::string("dlopen libnccl.so.2 failed: ") + dlerror();
    return api;
  }
#define SYM(field, name)                                                     \
  api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name));         \
  if (!api.field) {                                                          \
    api.err = std::string("missing NCCL symbol ") + name;                    \
    return api;                                                              \
  }
  SYM(GetUniqueId, "ncclGetUniqueId");
  SYM(CommInitRank, "ncclCommInitRank");
  SYM(CommDestroy, "ncclCommDestroy");
  SYM(GroupStart, "ncclGroupStart");
  SYM(GroupEnd, "ncclGroupEnd");
  SYM(Send, "ncclSend");
  SYM(Recv, "ncclRecv");
  SYM(AllGather, "ncclAllGather");
  SYM(AllReduce, "ncclAllReduce");
  SYM(GetErrorString, "ncclGetErrorString");
  SYM(CommGetAsyncError, "ncclCommGetAsyncError");
#undef SYM
  api.ok = true;
  return api;
}

// ---------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------
constexpr int kBucketThreads = 1024;

// Single CTA over the T local rows (T <= 16384):
//   ad_local[r] = a if this rank processes row r in place, else -1
//   send_idx    = the other rows, bucketed by owner rank (stable, local order)
//   counts[o]   = rows for owner o (0 for this rank); counts[world] = hash
//                 (layout hash of the call: every rank must pass the same)
// loopback != 0 (test knob LORA_SHARD_LOOPBACK=1) sends this rank's own rows
// through the exchange as well, so a single GPU exercises the NCCL path.
// Out-of-range ids are flagged and dropped (never sent, never applied).
__global__ void __launch_bounds__(kBucketThreads, 1)
    bucket_kernel(const int32_t* __restrict__ ad, const int32_t* __restrict__ ex, int T, Placement pl, int n_adapters,
                  int E, int loopback, int32_t* __restrict__ ad_local,
                  int32_t* __restrict__ send_idx, int32_t* __restrict__ counts, int* __restrict__ err, int hash) {
  __shared__ int s_tmp[32];
  __shared__ int s_base;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int chunk = (T + kBucketThreads - 1) / kBucketThreads;
  const int r0 = min(tid * chunk, T), r1 = min(r0 + chunk, T);
  if (tid == 0) s_base = 0;
  // a row is routable iff both ids are in range: a in [0, n_adapters), e in [0, E)
  auto routable = [&](int r, int a) {
    if (a < 0 || a >= n_adapters) return false;
    const int e = ex ? ex[r] : 0;
    return e >= 0 && e < E;
  };
  int bad = 0;
  if (tid == 0) counts[pl.world] = hash;
  for (int r = r0; r < r1; ++r) {
    const int a = ad[r];
    const bool ok = a == -1 || routable(r, a);
    if (!ok) bad = 1;
    ad_local[r] = (!loopback && ok && a >= 0 && pl.owner_unit(a, ex ? ex[r] : 0) == pl.rank) ? a : -1;
  }
  if (bad) atomicOr(err, 1);
  __syncthreads();
  for (int o = 0; o < pl.world; ++o) {
    if (o == pl.rank && !loopback) {
      if (tid == 0) counts[o] = 0;
      continue;
    }
    int c = 0;
    for (int r = r0; r < r1; ++r) {
      const int a = ad[r];
      c += (routable(r, a) && pl.owner_unit(a, ex ? ex[r] : 0) == o);
    }
    // block exclusive scan of c
    int x = c;
    for (int d = 1; d < 32; d <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= d) x += y;
    }
    if (lane == 31) s_tmp[warp] = x;
    __syncthreads();
    if (warp == 0) {
      int w = s_tmp[lane];
      for (int d = 1; d < 32; d <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, w, d);
        if (lane >= d) w += y;
      }
      s_tmp[lane] = w;
    }
    __syncthreads();
    int pos = s_base + (warp ? s_tmp[warp - 1] : 0) + x - c;
    const int tot = s_tmp[31];
    for (int r = r0; r < r1; ++r) {
      const int a = ad[r];
      if (routable(r, a) && pl.owner_unit(a, ex ? ex[r] : 0) == o) send_idx[pos++] = r;
    }
    __syncthreads();
    if (tid == 0) {
      counts[o] = tot;
      s_base += tot;
    }
    __syncthreads();
  }
}

// out[j] = in[idx[j]] (4-byte words)
__global__ void gather_words_kernel(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                                    const int32_t* __restrict__ idx, int n) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) out[j] = in[idx[j]];
}

// out[j][:] = in[idx[j]][:], rows of `chunks` 16-byte chunks; one block row per output row
__global__ void gather_rows16_kernel(const uint4* __restrict__ in, uint4* __restrict__ out,
                                     const int32_t* __restrict__ idx, int n, int chunks) {
  for (int j = blockIdx.y; j < n; j += gridDim.y) {
    const uint4* src = in + (long long)idx[j] * chunks;
    uint4* dst = out + (long long)j * chunks;
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < chunks; c += gridDim.x * blockDim.x) dst[c] = src[c];
  }
}

// y[idx[j]][c..c+4] = round(y + d[j][c..c+4]); d is fp32 (d_bf16 == 0) or bf16
__global__ void scatter_add4_kernel(void* __restrict__ y, int y_fp32, const void* __restrict__ d, int d_bf16,
                                    const int32_t* __restrict__ idx, int n, int width) {
  const int q4 = width >> 2;
  for (int j = blockIdx.y; j < n; j += gridDim.y) {
    const long long row = idx[j];
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < q4; c += gridDim.x * blockDim.x) {
      float4 v;
      if (d_bf16) {
        const uint2 b = reinterpret_cast<const uint2*>(d)[(long long)j * q4 + c];
        v = make_float4(bf16lo(b.x), bf16hi(b.x), bf16lo(b.y), bf16hi(b.y));
      } else {
        v = reinterpret_cast<const float4*>(d)[(long long)j * q4 + c];
      }
      if (y_fp32) {
        float4* p = reinterpret_cast<float4*>(y) + row * q4 + c;
        float4 o = *p;
        o.x += v.x; o.y += v.y; o.z += v.z; o.w += v.w;
        *p = o;
      } else {
        uint2* p = reinterpret_cast<uint2*>(y) + row * q4 + c;
        const uint2 o = *p;
        uint2 r;
        r.x = pack_bf16x2_rn(bf16lo(o.x) + v.x, bf16hi(o.x) + v.y);
        r.y = pack_bf16x2_rn(bf16lo(o.y) + v.z, bf16hi(o.y) + v.w);
        *p = r;
      }
    }
  }
}

int grid_of(long long n) {
  long long g = (n + 255) / 256;
  return (int)(g < 1 ? 1 : (g > 148 * 16 ? 148 * 16 : g));
}

// ---------------------------------------------------------------------------
// push path: control area and kernels
// ---------------------------------------------------------------------------
// Per-rank control area (library memory, IPC-mapped by every peer).  Peers
// write only their own slots: flag_cnt[p] / mbox[.][p] by source p,
// flag_done[q] by owner q.  The send arrays are this rank's, read by owners.
struct ShardCtl {
  unsigned int epoch;                              // this rank's apply counter (local)
  int stride;                                      // this rank's max_rows: the send arrays' length (read by owners)
  unsigned int pad_[6];
  unsigned int flag_cnt[kMaxWorld];                // source p's count row for epoch v is in mbox
  unsigned int flag_done[kMaxWorld];               // owner q finished pushing into this rank's y
  int mbox[2][kMaxWorld][kMaxWorld + 1];           // [epoch & 1][source p][owner q | layout hash]
};
static_assert(sizeof(ShardCtl) % 16 == 0, "control area alignment");
// send arrays after the header: send_row / send_a / send_e [max_rows] each
LORA_DEVINL int32_t* ctl_send(ShardCtl* c, int max_rows, int which) {
  return reinterpret_cast<int32_t*>(c + 1) + (size_t)which * max_rows;
}

struct PeerCtl {
  ShardCtl* p[kMaxWorld];  // every rank's control area (own: local pointer)
};

enum { kErrId = 1, kErrPeer = 2, kErrLayout = 4 };

LORA_DEVINL unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
LORA_DEVINL unsigned int ld_acquire_sys(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
LORA_DEVINL void st_release_sys(unsigned int* p, unsigned int v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// wait until *flag has reached epoch v (monotonic counters); false on timeout
LORA_DEVINL bool wait_flag(const unsigned int* flag, unsigned int v, unsigned long long timeout_ns) {
  const unsigned long long t0 = globaltimer_ns();
  while ((int)(ld_acquire_sys(flag) - v) < 0) {
    if (globaltimer_ns() - t0 > timeout_ns) return false;
    __nanosleep(64);
  }
  return true;
}

// 1 CTA.  After bucket_kernel: epoch += 1; the send list (local row, a, e in
// owner order) into this rank's control area; then to every peer q: this
// rank's count row + layout hash into q's mailbox, release flag.
__global__ void __launch_bounds__(1024) push_announce_kernel(PeerCtl pc, int me, int G, int max_rows,
                                                             const int32_t* __restrict__ counts,
                                                             const int32_t* __restrict__ send_idx,
                                                             const int32_t* __restrict__ ad,
                                                             const int32_t* __restrict__ ex) {
  __shared__ unsigned int s_epoch;
  ShardCtl* mine = pc.p[me];
  if (threadIdx.x == 0) {
    s_epoch = mine->epoch + 1;
    mine->epoch = s_epoch;
  }
  int n_send = 0;
  for (int q = 0; q < G; ++q) n_send += counts[q];
  int32_t* srow = ctl_send(mine, max_rows, 0);
  int32_t* sa = ctl_send(mine, max_rows, 1);
  int32_t* se = ctl_send(mine, max_rows, 2);
  for (int j = threadIdx.x; j < n_send; j += blockDim.x) {
    const int r = send_idx[j];
    srow[j] = r;
    sa[j] = ad[r];
    se[j] = ex ? ex[r] : 0;
  }
  __syncthreads();
  const unsigned int v = s_epoch;
  if (threadIdx.x < G) {
    const int q = threadIdx.x;
    int* mb = pc.p[q]->mbox[v & 1][me];
    for (int k = 0; k <= G; ++k) mb[k] = counts[k];
    __threadfence_system();  // the send arrays (whole CTA, ordered by the barrier) and the row before the flag
    st_release_sys(&pc.p[q]->flag_cnt[me], v);
  }
}

// 1 CTA (owner side, second stream).  Waits for every source's count row of
// this epoch; received rows: by source rank ascending, then each source's
// send order (R18).  Pulls each received row's ids from its source's
// control area and records its origin (source << 24 | source-local row).
// *n_recv = the received row count (0 on a timeout or a layout mismatch, with
// the sticky error flag set).
__global__ void __launch_bounds__(1024) push_recv_prep_kernel(PeerCtl pc, int me, int G, int max_rows, int hash,
                                                              int32_t* __restrict__ ids_a, int32_t* __restrict__ ids_e,
                                                              int32_t* __restrict__ origin, int* __restrict__ n_recv,
                                                              int cap, int* __restrict__ err,
                                                              unsigned long long timeout_ns) {
  __shared__ int s_off[kMaxWorld + 1], s_base[kMaxWorld], s_ok;
  ShardCtl* mine = pc.p[me];
  const unsigned int v = mine->epoch;  // set by this rank's announce (same stream order)
  if (threadIdx.x == 0) s_ok = 1;
  __syncthreads();
  if (threadIdx.x < G) {
    if (!wait_flag(&mine->flag_cnt[threadIdx.x], v, timeout_ns)) {
      atomicOr(err, kErrPeer);
      s_ok = 0;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int off = 0;
    for (int p = 0; p < G; ++p) {
      const volatile int* row = mine->mbox[v & 1][p];
      if (s_ok && row[G] != hash) {
        atomicOr(err, kErrLayout);
        s_ok = 0;
      }
      int base = 0;
      for (int q = 0; q < me; ++q) base += row[q];  // p's rows for owners before me
      s_base[p] = base;
      s_off[p] = off;
      off += row[me];
    }
    if (!s_ok || off > cap) {
      if (off > cap) atomicOr(err, kErrLayout);
      for (int p = 0; p <= G; ++p) s_off[p] = 0;
      off = 0;
    }
    s_off[G] = off;
    *n_recv = off;
  }
  __syncthreads();
  const int n = s_off[G];
  for (int r = threadIdx.x; r < n; r += blockDim.x) {
    int p = 0;
    while (p + 1 < G && s_off[p + 1] <= r) ++p;
    ShardCtl* src = pc.p[p];
    const int j = s_base[p] + (r - s_off[p]);
    const int sstride = src->stride;  // the source's own max_rows (ranks may differ)
    ids_a[r] = ctl_send(src, sstride, 1)[j];
    ids_e[r] = ctl_send(src, sstride, 2)[j];
    origin[r] = (p << kOriginRowBits) | ctl_send(src, sstride, 0)[j];
  }
}

// owner side, after its pushes: release flag "done for epoch v" into every peer
__global__ void push_done_kernel(PeerCtl pc, int me, int G) {
  const unsigned int v = pc.p[me]->epoch;
  __threadfence_system();
  if (threadIdx.x < G) st_release_sys(&pc.p[threadIdx.x]->flag_done[me], v);
}

// source side: wait until every owner has pushed this epoch's deltas
__global__ void push_wait_kernel(PeerCtl pc, int me, int G, int* err, unsigned long long timeout_ns) {
  ShardCtl* mine = pc.p[me];
  const unsigned int v = mine->epoch;
  if (threadIdx.x < G && !wait_flag(&mine->flag_done[threadIdx.x], v, timeout_ns)) atomicOr(err, kErrPeer);
}

}  // namespace

// ---------------------------------------------------------------------------
// host state
// ---------------------------------------------------------------------------
struct RegBuf {
  char* ptr;
  size_t bytes;
};

struct ShardState {
  ncclComm_t comm = nullptr;
  cudaStream_t cs = nullptr;  // communication stream
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  void* buf = nullptr;        // device scratch (grown on demand; NCCL path)
  size_t bytes = 0;
  lora_plan* plan = nullptr;        // owner-side plan over received rows (capacity max_rows * world)
  lora_plan* local_plan = nullptr;  // plan over this rank's rows processed in place
  bool fp32_return = false;
  bool loopback = false;
  // host control plane (lora_server_create_sharded_host): no NCCL at all
  lora_host_allgather_fn host_ag = nullptr;
  void* host_ctx = nullptr;
  int32_t* h_cnt = nullptr;  // pinned [world][world + 1] counts (async read-back, NCCL path)
  // push path: registered buffers and the control areas
  ShardCtl* ctl = nullptr;                 // this rank's control area (IPC-exported)
  size_t ctl_bytes = 0;
  PeerCtl peer_ctl{};
  std::vector<RegBuf> reg;                 // this rank's registered buffers, in registration order
  std::vector<char*> reg_peer;             // [k * world + p] base of buffer k on rank p
  char** d_reg = nullptr;                  // device copy of reg_peer
  std::vector<void*> opened;               // IPC mappings to close at destroy
  int32_t* d_push = nullptr;               // owner side: [3][Rmax] ids_a | ids_e | origin, + n_recv
  unsigned long long timeout_ns = 10ull * 1000 * 1000 * 1000;
};

// Control plane.  Blocking all-gather of small host blobs (IPC handles,
// agreement flags): the caller's host collective, or NCCL through a device
// scratch buffer.
static lora_status_t ctl_allgather(lora_server* s, const void* send_h, void* recv_h, size_t bytes, cudaStream_t st) {
  ShardState* sh = s->shard;
  const int G = s->world, me = s->shard_rank;
  if (sh->host_ag) {
    cudaStreamSynchronize(st);
    if (sh->host_ag(sh->host_ctx, send_h, recv_h, (int64_t)bytes) != 0)
      return fail(s, LORA_ERR_NCCL, "host all-gather callback failed");
    return LORA_OK;
  }
  NcclApi& api = nccl();
  char* d = nullptr;
  if (cudaMalloc(&d, bytes * G) != cudaSuccess) return fail(s, LORA_ERR_OOM, "control buffer");
  cudaMemcpy(d + bytes * me, send_h, bytes, cudaMemcpyHostToDevice);
  const ncclResult_t r = api.AllGather(d + bytes * me, d, bytes, ncclUint8, sh->comm, st);
  cudaStreamSynchronize(st);
  if (r == ncclSuccess) cudaMemcpy(recv_h, d, bytes * G, cudaMemcpyDeviceToHost);
  cudaFree(d);
  return r == ncclSuccess ? LORA_OK : fail(s, LORA_ERR_NCCL, std::string("all-gather: ") + api.GetErrorString(r));
}

// Release the peer mappings, the control area and the registration tables.
static void push_release(ShardState* sh) {
  for (void* p : sh->opened) cudaIpcCloseMemHandle(p);
  sh->opened.clear();
  cudaFree(sh->ctl);
  cudaFree(sh->d_reg);
  cudaFree(sh->d_push);
  sh->ctl = nullptr;
  sh->d_reg = nullptr;
  sh->d_push = nullptr;
  sh->reg.clear();
  sh->reg_peer.clear();
  sh->peer_ctl = PeerCtl{};
}

void lora_shard_free(lora_server* s) {
  if (!s || !s->shard) return;
  ShardState* sh = s->shard;
  push_release(sh);
  if (sh->h_cnt) cudaFreeHost(sh->h_cnt);
  if (sh->comm && nccl().ok) nccl().CommDestroy(sh->comm);
  cudaFree(sh->buf);
  if (sh->plan) plan_destroy_impl(sh->plan);
  if (sh->local_plan) plan_destroy_impl(sh->local_plan);
  for (auto& e : sh->ev)
    if (e) cudaEventDestroy(e);
  if (sh->cs) cudaStreamDestroy(sh->cs);
  delete sh;
  s->shard = nullptr;
}

// sticky-flag bits beyond "bad id" (lora_server_check); NCCL asynchronous errors
lora_status_t lora_shard_check_flags(lora_server* s, int flag) {
  if (flag & kErrLayout)
    return fail(s, LORA_ERR_PEER, "sharded apply: ranks disagreed on the call's layout (slots / buffers / dtype)");
  if (flag & kErrPeer) return fail(s, LORA_ERR_PEER, "sharded apply: a peer did not signal in time");
  if (s->shard && s->shard->comm && nccl().ok && nccl().CommGetAsyncError) {
    ncclResult_t ar = ncclSuccess;
    if (nccl().CommGetAsyncError(s->shard->comm, &ar) == ncclSuccess && ar != ncclSuccess && ar != ncclInProgress)
      return fail(s, LORA_ERR_NCCL, std::string("NCCL asynchronous error: ") + nccl().GetErrorString(ar));
  }
  return LORA_OK;
}

extern "C" lora_status_t lora_shard_layout(const int64_t* counts, int32_t world, int32_t rank, int64_t* send_off,
                                           int64_t* recv_off) {
  if (!counts || !send_off || !recv_off || world < 1 || rank < 0 || rank >= world)
    return fail(nullptr, LORA_ERR_INVALID_ARG, "lora_shard_layout: bad argument");
  send_off[0] = 0;
  recv_off[0] = 0;
  for (int p = 0; p < world; ++p) {
    if (counts[(size_t)rank * world + p] < 0 || counts[(size_t)p * world + rank] < 0)
      return fail(nullptr, LORA_ERR_INVALID_ARG, "lora_shard_layout: negative count");
    send_off[p + 1] = send_off[p] + counts[(size_t)rank * world + p];  // my rows for owner p
    recv_off[p + 1] = recv_off[p] + counts[(size_t)p * world + rank];  // rows source p sends me
  }
  return LORA_OK;
}

extern "C" lora_status_t lora_shard_peer_rows(const int64_t* counts, int32_t world, int32_t rank, int64_t* in_rowbase,
                                              int64_t* out_rowbase) {
  if (!counts || !in_rowbase || !out_rowbase || world < 1 || rank < 0 || rank >= world)
    return fail(nullptr, LORA_ERR_INVALID_ARG, "lora_shard_peer_rows: bad argument");
  std::vector<int64_t> so(world + 1), ro(world + 1);
  lora_status_t st = lora_shard_layout(counts, world, rank, so.data(), ro.data());
  if (st != LORA_OK) return st;
  for (int p = 0; p < world; ++p) {
    int64_t before_me_in_p = 0, before_me_at_p = 0;
    for (int q = 0; q < rank; ++q) before_me_in_p += counts[(size_t)p * world + q];  // p's rows for owners < rank
    for (int q = 0; q < rank; ++q) before_me_at_p += counts[(size_t)q * world + p];  // owner p's rows from sources < rank
    in_rowbase[p] = before_me_in_p - ro[p];
    out_rowbase[p] = before_me_at_p - so[p];
  }
  return LORA_OK;
}

extern "C" lora_status_t lora_nccl_unique_id(void* out128) {
  if (!out128) return fail(nullptr, LORA_ERR_INVALID_ARG, "NULL out");
  NcclApi& api = nccl();
  if (!api.ok) return fail(nullptr, LORA_ERR_NCCL, api.err);
  ncclUniqueId id;
  ncclResult_t r = api.GetUniqueId(&id);
  if (r != ncclSuccess) return fail(nullptr, LORA_ERR_NCCL, api.GetErrorString(r));
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  std::memcpy(out128, &id, 128);
  return LORA_OK;
}

static lora_status_t create_sharded_impl(const lora_config_t* cfg, int32_t rank, int32_t world,
                                         const void* nccl_unique_id, lora_host_allgather_fn host_ag, void* host_ctx,
                                         lora_server_t** out);

extern "C" lora_status_t lora_server_create_sharded(const lora_config_t* cfg, int32_t rank, int32_t world,
                                                    const void* nccl_unique_id, lora_server_t** out) {
  if (!nccl_unique_id) return fail(nullptr, LORA_ERR_INVALID_ARG, "lora_server_create_sharded: NULL unique id");
  return create_sharded_impl(cfg, rank, world, nccl_unique_id, nullptr, nullptr, out);
}

extern "C" lora_status_t lora_server_create_sharded_host(const lora_config_t* cfg, int32_t rank, int32_t world,
                                                         lora_host_allgather_fn allgather, void* ctx,
                                                         lora_server_t** out) {
  if (!allgather) return fail(nullptr, LORA_ERR_INVALID_ARG, "lora_server_create_sharded_host: NULL all-gather");
  return create_sharded_impl(cfg, rank, world, nullptr, allgather, ctx, out);
}

static lora_status_t create_sharded_impl(const lora_config_t* cfg, int32_t rank, int32_t world,
                                         const void* nccl_unique_id, lora_host_allgather_fn host_ag, void* host_ctx,
                                         lora_server_t** out) {
  if (!cfg || !out || world < 1 || rank < 0 || rank >= world)
    return fail(nullptr, LORA_ERR_INVALID_ARG, "lora_server_create_sharded: bad argument");
  if (world > kMaxWorld) return fail(nullptr, LORA_ERR_UNSUPPORTED, "world > 8 (one NVLink domain of B200s)");
  if ((long long)cfg->max_rows * world > kMaxPlanRows)  // the owner's plan holds every rank's rows at worst
    return fail(nullptr, LORA_ERR_UNSUPPORTED, "max_rows * world must be <= 32768 (owner-side plan capacity)");
  if (cfg->max_rows >= (1 << kOriginRowBits)) return fail(nullptr, LORA_ERR_UNSUPPORTED, "max_rows too large");
  if (cfg->n_replicated < 0) return fail(nullptr, LORA_ERR_INVALID_ARG, "n_replicated < 0");
  NcclApi& api = nccl();
  if (!host_ag && !api.ok) return fail(nullptr, LORA_ERR_NCCL, api.err);
  lora_status_t st = create_common_sharded(cfg, world, rank, out, cfg->n_replicated, cfg->expert_parallel);
  if (st != LORA_OK) return st;
  lora_server* s = *out;
  s->shard = new ShardState();
  ShardState* sh = s->shard;
  sh->host_ag = host_ag;
  sh->host_ctx = host_ctx;
  const char* f32 = std::getenv("LORA_SHARD_FP32");
  sh->fp32_return = f32 && f32[0] && std::strcmp(f32, "0") != 0;
  const char* lb = std::getenv("LORA_SHARD_LOOPBACK");
  sh->loopback = lb && lb[0] && std::strcmp(lb, "0") != 0;
  if (const char* to = std::getenv("LORA_SHARD_TIMEOUT_MS"))
    sh->timeout_ns = (unsigned long long)std::max(1L, std::atol(to)) * 1000000ull;
  cudaSetDevice(s->device);
  bool ok = cudaStreamCreateWithFlags(&sh->cs, cudaStreamNonBlocking) == cudaSuccess;
  for (auto& e : sh->ev) ok = ok && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess;
  ok = ok && cudaMallocHost(&sh->h_cnt, sizeof(int32_t) * world * (world + 1)) == cudaSuccess;
  if (!ok) {
    lora_server_destroy(s);
    *out = nullptr;
    return fail(nullptr, LORA_ERR_CUDA, "stream / event / pinned allocation failed");
  }
  if (!host_ag) {
    ncclUniqueId id;
    std::memcpy(&id, nccl_unique_id, 128);
    ncclResult_t r = api.CommInitRank(&sh->comm, world, id, rank);
    if (r != ncclSuccess) {
      std::string m = std::string("ncclCommInitRank: ") + api.GetErrorString(r);
      lora_server_destroy(s);
      *out = nullptr;
      return fail(nullptr, LORA_ERR_NCCL, m);
    }
  }
  st = plan_create_impl(s, cfg->max_rows * world, &sh->plan);
  if (st == LORA_OK) st = plan_create_impl(s, cfg->max_rows, &sh->local_plan);
  if (st != LORA_OK) {
    std::string m = s->last_error;
    lora_server_destroy(s);
    *out = nullptr;
    return fail(nullptr, st, m);
  }
  // the owner plan's tcgen05 shrink split follows the typical received count
  // (about one rank's rows), not its capacity
  sh->plan->T_hint = cfg->max_rows;
  return LORA_OK;
}

// ---------------------------------------------------------------------------
// registration (collective): CUDA IPC export of the allocation holding each
// buffer, all-gathered; every peer's allocations mapped once each
// ---------------------------------------------------------------------------
typedef CUresult (*PFN_memGetAddressRange)(CUdeviceptr*, size_t*, CUdeviceptr);
static PFN_memGetAddressRange address_range_fn() {
  static PFN_memGetAddressRange fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    cudaGetLastError();
    return reinterpret_cast<PFN_memGetAddressRange>(f);
  }();
  return fn;
}

struct RegInfo {  // one exported buffer (all-gathered)
  cudaIpcMemHandle_t h;
  int64_t offset;   // buffer start - allocation base
  int64_t bytes;
};

// export one buffer: handle of its allocation + offset (ok = false on failure)
static bool export_buffer(const void* ptr, size_t bytes, RegInfo& ri) {
  std::memset(&ri, 0, sizeof(ri));
  auto range = address_range_fn();
  CUdeviceptr base = 0;
  size_t size = 0;
  if (!range || range(&base, &size, reinterpret_cast<CUdeviceptr>(ptr)) != CUDA_SUCCESS) return false;
  if (reinterpret_cast<uintptr_t>(ptr) + bytes > base + size) return false;
  if (cudaIpcGetMemHandle(&ri.h, reinterpret_cast<void*>(base)) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  ri.offset = (int64_t)(reinterpret_cast<uintptr_t>(ptr) - base);
  ri.bytes = (int64_t)bytes;
  return true;
}

extern "C" lora_status_t lora_shard_register(lora_server_t* s, int32_t n, void* const* ptrs, const int64_t* bytes,
                                             void* stream) {
  if (!s) return fail(nullptr, LORA_ERR_INVALID_ARG, "server is NULL");
  if (!s->shard) return fail(s, LORA_ERR_INVALID_ARG, "not a sharded server");
  if (n < 0 || (n > 0 && (!ptrs || !bytes))) return fail(s, LORA_ERR_INVALID_ARG, "bad buffer list");
  ShardState* sh = s->shard;
  const int G = s->world, me = s->shard_rank;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (cudaSetDevice(s->device) != cudaSuccess) return fail(s, LORA_ERR_CUDA, "cudaSetDevice");
  cudaStreamSynchronize(st);
  cudaStreamSynchronize(sh->cs);
  int ok = 1;
  for (int i = 0; i < n; ++i)
    if (!ptrs[i] || bytes[i] <= 0) ok = 0;
  // the control area (first registration)
  bool new_ctl = false;
  if (!sh->ctl) {
    sh->ctl_bytes = sizeof(ShardCtl) + sizeof(int32_t) * 3 * (size_t)s->max_rows;
    const int stride = s->max_rows;
    if (cudaMalloc(&sh->ctl, sh->ctl_bytes) != cudaSuccess ||
        cudaMemset(sh->ctl, 0, sh->ctl_bytes) != cudaSuccess ||
        cudaMemcpy(&sh->ctl->stride, &stride, sizeof(int), cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMalloc(&sh->d_push, sizeof(int32_t) * (3 * (size_t)s->max_rows * G + 4)) != cudaSuccess) {
      cudaGetLastError();
      ok = 0;
    }
    new_ctl = true;
  }
  // blob: [n | ok | pad] [ctl RegInfo] [n RegInfo]
  const size_t blob = 16 + sizeof(RegInfo) * (1 + (size_t)n);
  std::vector<char> mine(blob, 0), all(blob * G, 0);
  RegInfo* ri = reinterpret_cast<RegInfo*>(mine.data() + 16);
  if (ok && new_ctl && !export_buffer(sh->ctl, sh->ctl_bytes, ri[0])) ok = 0;
  for (int i = 0; i < n && ok; ++i)
    if (!export_buffer(ptrs[i], (size_t)bytes[i], ri[1 + i])) ok = 0;
  reinterpret_cast<int32_t*>(mine.data())[0] = n;
  reinterpret_cast<int32_t*>(mine.data())[1] = ok;
  lora_status_t rc = ctl_allgather(s, mine.data(), all.data(), blob, st);
  if (rc != LORA_OK) return rc;
  for (int p = 0; p < G; ++p) {
    const int32_t* hd = reinterpret_cast<const int32_t*>(all.data() + blob * p);
    if (hd[0] != n) ok = 0;  // every rank must register the same number of buffers
    if (!hd[1]) ok = 0;
  }
  // map every peer's allocations (each distinct handle once per peer)
  std::vector<char*> ctl_peer(G, nullptr), peer_base((size_t)n * G, nullptr);
  std::vector<std::pair<std::string, void*>> mapped;
  auto open = [&](const cudaIpcMemHandle_t& h) -> char* {
    const std::string key(reinterpret_cast<const char*>(&h), sizeof(h));
    for (auto& m : mapped)
      if (m.first == key) return static_cast<char*>(m.second);
    void* a = nullptr;
    if (cudaIpcOpenMemHandle(&a, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    mapped.push_back({key, a});
    sh->opened.push_back(a);
    return static_cast<char*>(a);
  };
  for (int p = 0; p < G && ok; ++p) {
    const RegInfo* pr = reinterpret_cast<const RegInfo*>(all.data() + blob * p + 16);
    if (p == me) {
      ctl_peer[p] = reinterpret_cast<char*>(sh->ctl);
      for (int i = 0; i < n; ++i) peer_base[(size_t)i * G + p] = static_cast<char*>(ptrs[i]);
      continue;
    }
    mapped.clear();  // handles are per exporting process
    if (new_ctl) {
      char* b = open(pr[0].h);
      if (!b) ok = 0;
      ctl_peer[p] = b ? b + pr[0].offset : nullptr;
    }
    for (int i = 0; i < n && ok; ++i) {
      char* b = open(pr[1 + i].h);
      if (!b) ok = 0;
      peer_base[(size_t)i * G + p] = b ? b + pr[1 + i].offset : nullptr;
    }
  }
  // every rank must agree that every mapping worked
  std::vector<int32_t> oks(G, 0);
  rc = ctl_allgather(s, &ok, oks.data(), sizeof(int32_t), st);
  if (rc != LORA_OK) return rc;
  for (int v : oks) ok = ok && v;
  if (!ok) {
    push_release(sh);
    return fail(s, LORA_ERR_UNSUPPORTED,
                "lora_shard_register: a buffer could not be exported or mapped on some rank (every rank released "
                "its registrations)");
  }
  if (new_ctl)
    for (int p = 0; p < G; ++p) sh->peer_ctl.p[p] = reinterpret_cast<ShardCtl*>(ctl_peer[p]);
  for (int i = 0; i < n; ++i) {
    sh->reg.push_back({static_cast<char*>(ptrs[i]), (size_t)bytes[i]});
    for (int p = 0; p < G; ++p) sh->reg_peer.push_back(peer_base[(size_t)i * G + p]);
  }
  cudaFree(sh->d_reg);
  sh->d_reg = nullptr;
  if (!sh->reg_peer.empty()) {
    if (cudaMalloc(&sh->d_reg, sizeof(char*) * sh->reg_peer.size()) != cudaSuccess ||
        cudaMemcpy(sh->d_reg, sh->reg_peer.data(), sizeof(char*) * sh->reg_peer.size(), cudaMemcpyHostToDevice) !=
            cudaSuccess)
      return fail(s, LORA_ERR_OOM, "registration table");
  }
  return LORA_OK;
}

#define CKS(call)                                                 \
  do {                                                            \
    cudaError_t _e = (call);                                      \
    if (_e != cudaSuccess) return cuda_fail(s, _e, #call);        \
  } while (0)
#define CKN(call)                                                                        \
  do {                                                                                   \
    ncclResult_t _r = (call);                                                            \
    if (_r != ncclSuccess) return fail(s, LORA_ERR_NCCL, std::string(#call ": ") + api.GetErrorString(_r)); \
  } while (0)

// index of a registered buffer starting at p (-1: none)
static int reg_index(const ShardState* sh, const void* p) {
  for (size_t k = 0; k < sh->reg.size(); ++k)
    if (sh->reg[k].ptr == p) return (int)k;
  return -1;
}

// FNV-1a over the call's layout: every rank must pass the same slots in the
// same order, the same registered-buffer roles and the same y dtype
static int layout_hash(int n, const int32_t* slots, const std::vector<int>& xk, const std::vector<int>& yk,
                       lora_dtype_t dt) {
  uint32_t h = 2166136261u;
  auto mix = [&](int v) {
    for (int b = 0; b < 4; ++b) {
      h ^= (uint32_t)((v >> (8 * b)) & 0xFF);
      h *= 16777619u;
    }
  };
  mix(n);
  mix((int)dt);
  for (int i = 0; i < n; ++i) {
    mix(slots[i]);
    mix(xk[i]);
    mix(yk[i]);
  }
  return (int)(h & 0x7FFFFFFF);
}

// ---------------------------------------------------------------------------
// the push path
// ---------------------------------------------------------------------------
static lora_status_t apply_sharded_push(lora_server* s, int n, const int32_t* slots, const void* const* x,
                                        const int32_t* adapter_ids, const int32_t* expert_ids, void* const* y,
                                        lora_dtype_t y_dtype, int T, cudaStream_t st, const std::vector<int>& xk,
                                        const std::vector<int>& yk) {
  ShardState* sh = s->shard;
  const int G = s->world, me = s->shard_rank;
  const int E = s->slots[slots[0]].E;
  const Placement pl = slot_placement(s, slots[0]);  // (EP_x-PP_y: the group of the call's layer)
  const bool in_group = !pl.ep || pl.erank() >= 0;   // ranks outside it serve nothing, send everything
  const long long Rmax = (long long)s->max_rows * G;
  const int hash = layout_hash(n, slots, xk, yk, y_dtype);
  // scratch: counts [G + 1], send_idx [max_rows], ad_local [max_rows]
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  const size_t o_counts = 0, o_send_idx = al(sizeof(int32_t) * (G + 1)),
               o_ad_local = o_send_idx + al(sizeof(int32_t) * s->max_rows),
               need = o_ad_local + al(sizeof(int32_t) * s->max_rows);
  if (need > sh->bytes) {
    cudaStreamSynchronize(st);
    cudaStreamSynchronize(sh->cs);
    cudaFree(sh->buf);
    sh->buf = nullptr;
    sh->bytes = 0;
    CKS(cudaMalloc(&sh->buf, need));
    sh->bytes = need;
  }
  char* base = static_cast<char*>(sh->buf);
  int32_t* d_counts = reinterpret_cast<int32_t*>(base + o_counts);
  int32_t* d_send_idx = reinterpret_cast<int32_t*>(base + o_send_idx);
  int32_t* d_ad_local = reinterpret_cast<int32_t*>(base + o_ad_local);
  int32_t* ids_a = sh->d_push;
  int32_t* ids_e = ids_a + Rmax;
  int32_t* origin = ids_e + Rmax;
  int* n_recv = origin + Rmax;

  // 1. bucket + announce
  int pi = prof_start(s, st);
  bucket_kernel<<<1, kBucketThreads, 0, st>>>(adapter_ids, expert_ids, T, pl, s->n_adapters, E, sh->loopback,
                                              d_ad_local, d_send_idx, d_counts, s->d_err, hash);
  push_announce_kernel<<<1, 1024, 0, st>>>(sh->peer_ctl, me, G, s->max_rows, d_counts, d_send_idx, adapter_ids,
                                           expert_ids);
  prof_stop(s, pi, kKShardBucket, st);
  CKS(cudaGetLastError());
  // 2. owner side on the communication stream (overlaps the in-place apply)
  CKS(cudaEventRecord(sh->ev[0], st));
  CKS(cudaStreamWaitEvent(sh->cs, sh->ev[0], 0));
  pi = prof_start(s, sh->cs);
  push_recv_prep_kernel<<<1, 1024, 0, sh->cs>>>(sh->peer_ctl, me, G, s->max_rows, hash, ids_a, ids_e, origin, n_recv,
                                                (int)Rmax, s->d_err, sh->timeout_ns);
  prof_stop(s, pi, kKShardGather, sh->cs);
  CKS(cudaGetLastError());
  lora_status_t rc = LORA_OK;
  if (in_group) {
    rc = plan_build_impl(s, sh->plan, ids_a, ids_e, (int)Rmax, E, sh->cs, n_recv);
    if (rc != LORA_OK) return rc;
  }
  CKS(cudaEventRecord(sh->ev[1], sh->cs));
  //    in-place rows (this rank's own or replicated units)
  if (in_group && T > 0) {
    rc = plan_build_impl(s, sh->local_plan, d_ad_local, expert_ids, T, E, st);
    if (rc != LORA_OK) return rc;
    rc = apply_multi_impl(s, sh->local_plan, n, slots, x, y, y_dtype, st);
    if (rc != LORA_OK) return rc;
  }
  // 3. owner apply: remote-x shrink, push-add expand
  CKS(cudaStreamWaitEvent(st, sh->ev[1], 0));
  if (in_group) {
    PushIn push{G, origin, sh->d_reg};
    std::vector<int16_t> xr(n), yr(n);
    for (int i = 0; i < n; ++i) {
      xr[i] = (int16_t)xk[i];
      yr[i] = (int16_t)yk[i];
    }
    rc = apply_multi_impl(s, sh->plan, n, slots, x, y, y_dtype, st, 3, &push, xr.data(), yr.data());
    if (rc != LORA_OK) return rc;
  }
  // 4. done -> peers; wait for every owner's pushes into this rank's y
  pi = prof_start(s, st);
  push_done_kernel<<<1, 32, 0, st>>>(sh->peer_ctl, me, G);
  push_wait_kernel<<<1, 32, 0, st>>>(sh->peer_ctl, me, G, s->d_err, sh->timeout_ns);
  prof_stop(s, pi, kKShardScatter, st);
  CKS(cudaGetLastError());
  if (s->debug_sync) CKS(cudaStreamSynchronize(st));
  return LORA_OK;
}

// ---------------------------------------------------------------------------
// the NCCL path (unregistered buffers)
// ---------------------------------------------------------------------------
static lora_status_t apply_sharded_nccl(lora_server* s, int n, const int32_t* slots, const void* const* x,
                                        const int32_t* adapter_ids, const int32_t* expert_ids, void* const* y,
                                        lora_dtype_t y_dtype, int T, cudaStream_t st) {
  NcclApi& api = nccl();
  const int G = s->world, me = s->shard_rank;
  const Placement pl = slot_placement(s, slots[0]);  // (EP_x-PP_y: the group of the call's layer)
  const bool in_group = !pl.ep || pl.erank() >= 0;
  ShardState* sh = s->shard;
  cudaStream_t cs = sh->cs;
  const int E = s->slots[slots[0]].E;
  const bool d_bf16 = (y_dtype == LORA_BF16) && !sh->fp32_return;
  const size_t dsz = d_bf16 ? 2 : 4;

  // distinct x buffers (send-buffer regions, one NCCL message each)
  std::vector<const void*> xd;
  std::vector<int> x_of(n);
  for (int i = 0; i < n; ++i) {
    int j = 0;
    while (j < (int)xd.size() && xd[j] != x[i]) ++j;
    if (j == (int)xd.size()) xd.push_back(x[i]);
    x_of[i] = j;
  }
  std::vector<int> x_hin(xd.size());
  for (int i = 0; i < n; ++i) x_hin[x_of[i]] = s->slots[slots[i]].h_in;
  // the message layout depends on this x de-duplication: every rank must get
  // the same pattern (checked through the hash word of the count exchange)
  std::vector<int> yk(n, 0);
  const int hash = layout_hash(n, slots, x_of, yk, y_dtype);

  // scratch layout (worst case: every rank sends every row to me -> G*T rows)
  const long long Rmax = (long long)s->max_rows * G;
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  size_t off = 0;
  const size_t o_counts = off; off += al(sizeof(int32_t) * (G + 1) * (G + 1));
  const size_t o_send_idx = off; off += al(sizeof(int32_t) * s->max_rows);
  const size_t o_ad_local = off; off += al(sizeof(int32_t) * s->max_rows);
  const size_t o_ids_send = off; off += al(sizeof(int32_t) * 2 * s->max_rows);
  const size_t o_ids_recv = off; off += al(sizeof(int32_t) * 2 * Rmax);
  std::vector<size_t> o_xs(xd.size()), o_xr(xd.size());
  for (size_t j = 0; j < xd.size(); ++j) {
    o_xs[j] = off; off += al((size_t)s->max_rows * x_hin[j] * 2);
    o_xr[j] = off; off += al((size_t)Rmax * x_hin[j] * 2);
  }
  std::vector<size_t> o_d(n), o_dr(n);
  for (int i = 0; i < n; ++i) {
    o_d[i] = off; off += al((size_t)Rmax * s->slots[slots[i]].h_out * dsz);         // owner-side deltas
    o_dr[i] = off; off += al((size_t)s->max_rows * s->slots[slots[i]].h_out * dsz);  // returned deltas
  }
  if (off > sh->bytes) {
    cudaStreamSynchronize(st);
    cudaStreamSynchronize(cs);
    cudaFree(sh->buf);
    sh->buf = nullptr;
    sh->bytes = 0;
    CKS(cudaMalloc(&sh->buf, off));
    sh->bytes = off;
  }
  char* base = static_cast<char*>(sh->buf);
  int32_t* d_counts = reinterpret_cast<int32_t*>(base + o_counts);  // [G+1] mine, then [G][G+1] gathered
  int32_t* d_send_idx = reinterpret_cast<int32_t*>(base + o_send_idx);
  int32_t* d_ad_local = reinterpret_cast<int32_t*>(base + o_ad_local);
  int32_t* d_ids_send = reinterpret_cast<int32_t*>(base + o_ids_send);  // [2][max_rows] (a | e) in send order
  int32_t* d_ids_recv = reinterpret_cast<int32_t*>(base + o_ids_recv);  // [2][Rmax]

  // 1. classify + bucket.  The previous call's comm-stream work (reads of the
  //    scratch) must be done before it is overwritten: ev[3] was recorded last.
  CKS(cudaStreamWaitEvent(st, sh->ev[3], 0));
  const int pi = prof_start(s, st);
  bucket_kernel<<<1, kBucketThreads, 0, st>>>(adapter_ids, expert_ids, T, pl, s->n_adapters, E, sh->loopback,
                                              d_ad_local, d_send_idx, d_counts, s->d_err, hash);
  prof_stop(s, pi, kKShardBucket, st);
  CKS(cudaGetLastError());
  // 2. counts exchange (all-gather) + the one host wait; the in-place rows'
  //    plan and apply are enqueued before the host waits for the matrix.
  CKN(api.AllGather(d_counts, d_counts + (G + 1), G + 1, ncclInt32, sh->comm, st));
  CKS(cudaMemcpyAsync(sh->h_cnt, d_counts + (G + 1), sizeof(int32_t) * G * (G + 1), cudaMemcpyDeviceToHost, st));
  CKS(cudaEventRecord(sh->ev[0], st));  // bucket outputs + counts ready (the pack waits on this)
  lora_status_t rc = LORA_OK;
  if (in_group && T > 0) {
    rc = plan_build_impl(s, sh->local_plan, d_ad_local, expert_ids, T, E, st);
    if (rc != LORA_OK) return rc;
    rc = apply_multi_impl(s, sh->local_plan, n, slots, x, y, y_dtype, st);
    if (rc != LORA_OK) return rc;
  }
  CKS(cudaEventSynchronize(sh->ev[0]));
  std::vector<int64_t> c64((size_t)G * G), so(G + 1), ro(G + 1);
  for (int p = 0; p < G; ++p) {
    if (sh->h_cnt[p * (G + 1) + G] != hash)  // every rank sees every hash: all fail together
      return fail(s, LORA_ERR_INVALID_ARG, "sharded apply: ranks disagree on the call's layout (slots / x buffers / "
                                           "dtype); nothing exchanged");
    for (int q = 0; q < G; ++q) c64[(size_t)p * G + q] = sh->h_cnt[p * (G + 1) + q];
  }
  lora_status_t lr = lora_shard_layout(c64.data(), G, me, so.data(), ro.data());
  if (lr != LORA_OK) return fail(s, lr, "count exchange produced an invalid matrix");
  const int n_send = (int)so[G], n_recv = (int)ro[G];
  if (n_recv > Rmax) return fail(s, LORA_ERR_INVALID_ARG, "received rows exceed capacity");
  bool exchange = false;  // every rank sees the same matrix, so every rank takes the same branch
  for (int64_t v : c64) exchange = exchange || v > 0;
  if (!exchange) {
    CKS(cudaEventRecord(sh->ev[3], st));
    return LORA_OK;
  }

  // 3. (comm stream) pack + grouped send/recv, overlapped with the in-place apply
  CKS(cudaStreamWaitEvent(cs, sh->ev[0], 0));
  if (n_send > 0) {
    const int pg = prof_start(s, cs);
    gather_words_kernel<<<grid_of(n_send), 256, 0, cs>>>(reinterpret_cast<const uint32_t*>(adapter_ids),
                                                          reinterpret_cast<uint32_t*>(d_ids_send), d_send_idx, n_send);
    if (expert_ids)
      gather_words_kernel<<<grid_of(n_send), 256, 0, cs>>>(reinterpret_cast<const uint32_t*>(expert_ids),
                                                            reinterpret_cast<uint32_t*>(d_ids_send + s->max_rows),
                                                            d_send_idx, n_send);
    else
      CKS(cudaMemsetAsync(d_ids_send + s->max_rows, 0, sizeof(int32_t) * n_send, cs));
    for (size_t j = 0; j < xd.size(); ++j) {
      const int chunks = x_hin[j] / 8;  // 16-byte chunks per bf16 row
      gather_rows16_kernel<<<dim3((chunks + 255) / 256, std::min(n_send, 65535)), 256, 0, cs>>>(
          static_cast<const uint4*>(xd[j]), reinterpret_cast<uint4*>(base + o_xs[j]), d_send_idx, n_send, chunks);
    }
    prof_stop(s, pg, kKShardGather, cs);
    CKS(cudaGetLastError());
  }
  CKN(api.GroupStart());
  for (int p = 0; p < G; ++p) {
    const size_t ns = so[p + 1] - so[p], nr = ro[p + 1] - ro[p];
    if (ns) {
      CKN(api.Send(d_ids_send + so[p], ns, ncclInt32, p, sh->comm, cs));
      CKN(api.Send(d_ids_send + s->max_rows + so[p], ns, ncclInt32, p, sh->comm, cs));
      for (size_t j = 0; j < xd.size(); ++j)
        CKN(api.Send(base + o_xs[j] + so[p] * x_hin[j] * 2, ns * x_hin[j], ncclBfloat16, p, sh->comm, cs));
    }
    if (nr) {
      CKN(api.Recv(d_ids_recv + ro[p], nr, ncclInt32, p, sh->comm, cs));
      CKN(api.Recv(d_ids_recv + Rmax + ro[p], nr, ncclInt32, p, sh->comm, cs));
      for (size_t j = 0; j < xd.size(); ++j)
        CKN(api.Recv(base + o_xr[j] + ro[p] * x_hin[j] * 2, nr * x_hin[j], ncclBfloat16, p, sh->comm, cs));
    }
  }
  CKN(api.GroupEnd());
  //    owner side, still on the communication stream: the received rows' plan
  if (n_recv > 0) {
    rc = plan_build_impl(s, sh->plan, d_ids_recv, d_ids_recv + Rmax, n_recv, E, cs);
    if (rc != LORA_OK) return rc;
  }
  CKS(cudaEventRecord(sh->ev[1], cs));

  // 4. received rows: delta-mode apply (n_recv > 0 only inside the call's group)
  CKS(cudaStreamWaitEvent(st, sh->ev[1], 0));
  if (n_recv > 0) {
    std::vector<const void*> xs(n);
    std::vector<void*> ds(n);
    for (int i = 0; i < n; ++i) {
      xs[i] = base + o_xr[x_of[i]];
      ds[i] = base + o_d[i];
    }
    rc = apply_multi_delta(s, sh->plan, n, slots, xs.data(), ds.data(), st, d_bf16);
    if (rc != LORA_OK) return rc;
  }
  // 5. (comm stream) return the deltas
  CKS(cudaEventRecord(sh->ev[2], st));
  CKS(cudaStreamWaitEvent(cs, sh->ev[2], 0));
  const ncclDataType_t dt = d_bf16 ? ncclBfloat16 : ncclFloat32;
  CKN(api.GroupStart());
  for (int p = 0; p < G; ++p) {
    const size_t ns = so[p + 1] - so[p], nr = ro[p + 1] - ro[p];
    for (int i = 0; i < n; ++i) {
      const int ho = s->slots[slots[i]].h_out;
      if (nr) CKN(api.Send(base + o_d[i] + ro[p] * ho * dsz, nr * ho, dt, p, sh->comm, cs));
      if (ns) CKN(api.Recv(base + o_dr[i] + so[p] * ho * dsz, ns * ho, dt, p, sh->comm, cs));
    }
  }
  CKN(api.GroupEnd());
  CKS(cudaEventRecord(sh->ev[3], cs));
  CKS(cudaStreamWaitEvent(st, sh->ev[3], 0));

  // 6. add the returned deltas at the origin rows
  if (n_send > 0) {
    for (int i = 0; i < n; ++i) {
      const int ho = s->slots[slots[i]].h_out;
      const int ps = prof_start(s, st);
      scatter_add4_kernel<<<dim3((ho / 4 + 255) / 256, std::min(n_send, 65535)), 256, 0, st>>>(
          y[i], y_dtype == LORA_FP32, base + o_dr[i], d_bf16 ? 1 : 0, d_send_idx, n_send, ho);
      prof_stop(s, ps, kKShardScatter, st);
    }
    CKS(cudaGetLastError());
  }
  CKS(cudaEventRecord(sh->ev[3], st));
  if (s->debug_sync) CKS(cudaStreamSynchronize(st));
  return LORA_OK;
}

extern "C" lora_status_t lora_apply_sharded(lora_server_t* s, int32_t n, const int32_t* slots, const void* const* x,
                                            const int32_t* adapter_ids, const int32_t* expert_ids, void* const* y,
                                            lora_dtype_t y_dtype, int32_t T, void* stream) {
  if (!s) return fail(nullptr, LORA_ERR_INVALID_ARG, "server is NULL");
  if (!s->shard) return fail(s, LORA_ERR_INVALID_ARG, "not a sharded server");
  if (n < 1 || !slots || !x || !y || (T > 0 && !adapter_ids)) return fail(s, LORA_ERR_INVALID_ARG, "NULL argument");
  if (T < 0 || T > s->max_rows) return fail(s, LORA_ERR_INVALID_ARG, "T must be in [0, max_rows]");
  if (y_dtype != LORA_BF16 && y_dtype != LORA_FP32) return fail(s, LORA_ERR_UNSUPPORTED, "y_dtype");
  if (n > kMaxTasks) return fail(s, LORA_ERR_UNSUPPORTED, "at most 128 slots per sharded apply");
  for (int i = 0; i < n; ++i)
    if (slots[i] < 0 || slots[i] >= (int)s->slots.size()) return fail(s, LORA_ERR_INVALID_ARG, "bad slot index");
  const int E = s->slots[slots[0]].E;
  for (int i = 0; i < n; ++i) {
    if (s->slots[slots[i]].E != E) return fail(s, LORA_ERR_INVALID_ARG, "slots of one call must share n_experts");
    if (slot_placement(s, slots[i]).gbase != slot_placement(s, slots[0]).gbase)
      return fail(s, LORA_ERR_INVALID_ARG, "EP_x-PP_y: the slots of one call must belong to one pipeline group");
  }
  ShardState* sh = s->shard;
  CKS(cudaSetDevice(s->device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // registered buffers -> the push path (x and y must lie inside their
  // registered buffers for T rows)
  std::vector<int> xk(n, -1), yk(n, -1);
  bool all_reg = sh->ctl != nullptr;
  for (int i = 0; i < n && all_reg; ++i) {
    xk[i] = reg_index(sh, x[i]);
    yk[i] = reg_index(sh, y[i]);
    const SlotInfo& si = s->slots[slots[i]];
    const size_t ysz = y_dtype == LORA_FP32 ? 4 : 2;
    all_reg = xk[i] >= 0 && yk[i] >= 0 && sh->reg[xk[i]].bytes >= (size_t)T * si.h_in * 2 &&
              sh->reg[yk[i]].bytes >= (size_t)T * si.h_out * ysz;
  }
  if (all_reg) return apply_sharded_push(s, n, slots, x, adapter_ids, expert_ids, y, y_dtype, T, st, xk, yk);
  // once buffers are registered every call must use registered x / y: a rank
  // taking the NCCL path while its peers push would block them (they time out)
  if (sh->ctl)
    return fail(s, LORA_ERR_INVALID_ARG,
                "this server has registered buffers: x[i] / y[i] must be registered buffer starts of >= T rows");
  if (sh->host_ag)
    return fail(s, LORA_ERR_INVALID_ARG, "host control plane: x and y must be registered (lora_shard_register)");
  if (!sh->comm) return fail(s, LORA_ERR_NCCL, "no NCCL communicator");
  return apply_sharded_nccl(s, n, slots, x, adapter_ids, expert_ids, y, y_dtype, T, st);
}
