// shard.cu -- the Sharded LoRA Server: LoRA Data Parallel over NCCL / NVLink.
//
// P:288-291 (Sec. 4.1, Table 1 DP row): "evenly distribute LoRA adapters
// across the server GPUs ... activations from client GPUs must be routed
// accordingly ... the server GPUs perform a collective coordination step to
// determine which activations should be processed by which GPUs."  Skewed
// adapter popularity concentrates activations on a few server GPUs;
// the n_replicated hottest adapters are therefore stored on every rank
// and their rows never leave their rank.
//
// One collective apply (every rank, same slot list):
//   1. classify the local rows: owner == this rank (replicated or own units)
//      -> processed in place; the rest bucketed by owner (stable)
//   2. all-gather of the G send counts -> full G x G matrix, read back
//      asynchronously; the in-place plan + apply are enqueued before the host
//      waits for it (the GPU works through the one host round trip)
//   3. (comm stream) pack of x rows and ids into the send buffer, transport
//      (P2P: a barrier; NCCL: grouped send/recv), then the owner side's ids
//      and plan -- all overlapped with the in-place apply
//   4. received rows: delta-mode apply (P2P: the shrink reads the x rows from
//      the sources' send buffers over NVLink)
//   5. deltas back (P2P: barrier, then each source pulls its deltas fused with
//      the add; NCCL: reverse send/recv, then y[origin row] = round(y + delta))
// Deltas travel as fp32 when y is fp32 (sharded == unsharded bit for bit,
// DESIGN.md R18) and as bf16 when y is bf16 (half the NVLink bytes, one extra
// rounding of the delta: DESIGN.md R19), unless LORA_SHARD_FP32=1.
// NCCL is loaded with dlopen("libnccl.so.2") (the copy torch already loaded),
// so the library itself has no link-time NCCL dependency.
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
//   counts[o]   = rows for owner o (0 for this rank)
// loopback != 0 (test knob LORA_SHARD_LOOPBACK=1) sends this rank's own rows
// through the exchange as well, so a single GPU exercises the NCCL path.
// Out-of-range ids are flagged and dropped (never sent, never applied).
__global__ void __launch_bounds__(kBucketThreads, 1)
    bucket_kernel(const int32_t* __restrict__ ad, const int32_t* __restrict__ ex, int T, Placement pl, int n_adapters,
                  int E, int loopback, int32_t* __restrict__ ad_local,
                  int32_t* __restrict__ send_idx, int32_t* __restrict__ counts, int* __restrict__ err) {
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

// Peer-to-peer transport (ShardState::p2p).  Owner side: the ids of received
// row r are read from source s's registered send buffer (NVLink peer mapping).
struct PeerRows {
  int G;
  int off[kMaxWorld + 1];   // row ranges per peer
  int rowbase[kMaxWorld];   // row in the peer's buffer = r + rowbase[p]
  const char* base[kMaxWorld];
};
LORA_DEVINL int peer_of(const PeerRows& pr, int r) {
  int p = 0;
  while (p + 1 < pr.G && pr.off[p + 1] <= r) ++p;
  return p;
}

// ids_recv[r] = a, ids_recv[Rmax + r] = e of received row r (send buffer ids: [2][max_rows])
__global__ void pull_ids_kernel(PeerRows pr, int max_rows, int32_t* __restrict__ ids_recv, long long Rmax, int n) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    const int p = peer_of(pr, r);
    const int32_t* ids = reinterpret_cast<const int32_t*>(pr.base[p]);
    const int row = r + pr.rowbase[p];
    ids_recv[r] = ids[row];
    ids_recv[Rmax + r] = ids[max_rows + row];
  }
}

// Source side: y[idx[j]] = round(y + delta) where the delta of send-order row j
// sits in owner p's registered delta buffer (peer mapping), row j + rowbase[p]
// of the slot region at byte offset slot_off.  The NVLink read is fused with
// the accumulate.  4 columns per thread.
__global__ void pull_scatter_add4_kernel(void* __restrict__ y, int y_fp32, PeerRows pr, long long slot_off, int d_bf16,
                                         const int32_t* __restrict__ idx, int n, int width) {
  const int q4 = width >> 2;
  for (int j = blockIdx.y; j < n; j += gridDim.y) {
    const long long row = idx[j];
    const int p = peer_of(pr, j);
    const long long drow = (long long)(j + pr.rowbase[p]) * q4;
    const char* dbase = pr.base[p] + slot_off;
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < q4; c += gridDim.x * blockDim.x) {
      float4 v;
      if (d_bf16) {
        const uint2 b = reinterpret_cast<const uint2*>(dbase)[drow + c];
        v = make_float4(bf16lo(b.x), bf16hi(b.x), bf16lo(b.y), bf16hi(b.y));
      } else {
        v = reinterpret_cast<const float4*>(dbase)[drow + c];
      }
      if (y_fp32) {
        float4* yp = reinterpret_cast<float4*>(y) + row * q4 + c;
        float4 o = *yp;
        o.x += v.x; o.y += v.y; o.z += v.z; o.w += v.w;
        *yp = o;
      } else {
        uint2* yp = reinterpret_cast<uint2*>(y) + row * q4 + c;
        const uint2 o = *yp;
        uint2 r;
        r.x = pack_bf16x2_rn(bf16lo(o.x) + v.x, bf16hi(o.x) + v.y);
        r.y = pack_bf16x2_rn(bf16lo(o.y) + v.z, bf16hi(o.y) + v.w);
        *yp = r;
      }
    }
  }
}

int grid_of(long long n) {
  long long g = (n + 255) / 256;
  return (int)(g < 1 ? 1 : (g > 148 * 16 ? 148 * 16 : g));
}

}  // namespace

struct ShardState {
  ncclComm_t comm = nullptr;
  cudaStream_t cs = nullptr;  // communication stream (pack + NCCL)
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  void* buf = nullptr;        // device scratch (grown on demand)
  size_t bytes = 0;
  lora_plan* plan = nullptr;        // owner-side plan over received rows (capacity max_rows * world)
  lora_plan* local_plan = nullptr;  // plan over this rank's rows processed in place
  bool fp32_return = false;
  bool loopback = false;
  // peer-to-peer transport: registered (IPC-exported) buffers, mapped on every rank
  bool p2p = true;
  void* sendbuf = nullptr;  // [2][max_rows] ids + per distinct x buffer [max_rows][h_in] bf16, send order
  void* dbuf = nullptr;     // per slot [Rmax][h_out] deltas of received rows
  size_t send_cap = 0, d_cap = 0;
  std::vector<char*> peer_send, peer_d;  // index = rank (own rank: the local pointers)
  int* d_bar = nullptr;                   // barrier word (NCCL all-reduce)
  // host control plane (lora_server_create_sharded_host): no NCCL at all
  lora_host_allgather_fn host_ag = nullptr;
  void* host_ctx = nullptr;
  int32_t* h_cnt = nullptr;  // pinned [world][world] counts (async read-back)
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

// Barrier in the order of `st`: an NCCL all-reduce of one word (no host
// sync), or -- host control plane -- a stream synchronize and a host barrier.
static lora_status_t ctl_barrier(lora_server* s, cudaStream_t st) {
  ShardState* sh = s->shard;
  if (sh->host_ag) {
    char b = 0;
    std::vector<char> all(s->world);
    return ctl_allgather(s, &b, all.data(), 1, st);
  }
  NcclApi& api = nccl();
  const ncclResult_t r = api.AllReduce(sh->d_bar, sh->d_bar, 1, ncclInt32, ncclSum, sh->comm, st);
  return r == ncclSuccess ? LORA_OK : fail(s, LORA_ERR_NCCL, std::string("barrier: ") + api.GetErrorString(r));
}

// Release the peer mappings and the registered buffers.
static void p2p_release(ShardState* sh, int me) {
  for (size_t p = 0; p < sh->peer_send.size(); ++p)
    if ((int)p != me) {
      if (sh->peer_send[p]) cudaIpcCloseMemHandle(sh->peer_send[p]);
      if (sh->peer_d[p]) cudaIpcCloseMemHandle(sh->peer_d[p]);
    }
  sh->peer_send.clear();
  sh->peer_d.clear();
  cudaFree(sh->sendbuf);
  cudaFree(sh->dbuf);
  sh->sendbuf = sh->dbuf = nullptr;
  sh->send_cap = sh->d_cap = 0;
}

void lora_shard_free(lora_server* s) {
  if (!s || !s->shard) return;
  ShardState* sh = s->shard;
  p2p_release(sh, s->shard_rank);
  cudaFree(sh->d_bar);
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
  if (world > kMaxWorld) return fail(nullptr, LORA_ERR_UNSUPPORTED, "host control plane: world > 8");
  return create_sharded_impl(cfg, rank, world, nullptr, allgather, ctx, out);
}

static lora_status_t create_sharded_impl(const lora_config_t* cfg, int32_t rank, int32_t world,
                                         const void* nccl_unique_id, lora_host_allgather_fn host_ag, void* host_ctx,
                                         lora_server_t** out) {
  if (!cfg || !out || world < 1 || rank < 0 || rank >= world)
    return fail(nullptr, LORA_ERR_INVALID_ARG, "lora_server_create_sharded: bad argument");
  if ((long long)cfg->max_rows * world > kMaxPlanRows)
    return fail(nullptr, LORA_ERR_UNSUPPORTED, "max_rows * world must be <= 16384 (owner-side plan capacity)");
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
  const char* tr = std::getenv("LORA_SHARD_TRANSPORT");
  sh->p2p = !(tr && std::strcmp(tr, "nccl") == 0);
  if (world > kMaxWorld) sh->p2p = false;
  if (host_ag) sh->p2p = true;  // the only transport without NCCL
  cudaSetDevice(s->device);
  bool ok = cudaStreamCreateWithFlags(&sh->cs, cudaStreamNonBlocking) == cudaSuccess;
  for (auto& e : sh->ev) ok = ok && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess;
  if (!ok) {
    lora_server_destroy(s);
    *out = nullptr;
    return fail(nullptr, LORA_ERR_CUDA, "stream / event creation failed");
  }
  ok = ok && cudaMalloc(&sh->d_bar, sizeof(int)) == cudaSuccess && cudaMemset(sh->d_bar, 0, sizeof(int)) == cudaSuccess;
  ok = ok && cudaMallocHost(&sh->h_cnt, sizeof(int32_t) * world * world) == cudaSuccess;
  if (!ok) {
    lora_server_destroy(s);
    *out = nullptr;
    return fail(nullptr, LORA_ERR_CUDA, "barrier word allocation failed");
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
  return LORA_OK;
}

// Grow the registered P2P buffers to (need_send, need_d) bytes -- collective:
// every rank computes the same sizes from the same slot list.  Exports IPC
// handles, all-gathers them over NCCL and maps every peer's buffers; if any
// rank cannot map a peer, every rank falls back to the NCCL transport.
static lora_status_t p2p_register(lora_server* s, size_t need_send, size_t need_d, cudaStream_t st) {
  ShardState* sh = s->shard;
  NcclApi& api = nccl();
  const int G = s->world, me = s->shard_rank;
  if (need_send <= sh->send_cap && need_d <= sh->d_cap) return LORA_OK;
  cudaStreamSynchronize(st);
  cudaStreamSynchronize(sh->cs);
  p2p_release(sh, me);
  need_send = std::max(need_send, (size_t)1 << 20);
  need_d = std::max(need_d, (size_t)1 << 20);
  if (cudaMalloc(&sh->sendbuf, need_send) != cudaSuccess || cudaMalloc(&sh->dbuf, need_d) != cudaSuccess) {
    cudaGetLastError();
    p2p_release(sh, me);
    return fail(s, LORA_ERR_OOM, "P2P buffer allocation failed");
  }
  sh->send_cap = need_send;
  sh->d_cap = need_d;
  sh->peer_send.assign(G, nullptr);
  sh->peer_d.assign(G, nullptr);
  sh->peer_send[me] = static_cast<char*>(sh->sendbuf);
  sh->peer_d[me] = static_cast<char*>(sh->dbuf);
  if (G == 1) return LORA_OK;
  // handle exchange: [G][2][64 bytes]
  // A rank whose export fails still takes part in both all-gathers (zeroed
  // handles, ok = 0), so every rank reaches the same decision instead of the
  // others blocking in the handle exchange.
  std::vector<cudaIpcMemHandle_t> h(2 * G);
  int ok = 1;
  if (cudaIpcGetMemHandle(&h[2 * me], sh->sendbuf) != cudaSuccess ||
      cudaIpcGetMemHandle(&h[2 * me + 1], sh->dbuf) != cudaSuccess) {
    cudaGetLastError();
    std::memset(&h[2 * me], 0, 2 * sizeof(cudaIpcMemHandle_t));
    ok = 0;
  }
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  std::vector<cudaIpcMemHandle_t> mine(h.begin() + 2 * me, h.begin() + 2 * me + 2);
  lora_status_t rc = ctl_allgather(s, mine.data(), h.data(), 128, st);
  if (rc != LORA_OK) return rc;
  for (int p = 0; p < G && ok; ++p) {
    if (p == me) continue;
    void* a = nullptr;
    void* b = nullptr;
    if (cudaIpcOpenMemHandle(&a, h[2 * p], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess ||
        cudaIpcOpenMemHandle(&b, h[2 * p + 1], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      ok = 0;
    }
    sh->peer_send[p] = static_cast<char*>(a);
    sh->peer_d[p] = static_cast<char*>(b);
  }
  // every rank must agree on the transport
  std::vector<int> oks(G, 0);
  rc = ctl_allgather(s, &ok, oks.data(), sizeof(int), st);
  if (rc != LORA_OK) return rc;
  for (int v : oks) ok = ok && v;
  if (!ok) {
    p2p_release(sh, me);
    if (sh->host_ag) return fail(s, LORA_ERR_UNSUPPORTED, "peer mapping failed and the host control plane has no fallback");
    sh->p2p = false;  // NCCL send/recv from now on, on every rank
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

extern "C" lora_status_t lora_apply_sharded(lora_server_t* s, int32_t n, const int32_t* slots, const void* const* x,
                                            const int32_t* adapter_ids, const int32_t* expert_ids, void* const* y,
                                            lora_dtype_t y_dtype, int32_t T, void* stream) {
  if (!s) return fail(nullptr, LORA_ERR_INVALID_ARG, "server is NULL");
  if (!s->shard) return fail(s, LORA_ERR_INVALID_ARG, "not a sharded server");
  if (n < 1 || !slots || !x || !y || (T > 0 && !adapter_ids)) return fail(s, LORA_ERR_INVALID_ARG, "NULL argument");
  if (T < 0 || T > s->max_rows) return fail(s, LORA_ERR_INVALID_ARG, "T must be in [0, max_rows]");
  if (y_dtype != LORA_BF16 && y_dtype != LORA_FP32) return fail(s, LORA_ERR_UNSUPPORTED, "y_dtype");
  for (int i = 0; i < n; ++i)
    if (slots[i] < 0 || slots[i] >= (int)s->slots.size()) return fail(s, LORA_ERR_INVALID_ARG, "bad slot index");
  const int E = s->slots[slots[0]].E;
  for (int i = 0; i < n; ++i)
    if (s->slots[slots[i]].E != E) return fail(s, LORA_ERR_INVALID_ARG, "slots of one call must share n_experts");
  NcclApi& api = nccl();
  const int G = s->world, me = s->shard_rank;
  const Placement pl = placement(s);
  ShardState* sh = s->shard;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaStream_t cs = sh->cs;
  CKS(cudaSetDevice(s->device));
  const bool d_bf16 = (y_dtype == LORA_BF16) && !sh->fp32_return;
  const size_t dsz = d_bf16 ? 2 : 4;

  // distinct x buffers
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

  // scratch layout (worst case: every rank sends every row to me -> G*T rows)
  const long long Rmax = (long long)s->max_rows * G;
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  size_t off = 0;
  const size_t o_counts = off; off += al(sizeof(int32_t) * G * (G + 1));
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
  int32_t* d_counts = reinterpret_cast<int32_t*>(base + o_counts);  // [G] mine, then [G][G] gathered
  int32_t* d_send_idx = reinterpret_cast<int32_t*>(base + o_send_idx);
  int32_t* d_ad_local = reinterpret_cast<int32_t*>(base + o_ad_local);
  int32_t* d_ids_send = reinterpret_cast<int32_t*>(base + o_ids_send);  // [2][max_rows] (a | e) in send order
  int32_t* d_ids_recv = reinterpret_cast<int32_t*>(base + o_ids_recv);  // [2][Rmax]

  // 1. classify + bucket.  The previous call's comm-stream work (reads of the
  //    scratch) must be done before it is overwritten: ev[3] was recorded last.
  CKS(cudaStreamWaitEvent(st, sh->ev[3], 0));
  if (T > 0) {
    const int pi = prof_start(s, st);
    bucket_kernel<<<1, kBucketThreads, 0, st>>>(adapter_ids, expert_ids, T, pl, s->n_adapters, E, sh->loopback, d_ad_local, d_send_idx, d_counts,
                                                 s->d_err);
    prof_stop(s, pi, kKShardBucket, st);
  } else {
    CKS(cudaMemsetAsync(d_counts, 0, sizeof(int32_t) * G, st));
  }
  CKS(cudaGetLastError());
  // 2. counts exchange (all-gather) + the one host wait.  NCCL control plane:
  //    the matrix comes back asynchronously into pinned memory; the in-place
  //    rows' plan and apply are enqueued before the host waits for it, so the
  //    GPU keeps working through the host round trip.
  std::vector<int32_t> cnt(G * G);
  if (!sh->host_ag) {
    CKN(api.AllGather(d_counts, d_counts + G, G, ncclInt32, sh->comm, st));
    CKS(cudaMemcpyAsync(sh->h_cnt, d_counts + G, sizeof(int32_t) * G * G, cudaMemcpyDeviceToHost, st));
  }
  CKS(cudaEventRecord(sh->ev[0], st));  // bucket outputs + counts ready (the pack waits on this)
  // 3. rows this rank stores the adapter of: applied in place (independent of the counts)
  lora_status_t rc = plan_build_impl(s, sh->local_plan, d_ad_local, expert_ids, T, E, st);
  if (rc != LORA_OK) return rc;
  if (T > 0) {
    rc = apply_multi_impl(s, sh->local_plan, n, slots, x, y, y_dtype, st);
    if (rc != LORA_OK) return rc;
  }
  if (sh->host_ag) {
    std::vector<int32_t> mine(G);
    CKS(cudaMemcpyAsync(mine.data(), d_counts, sizeof(int32_t) * G, cudaMemcpyDeviceToHost, st));
    const lora_status_t cr = ctl_allgather(s, mine.data(), cnt.data(), sizeof(int32_t) * G, st);
    if (cr != LORA_OK) return cr;
  } else {
    CKS(cudaEventSynchronize(sh->ev[0]));
    std::memcpy(cnt.data(), sh->h_cnt, sizeof(int32_t) * G * G);
  }
  std::vector<int64_t> c64(cnt.begin(), cnt.end()), so(G + 1), ro(G + 1);
  lora_status_t lr = lora_shard_layout(c64.data(), G, me, so.data(), ro.data());
  if (lr != LORA_OK) return fail(s, lr, "count exchange produced an invalid matrix");
  const int n_send = (int)so[G], n_recv = (int)ro[G];
  if (n_recv > Rmax) return fail(s, LORA_ERR_INVALID_ARG, "received rows exceed capacity");
  // every rank sees the same matrix, so every rank takes the same branch
  bool exchange = false;
  for (int v : cnt) exchange = exchange || v > 0;

  // peer-to-peer transport: registered buffer layout (identical on every rank)
  size_t p_need_send = 0, p_need_d = 0;
  std::vector<size_t> p_xo(xd.size()), p_doff(n);
  p_need_send = al(sizeof(int32_t) * 2 * s->max_rows);
  for (size_t j = 0; j < xd.size(); ++j) {
    p_xo[j] = p_need_send;
    p_need_send += al((size_t)s->max_rows * x_hin[j] * 2);
  }
  for (int i = 0; i < n; ++i) {
    p_doff[i] = p_need_d;
    p_need_d += al((size_t)Rmax * s->slots[slots[i]].h_out * dsz);
  }
  if (exchange && sh->p2p) {
    const lora_status_t rr = p2p_register(s, p_need_send, p_need_d, st);
    if (rr != LORA_OK) return rr;
  }
  const bool p2p = exchange && sh->p2p;
  // row maps: my send-order rows for owner p; rows I receive from source p
  PeerRows pr_in{}, pr_out{};
  if (p2p) {
    pr_in.G = pr_out.G = G;
    for (int p = 0; p <= G; ++p) {
      pr_in.off[p] = (int)ro[p];
      pr_out.off[p] = (int)so[p];
    }
    std::vector<int64_t> rb_in(G), rb_out(G);
    lora_shard_peer_rows(c64.data(), G, me, rb_in.data(), rb_out.data());
    for (int p = 0; p < G; ++p) {
      pr_in.rowbase[p] = (int)rb_in[p];
      pr_in.base[p] = sh->peer_send[p];
      pr_out.rowbase[p] = (int)rb_out[p];
      pr_out.base[p] = sh->peer_d[p];
    }
  }

  // 3. (comm stream) pack + dispatch, overlapped with the in-place apply
  if (exchange) {
    CKS(cudaStreamWaitEvent(cs, sh->ev[0], 0));
    // P2P: pack straight into the registered send buffer the owners read from
    int32_t* ids_dst = p2p ? static_cast<int32_t*>(sh->sendbuf) : d_ids_send;
    if (n_send > 0) {
      const int pi = prof_start(s, cs);
      gather_words_kernel<<<grid_of(n_send), 256, 0, cs>>>(reinterpret_cast<const uint32_t*>(adapter_ids),
                                                            reinterpret_cast<uint32_t*>(ids_dst), d_send_idx,
                                                            n_send);
      if (expert_ids)
        gather_words_kernel<<<grid_of(n_send), 256, 0, cs>>>(reinterpret_cast<const uint32_t*>(expert_ids),
                                                              reinterpret_cast<uint32_t*>(ids_dst + s->max_rows),
                                                              d_send_idx, n_send);
      else
        CKS(cudaMemsetAsync(ids_dst + s->max_rows, 0, sizeof(int32_t) * n_send, cs));
      for (size_t j = 0; j < xd.size(); ++j) {
        const int chunks = x_hin[j] / 8;  // 16-byte chunks per bf16 row
        gather_rows16_kernel<<<dim3((chunks + 255) / 256, std::min(n_send, 65535)), 256, 0, cs>>>(
            static_cast<const uint4*>(xd[j]),
            reinterpret_cast<uint4*>(p2p ? static_cast<char*>(sh->sendbuf) + p_xo[j] : base + o_xs[j]), d_send_idx,
            n_send, chunks);
      }
      prof_stop(s, pi, kKShardGather, cs);
      CKS(cudaGetLastError());
    }
    if (p2p) {
      // every source's send buffer complete before any owner reads it
      const lora_status_t br = ctl_barrier(s, cs);
      if (br != LORA_OK) return br;
    } else {
      if (sh->host_ag) return fail(s, LORA_ERR_UNSUPPORTED, "host control plane needs the peer-to-peer transport");
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
    }
    // owner side, still on the communication stream: the received rows' ids
    // (P2P: pulled from the sources' send buffers) and their plan -- built
    // while the in-place apply runs on the caller's stream
    if (p2p && n_recv > 0) {
      pull_ids_kernel<<<grid_of(n_recv), 256, 0, cs>>>(pr_in, s->max_rows, d_ids_recv, Rmax, n_recv);
      CKS(cudaGetLastError());
    }
    const lora_status_t pr = plan_build_impl(s, sh->plan, d_ids_recv, d_ids_recv + Rmax, n_recv, E, cs);
    if (pr != LORA_OK) return pr;
    CKS(cudaEventRecord(sh->ev[1], cs));
  }

  if (!exchange) {
    CKS(cudaEventRecord(sh->ev[3], st));
    return LORA_OK;
  }

  // 5. received rows: owner-side plan + delta-mode apply
  CKS(cudaStreamWaitEvent(st, sh->ev[1], 0));
  if (n_recv > 0) {
    std::vector<const void*> xs(n);
    std::vector<void*> ds(n);
    std::vector<long long> xo(n);
    RemoteIn rin{};
    if (p2p) {
      // the shrink kernels read each received x row from its source's send
      // buffer over NVLink (the dispatch is fused into the shrink's loads)
      rin.G = G;
      for (int p = 0; p <= G; ++p) rin.ro[p] = pr_in.off[p];
      for (int p = 0; p < G; ++p) {
        rin.rowbase[p] = pr_in.rowbase[p];
        rin.src[p] = sh->peer_send[p];
      }
    }
    for (int i = 0; i < n; ++i) {
      xs[i] = p2p ? sh->sendbuf : base + o_xr[x_of[i]];
      xo[i] = p2p ? (long long)p_xo[x_of[i]] : 0;
      ds[i] = p2p ? static_cast<char*>(sh->dbuf) + p_doff[i] : base + o_d[i];
    }
    rc = apply_multi_delta(s, sh->plan, n, slots, xs.data(), ds.data(), st, d_bf16, p2p ? &rin : nullptr,
                           p2p ? xo.data() : nullptr);
    if (rc != LORA_OK) return rc;
  }
  if (p2p) {
    // every owner's deltas complete before any source reads them
    const lora_status_t br = ctl_barrier(s, st);
    if (br != LORA_OK) return br;
    if (n_send > 0) {
      for (int i = 0; i < n; ++i) {
        const int ho = s->slots[slots[i]].h_out;
        const int pi = prof_start(s, st);
        pull_scatter_add4_kernel<<<dim3((ho / 4 + 255) / 256, std::min(n_send, 65535)), 256, 0, st>>>(
            y[i], y_dtype == LORA_FP32, pr_out, (long long)p_doff[i], d_bf16 ? 1 : 0, d_send_idx, n_send, ho);
        prof_stop(s, pi, kKShardScatter, st);
      }
      CKS(cudaGetLastError());
    }
    CKS(cudaEventRecord(sh->ev[3], st));
    if (s->debug_sync) CKS(cudaStreamSynchronize(st));
    return LORA_OK;
  }

  // 6. (comm stream) return the deltas
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

  // 7. add the returned deltas at the origin rows
  if (n_send > 0) {
    for (int i = 0; i < n; ++i) {
      const int ho = s->slots[slots[i]].h_out;
      const int pi = prof_start(s, st);
      scatter_add4_kernel<<<dim3((ho / 4 + 255) / 256, std::min(n_send, 65535)), 256, 0, st>>>(
          y[i], y_dtype == LORA_FP32, base + o_dr[i], d_bf16 ? 1 : 0, d_send_idx, n_send, ho);
      prof_stop(s, pi, kKShardScatter, st);
    }
    CKS(cudaGetLastError());
  }
  CKS(cudaEventRecord(sh->ev[3], st));
  if (s->debug_sync) CKS(cudaStreamSynchronize(st));
  return LORA_OK;
}
