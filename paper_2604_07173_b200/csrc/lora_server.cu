// lora_server.cu -- the C-ABI (include/lora_server.h) and the host runtime:
// weight store, plans/workspace, size-based path dispatch.
//
// Operation: y[i,:] += s_{a_i} * (x[i,:] A_{a_i,e_i}) B_{a_i,e_i}
// (Sec. 2.2, Sec. 2.3, Fig. 4b, Sec. 4.1).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <new>
#include <set>
#include <string>
#include <vector>

#include "server.h"

using namespace lora;

namespace {
thread_local std::string g_thread_error = "";

bool env_flag(const char* name) {
  const char* v = std::getenv(name);
  return v && v[0] && std::strcmp(v, "0") != 0;
}

// largest divisor of n that is a multiple of `mult` and <= cap (>= mult; n % mult == 0)
int best_divisor(int n, int mult, int cap) {
  int best = mult;
  for (int d = mult; d <= n && d <= cap; d += mult)
    if (n % d == 0) best = d;
  return best;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
}  // namespace

namespace lora {

lora_status_t fail(lora_server* s, lora_status_t st, const std::string& msg) {
  if (s)
    s->last_error = msg;
  else
    g_thread_error = msg;
  g_thread_error = msg;
  return st;
}

lora_status_t cuda_fail(lora_server* s, cudaError_t e, const char* where) {
  return fail(s, LORA_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

}  // namespace lora

#define CK(s, call)                                          \
  do {                                                       \
    cudaError_t _e = (call);                                 \
    if (_e != cudaSuccess) return lora::cuda_fail((s), _e, #call); \
  } while (0)

// ---------------------------------------------------------------------------
// server
// ---------------------------------------------------------------------------
static lora_status_t validate_config(const lora_config_t* cfg) {
  if (!cfg) return fail(nullptr, LORA_ERR_INVALID_ARG, "cfg is NULL");
  if (cfg->n_slots < 1 || !cfg->h_in || !cfg->h_out || !cfg->n_experts)
    return fail(nullptr, LORA_ERR_INVALID_ARG, "n_slots < 1 or NULL shape arrays");
  if (cfg->rank != 8 && cfg->rank != 16 && cfg->rank != 32 && cfg->rank != 64 && cfg->rank != 128)
    return fail(nullptr, LORA_ERR_UNSUPPORTED, "rank must be 8, 16, 32, 64 or 128");
  if (cfg->n_adapters < 1) return fail(nullptr, LORA_ERR_INVALID_ARG, "n_adapters < 1");
  if (cfg->max_rows < 1 || cfg->max_rows > kMaxPlanRows)
    return fail(nullptr, LORA_ERR_UNSUPPORTED, "max_rows must be in [1, 32768]");
  for (int i = 0; i < cfg->n_slots; ++i) {
    if (cfg->h_in[i] < 64 || cfg->h_in[i] % 64 || cfg->h_out[i] < 64 || cfg->h_out[i] % 64)
      return fail(nullptr, LORA_ERR_UNSUPPORTED, "h_in / h_out must be positive multiples of 64");
    if (cfg->n_experts[i] < 1) return fail(nullptr, LORA_ERR_INVALID_ARG, "n_experts < 1");
    if ((long long)cfg->n_adapters * cfg->n_experts[i] >= (1LL << 31))
      return fail(nullptr, LORA_ERR_UNSUPPORTED, "n_adapters * E must fit in int32");
  }
  if (cfg->scale)
    for (int a = 0; a < cfg->n_adapters; ++a)
      if (!std::isfinite(cfg->scale[a])) return fail(nullptr, LORA_ERR_INVALID_ARG, "non-finite scale");
  return LORA_OK;
}

static void free_server(lora_server* s) {
  if (!s) return;
  if (s->internal_plan) plan_destroy_impl(s->internal_plan);
  for (auto hp : s->host_plans) plan_destroy_impl(hp);
  for (auto& sl : s->slots) {
    cudaFree(sl.At);
    cudaFree(sl.Bt);
  }
  cudaFree(s->d_scale);
  cudaFree(s->d_err);
  cudaFree(s->h2d_buf);
  for (auto p : s->hostA) cudaFreeHost(p);
  for (auto p : s->hostB) cudaFreeHost(p);
  cudaFree(s->d_cache);
  for (auto ev : s->slot_ready) cudaEventDestroy(ev);
  for (auto ev : s->events) cudaEventDestroy(ev);
  for (auto ev : s->prof_pool) cudaEventDestroy(ev);
  if (s->copy_stream) cudaStreamDestroy(s->copy_stream);
  if (s->d2h_stream) cudaStreamDestroy(s->d2h_stream);
  if (s->side_stream) cudaStreamDestroy(s->side_stream);
  if (s->ev_fork) cudaEventDestroy(s->ev_fork);
  if (s->ev_join) cudaEventDestroy(s->ev_join);
  delete s;
}

// allocate the store; world/rank select the owned adapters (a mod world == rank)
static lora_status_t create_common(const lora_config_t* cfg, int world, int rank, lora_server** out, int n_hot,
                                   int ep = 0) {
  lora_status_t v = validate_config(cfg);
  if (v != LORA_OK) return v;
  if (!out) return fail(nullptr, LORA_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || cfg->device < 0 || cfg->device >= ndev)
    return fail(nullptr, LORA_ERR_CUDA, "no such CUDA device");
  CK(nullptr, cudaSetDevice(cfg->device));
  int major = 0, minor = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, cfg->device);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, cfg->device);
  if (major != 10 || minor != 0)
    return fail(nullptr, LORA_ERR_UNSUPPORTED, "this library is built for sm_100a (B200) only");

  lora_server* s = new (std::nothrow) lora_server();
  if (!s) return fail(nullptr, LORA_ERR_OOM, "host allocation failed");
  s->device = cfg->device;
  s->r = cfg->rank;
  s->n_adapters = cfg->n_adapters;
  s->world = world;
  s->shard_rank = rank;
  s->ep = (world > 1 && ep) ? 1 : 0;
  s->n_hot = (world > 1 && !s->ep) ? std::max(0, std::min(n_hot, cfg->n_adapters)) : 0;
  if (s->ep)
    for (int i = 1; i < cfg->n_slots; ++i)
      if (cfg->n_experts[i] != cfg->n_experts[0]) {
        delete s;
        return fail(nullptr, LORA_ERR_UNSUPPORTED, "expert parallel needs one expert count for every slot");
      }
  if (s->ep) {
    s->pp = cfg->pp_stages > 1 ? cfg->pp_stages : 1;
    if (world % s->pp) {
      delete s;
      return fail(nullptr, LORA_ERR_INVALID_ARG, "pp_stages must divide the world size");
    }
  }
  s->slot_layer.assign(cfg->n_slots, 0);
  if (cfg->slot_layer)
    for (int i = 0; i < cfg->n_slots; ++i) {
      if (cfg->slot_layer[i] < 0) {
        delete s;
        return fail(nullptr, LORA_ERR_INVALID_ARG, "negative slot_layer");
      }
      s->slot_layer[i] = cfg->slot_layer[i];
    }
  s->n_adapters_local = placement(s).n_local(cfg->n_adapters);
  if (world == 1 && cfg->n_resident > 0 && cfg->n_resident < cfg->n_adapters) s->n_resident = cfg->n_resident;
  // device store: every local adapter, or the cache slots
  const int store_adapters = s->n_resident ? s->n_resident : s->n_adapters_local;
  s->max_rows = cfg->max_rows;
  s->debug_sync = env_flag("LORA_DEBUG_SYNC");
  if (const char* e = std::getenv("LORA_SMALL_SEG_MAX")) s->small_seg_max = std::atoi(e);
  if (const char* e = std::getenv("LORA_TC_KI_MAX")) s->tc_ki_max = std::max(128, std::atoi(e));
  if (const char* e = std::getenv("LORA_TC_CI_MAX")) s->tc_ci_max = std::atoi(e);
  if (const char* e = std::getenv("LORA_TC_CAP_K")) s->tc_cap_k = std::atoi(e);
  if (const char* e = std::getenv("LORA_TCE_FLAGS")) s->tc_flags = std::atoi(e);
  if (const char* e = std::getenv("LORA_TC_PAIR")) s->tc_pair = std::atoi(e) != 0;
  if (const char* e = std::getenv("LORA_TC_LPT")) s->tc_lpt = std::atoi(e) != 0;
  if (const char* e = std::getenv("LORA_PDL_TC")) s->pdl_tc = std::atoi(e) != 0;
  cudaDeviceGetAttribute(&s->sm_count, cudaDevAttrMultiProcessorCount, cfg->device);
  s->simt_split_items = 2 * 2 * s->sm_count;  // fewer whole-K items than 2 per CUDA-core CTA: split K
  // r = 16: the CUDA-core kernels beat the tcgen05 chain on decode batches
  // (measured, config-3 shapes at 512 tokens: 179 vs 204 us), so tcgen05
  // takes the large segments of prefill-sized batches only; r = 32 / 128
  // gain from it at decode sizes too (286 -> 277 us, 943 -> 898 us)
  if (s->r <= 16) s->tc_min_rows = 2048;
  if (const char* e = std::getenv("LORA_TC_MIN_ROWS")) s->tc_min_rows = std::atoi(e);
  if (const char* e = std::getenv("LORA_SIMT_SPLIT")) s->simt_split_items = std::atoi(e);
  if (const char* e = std::getenv("LORA_GROUP_ROWS")) s->group_rows = std::max(1, std::min(lora::kGroupRows, std::atoi(e)));
  if (cudaStreamCreateWithFlags(&s->side_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&s->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&s->ev_join, cudaEventDisableTiming) != cudaSuccess) {
    free_server(s);
    return fail(nullptr, LORA_ERR_CUDA, "stream / event creation failed");
  }
  s->concurrent_tc = !env_flag("LORA_SERIAL");

  const int r = cfg->rank;
  int kc_prefix = 0;
  for (int i = 0; i < cfg->n_slots; ++i) {
    SlotInfo sl;
    sl.h_in = cfg->h_in[i];
    sl.h_out = cfg->h_out[i];
    sl.E = cfg->n_experts[i];
    sl.units = s->n_resident ? (long long)store_adapters * sl.E
                             : slot_placement(s, i).n_local_units(cfg->n_adapters, sl.E);
    // shrink items of ~128 KB of A, expand items of ~128 KB of B
    sl.KI = best_divisor(sl.h_in, 64, std::max(64, 65536 / r));
    sl.SJ = best_divisor(sl.KI, 64, simt_sj_max(r));
    sl.n_kc = sl.h_in / sl.KI;
    sl.CI = best_divisor(sl.h_out, 64, std::max(64, 65536 / r));
    sl.SC = best_divisor(sl.CI, 64, simt_sc_max(r));
    sl.n_ci = sl.h_out / sl.CI;
    sl.kc_prefix = kc_prefix;
    kc_prefix += sl.n_kc;
    // (a hybrid EP_x-PP_y rank stores no unit of the other groups' layers: 16 bytes)
    const size_t a_bytes = std::max<size_t>(16, (size_t)sl.units * sl.h_in * r * 2),
                 b_bytes = std::max<size_t>(16, (size_t)sl.units * sl.h_out * r * 2);
    if (cudaMalloc(&sl.At, a_bytes) != cudaSuccess || cudaMalloc(&sl.Bt, b_bytes) != cudaSuccess) {
      cudaGetLastError();
      s->slots.push_back(sl);
      free_server(s);
      return fail(nullptr, LORA_ERR_OOM, "weight store allocation failed (slot " + std::to_string(i) + ")");
    }
    s->slots.push_back(sl);
    if (cudaMemset(sl.At, 0, a_bytes) != cudaSuccess || cudaMemset(sl.Bt, 0, b_bytes) != cudaSuccess) {
      free_server(s);
      return fail(nullptr, LORA_ERR_CUDA, "cudaMemset of the store failed");
    }
  }
  s->total_kc = kc_prefix;
  std::vector<float> sc(cfg->n_adapters, 1.0f);
  if (cfg->scale) std::memcpy(sc.data(), cfg->scale, sizeof(float) * cfg->n_adapters);
  if (cudaMalloc(&s->d_scale, sizeof(float) * cfg->n_adapters) != cudaSuccess ||
      cudaMalloc(&s->d_err, sizeof(int)) != cudaSuccess) {
    free_server(s);
    return fail(nullptr, LORA_ERR_OOM, "allocation failed");
  }
  cudaMemcpy(s->d_scale, sc.data(), sizeof(float) * cfg->n_adapters, cudaMemcpyHostToDevice);
  cudaMemset(s->d_err, 0, sizeof(int));
  if (s->n_resident) {
    // pinned host backing store in the kernel layout, cache table (all absent)
    for (int i = 0; i < cfg->n_slots; ++i) {
      const SlotInfo& sl = s->slots[i];
      uint16_t* ha = nullptr;
      uint16_t* hb = nullptr;
      const size_t na = (size_t)cfg->n_adapters * sl.E * sl.h_in * r, nb = (size_t)cfg->n_adapters * sl.E * sl.h_out * r;
      if (cudaMallocHost(&ha, na * 2) != cudaSuccess || cudaMallocHost(&hb, nb * 2) != cudaSuccess) {
        cudaGetLastError();
        if (ha) cudaFreeHost(ha);
        free_server(s);
        return fail(nullptr, LORA_ERR_OOM, "pinned host backing store allocation failed");
      }
      std::memset(ha, 0, na * 2);
      std::memset(hb, 0, nb * 2);
      s->hostA.push_back(ha);
      s->hostB.push_back(hb);
      cudaEvent_t ev;
      if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) {
        free_server(s);
        return fail(nullptr, LORA_ERR_CUDA, "event creation failed");
      }
      s->slot_ready.push_back(ev);
    }
    s->slot_pending.assign(cfg->n_slots, 0);
    s->h_cache.assign(cfg->n_adapters, -1);
    s->cache_owner.assign(s->n_resident, -1);
    s->cache_use.assign(s->n_resident, 0);
    if (cudaMalloc(&s->d_cache, sizeof(int32_t) * cfg->n_adapters) != cudaSuccess ||
        cudaMemcpy(s->d_cache, s->h_cache.data(), sizeof(int32_t) * cfg->n_adapters, cudaMemcpyHostToDevice) !=
            cudaSuccess) {
      free_server(s);
      return fail(nullptr, LORA_ERR_OOM, "cache table allocation failed");
    }
  }
  lora_status_t ps = plan_create_impl(s, cfg->max_rows, &s->internal_plan);
  if (ps != LORA_OK) {
    std::string m = s->last_error;
    free_server(s);
    return fail(nullptr, ps, m);
  }
  if (cudaDeviceSynchronize() != cudaSuccess) {
    free_server(s);
    return fail(nullptr, LORA_ERR_CUDA, "device synchronisation after create failed");
  }
  *out = s;
  return LORA_OK;
}

lora_status_t create_common_sharded(const lora_config_t* cfg, int world, int rank, lora_server** out, int n_hot,
                                    int ep) {
  return create_common(cfg, world, rank, out, n_hot, ep);
}

// delta mode for the sharded owner: d[i] receives s*(xA)B (stored, not added) as fp32 or bf16
namespace lora {
// Programmatic dependent launch of the shrink / expand / v-reduce kernels
// (prologues and the expand's first weight copies overlapping the previous
// kernel's tail).  Measured in round 2: with a single kernel chain (Llama
// decode, r = 16) 0.412 -> 0.407 ms; with the tcgen05 chain running
// concurrently on the side stream the early CTAs compete with the other
// chain (Mixtral decode 0.488 -> 0.565 ms), so apply_multi_impl allows it
// only when the apply does not fork (LORA_PDL=0 disables it everywhere).
thread_local bool g_pdl_allow = false;
bool pdl_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("LORA_PDL");
    return !(v && v[0] == '0');
  }();
  return on && g_pdl_allow;
}
}  // namespace lora

lora_status_t apply_multi_delta(lora_server* s, const lora_plan* p, int n, const int32_t* slots, const void* const* x,
                                void* const* d, cudaStream_t st, bool bf16) {
  return apply_multi_impl(s, p, n, slots, x, d, bf16 ? LORA_BF16 : LORA_FP32, st, bf16 ? 2 : 1);
}

static lora_status_t cache_reset(lora_server* s);

static lora_status_t load_slot(lora_server* s, int slot, int a_begin, int n, const void* A, const void* B,
                               int on_device, cudaStream_t st) {
  SlotInfo& sl = s->slots[slot];
  const int r = s->r;
  const size_t a_unit = (size_t)sl.h_in * r, b_unit = (size_t)sl.h_out * r;  // elements
  // stage one adapter at a time (E units) through a device buffer, relayout into the store
  uint16_t* stage = nullptr;
  const size_t stage_elems = (size_t)sl.E * std::max(a_unit, b_unit);
  CK(s, cudaMalloc(&stage, stage_elems * 2));
  lora_status_t rc = LORA_OK;
  const Placement pl = slot_placement(s, slot);
  for (int i = 0; i < n && rc == LORA_OK; ++i) {
    const int a = a_begin + i;
    // the owned experts of adapter a, as runs of consecutive units in the store
    // (all E for the adapter-level placements, every world-th one for EP)
    for (int e = 0; e < sl.E && rc == LORA_OK; ++e) {
      if (!pl.owns_unit(a, e)) continue;
      const int run = pl.ep ? 1 : sl.E;  // adapter-level: one run of E units
      // cache mode: relayout in cache slot 0's area, then into the host backing store
      const long long lu = s->n_resident ? 0 : pl.local_unit(a, e, sl.E);
      for (int pass = 0; pass < 2; ++pass) {
        const void* src = pass == 0 ? A : B;
        if (!src) continue;
        const size_t ue = pass == 0 ? a_unit : b_unit;
        const uint16_t* from = static_cast<const uint16_t*>(src) + ((size_t)i * sl.E + e) * ue;
        cudaError_t err = cudaMemcpyAsync(stage, from, (size_t)run * ue * 2,
                                          on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st);
        if (err == cudaSuccess)
          err = pass == 0 ? launch_relayout_A(stage, sl.At + lu * a_unit, run, sl.h_in, r, st)
                          : launch_relayout_B(stage, sl.Bt + lu * b_unit, run, sl.h_out, r, st);
        if (err == cudaSuccess && s->n_resident) {
          uint16_t* host = pass == 0 ? s->hostA[slot] + (size_t)a * sl.E * a_unit : s->hostB[slot] + (size_t)a * sl.E * b_unit;
          err = cudaMemcpyAsync(host, pass == 0 ? sl.At : sl.Bt, (size_t)run * ue * 2, cudaMemcpyDeviceToHost, st);
        }
        if (err == cudaSuccess) err = cudaStreamSynchronize(st);
        if (err != cudaSuccess) rc = cuda_fail(s, err, "lora_server_load");
      }
      if (!pl.ep) break;  // the run covered every expert of the adapter
    }
  }
  cudaFree(stage);
  if (rc == LORA_OK && s->n_resident) rc = cache_reset(s);
  return rc;
}

extern "C" lora_status_t lora_server_create(const lora_config_t* cfg, const void* const* A, const void* const* B,
                                            int weights_on_device, lora_server_t** out) {
  // Test hook LORA_FAKE_WORLD="world,rank[,ep[,n_hot]]": store only what that
  // rank of a sharded server would own (no communicator; rows of units it
  // does not own are rejected like out-of-range ids), so the sharded store
  // layouts can be checked against the oracle on one GPU.
  // (",pp" -- a fifth field -- overrides cfg->pp_stages: hybrid EP_x-PP_y)
  int fw = 1, fr = 0, fep = 0, fhot = 0, fpp = 0;
  if (const char* f = std::getenv("LORA_FAKE_WORLD")) {
    if (std::sscanf(f, "%d,%d,%d,%d,%d", &fw, &fr, &fep, &fhot, &fpp) < 2 || fw < 1 || fr < 0 || fr >= fw) {
      fw = 1;
      fr = 0;
    }
  }
  lora_config_t cfg2;
  if (cfg) {
    cfg2 = *cfg;
    if (fpp > 0) cfg2.pp_stages = fpp;
    cfg = &cfg2;
  }
  lora_status_t st = create_common(cfg, fw, fr, out, fhot, fep);
  if (st != LORA_OK) return st;
  lora_server* s = *out;
  for (int i = 0; i < cfg->n_slots; ++i) {
    const void* a = A ? A[i] : nullptr;
    const void* b = B ? B[i] : nullptr;
    if (!a && !b) continue;
    st = load_slot(s, i, 0, cfg->n_adapters, a, b, weights_on_device, nullptr);
    if (st != LORA_OK) {
      std::string m = s->last_error;
      free_server(s);
      *out = nullptr;
      return fail(nullptr, st, m);
    }
  }
  return LORA_OK;
}

extern "C" lora_status_t lora_server_load(lora_server_t* s, int32_t slot, int32_t adapter_begin, int32_t n,
                                          const void* A, const void* B, int on_device, void* stream) {
  if (!s) return fail(nullptr, LORA_ERR_INVALID_ARG, "server is NULL");
  if (slot < 0 || slot >= (int)s->slots.size()) return fail(s, LORA_ERR_INVALID_ARG, "bad slot");
  if (adapter_begin < 0 || n < 0 || (long long)adapter_begin + n > s->n_adapters)
    return fail(s, LORA_ERR_INVALID_ARG, "adapter range out of bounds");
  if (!A && !B) return fail(s, LORA_ERR_INVALID_ARG, "A and B are both NULL");
  CK(s, cudaSetDevice(s->device));
  return load_slot(s, slot, adapter_begin, n, A, B, on_device, static_cast<cudaStream_t>(stream));
}

extern "C" lora_status_t lora_server_fill_synthetic(lora_server_t* s, uint64_t seed, void* stream) {
  if (!s) return fail(nullptr, LORA_ERR_INVALID_ARG, "server is NULL");
  CK(s, cudaSetDevice(s->device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (s->n_resident) {
    // generate n_resident adapters at a time in the device cache area, copy them
    // to the host backing store; the cache is empty afterwards
    CK(s, cudaStreamSynchronize(st));
    for (size_t i = 0; i < s->slots.size(); ++i) {
      SlotInfo& sl = s->slots[i];
      const size_t ua = (size_t)sl.E * sl.h_in * s->r, ub = (size_t)sl.E * sl.h_out * s->r;  // per adapter
      for (int a0 = 0; a0 < s->n_adapters; a0 += s->n_resident) {
        const int na = std::min(s->n_resident, s->n_adapters - a0);
        CK(s, launch_fill_store(sl.At, sl.Bt, sl.h_in, sl.h_out, sl.E, s->r, (long long)na * sl.E, (int)i, seed,
                                Placement{1, 0, 0}, s->n_adapters, st, a0));
        CK(s, cudaMemcpyAsync(s->hostA[i] + (size_t)a0 * ua, sl.At, (size_t)na * ua * 2, cudaMemcpyDeviceToHost, st));
        CK(s, cudaMemcpyAsync(s->hostB[i] + (size_t)a0 * ub, sl.Bt, (size_t)na * ub * 2, cudaMemcpyDeviceToHost, st));
      }
    }
    CK(s, cudaStreamSynchronize(st));
    return cache_reset(s);
  }
  for (size_t i = 0; i < s->slots.size(); ++i) {
    SlotInfo& sl = s->slots[i];
    CK(s, launch_fill_store(sl.At, sl.Bt, sl.h_in, sl.h_out, sl.E, s->r, sl.units, (int)i, seed,
                            slot_placement(s, (int)i), s->n_adapters, st));
  }
  return LORA_OK;
}

// ---------------------------------------------------------------------------
// resident-adapter cache (cfg->n_resident > 0; P:519-531 layer-wise loading)
// ---------------------------------------------------------------------------
static lora_status_t cache_reset(lora_server* s) {
  std::fill(s->h_cache.begin(), s->h_cache.end(), -1);
  std::fill(s->cache_owner.begin(), s->cache_owner.end(), -1);
  std::fill(s->cache_use.begin(), s->cache_use.end(), 0);
  CK(s, cudaMemcpy(s->d_cache, s->h_cache.data(), sizeof(int32_t) * s->n_adapters, cudaMemcpyHostToDevice));
  return LORA_OK;
}

extern "C" lora_status_t lora_server_require(lora_server_t* s, const int32_t* adapters, int32_t n, int32_t* n_loaded,
                                             void* stream) {
  if (!s) return fail(nullptr, LORA_ERR_INVALID_ARG, "server is NULL");
  if (n_loaded) *n_loaded = 0;
  if (!s->n_resident || n <= 0) return LORA_OK;
  if (!adapters) return fail(s, LORA_ERR_INVALID_ARG, "adapters is NULL");
  std::vector<int> need;
  for (int i = 0; i < n; ++i) {
    const int a = adapters[i];
    if (a < 0) continue;  // no LoRA
    if (a >= s->n_adapters) return fail(s, LORA_ERR_INVALID_ARG, "adapter id out of range");
    need.push_back(a);
  }
  std::sort(need.begin(), need.end());
  need.erase(std::unique(need.begin(), need.end()), need.end());
  if ((int)need.size() > s->n_resident)
    return fail(s, LORA_ERR_UNSUPPORTED, "more distinct adapters than resident cache slots");
  CK(s, cudaSetDevice(s->device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const long long tick = ++s->cache_tick;
  std::vector<std::pair<int, int>> loads;  // (adapter, cache slot)
  for (int a : need)
    if (s->h_cache[a] >= 0) s->cache_use[s->h_cache[a]] = tick;
  for (int a : need) {
    if (s->h_cache[a] >= 0) continue;
    int victim = -1;
    for (int c = 0; c < s->n_resident; ++c) {  // an empty slot, else the least recently required
      if (s->cache_owner[c] < 0) {
        victim = c;
        break;
      }
      if (s->cache_use[c] < tick && (victim < 0 || s->cache_use[c] < s->cache_use[victim])) victim = c;
    }
    if (victim < 0) return fail(s, LORA_ERR_UNSUPPORTED, "no evictable cache slot");
    if (s->cache_owner[victim] >= 0) s->h_cache[s->cache_owner[victim]] = -1;
    s->cache_owner[victim] = a;
    s->cache_use[victim] = tick;
    s->h_cache[a] = victim;
    loads.push_back({a, victim});
  }
  if (loads.empty()) return LORA_OK;
  if (!s->copy_stream) CK(s, cudaStreamCreateWithFlags(&s->copy_stream, cudaStreamNonBlocking));
  if (s->events.empty()) {
    cudaEvent_t e;
    CK(s, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    s->events.push_back(e);
  }
  // evicted slots may still be read by work already queued on `stream`
  CK(s, cudaEventRecord(s->events[0], st));
  CK(s, cudaStreamWaitEvent(s->copy_stream, s->events[0], 0));
  for (size_t i = 0; i < s->slots.size(); ++i) {  // slot (layer) order: the first layers land first
    SlotInfo& sl = s->slots[i];
    const size_t ua = (size_t)sl.E * sl.h_in * s->r, ub = (size_t)sl.E * sl.h_out * s->r;
    for (auto& ac : loads) {
      CK(s, cudaMemcpyAsync(sl.At + (size_t)ac.second * ua, s->hostA[i] + (size_t)ac.first * ua, ua * 2,
                            cudaMemcpyHostToDevice, s->copy_stream));
      CK(s, cudaMemcpyAsync(sl.Bt + (size_t)ac.second * ub, s->hostB[i] + (size_t)ac.first * ub, ub * 2,
                            cudaMemcpyHostToDevice, s->copy_stream));
    }
    CK(s, cudaEventRecord(s->slot_ready[i], s->copy_stream));
    s->slot_pending[i] = 1;
  }
  // the new table, in stream order (pageable source: copied out at the call)
  CK(s, cudaMemcpyAsync(s->d_cache, s->h_cache.data(), sizeof(int32_t) * s->n_adapters, cudaMemcpyHostToDevice, st));
  if (n_loaded) *n_loaded = (int32_t)loads.size();
  return LORA_OK;
}

extern "C" lora_status_t lora_server_destroy(lora_server_t* s) {
  if (!s) return LORA_OK;
  cudaSetDevice(s->device);
  cudaDeviceSynchronize();
  lora_shard_free(s);
  free_server(s);
  return LORA_OK;
}

extern "C" lora_status_t lora_server_set_small_seg_max(lora_server_t* s, int32_t n) {
  if (!s) return fail(nullptr, LORA_ERR_INVALID_ARG, "server is NULL");
  s->small_seg_max = n;
  return LORA_OK;
}

extern "C" lora_status_t lora_server_set_concurrent(lora_server_t* s, int32_t on) {
  if (!s) return fail(nullptr, LORA_ERR_INVALID_ARG, "server is NULL");
  s->concurrent_tc = on != 0;
  return LORA_OK;
}

extern "C" lora_status_t lora_server_check(lora_server_t* s, void* stream) {
  if (!s) return fail(nullptr, LORA_ERR_INVALID_ARG, "server is NULL");
  CK(s, cudaSetDevice(s->device));
  CK(s, cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  int flag = 0;
  CK(s, cudaMemcpy(&flag, s->d_err, sizeof(int), cudaMemcpyDeviceToHost));
  if (flag) CK(s, cudaMemset(s->d_err, 0, sizeof(int)));
  if (s->shard) {  // peer timeouts / layout mismatches of the push path, NCCL asynchronous errors
    const lora_status_t sr = lora_shard_check_flags(s, flag);
    if (sr != LORA_OK) return sr;
  }
  if (flag & 1) return fail(s, LORA_ERR_ID_OUT_OF_RANGE, "an adapter or expert id was out of range (row skipped)");
  return LORA_OK;
}

extern "C" const char* lora_last_error(const lora_server_t* s) {
  return s ? s->last_error.c_str() : g_thread_error.c_str();
}

extern "C" const char* lora_version(void) { return "infinilora-b200 0.1 (sm_100a)"; }

// ---------------------------------------------------------------------------
// plans
// ---------------------------------------------------------------------------
namespace lora {

lora_status_t plan_create_impl(lora_server* s, int max_rows, lora_plan** out) {
  if (max_rows < 1 || max_rows > kMaxPlanRows) return fail(s, LORA_ERR_UNSUPPORTED, "max_rows must be in [1, 32768]");
  lora_plan* p = new (std::nothrow) lora_plan();
  if (!p) return fail(s, LORA_ERR_OOM, "host allocation failed");
  p->s = s;
  p->max_rows = max_rows;
  p->world = s->world;
  PlanDev& d = p->dev;
  d.max_rows = max_rows;
  bool ok = cudaMalloc(&d.perm, sizeof(int32_t) * max_rows) == cudaSuccess &&
            cudaMalloc(&d.seg_off, sizeof(int32_t) * (max_rows + 1)) == cudaSuccess &&
            cudaMalloc(&d.seg_key, sizeof(int32_t) * max_rows) == cudaSuccess &&
            cudaMalloc(&d.counts, sizeof(int32_t) * kCntWords) == cudaSuccess &&
            cudaMalloc(&d.groups, sizeof(int4) * max_rows) == cudaSuccess &&
            cudaMalloc(&d.tiles, sizeof(int4) * max_rows) == cudaSuccess &&
            cudaMalloc(&d.vpart, sizeof(float) * (size_t)s->total_kc * max_rows * s->r) == cudaSuccess &&
            cudaMalloc(&d.vbf, sizeof(uint16_t) * s->slots.size() * (size_t)max_rows * std::max(s->r, 16)) == cudaSuccess &&
            cudaMalloc(&d.wctr, sizeof(unsigned long long) * kWorkSlots) == cudaSuccess &&
            cudaMalloc(&d.wdone, sizeof(unsigned int) * kWorkSlots) == cudaSuccess &&
            cudaMalloc(&d.gcnt, sizeof(unsigned int) * kMaxTasks * (size_t)max_rows) == cudaSuccess;
  if (ok) {  // multi-CTA segmenter scratch (used for T >= kSegMultiMin)
    const size_t cap = (size_t)(max_rows + 4095) / 4096 * 4096;  // whole CTAs of rows
    ok = cudaMalloc(&d.lsort, sizeof(uint32_t) * cap) == cudaSuccess &&
         cudaMalloc(&d.lrank, sizeof(int32_t) * cap) == cudaSuccess &&
         cudaMalloc(&d.hist, sizeof(int32_t) * kSegHistMax) == cudaSuccess &&
         cudaMalloc(&d.offs, sizeof(int32_t) * kSegHistMax) == cudaSuccess;
    if (ok) cudaMemset(d.hist, 0, sizeof(int32_t) * kSegHistMax);
  }
  if (!ok) {
    cudaGetLastError();
    plan_destroy_impl(p);
    return fail(s, LORA_ERR_OOM, "plan allocation failed");
  }
  cudaMemset(d.counts, 0, sizeof(int32_t) * kCntWords);
  cudaMemset(d.wctr, 0, sizeof(unsigned long long) * kWorkSlots);
  cudaMemset(d.wdone, 0, sizeof(unsigned int) * kWorkSlots);
  cudaMemset(d.gcnt, 0, sizeof(unsigned int) * kMaxTasks * (size_t)max_rows);
  cudaMemset(d.seg_off, 0, sizeof(int32_t) * (max_rows + 1));
  *out = p;
  return LORA_OK;
}

void plan_destroy_impl(lora_plan* p) {
  if (!p) return;
  cudaFree(p->dev.perm);
  cudaFree(p->dev.seg_off);
  cudaFree(p->dev.seg_key);
  cudaFree(p->dev.counts);
  cudaFree(p->dev.groups);
  cudaFree(p->dev.tiles);
  cudaFree(p->dev.vpart);
  cudaFree(p->dev.vbf);
  cudaFree(p->dev.wctr);
  cudaFree(p->dev.wdone);
  cudaFree(p->dev.gcnt);
  cudaFree(p->dev.lsort);
  cudaFree(p->dev.lrank);
  cudaFree(p->dev.hist);
  cudaFree(p->dev.offs);
  delete p;
}

// tcgen05 path: rank 8 / 16 / 32 / 64 / 128, every slot's item widths multiples of the 128-wide MMA tiles
static bool tc_enabled(const lora_server* s) {
  if (!tc_available() || !tc_rank_supported(s->r) || s->small_seg_max < 0) return false;
  for (const auto& sl : s->slots)
    if (sl.KI % 128 || sl.CI % 128) return false;
  return true;
}

lora_status_t plan_build_impl(lora_server* s, lora_plan* p, const int32_t* adapter_ids, const int32_t* expert_ids,
                              int T, int E, cudaStream_t st, const int* T_dev) {
  if (T < 0 || T > p->max_rows) return fail(s, LORA_ERR_INVALID_ARG, "T must be in [0, max_rows]");
  if (E < 1) return fail(s, LORA_ERR_INVALID_ARG, "n_experts < 1");
  if (T > 0 && !adapter_ids) return fail(s, LORA_ERR_INVALID_ARG, "adapter_ids is NULL");
  SegParams sp;
  sp.small_max = s->small_seg_max < 0 ? kMaxPlanRows : s->small_seg_max;
  sp.tc_enabled = tc_enabled(s) ? 1 : 0;
  sp.tc_min_rows = s->tc_min_rows;
  sp.tile_rows = kTileRows;
  sp.group_rows = s->group_rows;
  CK(s, cudaSetDevice(s->device));
  const int pi = prof_start(s, st);
  sp.pl = placement(s);
  sp.cache = s->d_cache;
  CK(s, launch_segment(adapter_ids, expert_ids, T, E, s->n_adapters, sp, p->dev, s->d_err, st, T_dev));
  prof_stop(s, pi, kKSegment, st);
  p->n_experts = E;
  p->T = T;
  if (s->debug_sync) {
    CK(s, cudaStreamSynchronize(st));
    int flag = 0;
    CK(s, cudaMemcpy(&flag, s->d_err, sizeof(int), cudaMemcpyDeviceToHost));
    if (flag) {
      cudaMemset(s->d_err, 0, sizeof(int));
      return fail(s, LORA_ERR_ID_OUT_OF_RANGE, "an adapter or expert id was out of range (LORA_DEBUG_SYNC)");
    }
  }
  return LORA_OK;
}

// item-range -> task lookup tables of a launch (kernels.h find_task_kc / find_task_ci)
static void fill_task_tables(MultiArgs& a) {
  for (int i = 0; i < a.n_tasks; ++i) {
    const SlotTask& t = a.t[i];
    for (int k = 0; k < t.n_kc && t.kc_base + k < kTaskTable; ++k) a.kc_task[t.kc_base + k] = (uint8_t)i;
    for (int k = 0; k < t.n_ci && t.ci_base + k < kTaskTable; ++k) a.ci_task[t.ci_base + k] = (uint8_t)i;
  }
}

lora_status_t apply_multi_impl(lora_server* s, const lora_plan* p, int n, const int32_t* slots, const void* const* x,
                               void* const* y, lora_dtype_t y_dtype, cudaStream_t st, int store, const PushIn* push,
                               const int16_t* xreg, const int16_t* yreg, bool zero_y) {
  if (!p || p->s != s) return fail(s, LORA_ERR_INVALID_ARG, "plan does not belong to this server");
  if (p->n_experts < 0) return fail(s, LORA_ERR_INVALID_ARG, "plan was never built");
  if (n < 0 || (n > 0 && (!slots || !x || !y))) return fail(s, LORA_ERR_INVALID_ARG, "bad slot list");
  if (y_dtype != LORA_BF16 && y_dtype != LORA_FP32) return fail(s, LORA_ERR_UNSUPPORTED, "y_dtype");
  std::set<int> seen;
  // byte ranges of every y (written) and every x (read) of the launch: the
  // slots' kernels run concurrently (two chains, any order of items), so a y
  // may overlap no other y and no x of ANY slot of the call
  std::vector<std::pair<uintptr_t, uintptr_t>> yr, xr;
  for (int i = 0; i < n; ++i) {
    const int sl = slots[i];
    if (sl < 0 || sl >= (int)s->slots.size()) return fail(s, LORA_ERR_INVALID_ARG, "bad slot index");
    if (!seen.insert(sl).second) return fail(s, LORA_ERR_INVALID_ARG, "duplicate slot in one multi apply");
    if (s->slots[sl].E != p->n_experts)
      return fail(s, LORA_ERR_INVALID_ARG, "slot n_experts differs from the plan's n_experts");
    if (s->ep && slot_placement(s, sl).gbase != placement(s).gbase)
      return fail(s, LORA_ERR_INVALID_ARG, "the slot's layer belongs to another pipeline group (EP_x-PP_y)");
    if (p->T > 0) {
      if (!x[i] || !y[i]) return fail(s, LORA_ERR_INVALID_ARG, "x or y is NULL");
      if (!aligned16(x[i]) || !aligned16(y[i])) return fail(s, LORA_ERR_INVALID_ARG, "x and y must be 16-byte aligned");
      const SlotInfo& si = s->slots[sl];
      const uintptr_t xb = reinterpret_cast<uintptr_t>(x[i]), yb = reinterpret_cast<uintptr_t>(y[i]);
      const size_t xl = (size_t)p->T * si.h_in * 2, yl = (size_t)p->T * si.h_out * (y_dtype == LORA_FP32 ? 4 : 2);
      if (!push) {  // (push: x rows and y rows live in the sources' registered buffers)
        xr.push_back({xb, xb + xl});
        yr.push_back({yb, yb + yl});
      }
    }
  }
  if (!yr.empty()) {
    std::sort(yr.begin(), yr.end());
    for (size_t k = 1; k < yr.size(); ++k)
      if (yr[k].first < yr[k - 1].second) return fail(s, LORA_ERR_INVALID_ARG, "y buffers of two slots overlap");
    // y ranges are disjoint and sorted (so are their ends): the last y starting
    // before an x range ends is the only one that can overlap it
    for (const auto& r : xr) {
      auto it = std::lower_bound(yr.begin(), yr.end(), std::make_pair(r.second, uintptr_t(0)));
      if (it != yr.begin() && std::prev(it)->second > r.first)
        return fail(s, LORA_ERR_INVALID_ARG, "an x buffer overlaps a y buffer of the same call");
    }
  }
  if (n == 0 || p->T == 0) return LORA_OK;
  CK(s, cudaSetDevice(s->device));
  if (zero_y)  // delta outputs (store modes): rows without an adapter get a zero delta
    for (int i = 0; i < n; ++i)
      CK(s, cudaMemsetAsync(y[i], 0, (size_t)p->T * s->slots[slots[i]].h_out * (y_dtype == LORA_FP32 ? 4 : 2), st));
  if (s->n_resident) {
    // resident cache: wait for the pending host->device copies of these slots only
    for (int i = 0; i < n; ++i)
      if (s->slot_pending[slots[i]]) {
        CK(s, cudaStreamWaitEvent(st, s->slot_ready[slots[i]], 0));
        s->slot_pending[slots[i]] = 0;
      }
  }
  // the segmenter makes tcgen05 tiles only when the large segments hold at
  // least tc_min_rows rows: a plan of fewer rows (p->T bounds them, also for
  // a device-side row count) runs the CUDA-core chain alone -- no side-stream
  // fork, no empty tcgen05 launches, PDL between its kernels
  const bool tc = tc_enabled(s) && p->T >= s->tc_min_rows;
  for (int b0 = 0; b0 < n; b0 += kMaxTasks) {
    const int nb = std::min(kMaxTasks, n - b0);
    MultiArgs args;
    std::memset(&args, 0, sizeof(args));
    args.n_tasks = nb;
    args.y_fp32 = y_dtype == LORA_FP32;
    args.y_store = store;
    args.tc_cap_k = s->concurrent_tc ? s->tc_cap_k : 0;
    args.tc_flags = s->tc_flags;
    args.simt_split_items = s->simt_split_items;
    std::memset(args.tc_pair, -1, sizeof(args.tc_pair));  // (set per tcgen05 shrink launch below)
    args.pl = placement(s);
    args.cache = s->d_cache;
    args.scale = s->d_scale;
    if (push) args.push = *push;
    int kc = 0, ci = 0;
    bool any_split = false;
    for (int i = 0; i < nb; ++i) {
      const SlotInfo& si = s->slots[slots[b0 + i]];
      SlotTask& t = args.t[i];
      t.At = si.At;
      t.Bt = si.Bt;
      t.x = static_cast<const uint16_t*>(x[b0 + i]);
      args.xreg[i] = xreg ? xreg[b0 + i] : 0;
      args.yreg[i] = yreg ? yreg[b0 + i] : 0;
      t.y = y[b0 + i];
      t.vpart_off = (long long)si.kc_prefix * p->max_rows * s->r;
      t.vbf_off = (long long)slots[b0 + i] * p->max_rows * std::max(s->r, 16);  // (r = 8: rows padded to K = 16)
      t.h_in = si.h_in;
      t.h_out = si.h_out;
      t.E = si.E;
      t.KI = si.KI;
      t.SJ = si.SJ;
      t.n_kc = si.n_kc;
      if (tc && (p->T_hint > 0 ? p->T_hint : p->T) >= kTcWideKRows) {
        // large batches have tcgen05 tiles enough to fill the GPU without
        // splitting K: a tile's item takes the whole h_in (measured best vs
        // 1024 / 4096 / 7168 caps: prefill 0.634 / 0.583 / 0.577 / 0.569 ms)
        // and writes v directly; no reduction pass
        // (never below the slot's own KI: the partial-sum regions are sized
        // and placed by the slot's n_kc)
        t.KI = best_divisor(si.h_in, 128, std::max(s->tc_ki_max, si.KI));
        t.n_kc = si.h_in / t.KI;
      }
      t.CI = si.CI;
      t.SC = si.SC;
      t.n_ci = si.n_ci;
      t.kc_base = kc;
      t.ci_base = ci;
      kc += t.n_kc;
      ci += si.n_ci;
      any_split |= t.n_kc > 1;
    }
    args.total_kc = kc;
    args.total_ci = ci;
    fill_task_tables(args);
    const int grid = s->sm_count;
    // The CUDA-core shrink hands out (task, group) items round-robin; order the
    // tasks by decreasing h_in so the longest items go first and the tail of
    // the launch is made of the shortest ones.
    MultiArgs sargs = args;
    {
      std::vector<int> order(nb);
      for (int i = 0; i < nb; ++i) order[i] = i;
      std::stable_sort(order.begin(), order.end(),
                       [&](int a, int b) { return args.t[a].h_in > args.t[b].h_in; });
      int kc2 = 0, ci2 = 0;
      for (int i = 0; i < nb; ++i) {
        sargs.t[i] = args.t[order[i]];
        sargs.xreg[i] = args.xreg[order[i]];
        sargs.yreg[i] = args.yreg[order[i]];
        sargs.t[i].kc_base = kc2;
        sargs.t[i].ci_base = ci2;
        kc2 += sargs.t[i].n_kc;
        ci2 += sargs.t[i].n_ci;
      }
      fill_task_tables(sargs);
    }
    if (tc && s->tc_ci_max > 0 && (p->T_hint > 0 ? p->T_hint : p->T) >= kTcWideKRows) {
      // large batches: tcgen05 expand items of up to tc_ci_max columns of one
      // tile (decode-sized batches have few tiles and keep the slot's CI)
      int ci3 = 0;
      for (int i = 0; i < nb; ++i) {
        SlotTask& t = args.t[i];
        t.CI = best_divisor(t.h_out, 128, s->tc_ci_max);
        t.n_ci = t.h_out / t.CI;
        t.ci_base = ci3;
        ci3 += t.n_ci;
      }
      args.total_ci = ci3;
      fill_task_tables(args);
    }
    // The tcgen05 chain and the CUDA-core chain touch disjoint rows: run the
    // tcgen05 chain on the side stream (fork/join with events, graph-capturable)
    // so its CTAs fill the SMs the persistent CUDA-core kernels leave idle.
    const bool fork = tc && s->concurrent_tc;
    cudaStream_t tst = fork ? s->side_stream : st;
    g_pdl_allow = !tc;  // (see pdl_enabled)
    if (fork) {
      CK(s, cudaEventRecord(s->ev_fork, st));
      CK(s, cudaStreamWaitEvent(tst, s->ev_fork, 0));
    }
    int pi;
    if (tc) {
      // gate + up (slots sharing x, h_in, KI): one item per pair (x gathered
      // once, N = 2r MMA); the partner's items are dropped from the shrink's
      // item space (env LORA_TC_PAIR=0 disables)
      MultiArgs targs = args;
      std::memset(targs.tc_pair, -1, sizeof(targs.tc_pair));
      if (s->tc_pair) {
        std::vector<char> taken(nb, 0);
        for (int i = 0; i < nb; ++i) {
          if (taken[i]) continue;
          for (int j = i + 1; j < nb; ++j) {
            const SlotTask &a = args.t[i], &b = args.t[j];
            if (!taken[j] && a.x == b.x && a.h_in == b.h_in && a.KI == b.KI && a.n_kc == b.n_kc && a.E == b.E &&
                args.xreg[i] == args.xreg[j]) {
              targs.tc_pair[i] = (int8_t)j;
              taken[i] = taken[j] = 1;
              break;
            }
          }
        }
        // item order longest first (decreasing h_in; a pair's items carry two
        // slots' A): a long item started last would set the launch's tail --
        // the tasks are permuted in targs (partners remapped)
        std::vector<int> ord(nb), pos(nb);
        for (int i = 0; i < nb; ++i) ord[i] = i;
        auto weight = [&](int i) { return (long long)args.t[i].h_in * (targs.tc_pair[i] >= 0 ? 2 : 1); };
        if (s->tc_lpt)
          std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return weight(a) > weight(b); });
        for (int i = 0; i < nb; ++i) pos[ord[i]] = i;
        MultiArgs perm_args = targs;
        for (int i = 0; i < nb; ++i) {
          perm_args.t[i] = targs.t[ord[i]];
          perm_args.xreg[i] = targs.xreg[ord[i]];
          perm_args.yreg[i] = targs.yreg[ord[i]];
          perm_args.tc_pair[i] = targs.tc_pair[ord[i]] >= 0 ? (int8_t)pos[targs.tc_pair[ord[i]]] : (int8_t)-1;
        }
        std::vector<char> ptaken(nb);
        for (int i = 0; i < nb; ++i) ptaken[i] = taken[ord[i]];
        targs = perm_args;
        int kc4 = 0;
        for (int i = 0; i < nb; ++i) {
          SlotTask& t = targs.t[i];
          const bool partner = ptaken[i] && targs.tc_pair[i] < 0;
          t.kc_base = kc4;
          kc4 += partner ? 0 : t.n_kc;
        }
        // (a partner keeps its n_kc: the primary's epilogue stores its v with it)
        targs.total_kc = kc4;
        for (int i = 0; i < nb; ++i) {
          const bool partner = ptaken[i] && targs.tc_pair[i] < 0;
          for (int k = 0; !partner && k < targs.t[i].n_kc && targs.t[i].kc_base + k < kTaskTable; ++k)
            targs.kc_task[targs.t[i].kc_base + k] = (uint8_t)i;
        }
      }
      g_pdl_allow = s->pdl_tc;  // tcgen05 chain on its own stream: shrink -> (vreduce) -> expand
      pi = prof_start(s, tst);
      CK(s, launch_tc_shrink(s->r, targs, p->dev, p->T, grid, tst));
      prof_stop(s, pi, kKTcShrink, tst);
      if (any_split) {  // tiles of a task with n_kc == 1 got their v from the shrink
        pi = prof_start(s, tst);
        CK(s, launch_tc_vreduce(s->r, args, p->dev, grid, tst));
        prof_stop(s, pi, kKTcVreduce, tst);
      }
      pi = prof_start(s, tst);
      CK(s, launch_tc_expand(s->r, args, p->dev, grid, tst));
      prof_stop(s, pi, kKTcExpand, tst);
      g_pdl_allow = !tc;
    }
    pi = prof_start(s, st);
    CK(s, launch_simt_shrink(s->r, sargs, p->dev, grid, st));
    prof_stop(s, pi, kKSimtShrink, st);
    pi = prof_start(s, st);
    CK(s, launch_simt_expand(s->r, args, p->dev, grid, st));
    prof_stop(s, pi, kKSimtExpand, st);
    g_pdl_allow = false;
    if (fork) {
      CK(s, cudaEventRecord(s->ev_join, tst));
      CK(s, cudaStreamWaitEvent(st, s->ev_join, 0));
    }
  }
  if (s->debug_sync) {
    CK(s, cudaStreamSynchronize(st));
    int flag = 0;
    CK(s, cudaMemcpy(&flag, s->d_err, sizeof(int), cudaMemcpyDeviceToHost));
    if (flag) {
      cudaMemset(s->d_err, 0, sizeof(int));
      return fail(s, LORA_ERR_ID_OUT_OF_RANGE, "an adapter or expert id was out of range (LORA_DEBUG_SYNC)");
    }
  }
  return LORA_OK;
}

}  // namespace lora

extern "C" lora_status_t lora_plan_create(lora_server_t* s, int32_t max_rows, lora_plan_t** out) {
  if (!s || !out) return fail(s, LORA_ERR_INVALID_ARG, "NULL argument");
  CK(s, cudaSetDevice(s->device));
  return plan_create_impl(s, max_rows, out);
}

extern "C" lora_status_t lora_plan_destroy(lora_plan_t* p) {
  if (!p) return LORA_OK;
  cudaSetDevice(p->s->device);
  cudaDeviceSynchronize();
  plan_destroy_impl(p);
  return LORA_OK;
}

extern "C" lora_status_t lora_plan_build(lora_server_t* s, lora_plan_t* p, const int32_t* adapter_ids,
                                         const int32_t* expert_ids, int32_t T, int32_t n_experts, void* stream) {
  if (!s || !p) return fail(s, LORA_ERR_INVALID_ARG, "NULL server or plan");
  if (p->s != s) return fail(s, LORA_ERR_INVALID_ARG, "plan does not belong to this server");
  return plan_build_impl(s, p, adapter_ids, expert_ids, T, n_experts, static_cast<cudaStream_t>(stream));
}

extern "C" lora_status_t lora_plan_export(const lora_plan_t* p, int32_t* perm, int32_t* seg_offsets,
                                          int32_t* seg_keys, int32_t* n_valid, int32_t* n_segs, void* stream) {
  if (!p || !n_valid || !n_segs) return fail(nullptr, LORA_ERR_INVALID_ARG, "NULL argument");
  lora_server* s = p->s;
  CK(s, cudaSetDevice(s->device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int32_t cnt[kCntWords];
  CK(s, cudaMemcpyAsync(cnt, p->dev.counts, sizeof(cnt), cudaMemcpyDeviceToHost, st));
  CK(s, cudaStreamSynchronize(st));
  *n_valid = cnt[kCntValid];
  *n_segs = cnt[kCntSegs];
  if (perm && cnt[kCntValid] > 0)
    CK(s, cudaMemcpyAsync(perm, p->dev.perm, sizeof(int32_t) * cnt[kCntValid], cudaMemcpyDeviceToDevice, st));
  if (seg_offsets)
    CK(s, cudaMemcpyAsync(seg_offsets, p->dev.seg_off, sizeof(int32_t) * (cnt[kCntSegs] + 1),
                          cudaMemcpyDeviceToDevice, st));
  if (seg_keys && cnt[kCntSegs] > 0)
    CK(s, cudaMemcpyAsync(seg_keys, p->dev.seg_key, sizeof(int32_t) * cnt[kCntSegs], cudaMemcpyDeviceToDevice, st));
  CK(s, cudaStreamSynchronize(st));
  return LORA_OK;
}

extern "C" lora_status_t lora_plan_stats(const lora_plan_t* p, int32_t* out4, void* stream) {
  if (!p || !out4) return fail(nullptr, LORA_ERR_INVALID_ARG, "NULL argument");
  lora_server* s = p->s;
  CK(s, cudaSetDevice(s->device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int32_t cnt[kCntWords];
  CK(s, cudaMemcpyAsync(cnt, p->dev.counts, sizeof(cnt), cudaMemcpyDeviceToHost, st));
  CK(s, cudaStreamSynchronize(st));
  out4[0] = cnt[kCntValid];
  out4[1] = cnt[kCntSegs];
  out4[2] = cnt[kCntGroups];
  out4[3] = cnt[kCntTiles];
  return LORA_OK;
}

extern "C" lora_status_t lora_apply_plan(lora_server_t* s, const lora_plan_t* p, int32_t slot, const void* x, void* y,
                                         lora_dtype_t y_dtype, void* stream) {
  if (!s) return fail(nullptr, LORA_ERR_INVALID_ARG, "server is NULL");
  if (s->shard) return fail(s, LORA_ERR_INVALID_ARG, "sharded server: use lora_apply_sharded");
  const void* xs[1] = {x};
  void* ys[1] = {y};
  return apply_multi_impl(s, p, 1, &slot, xs, ys, y_dtype, static_cast<cudaStream_t>(stream));
}

extern "C" lora_status_t lora_apply_plan_multi(lora_server_t* s, const lora_plan_t* p, int32_t n, const int32_t* slots,
                                               const void* const* x, void* const* y, lora_dtype_t y_dtype,
                                               void* stream) {
  if (!s) return fail(nullptr, LORA_ERR_INVALID_ARG, "server is NULL");
  if (s->shard) return fail(s, LORA_ERR_INVALID_ARG, "sharded server: use lora_apply_sharded");
  return apply_multi_impl(s, p, n, slots, x, y, y_dtype, static_cast<cudaStream_t>(stream));
}

extern "C" lora_status_t lora_apply_plan_multi_delta(lora_server_t* s, const lora_plan_t* p, int32_t n,
                                                     const int32_t* slots, const void* const* x, void* const* delta,
                                                     lora_dtype_t delta_dtype, void* stream) {
  if (!s) return fail(nullptr, LORA_ERR_INVALID_ARG, "server is NULL");
  if (s->shard) return fail(s, LORA_ERR_INVALID_ARG, "sharded server: use lora_apply_sharded");
  if (delta_dtype != LORA_BF16 && delta_dtype != LORA_FP32) return fail(s, LORA_ERR_UNSUPPORTED, "delta_dtype");
  return apply_multi_impl(s, p, n, slots, x, delta, delta_dtype, static_cast<cudaStream_t>(stream),
                          delta_dtype == LORA_BF16 ? 2 : 1, nullptr, nullptr, nullptr, true);
}

extern "C" lora_status_t lora_apply(lora_server_t* s, int32_t slot, const void* x, const int32_t* adapter_ids,
                                    const int32_t* expert_ids, void* y, lora_dtype_t y_dtype, int32_t T,
                                    void* stream) {
  if (!s) return fail(nullptr, LORA_ERR_INVALID_ARG, "server is NULL");
  if (s->shard) return fail(s, LORA_ERR_INVALID_ARG, "sharded server: use lora_apply_sharded");
  if (slot < 0 || slot >= (int)s->slots.size()) return fail(s, LORA_ERR_INVALID_ARG, "bad slot index");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  lora_status_t rc = plan_build_impl(s, s->internal_plan, adapter_ids, expert_ids, T, s->slots[slot].E, st);
  if (rc != LORA_OK) return rc;
  const void* xs[1] = {x};
  void* ys[1] = {y};
  return apply_multi_impl(s, s->internal_plan, 1, &slot, xs, ys, y_dtype, st);
}

// ---------------------------------------------------------------------------
// end-to-end with host buffers
// ---------------------------------------------------------------------------
static lora_status_t apply_multi_host_impl(lora_server_t* s, int32_t n, const int32_t* slots,
                                          const void* const* x_host, const int32_t* adapter_ids_host,
                                          const int32_t* expert_ids_host, void* const* y_host, lora_dtype_t y_dtype,
                                          int32_t T, void* stream, bool delta) {
  if (!s) return fail(nullptr, LORA_ERR_INVALID_ARG, "server is NULL");
  if (s->shard) return fail(s, LORA_ERR_INVALID_ARG, "sharded server: use lora_apply_sharded");
  if (n < 1 || !slots || !x_host || !y_host || (T > 0 && !adapter_ids_host))
    return fail(s, LORA_ERR_INVALID_ARG, "NULL argument");
  if (T < 0 || T > s->max_rows) return fail(s, LORA_ERR_INVALID_ARG, "T must be in [0, max_rows]");
  if (y_dtype != LORA_BF16 && y_dtype != LORA_FP32) return fail(s, LORA_ERR_UNSUPPORTED, "y_dtype");
  for (int i = 0; i < n; ++i) {
    if (slots[i] < 0 || slots[i] >= (int)s->slots.size()) return fail(s, LORA_ERR_INVALID_ARG, "bad slot index");
    if (s->slots[slots[i]].E != s->slots[slots[0]].E)
      return fail(s, LORA_ERR_INVALID_ARG, "all slots of one call must share n_experts");
  }
  if (T == 0) return LORA_OK;
  CK(s, cudaSetDevice(s->device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t ysz = y_dtype == LORA_FP32 ? 4 : 2;
  // Pipelined executor over (row chunk, slot group) pieces.  The rows are cut
  // into RC chunks (1 for small batches, up to 4) and each chunk's slots into
  // groups of >= 32 MB of upload; per piece: its x rows (first use of the x
  // buffer in the row chunk) and y rows go host->device on the copy stream,
  // the piece is applied on the caller's stream with the row chunk's plan
  // (built once from that chunk's ids), and its y rows go device->host on a
  // third stream -- piece p+1's upload, piece p's apply and piece p-1's
  // download overlap (the two copy directions use separate copy engines), so
  // the PCIe time is exposed only for the first piece's upload and the last
  // piece's download.  Row chunks re-stream the weights of the units they
  // touch (one apply per chunk): GPU time grows, far below the PCIe time at
  // the sizes where RC > 1.  Each row's arithmetic depends only on its
  // segment's route (CUDA-core / tcgen05), decided per chunk.  The caller's
  // stream waits for the last download: the call stays stream-ordered.
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  std::vector<const void*> xd;  // distinct x host pointers
  std::vector<int> x_of(n);
  for (int i = 0; i < n; ++i) {
    auto it = std::find(xd.begin(), xd.end(), x_host[i]);
    if (it == xd.end()) {
      x_of[i] = (int)xd.size();
      xd.push_back(x_host[i]);
    } else {
      x_of[i] = (int)(it - xd.begin());
    }
  }
  std::vector<size_t> x_off(xd.size()), y_off(n);
  size_t off = al((size_t)T * 4) * 2;
  std::vector<int> x_hin(xd.size());
  for (int i = 0; i < n; ++i) x_hin[x_of[i]] = s->slots[slots[i]].h_in;
  for (size_t j = 0; j < xd.size(); ++j) {
    x_off[j] = off;
    off += al((size_t)T * x_hin[j] * 2);
  }
  for (int i = 0; i < n; ++i) {
    y_off[i] = off;
    off += al((size_t)T * s->slots[slots[i]].h_out * ysz);
  }
  if (off > s->h2d_bytes) {
    cudaStreamSynchronize(st);
    cudaFree(s->h2d_buf);
    s->h2d_buf = nullptr;
    s->h2d_bytes = 0;
    CK(s, cudaMalloc(&s->h2d_buf, off));
    s->h2d_bytes = off;
  }
  if (!s->copy_stream) CK(s, cudaStreamCreateWithFlags(&s->copy_stream, cudaStreamNonBlocking));
  if (!s->d2h_stream) CK(s, cudaStreamCreateWithFlags(&s->d2h_stream, cudaStreamNonBlocking));
  // row chunks: RC = clamp(T / 2048, 1, 4) (env LORA_HOST_ROW_CHUNKS), one plan each
  int RC = std::max(1, std::min(4, T / 2048));
  if (const char* e = std::getenv("LORA_HOST_ROW_CHUNKS")) RC = std::max(1, std::min(8, std::atoi(e)));
  RC = std::min(RC, T);
  while ((int)s->host_plans.size() < RC) {
    lora_plan* hp = nullptr;
    const lora_status_t pc = plan_create_impl(s, s->max_rows, &hp);
    if (pc != LORA_OK) return pc;
    s->host_plans.push_back(hp);
  }
  std::vector<int> r0(RC + 1);
  for (int c = 0; c <= RC; ++c) r0[c] = (int)((long long)T * c / RC);
  // pieces: per row chunk, consecutive slots cut at >= max(1/8 of the chunk's upload, 32 MB)
  struct Piece {
    int rc, s0, s1;
  };
  std::vector<Piece> pieces;
  std::vector<std::vector<char>> x_first(RC, std::vector<char>(n, 0));
  for (int c = 0; c < RC; ++c) {
    const size_t rows = (size_t)(r0[c + 1] - r0[c]);
    std::vector<size_t> up(n);
    std::vector<char> seen(xd.size(), 0);
    size_t total = 0;
    for (int i = 0; i < n; ++i) {
      up[i] = delta ? 0 : rows * s->slots[slots[i]].h_out * ysz;
      if (!seen[x_of[i]]) {
        seen[x_of[i]] = 1;
        x_first[c][i] = 1;
        up[i] += rows * x_hin[x_of[i]] * 2;
      }
      total += up[i];
    }
    const size_t target = std::max<size_t>(total / 8, (size_t)32 << 20);
    int start = 0;
    size_t acc = 0;
    for (int i = 0; i < n; ++i) {
      acc += up[i];
      if (acc >= target || i == n - 1) {
        pieces.push_back({c, start, i + 1});
        start = i + 1;
        acc = 0;
      }
    }
  }
  const int n_pieces = (int)pieces.size();
  while ((int)s->events.size() < 2 * n_pieces + 2) {
    cudaEvent_t e;
    CK(s, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    s->events.push_back(e);
  }
  cudaEvent_t ev_start = s->events[0], ev_ids = s->events[1];
  char* base = static_cast<char*>(s->h2d_buf);
  int32_t* d_ad = reinterpret_cast<int32_t*>(base);
  int32_t* d_ex = reinterpret_cast<int32_t*>(base + al((size_t)T * 4));
  // the copy streams start after whatever the caller queued on `stream`
  CK(s, cudaEventRecord(ev_start, st));
  CK(s, cudaStreamWaitEvent(s->copy_stream, ev_start, 0));
  CK(s, cudaStreamWaitEvent(s->d2h_stream, ev_start, 0));
  CK(s, cudaMemcpyAsync(d_ad, adapter_ids_host, (size_t)T * 4, cudaMemcpyHostToDevice, s->copy_stream));
  if (expert_ids_host)
    CK(s, cudaMemcpyAsync(d_ex, expert_ids_host, (size_t)T * 4, cudaMemcpyHostToDevice, s->copy_stream));
  CK(s, cudaEventRecord(ev_ids, s->copy_stream));
  CK(s, cudaStreamWaitEvent(st, ev_ids, 0));
  const int E = s->slots[slots[0]].E;
  for (int c = 0; c < RC; ++c) {
    lora_status_t rc = plan_build_impl(s, s->host_plans[c], d_ad + r0[c], expert_ids_host ? d_ex + r0[c] : nullptr,
                                       r0[c + 1] - r0[c], E, st);
    if (rc != LORA_OK) return rc;
  }
  std::vector<const void*> xs(n);
  std::vector<void*> ys(n);
  for (int pi = 0; pi < n_pieces; ++pi) {
    const Piece& pc = pieces[pi];
    const int a = r0[pc.rc], rows = r0[pc.rc + 1] - a;
    cudaEvent_t ev_in = s->events[2 + 2 * pi], ev_done = s->events[3 + 2 * pi];
    for (int i = pc.s0; i < pc.s1; ++i) {
      const size_t hi = (size_t)x_hin[x_of[i]], ho = (size_t)s->slots[slots[i]].h_out;
      if (x_first[pc.rc][i])
        CK(s, cudaMemcpyAsync(base + x_off[x_of[i]] + (size_t)a * hi * 2,
                              static_cast<const char*>(xd[x_of[i]]) + (size_t)a * hi * 2, (size_t)rows * hi * 2,
                              cudaMemcpyHostToDevice, s->copy_stream));
      if (!delta)
        CK(s, cudaMemcpyAsync(base + y_off[i] + (size_t)a * ho * ysz,
                              static_cast<const char*>(y_host[i]) + (size_t)a * ho * ysz, (size_t)rows * ho * ysz,
                              cudaMemcpyHostToDevice, s->copy_stream));
      xs[i] = base + x_off[x_of[i]] + (size_t)a * hi * 2;
      ys[i] = base + y_off[i] + (size_t)a * ho * ysz;
    }
    CK(s, cudaEventRecord(ev_in, s->copy_stream));
    CK(s, cudaStreamWaitEvent(st, ev_in, 0));
    const lora_status_t rc = apply_multi_impl(s, s->host_plans[pc.rc], pc.s1 - pc.s0, slots + pc.s0, xs.data() + pc.s0,
                                              ys.data() + pc.s0, y_dtype, st, delta ? (y_dtype == LORA_BF16 ? 2 : 1) : 0,
                                              nullptr, nullptr, nullptr, delta);
    if (rc != LORA_OK) return rc;
    CK(s, cudaEventRecord(ev_done, st));
    CK(s, cudaStreamWaitEvent(s->d2h_stream, ev_done, 0));
    for (int i = pc.s0; i < pc.s1; ++i) {
      const size_t ho = (size_t)s->slots[slots[i]].h_out;
      CK(s, cudaMemcpyAsync(static_cast<char*>(y_host[i]) + (size_t)a * ho * ysz, ys[i], (size_t)rows * ho * ysz,
                            cudaMemcpyDeviceToHost, s->d2h_stream));
    }
  }
  // join: the caller's stream completes after the last download
  CK(s, cudaEventRecord(ev_start, s->d2h_stream));
  CK(s, cudaStreamWaitEvent(st, ev_start, 0));
  return LORA_OK;
}

extern "C" lora_status_t lora_apply_multi_host(lora_server_t* s, int32_t n, const int32_t* slots,
                                               const void* const* x_host, const int32_t* adapter_ids_host,
                                               const int32_t* expert_ids_host, void* const* y_host,
                                               lora_dtype_t y_dtype, int32_t T, void* stream) {
  return apply_multi_host_impl(s, n, slots, x_host, adapter_ids_host, expert_ids_host, y_host, y_dtype, T, stream,
                               false);
}

extern "C" lora_status_t lora_apply_multi_host_delta(lora_server_t* s, int32_t n, const int32_t* slots,
                                                     const void* const* x_host, const int32_t* adapter_ids_host,
                                                     const int32_t* expert_ids_host, void* const* delta_host,
                                                     lora_dtype_t delta_dtype, int32_t T, void* stream) {
  return apply_multi_host_impl(s, n, slots, x_host, adapter_ids_host, expert_ids_host, delta_host, delta_dtype, T,
                               stream, true);
}

// ---------------------------------------------------------------------------
// per-launch profiling with CUDA events on the launching stream
// ---------------------------------------------------------------------------
int prof_start(lora_server* s, cudaStream_t st) {
  if (!s->prof_on || s->prof_recs.size() * 2 + 2 > s->prof_pool.size()) return -1;
  const int i = (int)s->prof_recs.size() * 2;
  if (cudaEventRecord(s->prof_pool[i], st) != cudaSuccess) return -1;
  return i;
}

void prof_stop(lora_server* s, int idx, int kind, cudaStream_t st) {
  if (idx < 0) return;
  if (cudaEventRecord(s->prof_pool[idx + 1], st) == cudaSuccess) s->prof_recs.push_back({idx, kind});
}

extern "C" lora_status_t lora_profile_enable(lora_server_t* s, int32_t max_launches) {
  if (!s) return fail(nullptr, LORA_ERR_INVALID_ARG, "server is NULL");
  CK(s, cudaSetDevice(s->device));
  s->prof_recs.clear();
  if (max_launches <= 0) {
    s->prof_on = false;
    return LORA_OK;
  }
  while ((int)s->prof_pool.size() < 2 * max_launches) {
    cudaEvent_t e;
    CK(s, cudaEventCreate(&e));
    s->prof_pool.push_back(e);
  }
  s->prof_on = true;
  return LORA_OK;
}

extern "C" lora_status_t lora_profile_read(lora_server_t* s, int32_t n_kinds, int32_t* launches, double* total_ms) {
  if (!s || !launches || !total_ms || n_kinds < 1) return fail(s, LORA_ERR_INVALID_ARG, "bad argument");
  CK(s, cudaSetDevice(s->device));
  for (int k = 0; k < n_kinds; ++k) {
    launches[k] = 0;
    total_ms[k] = 0.0;
  }
  for (auto& r : s->prof_recs) {
    CK(s, cudaEventSynchronize(s->prof_pool[r.first + 1]));
    float ms = 0.f;
    CK(s, cudaEventElapsedTime(&ms, s->prof_pool[r.first], s->prof_pool[r.first + 1]));
    if (r.second < n_kinds) {
      launches[r.second] += 1;
      total_ms[r.second] += ms;
    }
  }
  s->prof_recs.clear();
  return LORA_OK;
}

extern "C" const char* lora_kernel_name(int32_t kind) {
  static const char* names[kKNumKinds] = {"segment",        "simt_shrink",   "tc05_shrink",  "simt_expand",
                                          "tc05_expand",    "shard_bucket",  "shard_gather", "shard_scatter_add",
                                          "tc05_vreduce"};
  return (kind >= 0 && kind < kKNumKinds) ? names[kind] : "unknown";
}

// synthetic activation rows (benchmarks / tests): dst bf16 [rows][width]
extern "C" lora_status_t lora_synth_fill_rows(void* dst, int64_t rows, int32_t width, uint64_t seed, uint32_t tag,
                                              int32_t shift, int64_t row_base, void* stream) {
  if (!dst || rows < 0 || width < 1) return fail(nullptr, LORA_ERR_INVALID_ARG, "bad argument");
  cudaError_t e = launch_fill_rows(static_cast<uint16_t*>(dst), rows, width, seed, tag, shift, row_base,
                                   static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(nullptr, e, "lora_synth_fill_rows");
  return LORA_OK;
}
