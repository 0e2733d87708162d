// server.h -- internal C++ definitions of the opaque C-ABI handles.
#pragma once

#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "../../include/lora_server.h"
#include "kernels.h"

struct SlotInfo {
  int h_in = 0, h_out = 0, E = 1;
  long long units = 0;     // local units = local adapters * E
  uint16_t* At = nullptr;  // store, shrink operand
  uint16_t* Bt = nullptr;  // store, expand operand
  int KI = 0, SJ = 0, n_kc = 0;
  int CI = 0, SC = 0, n_ci = 0;
  int kc_prefix = 0;       // sum of n_kc over previous slots (workspace offset)
};

struct ShardState;  // shard.cu

struct lora_server {
  int device = 0;
  int r = 0;
  int n_adapters = 0;
  int n_adapters_local = 0;
  int max_rows = 0;
  int sm_count = 148;
  int small_seg_max = 8;
  int tc_cap_k = 2;        // tcgen05 CTAs per tile when both chains run (measured 1/2/4/8 with the staged-tile expand: Mixtral decode 0.478/0.482/0.489/0.494 ms, prefill 0.576/0.561/-/- ms; env LORA_TC_CAP_K, 0 = all SMs)
  int tc_ci_max = 8192;    // tcgen05 expand: max h_out per item (measured best of 1024..8192; env LORA_TC_CI_MAX, 0 = slot CI)
  int tc_flags = 1;         // tcgen05 expand L2 policies (MultiArgs::tc_flags; env LORA_TCE_FLAGS): Bt evict_last (measured prefill 0.550 -> 0.529 ms; y evict_first hints slower)
  int group_rows = 8;           // rows per CUDA-core group (kGroupRows; env LORA_GROUP_ROWS, smaller only)
  int tc_min_rows = 256;    // segmenter: tcgen05 tiles only with at least this many rows in large segments (env LORA_TC_MIN_ROWS)
  int simt_split_items = 0;  // MultiArgs::simt_split_items (set at create: 8 items per CUDA-core CTA; env LORA_SIMT_SPLIT)
  bool tc_pair = true;
  bool pdl_tc = false;      // PDL between the tcgen05 chain's kernels on a forking apply (env LORA_PDL_TC=1)
  bool tc_lpt = true;       // tcgen05 shrink items longest first (env LORA_TC_LPT=0: slot order)      // tcgen05 shrink: slots sharing x in one N = 2r MMA (env LORA_TC_PAIR=0: off)
  int tc_ki_max = 1 << 20;  // large-batch tcgen05 shrink: max h_in per item, default the whole h_in (env LORA_TC_KI_MAX)
  int world = 1, shard_rank = 0;
  int n_hot = 0;  // adapters [0, n_hot) replicated on every rank of a sharded server
  int ep = 0;     // 1: expert-parallel ownership (unit (a, e) on rank gbase + e mod x)
  int pp = 1;     // ep: pipeline stages y of EP_x-PP_y (x = world / y ranks per group)
  std::vector<int> slot_layer;  // layer of each slot (group = layer mod pp)
  bool debug_sync = false;
  std::vector<SlotInfo> slots;
  int total_kc = 0;        // sum of n_kc over all slots
  float* d_scale = nullptr;
  int* d_err = nullptr;
  lora_plan_t* internal_plan = nullptr;
  std::vector<lora_plan_t*> host_plans;  // lora_apply_multi_host: one plan per row chunk
  std::string last_error;
  // staging for lora_apply_multi_host (grown lazily)
  void* h2d_buf = nullptr;
  size_t h2d_bytes = 0;
  cudaStream_t copy_stream = nullptr;   // lora_apply_multi_host: host -> device copies
  cudaStream_t d2h_stream = nullptr;    // lora_apply_multi_host: device -> host copies
  // tcgen05 kernels run on a side stream forked from / joined to the caller's
  // stream, concurrently with the CUDA-core kernels (independent rows)
  cudaStream_t side_stream = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  bool concurrent_tc = true;  // env LORA_SERIAL=1 keeps everything on the caller's stream
  std::vector<cudaEvent_t> events;      // lora_apply_multi_host pipeline events (grown on demand)
  ShardState* shard = nullptr;
  // resident-adapter cache (n_resident > 0): host backing store per slot in the
  // kernel layout, device cache-slot table, LRU state, per-slot load events
  int n_resident = 0;
  std::vector<uint16_t*> hostA, hostB;  // pinned, [n_adapters][E][...] per slot
  int32_t* d_cache = nullptr;           // [n_adapters] cache slot or -1
  std::vector<int32_t> h_cache;         // host mirror of d_cache
  std::vector<int> cache_owner;         // [n_resident] adapter in each cache slot, -1 empty
  std::vector<long long> cache_use;     // [n_resident] last require tick
  long long cache_tick = 0;
  std::vector<cudaEvent_t> slot_ready;  // per slot: its copies done
  std::vector<char> slot_pending;       // per slot: a wait is owed by the next apply
  // per-launch CUDA-event profiling (lora_profile_enable / lora_profile_read)
  bool prof_on = false;
  std::vector<cudaEvent_t> prof_pool;
  std::vector<std::pair<int, int>> prof_recs;  // (event index, kernel kind)
};

// kernel kinds reported by lora_profile_read
enum { kKSegment = 0, kKSimtShrink = 1, kKTcShrink = 2, kKSimtExpand = 3, kKTcExpand = 4, kKShardBucket = 5,
       kKShardGather = 6, kKShardScatter = 7, kKTcVreduce = 8, kKNumKinds = 9 };
int prof_start(lora_server* s, cudaStream_t st);
void prof_stop(lora_server* s, int idx, int kind, cudaStream_t st);

struct lora_plan {
  lora_server* s = nullptr;
  lora::PlanDev dev{};
  int max_rows = 0;
  int n_experts = -1;  // E the plan was last built with (-1: never built)
  int T = 0;
  int T_hint = 0;      // > 0: row count to size the tcgen05 split by (device-side row counts: the capacity is T)
  int world = 1;
};

namespace lora {
lora_status_t fail(lora_server* s, lora_status_t st, const std::string& msg);
lora_status_t cuda_fail(lora_server* s, cudaError_t e, const char* where);
lora_status_t apply_multi_impl(lora_server* s, const lora_plan* p, int n, const int32_t* slots,
                               const void* const* x, void* const* y, lora_dtype_t y_dtype, cudaStream_t st,
                               int store = 0, const PushIn* push = nullptr, const int16_t* xreg = nullptr,
                               const int16_t* yreg = nullptr, bool zero_y = false);
lora_status_t plan_build_impl(lora_server* s, lora_plan* p, const int32_t* adapter_ids, const int32_t* expert_ids,
                              int T, int E, cudaStream_t st, const int* T_dev = nullptr);
lora_status_t plan_create_impl(lora_server* s, int max_rows, lora_plan** out);
void plan_destroy_impl(lora_plan* p);
}  // namespace lora

// shard.cu / lora_server.cu cross-file helpers (C++ linkage)
void lora_shard_free(lora_server* s);
lora_status_t lora_shard_check_flags(lora_server* s, int flag);  // sticky-flag bits of the sharded path, NCCL errors
lora_status_t create_common_sharded(const lora_config_t* cfg, int world, int rank, lora_server** out, int n_hot,
                                    int ep);
// this rank's placement (ep: its own group)
inline lora::Placement placement(const lora_server* s) {
  lora::Placement p{s->world, s->shard_rank, s->n_hot, s->ep};
  if (s->ep) {
    p.x = s->world / s->pp;
    p.gbase = (s->shard_rank / p.x) * p.x;
  }
  return p;
}
// placement of one slot's units (ep: the group of the slot's layer)
inline lora::Placement slot_placement(const lora_server* s, int slot) {
  lora::Placement p = placement(s);
  if (s->ep) p.gbase = (s->slot_layer[slot] % s->pp) * p.x;
  return p;
}
lora_status_t apply_multi_delta(lora_server* s, const lora_plan* p, int n, const int32_t* slots,
                                const void* const* x, void* const* d, cudaStream_t st, bool bf16);
