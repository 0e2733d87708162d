// kernels.h -- internal (non-ABI) declarations shared by the .cu files of the
// CUDA path: device-side plan view, per-launch task descriptors, launchers.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace lora {

constexpr int kMaxPlanRows = 32768;  // plan capacity (rows); above kMaxOneCtaRows the multi-CTA segmenter runs
constexpr int kMaxOneCtaRows = 16384;  // single-CTA segmenter capacity (128 KB of composites)
constexpr int kSegMultiMin = 4096;   // T at or above which the multi-CTA segmenter runs
constexpr int kSegHistMax = 1 << 18; // K * C bound of the multi-CTA segmenter's histogram
constexpr int kTcWideKRows = 4096;  // plan rows from which tcgen05 shrink items take the whole h_in
constexpr int kGroupRows = 8;        // rows per CUDA-core work group
constexpr int kTileRows = 128;       // rows per tcgen05 tile (UMMA M / N)
constexpr int kMaxTasks = 128;       // slots per multi-slot launch (param space; 32 layers x q,k,v,o)
constexpr int kTaskTable = 2048;     // item-range -> task lookup entries (param space)

enum { kCntValid = 0, kCntSegs = 1, kCntGroups = 2, kCntTiles = 3, kCntWords = 8 };
// work-counter slots of the persistent kernels
enum { kWqSimtShrink = 0, kWqSimtExpand = 1, kWqTcShrink = 2, kWqTcExpand = 3, kWorkSlots = 8 };

// Unit placement of a (sharded) server; a unit is (adapter a, expert e).
//  * LoRA Data Parallel (ep = 0): adapters [0, n_hot) are
//    replicated on every rank (popularity-aware placement);
//    adapter a >= n_hot is owned by rank (a - n_hot) mod world, all experts.
//  * Expert parallel (ep = 1, Table 1 EP row):
//    unit (a, e) is owned by rank gbase + e mod x, every adapter (all slots of
//    the server share one expert count, checked at create).  Pure EP: x =
//    world, gbase = 0.  Hybrid EP_x-PP_y (Table 1 last row): the
//    world is y groups of x ranks, layer l belongs to group l mod y
//    (interleaved), gbase = (l mod y) * x; ranks outside the group store no
//    unit of that layer.
// An unsharded server is {1, 0, 0, 0, 1, 0}.
struct Placement {
  int world, rank, n_hot, ep;
  int x = 1;      // ep: expert-parallel degree (ranks per group)
  int gbase = 0;  // ep: first rank of the group that owns this layer
  // adapter-level view (ep = 0)
  __host__ __device__ bool owns(int a) const { return a < n_hot || (a - n_hot) % world == rank; }
  __host__ __device__ int owner(int a) const { return a < n_hot ? rank : (a - n_hot) % world; }
  __host__ __device__ long long local_index(int a) const {
    return a < n_hot ? (long long)a : (long long)n_hot + (a - n_hot) / world;
  }
  // inverse of local_index for an owned adapter
  __host__ __device__ long long global_adapter(long long li) const {
    return li < n_hot ? li : (long long)n_hot + (li - n_hot) * world + rank;
  }
  // adapters stored on this rank (ep = 0)
  __host__ __device__ int n_local(int n_adapters) const {
    const int h = n_hot < n_adapters ? n_hot : n_adapters;
    const int rest = n_adapters - h;
    return h + (rest > rank ? (rest - rank + world - 1) / world : 0);
  }
  // this rank's position in the owning group (ep), -1 if outside it
  __host__ __device__ int erank() const { return (rank >= gbase && rank < gbase + x) ? rank - gbase : -1; }
  // unit-level view (both modes)
  __host__ __device__ int experts_local(int E) const {
    if (!ep) return E;
    const int r = erank();
    return (r >= 0 && E > r) ? (E - 1 - r) / x + 1 : 0;
  }
  __host__ __device__ bool owns_unit(int a, int e) const { return ep ? gbase + e % x == rank : owns(a); }
  __host__ __device__ int owner_unit(int a, int e) const { return ep ? gbase + e % x : owner(a); }
  __host__ __device__ long long local_unit(int a, int e, int E) const {
    return ep ? (long long)a * experts_local(E) + e / x : local_index(a) * E + e;
  }
  // inverse of local_unit: global key a*E+e of local unit u (-1: none)
  __host__ __device__ long long global_key(long long u, int E, int n_adapters) const {
    const int el = experts_local(E);
    if (el == 0) return -1;
    const long long al = u / el, ei = u - al * el;
    const long long a = ep ? al : global_adapter(al);
    const long long e = ep ? ei * x + erank() : ei;
    return a < n_adapters ? a * E + e : -1;
  }
  // units stored on this rank
  __host__ __device__ long long n_local_units(int n_adapters, int E) const {
    return ep ? (long long)n_adapters * experts_local(E) : (long long)n_local(n_adapters) * E;
  }
};

// Device view of a plan (all device pointers).
struct PlanDev {
  int32_t* perm;     // [max_rows]   sorted position -> original row
  int32_t* seg_off;  // [max_rows+1]
  int32_t* seg_key;  // [max_rows]   key a*E+e
  int32_t* counts;   // [kCntWords]
  int4* groups;      // [max_rows]   CUDA-core groups {row_begin, nrows, key, seg}
  int4* tiles;       // [max_rows]   tcgen05 tiles    {row_begin, nrows, key, seg}
  float* vpart;      // shrink partial sums, per slot region [n_kc][max_rows][r]
  uint16_t* vbf;     // tcgen05 path: complete v rounded to bf16, per slot region [max_rows][r]
  unsigned long long* wctr;  // [kWorkSlots] dynamic item counters of the persistent kernels (self-resetting)
  unsigned int* wdone;       // [kWorkSlots] finished-CTA counters
  // multi-CTA segmenter scratch
  uint32_t* lsort;           // [max_rows rounded up to 4096] per-CTA sorted composites (key << 12 | local row)
  int32_t* lrank;            // [same] rank of each sorted entry inside its key's run
  int32_t* hist;             // [kSegHistMax] run lengths, key-major [K][C] (kept zero between builds)
  int32_t* offs;             // [kSegHistMax] exclusive prefix of hist
  unsigned int* gcnt;        // [kMaxTasks][max_rows] K-split CUDA-core shrink: arrivals per (task, group), self-resetting
  int max_rows;
};

struct SegParams {
  int small_max;   // segments with more rows than this go to tcgen05 (if enabled)
  int tc_enabled;  // a tcgen05 rank (16 / 32 / 64 / 128) and not forced off
  int tc_min_rows; // tcgen05 tiles only if the large segments hold at least this many rows in total
  int tile_rows;
  int group_rows;   // rows per CUDA-core group (<= kGroupRows; env LORA_GROUP_ROWS, a test / tuning hook)
  Placement pl;    // rows whose adapter this rank does not store are rejected (flagged)
  const int32_t* cache;  // resident-cache mode: [n_adapters] cache slot or -1 (not resident: rejected)
};

// key a*E+e -> unit index in the device store: the adapter's resident cache
// slot (cache mode) or its local index under the placement
__host__ __device__ inline long long store_unit(int key, int E, const Placement& pl, const int32_t* cache) {
  const int a = key / E, e = key - a * E;
#ifdef __CUDA_ARCH__
  if (cache) return (long long)__ldg(cache + a) * E + e;
#else
  if (cache) return (long long)cache[a] * E + e;
#endif
  return pl.local_unit(a, e, E);
}

// One slot inside a (multi-slot) launch.
struct SlotTask {
  const uint16_t* At;  // weight store, shrink operand
  const uint16_t* Bt;  // weight store, expand operand
  const uint16_t* x;   // bf16 [T][h_in]
  void* y;             // bf16 / fp32 [T][h_out]
  long long vpart_off; // float offset of this slot's partial-sum region
  long long vbf_off;   // element offset of this slot's bf16 v region
  int h_in, h_out, E;
  int KI, SJ, n_kc;    // shrink: j-range per item, j per stage, items per row group
  int CI, SC, n_ci;    // expand: c-range per item, c rows per stage, items per row group
  int kc_base, ci_base;// prefix over tasks of n_kc / n_ci
};

// Owner side of a sharded apply over registered buffers (shard.cu, the push
// path): received row r was sent by source rank origin[r] >> 24 from its
// local row origin[r] & 0xFFFFFF.  The shrink kernels read that x row straight
// from the source's registered x buffer and the expand epilogues add the
// delta straight into the source's registered y row (NVLink peer mappings),
// so neither the rows nor the deltas are staged anywhere.
constexpr int kMaxWorld = 8;
constexpr int kOriginRowBits = 24;
struct PushIn {
  int G;                     // 0: local rows (t.x / t.y + row)
  const int32_t* origin;     // [rows] (source << 24) | source-local row
  char* const* reg;          // device [n_reg * G]: base of registered buffer k on rank p
};

struct MultiArgs {
  int n_tasks;
  int total_kc, total_ci;  // sums of n_kc / n_ci
  int y_fp32;
  int y_store;             // 0: y += delta; sharded delta mode stores s*(xA)B into y: 1 as fp32, 2 as bf16;
                           // 3 (push): adds it into the source's y row (red.add over NVLink)
  int tc_cap_k;            // > 0: tcgen05 kernels use at most max(8, tiles * tc_cap_k) CTAs (rest exit at once)
  int simt_split_items;    // CUDA-core shrink: split each group's h_in into n_kc items (partials + a
                           // deterministic last-arriver sum) when groups * tasks < this (0: never)
  int tc_flags;            // L2 policies (env LORA_TCE_FLAGS): tcgen05 expand bit 0 Bt evict_last (else
                           // evict_first), bit 1 y loads evict_first, bit 2 y stores evict_first; CUDA-core
                           // kernels bit 3 expand B evict_last, bit 4 shrink A evict_last (else evict_first)
  Placement pl;            // adapter placement (unit = pl.local_index(a)*E + e)
  const int32_t* cache;    // resident-cache mode: unit = cache[a]*E + e (nullptr: placement)
  const float* scale;      // [n_adapters] s_a
  SlotTask t[kMaxTasks];
  // task of each global shrink chunk (kc) / expand column range (ci) index,
  // filled by the host when total_kc / total_ci <= kTaskTable
  uint8_t kc_task[kTaskTable];
  uint8_t ci_task[kTaskTable];
  int8_t tc_pair[kMaxTasks];   // tcgen05 shrink launch: partner task sharing this task's x / h_in / KI (its
                               // A tiles ride in the same N = 2r MMA; the partner has no items), -1 none
  PushIn push;                 // sharded owner over registered buffers (G = 0 otherwise)
  int16_t xreg[kMaxTasks];     // push: registered-buffer index of each task's x and y
  int16_t yreg[kMaxTasks];
};

#ifdef __CUDACC__
// address of x row `row` of task t (local, or -- REMOTE -- the origin row in
// its source's registered x buffer); REMOTE is a compile-time kernel variant
// so the local path is unchanged
template <bool REMOTE>
__device__ __forceinline__ const uint16_t* x_row(const MultiArgs& a, int task, int row) {
  const SlotTask& t = a.t[task];
  if (!REMOTE) return t.x + (long long)row * t.h_in;
  const int o = __ldg(a.push.origin + row);
  const char* base = a.push.reg[a.xreg[task] * a.push.G + (o >> kOriginRowBits)];
  return reinterpret_cast<const uint16_t*>(base) + (long long)(o & ((1 << kOriginRowBits) - 1)) * t.h_in;
}
// push mode: element 0 of the origin row of received row `row` in its source's
// registered y buffer (bf16 or fp32, esz bytes per element)
__device__ __forceinline__ char* y_push_row(const MultiArgs& a, int task, int row, int esz) {
  const SlotTask& t = a.t[task];
  const int o = __ldg(a.push.origin + row);
  char* base = a.push.reg[a.yreg[task] * a.push.G + (o >> kOriginRowBits)];
  return base + (long long)(o & ((1 << kOriginRowBits) - 1)) * t.h_out * esz;
}
// task owning global expand column-range index g (ci_base prefix)
__device__ __forceinline__ int find_task_ci(const MultiArgs& a, int g) {
  if (a.total_ci <= kTaskTable) return a.ci_task[g];
  int lo = 0, hi = a.n_tasks - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (a.t[mid].ci_base <= g) lo = mid; else hi = mid - 1;
  }
  return lo;
}
// task owning global shrink chunk index g (kc_base prefix)
__device__ __forceinline__ int find_task_kc(const MultiArgs& a, int g) {
  if (a.total_kc <= kTaskTable) return a.kc_task[g];
  int lo = 0, hi = a.n_tasks - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (a.t[mid].kc_base <= g) lo = mid; else hi = mid - 1;
  }
  return lo;
}
#endif

// launchers (return cudaGetLastError())
// T_dev != nullptr: the row count is *T_dev (<= T, read on the device; T is the capacity)
cudaError_t launch_segment(const int32_t* adapter_ids, const int32_t* expert_ids, int T, int E, int n_adapters,
                           const SegParams& sp, const PlanDev& pd, int* err_flag, cudaStream_t stream,
                           const int* T_dev = nullptr);
cudaError_t launch_simt_shrink(int rank, const MultiArgs& args, const PlanDev& pd, int grid, cudaStream_t stream);
cudaError_t launch_simt_expand(int rank, const MultiArgs& args, const PlanDev& pd, int grid, cudaStream_t stream);
// tcgen05 chain at rank 16 / 32 / 64 / 128 (tc_rank_supported)
cudaError_t launch_tc_shrink(int rank, const MultiArgs& args, const PlanDev& pd, int x_rows, int grid,
                             cudaStream_t stream);
cudaError_t launch_tc_vreduce(int rank, const MultiArgs& args, const PlanDev& pd, int grid, cudaStream_t stream);
cudaError_t launch_tc_expand(int rank, const MultiArgs& args, const PlanDev& pd, int grid, cudaStream_t stream);
bool tc_available();
bool tc_rank_supported(int rank);

// synthetic fill / weight relayout (synth_fill.cu)
cudaError_t launch_fill_store(uint16_t* At, uint16_t* Bt, int h_in, int h_out, int E, int r, long long units,
                              int slot, unsigned long long seed, const Placement& pl, int n_adapters,
                              cudaStream_t stream, long long adapter_base = 0);
cudaError_t launch_fill_rows(uint16_t* dst, long long rows, int width, unsigned long long seed, unsigned tag,
                             int shift, long long row_base, cudaStream_t stream);
cudaError_t launch_relayout_A(const uint16_t* src, uint16_t* At, long long units, int h_in, int r,
                              cudaStream_t stream);
cudaError_t launch_relayout_B(const uint16_t* src, uint16_t* Bt, long long units, int h_out, int r,
                              cudaStream_t stream);

// simt kernel smem requirement (for host-side validation)
int simt_shrink_smem(int rank);
int simt_expand_smem(int rank);
int simt_sj_max(int rank);
int simt_sc_max(int rank);

}  // namespace lora
