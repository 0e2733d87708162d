/*
 * lora_server.h -- C-ABI of the B200-native multi-LoRA delta hot path
 * (InfiniLoRA, arxiv 2604.07173: the LoRA Server's data-parallel compute).
 *
 * Citations: P:n = PAPER.md line n (section / equation / figure).
 *
 * The operation (Sec. 2.2, Sec. 2.3, Fig. 4b, Sec. 4.1):
 *   for every activation row i carrying adapter id a_i and routed expert e_i,
 *       y[i,:] += s_{a_i} * (x[i,:] A_{a_i,e_i}) B_{a_i,e_i}
 *   A_{a,e} in R^{h_in x r}, B_{a,e} in R^{r x h_out} (paper orientation),
 *   rows with a_i = -1 carry no LoRA and are left bit-identical.
 * Steps: a1 segment (stable sort by key a*E+e) -> a2 shrink
 * v = x A -> a3 expand d = s v B -> a4 scatter-accumulate y[perm] += d.
 *
 * Terms
 *   slot  one LoRA'd projection (e.g. layer 0 "gate" 4096->14336 with E=8
 *         experts, or layer 3 "q" 4096->4096 with E=1).  The paper's
 *         adapter space n x l x e is (adapter, slot, expert) here.
 *   unit  (slot, adapter a, expert e): one A/B pair; unit id in a slot = a*E+e.
 *   row   one activation vector; for MoE a (token, routed expert) pair, so a
 *         batch of b tokens with top-k routing has T = b*k rows.
 *
 * Conventions (all functions)
 *   - bf16 tensors are passed as raw 16-bit patterns (uint16).
 *   - Every function returns lora_status_t and never throws / aborts.
 *   - Host-detectable argument errors enqueue NOTHING and return
 *     LORA_ERR_INVALID_ARG (or _UNSUPPORTED); lora_last_error() explains.
 *   - Device-detectable id errors (adapter id outside [-1, n_adapters) or
 *     expert id outside [0, E)) skip the row (treated as a = -1) and set a
 *     sticky device flag, reported by lora_server_check() -- or immediately
 *     if the environment variable LORA_DEBUG_SYNC=1 is set.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *   - Single-GPU apply is fully asynchronous: no host synchronisation, no
 *     allocation, so it can be captured into a CUDA graph.
 *   - A server / plan handle is not thread-safe.  A plan owns its workspace,
 *     so concurrent applies need one plan per stream.
 */
#ifndef LORA_SERVER_H_
#define LORA_SERVER_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct lora_server lora_server_t; /* opaque */
typedef struct lora_plan lora_plan_t;     /* opaque, reusable segmentation + workspace */

typedef enum {
  LORA_OK = 0,
  LORA_ERR_INVALID_ARG = 1,
  LORA_ERR_OOM = 2,
  LORA_ERR_CUDA = 3,
  LORA_ERR_ID_OUT_OF_RANGE = 4,
  LORA_ERR_UNSUPPORTED = 5,
  LORA_ERR_NCCL = 6,
  LORA_ERR_PEER = 7   /* sharded push path: a peer did not signal in time, or ranks disagreed on a call */
} lora_status_t;

typedef enum { LORA_BF16 = 0, LORA_FP32 = 1 } lora_dtype_t;

typedef struct {
  int32_t n_slots;           /* number of LoRA'd projections, >= 1 */
  const int32_t *h_in;       /* [n_slots] input width;  multiple of 64 */
  const int32_t *h_out;      /* [n_slots] output width; multiple of 64 */
  const int32_t *n_experts;  /* [n_slots] E (1 for dense slots), >= 1 */
  int32_t rank;              /* r, uniform (one rank per model): 8, 16, 32, 64 or 128 ("r typically 32-128") */
  int32_t n_adapters;        /* global adapter count n */
  const float *scale;        /* [n_adapters] host fp32 s_a; NULL => all 1.0 (R1) */
  int32_t max_rows;          /* capacity (rows) of the internal plan; 0 < max_rows <= 32768 (sharded: max_rows * world <= 32768) */
  int32_t device;            /* CUDA device ordinal */
  int32_t n_replicated;      /* sharded servers only: adapters [0, n_replicated) are stored on
                                every rank (popularity-aware placement for skewed traffic,
                                P:291; adapter ids are assumed ordered by popularity); 0 =
                                plain striping.  Ignored by lora_server_create. */
  int32_t expert_parallel;   /* sharded servers: 0 => LoRA Data Parallel (adapter striping, with
                                n_replicated); 1 => expert parallel: unit (a, e) owned by rank
                                e mod world, every adapter (all slots must share one
                                expert count).  Ignored by lora_server_create. */
  int32_t n_resident;        /* single-GPU servers: 0 => every adapter resident in device memory;
                                0 < n_resident < n_adapters => resident-adapter cache (P:519-531,
                                Sec. 5.3): all adapters live in pinned host memory in the kernel
                                layout, n_resident of them in device memory; lora_server_require
                                makes a batch's adapters resident (LRU eviction, per-slot async
                                host->device copies that the applies of each slot wait for). */
  int32_t pp_stages;         /* sharded servers with expert_parallel: y pipeline stages of hybrid
                                EP_x-PP_y: the world is y groups of x = world / y ranks,
                                layer l belongs to group l mod y (interleaved), unit (a, e) of a
                                layer-l slot is owned by rank (l mod y) * x + e mod x.  0 or 1 =
                                pure expert parallel.  world % y == 0. */
  const int32_t *slot_layer; /* [n_slots] layer index of each slot (hybrid placement); NULL = 0 */
} lora_config_t;

/* ------------------------------------------------------------------------- */
/* Server: weight store                                                       */
/* ------------------------------------------------------------------------- */

/* Create a server and allocate its device weight store (all units of all
 * slots).  A / B may be NULL (weights stay zero until lora_server_load or
 * lora_server_fill_synthetic); otherwise A[slot] points to bf16 bits laid out
 * [n_adapters][E][h_in][r] and B[slot] to [n_adapters][E][r][h_out] (P:165
 * orientation), in device memory if weights_on_device != 0 else host memory.
 * The weights are copied into library-owned memory (re-laid-out for the
 * kernels); the caller may free its buffers when the call returns.
 * Errors: INVALID_ARG (bad config), UNSUPPORTED (rank or widths), OOM, CUDA. */
lora_status_t lora_server_create(const lora_config_t *cfg, const void *const *A, const void *const *B,
                                 int weights_on_device, lora_server_t **out);

/* Overwrite adapters [adapter_begin, adapter_begin+n) of one slot.  A / B use
 * the create() layout restricted to those adapters ([n][E][h_in][r] and
 * [n][E][r][h_out]).  Synchronises `stream` before returning.  On a sharded
 * server, adapters the rank does not own are skipped. */
lora_status_t lora_server_load(lora_server_t *s, int32_t slot, int32_t adapter_begin, int32_t n,
                               const void *A, const void *B, int on_device, void *stream);

/* Fill every unit of every slot from the counter-based generator described in
 * DESIGN.md "Input recipe" (seeded, bf16-exact values; used for benchmarks
 * whose weights do not fit through PCIe).  Async on `stream`. */
lora_status_t lora_server_fill_synthetic(lora_server_t *s, uint64_t seed, void *stream);

/* Synchronise the device, free everything. */
lora_status_t lora_server_destroy(lora_server_t *s);

/* Segments with more than `n` rows go to the tcgen05/TMEM kernels, the rest
 * to the CUDA-core kernels (default: env LORA_SMALL_SEG_MAX, else 8).  n < 0
 * forces the CUDA-core path for every segment.  The tcgen05 path runs at
 * every rank (8 with zero-padded MMAs), when the large segments of a batch
 * hold at least LORA_TC_MIN_ROWS rows together (default 2048 at ranks 8 and
 * 16, else 256).  Takes effect at the
 * next lora_plan_build. */
lora_status_t lora_server_set_small_seg_max(lora_server_t *s, int32_t n);

/* Resident-adapter cache (cfg->n_resident > 0): make the n adapters in
 * `adapters` (host ids, duplicates allowed, at most n_resident distinct)
 * resident before the next applies.  Missing adapters take free cache slots
 * or evict the least recently required adapters not in this set; their
 * weights are copied host->device on an internal copy stream, slot by slot
 * (layer-wise), after the work already queued on `stream`; every later apply
 * of a slot on `stream` waits only for that slot's copies, so loading the
 * next layers overlaps applying the first.  *n_loaded (may be NULL) receives
 * the number of adapters copied.  Rows whose adapter is not resident at plan
 * build are treated as out of range (skipped and flagged).  Without a cache:
 * no-op.  Single stream per server. */
lora_status_t lora_server_require(lora_server_t *s, const int32_t *adapters, int32_t n, int32_t *n_loaded,
                                  void *stream);

/* on != 0 (default; env LORA_SERIAL=1 at create sets 0): the tcgen05 chain of
 * an apply runs on an internal side stream forked from / joined to the
 * caller's stream, concurrently with the CUDA-core chain (disjoint rows).
 * on == 0 serialises every kernel on the caller's stream (the per-kernel
 * profiling mode bench.py uses for roofline durations).  Results are
 * identical either way. */
lora_status_t lora_server_set_concurrent(lora_server_t *s, int32_t on);

/* Sticky device error check: synchronises `stream`; returns
 * LORA_ERR_ID_OUT_OF_RANGE (and clears the flag) if any apply since the last
 * check met an out-of-range id, LORA_ERR_CUDA on a CUDA error, else LORA_OK. */
lora_status_t lora_server_check(lora_server_t *s, void *stream);

/* Human-readable reason for the last failing call on `s` (NULL => the calling
 * thread's last create / argument error).  Never NULL. */
const char *lora_last_error(const lora_server_t *s);

/* ------------------------------------------------------------------------- */
/* Plans: a1 segmentation, reusable across the slots of one unit of work       */
/* ------------------------------------------------------------------------- */

/* Allocate a plan for up to max_rows rows (<= 32768) plus the workspace of
 * every slot (so one plan serves any sequence of slots). */
lora_status_t lora_plan_create(lora_server_t *s, int32_t max_rows, lora_plan_t **out);
lora_status_t lora_plan_destroy(lora_plan_t *p);

/* a1: stable segmentation of T rows (device pointers adapter_ids[T],
 * expert_ids[T] or NULL => e = 0) by key a*E + e with E = n_experts; rows with
 * a = -1 are dropped; ties broken by ascending row index (R9).
 * Builds perm / seg_offsets / seg_keys and the device work lists; the segment
 * count stays on the device.  T = 0 is a no-op plan.  Async. */
lora_status_t lora_plan_build(lora_server_t *s, lora_plan_t *p, const int32_t *adapter_ids,
                              const int32_t *expert_ids, int32_t T, int32_t n_experts, void *stream);

/* Copy the plan's indices out (bit-exact contract): perm[n_valid],
 * seg_offsets[n_segs+1], seg_keys[n_segs] into DEVICE buffers sized
 * max_rows / max_rows+1 / max_rows; n_valid / n_segs into HOST ints.
 * Synchronises `stream`. */
lora_status_t lora_plan_export(const lora_plan_t *p, int32_t *perm, int32_t *seg_offsets,
                               int32_t *seg_keys, int32_t *n_valid, int32_t *n_segs, void *stream);

/* Work-list sizes of the last build (host ints, synchronises `stream`):
 * out[0] valid rows, out[1] segments, out[2] CUDA-core row groups (<= 8 rows),
 * out[3] tcgen05 row tiles (<= 128 rows). */
lora_status_t lora_plan_stats(const lora_plan_t *p, int32_t *out4, void *stream);

/* ------------------------------------------------------------------------- */
/* Apply: a2 shrink, a3 expand, a4 scatter-accumulate                          */
/* ------------------------------------------------------------------------- */

/* One slot: y[T][h_out] (bf16 or fp32, device, read-modify-written in place)
 * += s * (x A) B for the rows of plan p; x is bf16 [T][h_in] (device).  The
 * slot's E must equal the plan's n_experts.  x and y must not overlap. */
lora_status_t lora_apply_plan(lora_server_t *s, const lora_plan_t *p, int32_t slot, const void *x,
                              void *y, lora_dtype_t y_dtype, void *stream);

/* Several slots sharing one plan in ONE set of launches (e.g. gate, up, down
 * of a MoE layer, or the 128 q/k/v/o slots of a Llama decode step).  slots[n]
 * must be distinct; x[i] / y[i] as in lora_apply_plan.  x buffers may be
 * shared between slots (e.g. q/k/v); every y byte range (T * h_out elements)
 * must be disjoint from every other y range and from every x range of the
 * call (the slots' kernels run concurrently) -- else LORA_ERR_INVALID_ARG,
 * nothing enqueued.  slots / x / y are host arrays. */
lora_status_t lora_apply_plan_multi(lora_server_t *s, const lora_plan_t *p, int32_t n,
                                    const int32_t *slots, const void *const *x, void *const *y,
                                    lora_dtype_t y_dtype, void *stream);

/* The deltas themselves, for a client that adds them to its own base output
 * ("returns the updated activations", "receive the computed
 * results ... followed by a final addition"): delta[i] row r = s_a * (x A) B
 * for rows with an adapter, 0 for rows without (a = -1, or flagged ids);
 * delta_dtype LORA_BF16 (each element rounded once) or LORA_FP32.  The delta
 * buffers [T][h_out] (device) are written, never read; same plan / slot / x
 * rules and errors as lora_apply_plan_multi (nothing enqueued on a host-side
 * error).  Equals lora_apply_plan_multi on a zero y, bit for bit. */
lora_status_t lora_apply_plan_multi_delta(lora_server_t *s, const lora_plan_t *p, int32_t n,
                                          const int32_t *slots, const void *const *x, void *const *delta,
                                          lora_dtype_t delta_dtype, void *stream);

/* Convenience: plan_build on the server's internal plan + apply_plan. */
lora_status_t lora_apply(lora_server_t *s, int32_t slot, const void *x, const int32_t *adapter_ids,
                         const int32_t *expert_ids, void *y, lora_dtype_t y_dtype, int32_t T,
                         void *stream);

/* End-to-end entry with HOST buffers (pinned for full async speed): copies
 * the ids and the n slots' x / y host->device into library staging buffers,
 * applies, and copies every y back device->host.  Pipelined: the rows are cut
 * into RC chunks (RC = clamp(T / 2048, 1, 4); env LORA_HOST_ROW_CHUNKS) with
 * one internal plan each, every row chunk's slots into groups of >= 32 MB of
 * upload; piece p+1's upload (internal copy stream), piece p's apply
 * (`stream`) and piece p-1's download (a second internal stream) overlap.
 * Row chunks re-read the weights their units need (one apply per chunk); the
 * segments, and so the kernel route of a row (CUDA-core / tcgen05), are those
 * of its row chunk.  Stream-ordered on `stream` at both ends; returns after
 * enqueueing, the caller synchronises `stream` before reading y.  Capacity:
 * T <= max_rows.  x[i] pointers may repeat (uploaded once). */
lora_status_t lora_apply_multi_host(lora_server_t *s, int32_t n, const int32_t *slots,
                                    const void *const *x_host, const int32_t *adapter_ids_host,
                                    const int32_t *expert_ids_host, void *const *y_host,
                                    lora_dtype_t y_dtype, int32_t T, void *stream);

/* The same pipeline returning the deltas (lora_apply_plan_multi_delta) into
 * HOST buffers delta_host[i] [T][h_out]: only x and the ids go up, the deltas
 * come down (no base output crosses PCIe). */
lora_status_t lora_apply_multi_host_delta(lora_server_t *s, int32_t n, const int32_t *slots,
                                          const void *const *x_host, const int32_t *adapter_ids_host,
                                          const int32_t *expert_ids_host, void *const *delta_host,
                                          lora_dtype_t delta_dtype, int32_t T, void *stream);

/* ------------------------------------------------------------------------- */
/* Sharded LoRA Server: LoRA Data Parallel (Sec. 4.1, Table 1 DP row) */
/* ------------------------------------------------------------------------- */

/* 128-byte NCCL unique id for rank 0 to broadcast (torch.distributed is the
 * bootstrap).  Fails with LORA_ERR_NCCL if libnccl.so.2 cannot be loaded. */
lora_status_t lora_nccl_unique_id(void *out128);

/* Create the rank-`rank` member of a world-`world` sharded server (world <=
 * 8: one NVLink / NVSwitch domain).  With h = cfg->n_replicated, adapters
 * a < h are stored on every rank and adapter a >= h is owned by rank
 * (a - h) mod world (LoRA Data Parallel striping); with
 * cfg->expert_parallel, unit (a, e) is owned by rank e mod world.
 * Each rank stores only what it owns.  Every rank must call this
 * collectively with the same config.  cfg->max_rows is this rank's row
 * capacity; its owner-side plan holds max_rows * world received rows (rows
 * beyond that are dropped and flagged), so an unbalanced deployment sizes
 * max_rows for the most loaded owner.  max_rows * world <= 32768. */
lora_status_t lora_server_create_sharded(const lora_config_t *cfg, int32_t rank, int32_t world,
                                         const void *nccl_unique_id, lora_server_t **out);

/* Host control plane for a sharded server without NCCL: a blocking host
 * all-gather supplied by the caller (e.g. an MPI / gloo / socket collective).
 * Every rank contributes `bytes` bytes from `send`; `recv` receives
 * world * bytes, rank-major.  Return 0 on success. */
typedef int (*lora_host_allgather_fn)(void *ctx, const void *send, void *recv, int64_t bytes);

/* As lora_server_create_sharded, with the control plane (IPC-handle and
 * agreement exchanges of lora_shard_register) on the caller's host all-gather
 * instead of NCCL.  Applies then need registered x / y buffers (the push path
 * runs without any host collective).  Peers may share a GPU (the
 * multi-process tests run two ranks on one B200). */
lora_status_t lora_server_create_sharded_host(const lora_config_t *cfg, int32_t rank, int32_t world,
                                              lora_host_allgather_fn allgather, void *ctx,
                                              lora_server_t **out);

/* Register n caller device buffers for the sharded push path (collective:
 * every rank registers the same number of buffers, in the same roles and
 * order, e.g. its x of gate/up, its x of down, then its y of gate, up, down).
 * Each buffer (ptrs[i], bytes[i] bytes, inside one cudaMalloc allocation --
 * torch's caching allocator qualifies; expandable segments do not) is
 * exported with CUDA IPC and mapped on every peer (NVLink peer access); the
 * first call also creates this rank's control area.  Registrations last
 * until lora_server_destroy; the caller keeps the buffers alive until then.
 * If any rank cannot export or map a buffer, every rank releases ALL its
 * registrations and returns LORA_ERR_UNSUPPORTED.  Synchronises `stream`. */
lora_status_t lora_shard_register(lora_server_t *s, int32_t n, void *const *ptrs, const int64_t *bytes,
                                  void *stream);

/* Collective apply on a sharded server: every rank passes its OWN rows
 * (T local rows, device pointers, same slot list on every rank).  Rows whose
 * unit this rank stores (its own or a replicated adapter) are applied in
 * place; the others are applied by their unit's owner.
 *
 * Push path -- every x[i] and y[i] is the start of a registered buffer (of
 * at least T rows), on every rank (one-sided pushes both ways;
 * receive / compute / send overlapped): the counts travel through
 * peer memory (device flags, no host synchronisation, CUDA-graph
 * capturable); the owner's shrink reads each routed x row directly from its
 * source's x over NVLink, and its expand epilogue adds the delta directly
 * into the source's y row (red.add: one writer per element; bf16 y: the
 * delta is rounded to bf16 first, R19; fp32 y: bit-identical to
 * the unsharded server when every row takes the same kernel route, R18,
 * except that a subnormal delta or sum is flushed to zero).  The call is
 * stream-ordered: when `stream` reaches its end, every owner has finished
 * adding into this rank's y.  A rank that does not arrive within
 * LORA_SHARD_TIMEOUT_MS (default 10000) makes the others skip its rows and
 * raise the sticky flag (lora_server_check -> LORA_ERR_PEER), as do ranks
 * whose calls disagree (slots, buffer roles, dtype).
 *
 * Otherwise (NCCL control plane only): grouped ncclSend/ncclRecv of the
 * routed x rows + ids and of the deltas (fp32 for an fp32 y, bf16 for a bf16
 * y unless LORA_SHARD_FP32=1), one host synchronisation for the count
 * matrix; ranks whose calls disagree all return LORA_ERR_INVALID_ARG before
 * any row moves.
 *
 * Rows with adapter id -1 stay local and untouched; out-of-range ids are
 * flagged and dropped (never sent, never applied).  n <= 128. */
lora_status_t lora_apply_sharded(lora_server_t *s, int32_t n, const int32_t *slots,
                                 const void *const *x, const int32_t *adapter_ids,
                                 const int32_t *expert_ids, void *const *y, lora_dtype_t y_dtype,
                                 int32_t T, void *stream);

/* Host-only helper (no GPU needed): given the world x world send-count
 * matrix counts[src*world+dst], fill this rank's send offsets
 * send_off[world+1] (into its owner-bucketed send buffer) and receive
 * offsets recv_off[world+1] (receive order: by source rank ascending).
 * Used by the sharded apply and by the CPU multi-process tests. */
lora_status_t lora_shard_layout(const int64_t *counts, int32_t world, int32_t rank,
                                int64_t *send_off, int64_t *recv_off);

/* Host-only helper (no GPU needed) for the peer-to-peer transport: from the
 * same count matrix, for every peer p:
 *   in_rowbase[p]:  received row r (from source p, r in [recv_off[p],
 *                   recv_off[p+1])) is row r + in_rowbase[p] of p's send
 *                   buffer (p's rows ordered by owner);
 *   out_rowbase[p]: this rank's send-order row j (for owner p) has its delta
 *                   in row j + out_rowbase[p] of owner p's delta buffer. */
lora_status_t lora_shard_peer_rows(const int64_t *counts, int32_t world, int32_t rank,
                                   int64_t *in_rowbase, int64_t *out_rowbase);

/* Synthetic activation rows for benchmarks and tests: dst is bf16 [rows][width]
 * (device), element (i, c) = the counter-based generator of DESIGN.md "Input
 * recipe" with major = row_base + i, minor = c, the given tag and shift.  Async. */
lora_status_t lora_synth_fill_rows(void *dst, int64_t rows, int32_t width, uint64_t seed, uint32_t tag,
                                   int32_t shift, int64_t row_base, void *stream);

/* ------------------------------------------------------------------------- */
/* Profiling: per-launch CUDA events on the launching stream                  */
/* ------------------------------------------------------------------------- */

/* Start recording a (start, end) event pair around every kernel launch of
 * this server (up to max_launches launches; <= 0 disables).  Clears records. */
lora_status_t lora_profile_enable(lora_server_t *s, int32_t max_launches);

/* Synchronise on the recorded events and return, per kernel kind k <
 * n_kinds, the number of launches and their summed device time in ms
 * (launches[k], total_ms[k]; host arrays).  Clears the records. */
lora_status_t lora_profile_read(lora_server_t *s, int32_t n_kinds, int32_t *launches, double *total_ms);

/* Name of kernel kind k (0 segment, 1 simt_shrink, 2 tc05_shrink,
 * 3 simt_expand, 4 tc05_expand, 5 shard_bucket, 6 shard_gather,
 * 7 shard_scatter_add, 8 tc05_vreduce; push path: 5 = bucket + announce,
 * 6 = recv-prep, 7 = done + wait); "unknown" otherwise. */
const char *lora_kernel_name(int32_t kind);

/* Library version string. */
const char *lora_version(void);

#ifdef __cplusplus
}
#endif
#endif /* LORA_SERVER_H_ */
