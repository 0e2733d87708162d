// common.cuh -- shared device helpers for the sm_100a multi-LoRA kernels.
//
// PTX wrappers (mbarrier, 1-D TMA bulk copies, cp.async, tcgen05), bf16
// helpers and the weight-store layout.  Product code only; the oracle shares
// nothing with this file.
#pragma once

#include <utility>

#include <cuda_runtime.h>
#include <stdint.h>

#define LORA_DEVINL __device__ __forceinline__

namespace lora {

constexpr int kWarp = 32;

// ---------------------------------------------------------------------------
// scalar helpers
// ---------------------------------------------------------------------------
LORA_DEVINL float bf16lo(uint32_t w) { return __uint_as_float(w << 16); }
LORA_DEVINL float bf16hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }
LORA_DEVINL float bf16_to_f32(uint16_t b) { return __uint_as_float(uint32_t(b) << 16); }

// round-to-nearest-even fp32 -> bf16 bits (hardware cvt.rn, one instruction)
LORA_DEVINL uint16_t f32_to_bf16_rne(float f) {
  uint16_t r;
  asm("cvt.rn.bf16.f32 %0, %1;" : "=h"(r) : "f"(f));
  return r;
}

// hardware round-to-nearest-even conversions (F2FP): one instruction per pair
LORA_DEVINL uint32_t pack_bf16x2_rn(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
LORA_DEVINL uint16_t bf16_rn(float f) {
  uint16_t r;
  asm("cvt.rn.bf16.f32 %0, %1;" : "=h"(r) : "f"(f));
  return r;
}

LORA_DEVINL uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

LORA_DEVINL int lane_id() { return threadIdx.x & 31; }
LORA_DEVINL int warp_id() { return threadIdx.x >> 5; }

// ---------------------------------------------------------------------------
// mbarrier
// ---------------------------------------------------------------------------
LORA_DEVINL void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
LORA_DEVINL void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
LORA_DEVINL void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
LORA_DEVINL void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
LORA_DEVINL bool mbar_try_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
LORA_DEVINL void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t b = smem_u32(bar);
  while (!mbar_try_wait(b, parity)) {
  }
}

// ---------------------------------------------------------------------------
// 1-D TMA bulk copies (cp.async.bulk) -- SASS UBLKCP
// ---------------------------------------------------------------------------
LORA_DEVINL uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
LORA_DEVINL uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
LORA_DEVINL uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// global -> shared, completion counted on `bar` (bytes multiple of 16, 16B aligned)
LORA_DEVINL void bulk_g2s(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
LORA_DEVINL void bulk_g2s_hint(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar,
                               uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
      "%4;" ::"r"(smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
// shared -> global bulk store (bulk-group completion)
LORA_DEVINL void bulk_s2g(void* gdst, const void* smem_src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
               "r"(smem_u32(smem_src)), "r"(bytes)
               : "memory");
}
LORA_DEVINL void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
LORA_DEVINL void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
LORA_DEVINL void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}

// ---------------------------------------------------------------------------
// cp.async (LDGSTS), 16 bytes, zero-fill when src_bytes == 0
// ---------------------------------------------------------------------------
LORA_DEVINL void cp_async16(void* smem_dst, const void* gsrc, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(smem_dst)), "l"(gsrc),
               "r"(src_bytes)
               : "memory");
}
LORA_DEVINL void cp_async16_u32(uint32_t smem_dst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_dst), "l"(gsrc) : "memory");
}
LORA_DEVINL void cp_async16_u32_hint(uint32_t smem_dst, const void* gsrc, uint64_t policy) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(smem_dst), "l"(gsrc),
               "l"(policy)
               : "memory");
}
LORA_DEVINL void st_global_v4_hint(void* p, uint4 v, uint64_t policy) {
  asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w), "l"(policy)
               : "memory");
}
LORA_DEVINL void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
LORA_DEVINL void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
// make generic-proxy smem writes visible to the async proxy (TMA / tcgen05)
LORA_DEVINL void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

LORA_DEVINL void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Programmatic dependent launch: a kernel launched with launch_pdl may start
// while its predecessor on the stream is still running; pdl_wait() blocks
// until that predecessor grid has completed (its writes visible), and
// pdl_launch_dependents() lets the next PDL kernel be scheduled.  Both are
// no-ops for kernels launched normally.
LORA_DEVINL void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
LORA_DEVINL void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" :::); }

// host: launch with programmatic stream serialization when LORA_PDL=1 (else a plain launch)
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// Push adds into a peer's (or this GPU's) registered y (sharded owner, one
// writer per element, so the add is the only update of the element and the
// result is deterministic).  System scope: the target may be another GPU's
// memory behind an NVLink peer mapping.  bf16: one rounding of y + d_bf16
// (d already rounded to bf16, R19); f32: red.add.f32 (FTZ on
// subnormal operands/results, the only difference from a local fp32 add).
LORA_DEVINL void red_add_bf16x8(void* p, uint4 v) {
  asm volatile("red.relaxed.sys.global.add.noftz.v4.bf16x2 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}
LORA_DEVINL void red_add_bf16x2(void* p, uint32_t v) {
  asm volatile("red.relaxed.sys.global.add.noftz.bf16x2 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
LORA_DEVINL void red_add_f32(void* p, float v) {
  asm volatile("red.relaxed.sys.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
LORA_DEVINL void red_add_f32x4(void* p, float4 v) {
  asm volatile("red.relaxed.sys.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}

// 128-bit loads
LORA_DEVINL uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}
LORA_DEVINL float4 lds128f(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}

// ---------------------------------------------------------------------------
// Dynamic work distribution for persistent kernels.
//
// One producer lane per CTA takes item indices from a global counter
// (atomicAdd) and publishes them to the CTA's consumer warps through a
// shared-memory ring guarded by mbarriers; -1 ends the stream.  CTAs that
// start late (another kernel still holds their SM) simply take fewer items.
// The last CTA to finish resets the counters, so every launch starts at 0.
// ---------------------------------------------------------------------------
template <int QD>
struct WorkQueue {
  long long* item;  // smem [QD]
  uint64_t* full;   // smem [QD], 1 arrival (producer)
  uint64_t* empty;  // smem [QD], one arrival per consumer warp
  LORA_DEVINL void init(int consumer_warps) {
    for (int i = 0; i < QD; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], consumer_warps);
    }
  }
};

struct QueuePos {
  int slot = 0;
  uint32_t phase = 0;
  LORA_DEVINL void advance(int qd) {
    if (++slot == qd) {
      slot = 0;
      phase ^= 1;
    }
  }
};

// producer lane: fetch the next item (or -1) and publish it.  (Fetching the
// following item ahead of time was measured slower: long items, worse tail.)
template <int QD>
LORA_DEVINL long long wq_push_next(WorkQueue<QD>& q, QueuePos& p, unsigned long long* counter, long long n_items) {
  long long it = (long long)atomicAdd(counter, 1ull);
  if (it >= n_items) it = -1;
  mbar_wait(&q.empty[p.slot], p.phase ^ 1);
  q.item[p.slot] = it;
  mbar_arrive(&q.full[p.slot]);
  p.advance(QD);
  return it;
}

// consumer warp: take the next item (all lanes get it; lane 0 releases the slot)
template <int QD>
LORA_DEVINL long long wq_pop(WorkQueue<QD>& q, QueuePos& p) {
  mbar_wait(&q.full[p.slot], p.phase);
  const long long it = q.item[p.slot];
  __syncwarp();
  if ((threadIdx.x & 31) == 0) mbar_arrive(&q.empty[p.slot]);
  p.advance(QD);
  return it;
}

// end of a persistent launch (call with all threads after a __syncthreads):
// the last CTA resets the item counter and the done counter
LORA_DEVINL void wq_finish(unsigned long long* counter, unsigned int* done) {
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(done, 1u) == gridDim.x - 1) {
      *counter = 0ull;
      *done = 0u;
      __threadfence();
    }
  }
}

// ---------------------------------------------------------------------------
// Weight-store layout
//
//   At (shrink operand): [U][h_in/64][r][64] bf16.  Each [r][64] tile has
//       128-byte rows (one rank index k per row, 64 consecutive j) and is
//       stored with the 128B swizzle already applied: 16-byte chunk q of row
//       k sits at chunk position q ^ (k & 7).  A contiguous run of tiles is
//       therefore the exact shared-memory image a 1-D bulk copy lands, and
//       it is the canonical SWIZZLE_128B K-major operand for tcgen05.
//   Bt (expand operand): [U][h_out][r] bf16, rows of r*2 bytes (one output
//       column c per row), swizzled with the pattern of that row width
//       (256B: q ^ ((c&3)<<1); 128B: q ^ (c&7); 64B: q ^ ((c>>1)&3);
//       32B: q ^ ((c>>2)&1); 16B: none).
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ int swz_row_chunk(int row, int chunk, int row_bytes) {
  // physical 16-byte chunk index inside a row of `row_bytes` bytes
  switch (row_bytes) {
    case 256: return chunk ^ ((row & 3) << 1);
    case 128: return chunk ^ (row & 7);
    case 64: return chunk ^ ((row >> 1) & 3);
    case 32: return chunk ^ ((row >> 2) & 1);
    default: return chunk;
  }
}

}  // namespace lora
