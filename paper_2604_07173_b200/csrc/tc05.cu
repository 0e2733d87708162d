// tc05.cu -- a2 shrink and a3+a4 expand on the 5th-generation tensor cores
// (tcgen05.mma, accumulators in TMEM) for LARGE segments.
//
// A segment with more than `small_seg_max` rows of one unit is a real dense
// contraction (prefill: 474-893 rows per unit; decode: the Zipf head).  The
// paper's SGMV "aggregat[es] tokens that share the same LoRA adapter into a
// single GEMM" on Hopper wgmma with swap-AB; here it is
// tcgen05 with one elected issuing thread, TMEM accumulators and mbarrier
// pipelines:
//
//   shrink item (task, kc, tile<=128 rows):
//       D[128 rows x r] (TMEM, fp32) = X_tile[128 x KI] . A_u[KI x r]
//       A operand = gathered activation rows (cp.async, manual 128B swizzle)
//       B operand = pre-swizzled At store tiles (1-D TMA bulk copy); gate + up
//                   in one N = 2r MMA (x gathered once)
//       epilogue: TMEM -> regs -> v (bf16, whole K) or vpart[kc][row][0:r]
//   expand item (task, ci, tile<=128 rows), per 128-column sub-tile:
//       D[128 rows x 128 cols] (TMEM lane = tile row) = v_tile[128 x r] . Bt_sub[128 cols x r]^T
//       A operand = v tile (bf16, pre-swizzled, 1-D TMA bulk copy per K block)
//       B operand = pre-swizzled Bt store rows (1-D TMA bulk copy; r = 128:
//                   re-tiled into two 64-wide K blocks by the producer warp)
//       epilogue: TMEM -> regs -> y[perm[n]][c] = round(y + s_a * D)
//
// Ranks 16 / 32 / 64 / 128 (template R): the x tiles and At tiles are K-major
// SWIZZLE_128B at every rank (64 k per atom, N = r rows); the expand's K = r
// operands use SWIZZLE_32B / 64B / 128B rows of min(2r, 128) bytes (KGeo).
// The instruction descriptor selects bf16 x bf16 -> fp32.
#include <cstdlib>
#include <cstring>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "kernels.h"

namespace lora {

namespace {

// ---------------------------------------------------------------------------
// tcgen05 PTX wrappers
// ---------------------------------------------------------------------------
LORA_DEVINL void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
LORA_DEVINL void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
LORA_DEVINL void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
LORA_DEVINL void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// D[tmem] (+)= A[smem] . B[smem]; bf16 inputs, fp32 accumulate
LORA_DEVINL void umma_bf16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accum)
      : "memory");
}
// arrive on an mbarrier when all previously issued tcgen05.mma of this thread complete
LORA_DEVINL void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// 32 lanes x 32 bit, 16 consecutive columns -> 16 registers
LORA_DEVINL void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// K-major, SWIZZLE_128B shared-memory matrix descriptor (sm_100 format)
LORA_DEVINL uint64_t sw128_desc(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);        // start address
  d |= (uint64_t)1 << 16;                            // LBO (ignored for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;                  // SBO: 8 rows x 128 B
  d |= (uint64_t)1 << 46;                            // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;                            // SWIZZLE_128B
  return d;
}

// instruction descriptor: bf16 x bf16 -> fp32, both K-major, shape M x N
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

LORA_DEVINL void cp_async_mbar_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

LORA_DEVINL uint8_t* align1024(uint8_t* p) {
  const uint32_t a = smem_u32(p);
  return p + (((a + 1023u) & ~1023u) - a);
}


constexpr int kQD = 4;  // work-queue depth

// K-major operand geometry of rank R in the expand MMA (K = R) and in the
// tcgen05 path's bf16 v store: rows of RB = min(2R, 128) bytes with the
// matching UMMA swizzle (SWIZZLE_32B / 64B / 128B for r = 16 / 32 / >= 64;
// 16-byte chunk c of row n at swz_row_chunk(n, c, RB)), r = 128 as KB = 2
// blocks of 64 k.  The Bt store rows of r <= 64 already have exactly this
// layout (common.cuh); r = 128 Bt rows are 256 bytes and are re-tiled into
// two SWIZZLE_128B blocks by the expand's producer warp.
template <int R>
struct KGeo {
  static_assert(R == 8 || R == 16 || R == 32 || R == 64 || R == 128, "tcgen05 ranks");
  // r = 8: K and N padded to 16 with zeros (the MMA's minimum), rows of 32 bytes
  static constexpr int RP = R < 16 ? 16 : R;         // padded rank
  static constexpr int RB = RP >= 64 ? 128 : RP * 2;  // bytes per row of one K block (= swizzle width)
  static constexpr int KB = RP >= 64 ? RP / 64 : 1;   // K blocks
  static constexpr int KPB = RB / 32;                 // 16-element MMA k-steps per K block
  static constexpr int CPB = RB / 16;                 // 16-byte chunks per row of a K block
};

// K-major shared-memory matrix descriptor (sm_100 format) for swizzle width
// RB (128 / 64 / 32 bytes): 8-row core groups RB * 8 bytes apart
template <int RB>
LORA_DEVINL uint64_t kmajor_desc(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);             // start address
  d |= (uint64_t)1 << 16;                                 // LBO (ignored for swizzled K-major)
  d |= (uint64_t)((RB * 8) >> 4) << 32;                   // SBO: 8 rows
  d |= (uint64_t)1 << 46;                                 // descriptor version (sm_100)
  d |= (uint64_t)(RB == 128 ? 2 : RB == 64 ? 4 : 6) << 61;  // SWIZZLE_128B / 64B / 32B
  return d;
}

// element offset of 16-byte chunk q (0 .. RP/8-1) of sorted row `row` (row n of
// its tile) in a slot's bf16 v region: [KB][max_rows][RB / 2]
template <int R>
LORA_DEVINL long long vbf_chunk(long long row, int n, int q, int max_rows) {
  using G = KGeo<R>;
  const int kb = q / G::CPB, c = q - kb * G::CPB;
  return (long long)kb * max_rows * (G::RB / 2) + row * (G::RB / 2) + swz_row_chunk(n, c, G::RB) * 8;
}

// x tensor maps of a tcgen05 shrink launch (one per task): 2-D [T rows][h_in]
// bf16, box {64 columns, 1 row}, SWIZZLE_128B -- the layout a TMA tile::gather4
// lands is then exactly the canonical SW128 K-major operand (row n of the tile
// at smem row n, 16-byte chunk q at q ^ (n & 7); measured, tools/gather4_probe.cu)
constexpr int kTcMapTasks = 8;
struct TcMaps {
  CUtensorMap x[kTcMapTasks];
  int use;  // 1: x rows by gather4 from one producer warp; 0: cp.async gathers
};

// 4 rows (r0..r3) x 64 columns from col of map into smem dst (512 bytes)
LORA_DEVINL void tma_gather4(uint32_t dst, const CUtensorMap* map, int col, int r0, int r1, int r2, int r3,
                             uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
      : "memory");
}

// CTAs that do work in a tcgen05 launch: with tc_cap_k > 0 a few tiles use a
// few SMs and leave the others to the concurrent CUDA-core chain
LORA_DEVINL bool tc_cta_idle(const MultiArgs& args, const PlanDev& pd) {
  if (args.tc_cap_k <= 0) return false;
  const long long cap = (long long)pd.counts[kCntTiles] * args.tc_cap_k;
  return blockIdx.x >= (cap < 8 ? 8 : cap);
}

// ===========================================================================
// shrink
// ===========================================================================
// PAIR: two slots that share x, h_in and the row plan (gate and up of a MoE
// layer) in one item -- the gathered x tile feeds one
// N = 2r MMA whose B operand is the two slots' A tiles back to back, so x is
// read once for both.
template <int R, bool PAIR>
struct ShrinkCfgT {
  static constexpr int EPI_WARPS = 4;   // warps 0-3: epilogue (TMEM lanes 0-127)
  static constexpr int MMA_WARP = 4;    // warp 4: TMEM alloc + MMA issue
  static constexpr int PROD_WARP0 = 5;  // warps 5-8: activation gather (+ weight bulk copy)
  static constexpr int PROD_THREADS = 128;
  static constexpr int THREADS = 9 * 32;
  static constexpr int KSTEP = 64;                         // K per SW128 atom
#ifndef LORA_TCS_KS
#define LORA_TCS_KS 2
#endif
#ifndef LORA_TCS_NST
#define LORA_TCS_NST 4
#endif
#ifndef LORA_TCS_LAG
#define LORA_TCS_LAG 1  // cp.async groups left in flight per producer thread (measured: config 5 tc shrink 130 -> 118 us vs 2, prefill equal)
#endif
#ifndef LORA_TCSP_NST
#define LORA_TCSP_NST 3
#endif
#ifndef LORA_TCS_NOINC
#define LORA_TCS_NOINC 1  // producers arrive with cp.async.mbarrier.arrive.noinc instead of waiting (measured: prefill tc shrink 140 -> 136 us, config 5 115 -> 110 us)
#endif
  static constexpr int KS_PER_STAGE = LORA_TCS_KS;         // k-steps per stage
  static constexpr int NW = PAIR ? 2 : 1;                  // A tiles per k-step
  static constexpr int X_SUB = kTileRows * 128;            // 16 KB per k-step
  static constexpr int NP = KGeo<R>::RP;                   // MMA N per slot (r = 8: rows 8-15 zero)
  static constexpr int W_SUB = NP * 128;                   // smem A rows of one k-step and slot (8 KB at r = 64)
  static constexpr int W_G = R * 128;                      // bytes of one k-step of a unit's At in global memory
  static constexpr int STAGE = KS_PER_STAGE * (X_SUB + NW * W_SUB);
  // r = 64: the measured depths; other ranks as many stages as fit (<= 6)
  static constexpr int NST_FIT = (220 * 1024) / STAGE > 6 ? 6 : (220 * 1024) / STAGE;
  static constexpr int NST = R == 64 ? (PAIR ? LORA_TCSP_NST : LORA_TCS_NST) : NST_FIT;
  static constexpr int LAG = LORA_TCS_LAG < NST - 1 ? LORA_TCS_LAG : NST - 1;  // cp.async groups kept in flight
  static constexpr int ACC_COLS = NW * NP;                 // N = r (pair: 2r)
  static constexpr int TMEM_COLS = 2 * ACC_COLS;           // 2 accumulators
  static constexpr int SMEM = 1024 + NST * STAGE + 256;
  static_assert(SMEM <= 227 * 1024, "shrink stages exceed shared memory");
};

// v row n of a tile (R fp32 sums) rounded to bf16 into the pre-swizzled
// expand operand (vbf_chunk layout)
template <int R>
LORA_DEVINL void store_vbf_row(uint16_t* vslot, long long row, int n, const float* v, int max_rows) {
#pragma unroll
  for (int q = 0; q < R / 8; ++q) {
    uint4 w;
    w.x = pack_bf16x2_rn(v[8 * q], v[8 * q + 1]);
    w.y = pack_bf16x2_rn(v[8 * q + 2], v[8 * q + 3]);
    w.z = pack_bf16x2_rn(v[8 * q + 4], v[8 * q + 5]);
    w.w = pack_bf16x2_rn(v[8 * q + 6], v[8 * q + 7]);
    *reinterpret_cast<uint4*>(vslot + vbf_chunk<R>(row, n, q, max_rows)) = w;
  }
  if constexpr (R < 16)  // the K padding of the expand operand
    *reinterpret_cast<uint4*>(vslot + vbf_chunk<R>(row, n, 1, max_rows)) = make_uint4(0, 0, 0, 0);
}

template <int R, bool REMOTE, bool PAIR>
__global__ void __launch_bounds__(9 * 32, 1)
    tc_shrink_kernel(const __grid_constant__ MultiArgs args, const PlanDev pd, const __grid_constant__ TcMaps maps) {
  using C = ShrinkCfgT<R, PAIR>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::NST * C::STAGE);
  uint64_t* full = bars;                  // [NST]  producers -> MMA
  uint64_t* empty = bars + C::NST;        // [NST]  MMA commit -> producers
  uint64_t* tfull = bars + 2 * C::NST;    // [2]    MMA commit -> epilogue
  uint64_t* tempty = tfull + 2;           // [2]    epilogue -> MMA
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  long long* wq_items = reinterpret_cast<long long*>(tmem_slot + 2);
  WorkQueue<kQD> wq{wq_items, reinterpret_cast<uint64_t*>(wq_items + kQD),
                    reinterpret_cast<uint64_t*>(wq_items + kQD) + kQD};

  pdl_wait();  // the plan (segmenter) is complete
  if (tc_cta_idle(args, pd)) {
    wq_finish(pd.wctr + kWqTcShrink, pd.wdone + kWqTcShrink);
    return;
  }
  const int warp = warp_id(), lane = lane_id();
  if (threadIdx.x == 0) {
    wq.init(C::EPI_WARPS + 1 + 3);  // epilogue, MMA and the producer warps that pop (warp PROD_WARP0 fetches)
    const bool g4 = !REMOTE && maps.use;
    for (int s = 0; s < C::NST; ++s) {
      mbar_init(&full[s], g4 ? 1 : C::PROD_THREADS + 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], C::EPI_WARPS * 32);
    }
    fence_mbar_init();
  }
  if (warp == C::MMA_WARP) tmem_alloc(tmem_slot, C::TMEM_COLS);
  if constexpr (C::NP != R) {
    // r = 8: A rows 8-15 of every slot of every stage stay zero (the bulk
    // copies fill rows 0-7 only)
    for (int s = 0; s < C::NST; ++s)
      for (int i = threadIdx.x; i < C::KS_PER_STAGE * C::NW * (C::W_SUB - C::W_G) / 16; i += C::THREADS) {
        const int per = (C::W_SUB - C::W_G) / 16, slot = i / per, o = i - slot * per;
        *reinterpret_cast<uint4*>(smem + s * C::STAGE + C::KS_PER_STAGE * C::X_SUB + slot * C::W_SUB + C::W_G +
                                  o * 16) = make_uint4(0, 0, 0, 0);
      }
    fence_proxy_async_smem();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  pdl_wait();               // the plan (segmenter) is complete
  pdl_launch_dependents();  // the v reduction may launch
  const int n_tiles = pd.counts[kCntTiles];
  const long long n_items = (long long)n_tiles * args.total_kc;

  if (warp >= C::PROD_WARP0) {
    // ===================== producers: gather X rows, bulk-copy W =====================
    const int pt = threadIdx.x - C::PROD_WARP0 * 32;  // 0..127
    int stage = 0;
    uint32_t phase = 0;
    int pend_stage[C::LAG + 1];
    int npend = 0;
    QueuePos qp;
    for (;;) {
      long long it = -1;
      if (warp == C::PROD_WARP0) {
        if (lane == 0) it = wq_push_next(wq, qp, pd.wctr + kWqTcShrink, n_items);
        it = __shfl_sync(0xffffffffu, it, 0);
      } else {
        it = wq_pop(wq, qp);
      }
      if (it < 0) break;
      const int kcg = (int)(it / n_tiles), ti = (int)(it - (long long)kcg * n_tiles);
      const int task = find_task_kc(args, kcg);
      const SlotTask& t = args.t[task];
      const int kc = kcg - t.kc_base;
      const int4 tile = pd.tiles[ti];
      const long long unit = store_unit(tile.z, t.E, args.pl, args.cache);
      const long long woff = (unit * (t.h_in >> 6) + ((kc * t.KI) >> 6)) * (long long)(R * 64);
      const uint16_t* wbase = t.At + woff;
      const int pj = PAIR ? args.tc_pair[task] : -1;          // partner slot (same x, h_in, plan)
      const uint16_t* wbase2 = pj >= 0 ? args.t[pj].At + woff : nullptr;
      const int n_st = t.KI / (C::KSTEP * C::KS_PER_STAGE);
      if (!PAIR && !REMOTE && maps.use) {
        // one warp: lane l gathers tile rows 4l .. 4l+3 (rows past the tile
        // repeat its first row; their accumulator rows are never read)
        if (warp != C::PROD_WARP0) continue;
        int rr[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int n = lane * 4 + i;
          rr[i] = pd.perm[tile.x + (n < tile.y ? n : 0)];
        }
        const CUtensorMap* xm = &maps.x[task];
        for (int st = 0; st < n_st; ++st) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sbase = smem + stage * C::STAGE;
          if (lane == 0) {
            mbar_arrive_expect_tx(&full[stage], C::KS_PER_STAGE * (C::W_G + C::X_SUB));
#pragma unroll
            for (int ks = 0; ks < C::KS_PER_STAGE; ++ks)
              bulk_g2s(sbase + C::KS_PER_STAGE * C::X_SUB + ks * C::W_SUB,
                       wbase + (long long)(st * C::KS_PER_STAGE + ks) * (R * 64), C::W_G, &full[stage]);
          }
          __syncwarp();
          const int col = kc * t.KI + st * C::KS_PER_STAGE * C::KSTEP;
#pragma unroll
          for (int ks = 0; ks < C::KS_PER_STAGE; ++ks)
            tma_gather4(smem_u32(sbase + ks * C::X_SUB + lane * 512), xm, col + ks * C::KSTEP, rr[0], rr[1], rr[2],
                        rr[3], &full[stage]);
          if (++stage == C::NST) {
            stage = 0;
            phase ^= 1;
          }
        }
        continue;
      }
      // this thread's rows / chunks: 128 rows x 8 chunks per k-step, 1024 copies / 128 threads;
      // thread pt always copies chunk q = pt & 7 of rows n = (pt >> 3) + 16 i
      const uint16_t* xsrc[8];
      uint32_t xbytes[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int n = (pt >> 3) + 16 * i;
        const bool valid = n < tile.y;
        xsrc[i] = (valid ? x_row<REMOTE>(args, task, pd.perm[tile.x + n]) : t.x) + (long long)kc * t.KI + (pt & 7) * 8;
        xbytes[i] = valid ? 16u : 0u;
      }
      for (int st = 0; st < n_st; ++st) {
        mbar_wait(&empty[stage], phase ^ 1);
        uint8_t* sbase = smem + stage * C::STAGE;
        if (pt == 0) {
          // W region of a stage: per k-step [NW][R rows x 128 B] -- for a pair the
          // two slots' A tiles back to back, one N = 2r operand
          // (A tiles evict_last when args.tc_flags bit 5: a unit's A is re-read by each of its tiles)
          const uint64_t wpol = (args.tc_flags & 32) ? policy_evict_last() : policy_evict_normal();
          if (pj >= 0) {
            mbar_arrive_expect_tx(&full[stage], C::KS_PER_STAGE * 2 * C::W_G);
#pragma unroll
            for (int ks = 0; ks < C::KS_PER_STAGE; ++ks) {
              uint8_t* wd = sbase + C::KS_PER_STAGE * C::X_SUB + ks * C::NW * C::W_SUB;
              const long long wo = (long long)(st * C::KS_PER_STAGE + ks) * (R * 64);
              bulk_g2s_hint(wd, wbase + wo, C::W_G, &full[stage], wpol);
              bulk_g2s_hint(wd + C::W_SUB, wbase2 + wo, C::W_G, &full[stage], wpol);
            }
          } else if (C::NW == 1 && C::NP == R) {
            mbar_arrive_expect_tx(&full[stage], C::KS_PER_STAGE * C::W_SUB);
            bulk_g2s_hint(sbase + C::KS_PER_STAGE * C::X_SUB, wbase + (long long)st * C::KS_PER_STAGE * (R * 64),
                          C::KS_PER_STAGE * C::W_SUB, &full[stage], wpol);
          } else {  // an unpaired task in a pair launch (or r = 8): one A tile per k-step, N = r
            mbar_arrive_expect_tx(&full[stage], C::KS_PER_STAGE * C::W_G);
#pragma unroll
            for (int ks = 0; ks < C::KS_PER_STAGE; ++ks)
              bulk_g2s_hint(sbase + C::KS_PER_STAGE * C::X_SUB + ks * C::NW * C::W_SUB,
                            wbase + (long long)(st * C::KS_PER_STAGE + ks) * (R * 64), C::W_G, &full[stage], wpol);
          }
        }
        const int j0 = st * C::KS_PER_STAGE * C::KSTEP;
#pragma unroll
        for (int ks = 0; ks < C::KS_PER_STAGE; ++ks) {
          uint8_t* xs = sbase + ks * C::X_SUB;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int n = (pt >> 3) + 16 * i, q = pt & 7;
            cp_async16(xs + n * 128 + ((q ^ (n & 7)) << 4), xsrc[i] + j0 + ks * C::KSTEP, xbytes[i]);
          }
        }
#if LORA_TCS_NOINC
        // the stage's barrier tracks this thread's copies itself: no wait here,
        // every stage of the ring can be in flight (the MMA thread fences the
        // async proxy after its wait)
        cp_async_mbar_arrive_noinc(&full[stage]);
#else
        cp_async_commit();
        pend_stage[npend++] = stage;
        if (npend > C::LAG) {
          cp_async_wait<C::LAG>();
          fence_proxy_async_smem();
          mbar_arrive(&full[pend_stage[0]]);
          for (int q = 0; q < npend - 1; ++q) pend_stage[q] = pend_stage[q + 1];
          --npend;
        }
#endif
        if (++stage == C::NST) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
#if !LORA_TCS_NOINC
    cp_async_wait<0>();
    fence_proxy_async_smem();
    for (int q = 0; q < npend; ++q) mbar_arrive(&full[pend_stage[q]]);
#else
    cp_async_wait<0>();
    (void)npend;
    (void)pend_stage;
#endif
  } else if (warp == C::MMA_WARP) {
    // ===================== MMA issuer =====================
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    QueuePos qp;
    for (;;) {
      const long long it = wq_pop(wq, qp);
      if (it < 0) break;
      const int kcg = (int)(it / n_tiles);
      const int task = find_task_kc(args, kcg);
      const SlotTask& t = args.t[task];
      const int n_st = t.KI / (C::KSTEP * C::KS_PER_STAGE);
      const uint32_t idesc = idesc_bf16(128, (PAIR && args.tc_pair[task] >= 0) ? 2 * C::NP : C::NP);
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem + acc * C::ACC_COLS;
      for (int st = 0; st < n_st; ++st) {
        mbar_wait(&full[stage], phase);
#if LORA_TCS_NOINC
        fence_proxy_async_smem();  // the producers' cp.async writes, seen through the barrier, to the MMA's async proxy
#endif
        tc_fence_after();
        if (lane == 0) {
          const uint32_t sbase = smem_u32(smem + stage * C::STAGE);
#pragma unroll
          for (int ks = 0; ks < C::KS_PER_STAGE; ++ks) {
            const uint32_t xa = sbase + ks * C::X_SUB;
            const uint32_t wa = sbase + C::KS_PER_STAGE * C::X_SUB + ks * C::NW * C::W_SUB;
#pragma unroll
            for (int k = 0; k < C::KSTEP / 16; ++k) {
              umma_bf16(d_tmem, sw128_desc(xa + k * 32), sw128_desc(wa + k * 32), idesc,
                        (st > 0 || ks > 0 || k > 0) ? 1u : 0u);
            }
          }
          umma_commit(&empty[stage]);
          if (st == n_st - 1) umma_commit(&tfull[acc]);
        }
        __syncwarp();
        if (++stage == C::NST) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  } else {
    // ===================== epilogue: TMEM -> vpart =====================
    int acc = 0;
    uint32_t acc_phase = 0;
    const int row_in_tile = warp * 32 + lane;  // TMEM lane
    QueuePos qp;
    for (;;) {
      const long long it = wq_pop(wq, qp);
      if (it < 0) break;
      const int kcg = (int)(it / n_tiles), ti = (int)(it - (long long)kcg * n_tiles);
      const int task = find_task_kc(args, kcg);
      const SlotTask& t = args.t[task];
      const int kc = kcg - t.kc_base;
      const int4 tile = pd.tiles[ti];
      const int pj = PAIR ? args.tc_pair[task] : -1;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      // columns [0, R) are this task's v, [R, 2R) the partner's (pair)
#pragma unroll 1
      for (int half = 0; half < (pj >= 0 ? 2 : 1); ++half) {
        const SlotTask& th = half ? args.t[pj] : t;
        float v[C::NP];
        const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + acc * C::ACC_COLS + half * C::NP;
#pragma unroll
        for (int c = 0; c < C::NP; c += 16) tmem_ld16(taddr + c, v + c);
        if (row_in_tile < tile.y) {
          if (t.n_kc == 1) {
            // the whole K in one accumulator: v rounded to bf16 here (no reduction pass)
            store_vbf_row<R>(pd.vbf + th.vbf_off, (long long)tile.x + row_in_tile, row_in_tile, v, pd.max_rows);
          } else {
            float4* dst = reinterpret_cast<float4*>(pd.vpart + th.vpart_off +
                                                    ((long long)kc * pd.max_rows + tile.x + row_in_tile) * R);
#pragma unroll
            for (int c = 0; c < R / 4; ++c) dst[c] = make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  wq_finish(pd.wctr + kWqTcShrink, pd.wdone + kWqTcShrink);
  if (warp == C::MMA_WARP) {
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

// ===========================================================================
// v reduction: the tcgen05 shrink leaves n_kc fp32 partials per row; sum them
// in fixed kc order, round once to bf16 and store each tile's rows already in
// the SWIZZLE_128B K-major layout (row n of a tile: 16-byte chunk q at
// q ^ (n & 7)), so the expand loads its MMA operand with one bulk copy.
// ===========================================================================
template <int R>
__global__ void __launch_bounds__(256) tc_vreduce_kernel(const __grid_constant__ MultiArgs args, const PlanDev pd) {
  pdl_wait();               // the tcgen05 shrink's partials are complete
  pdl_launch_dependents();
  const int n_tiles = pd.counts[kCntTiles];
  const long long per_task = (long long)n_tiles * kTileRows * (R / 8);
  const long long total = per_task * args.n_tasks;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int task = (int)(i / per_task);
    const long long rem = i - (long long)task * per_task;
    const int ti = (int)(rem / (kTileRows * (R / 8)));
    const int within = (int)(rem - (long long)ti * (kTileRows * (R / 8)));
    const int n = within / (R / 8), q = within - n * (R / 8);
    const int4 tile = pd.tiles[ti];
    if (n >= tile.y) continue;
    const SlotTask& t = args.t[task];
    if (t.n_kc == 1) continue;  // written by the shrink epilogue
    const float* src = pd.vpart + t.vpart_off + ((long long)tile.x + n) * R + q * 8;
    float s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int kc = 0; kc < t.n_kc; ++kc) {
      const float4* p4 = reinterpret_cast<const float4*>(src + (long long)kc * pd.max_rows * R);
      const float4 a = p4[0], b = p4[1];
      s[0] += a.x; s[1] += a.y; s[2] += a.z; s[3] += a.w;
      s[4] += b.x; s[5] += b.y; s[6] += b.z; s[7] += b.w;
    }
    uint4 w;
    w.x = pack_bf16x2_rn(s[0], s[1]);
    w.y = pack_bf16x2_rn(s[2], s[3]);
    w.z = pack_bf16x2_rn(s[4], s[5]);
    w.w = pack_bf16x2_rn(s[6], s[7]);
    *reinterpret_cast<uint4*>(pd.vbf + t.vbf_off + vbf_chunk<R>((long long)tile.x + n, n, q, pd.max_rows)) = w;
    if constexpr (R < 16)  // the K padding of the expand operand
      *reinterpret_cast<uint4*>(pd.vbf + t.vbf_off + vbf_chunk<R>((long long)tile.x + n, n, 1, pd.max_rows)) =
          make_uint4(0, 0, 0, 0);
  }
}

LORA_DEVINL void tmem_ld16_nowait(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
}
LORA_DEVINL void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

LORA_DEVINL void tmem_ld8_nowait(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr)
               : "memory");
}
LORA_DEVINL void tmem_ld32_nowait(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
}

// 2 x 256-bit global load / store (64 contiguous bytes; full 32-byte sectors)
LORA_DEVINL void ldg256x2(const void* p, uint32_t* r) {
  asm volatile("ld.global.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "l"(p));
  asm volatile("ld.global.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
               : "l"(static_cast<const char*>(p) + 32));
}
LORA_DEVINL void stg256x2(void* p, const uint32_t* w) {
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(w[0]), "r"(w[1]), "r"(w[2]),
               "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
               : "memory");
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(static_cast<char*>(p) + 32), "r"(w[8]),
               "r"(w[9]), "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]), "r"(w[15])
               : "memory");
}

// ===========================================================================
// expand.  Per 128-column sub-tile: D[128 rows x 128 cols] = v_tile . Bt_sub^T
// in TMEM (four accumulators): TMEM lane = tile row, so every epilogue thread
// owns one row and 32 consecutive output columns -- it reads its 64-byte
// y segment (two 256-bit loads, issued one sub-tile ahead), adds s_a * D and
// writes the segment back with two 256-bit stores.  No transposing staging
// tile, every access a full 32-byte sector.  16 epilogue warps: TMEM lane quadrant = warp % 4,
// column block = warp / 4.
// ===========================================================================
template <int R>
struct ExpandCfg {
  using G = KGeo<R>;
  static constexpr int EPI_WARPS = 16;
  static constexpr int EPI_THREADS = EPI_WARPS * 32;
  static constexpr int TMA_WARP = 16;   // warp 16: v tile + Bt bulk copies
  static constexpr int MMA_WARP = 17;   // warp 17: TMEM alloc + MMA
  static constexpr int THREADS = 18 * 32;
  static constexpr int MSUB = 128;                     // output columns per MMA (N)
  static constexpr int B_SUB = MSUB * G::RP * 2;       // smem Bt rows of a sub-tile (16 KB at r = 64)
  // r = 128: the producer warp re-tiles the 256-byte Bt rows into two
  // SWIZZLE_128B K blocks with cp.async (all 32 lanes arrive on the stage);
  // r = 8: the 16-byte rows go to the data chunk of 32-byte SWIZZLE_32B rows
  // whose other chunk stays zero (K padded to 16)
  static constexpr bool BT_RETILE = R > 64 || R < 16;
#ifndef LORA_TCE_NST
#define LORA_TCE_NST 2
#endif
#ifndef LORA_TCE_YD
#define LORA_TCE_YD 4
#endif
#ifndef LORA_TCE128_NST
#define LORA_TCE128_NST 2
#endif
#ifndef LORA_TCE128_VB
#define LORA_TCE128_VB 2  // r = 128 (shared memory: 2 x 32 KB Bt + VB x 32 KB v + (YD + 1) x 32 KB y):
#endif                    // measured VB 2 / YD 2 444 us, VB 1 / YD 3 452 us, NST 3 / YD 2 452 us (prefill shapes)
#ifndef LORA_TCE128_YD
#define LORA_TCE128_YD 2
#endif
  static constexpr int NST = R > 64 ? LORA_TCE128_NST : LORA_TCE_NST;
  static constexpr int V_TILE = kTileRows * G::RP * 2; // v tile, M = 128 rows x K = r (16 KB at r = 64)
  static constexpr int VB = R > 64 ? LORA_TCE128_VB : 2;  // v tile buffers
  // bf16 output: y tiles [128 rows][128 cols] (16-byte chunks XOR-swizzled by
  // row) in a ring of YS slots, fetched YD-1 sub-tiles ahead
  static constexpr int YD = R > 64 ? LORA_TCE128_YD : LORA_TCE_YD;
  static constexpr int YS = YD + 1;
  static constexpr int Y_TILE = kTileRows * MSUB * 2;  // 32 KB
  static constexpr int NACC = 4;
  static constexpr int ACC_COLS = MSUB;                // N columns per accumulator
  static constexpr int TMEM_COLS = NACC * ACC_COLS;    // 512
  static constexpr int SMEM = 1024 + NST * B_SUB + VB * V_TILE + YS * Y_TILE + 512;
  static_assert(SMEM <= 227 * 1024, "expand stages exceed shared memory");
};

// output mode M (compile time): 0 bf16 accumulate, 1 fp32 delta store, 2 bf16
// delta store (sharded), 3 fp32 accumulate, 4 / 5 bf16 / fp32 push (sharded
// owner: the delta is added into the origin row of the source's registered y
// with red.add over NVLink)
template <int R, int M>
__global__ void __launch_bounds__(18 * 32, 1)
    tc_expand_kernel(const __grid_constant__ MultiArgs args, const PlanDev pd) {
  using C = ExpandCfg<R>;
  using G = KGeo<R>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* vtile = smem + C::NST * C::B_SUB;   // [VB][V_TILE] swizzled MMA operand A
  uint8_t* yring = vtile + C::VB * C::V_TILE;  // [YS][Y_TILE] bf16 y tiles (bf16 output modes)
  uint64_t* bars = reinterpret_cast<uint64_t*>(yring + C::YS * C::Y_TILE);
  uint64_t* full = bars;                       // [NST] Bt landed
  uint64_t* empty = bars + C::NST;             // [NST] MMA done with Bt stage
  uint64_t* vfull = bars + 2 * C::NST;         // [2]  v tile landed
  uint64_t* vempty = vfull + 2;                // [2]  MMA done with the v tile
  uint64_t* tfull = vempty + 2;                // [NACC] accumulator ready
  uint64_t* tempty = tfull + C::NACC;          // [NACC] accumulator drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + C::NACC);
  long long* wq_items = reinterpret_cast<long long*>(tmem_slot + 2);
  WorkQueue<kQD> wq{wq_items, reinterpret_cast<uint64_t*>(wq_items + kQD),
                    reinterpret_cast<uint64_t*>(wq_items + kQD) + kQD};

  if (tc_cta_idle(args, pd)) {
    wq_finish(pd.wctr + kWqTcExpand, pd.wdone + kWqTcExpand);
    return;
  }
  const int warp = warp_id(), lane = lane_id();
  if (threadIdx.x == 0) {
    wq.init(C::EPI_WARPS + 1);  // epilogue + MMA warps pop; the TMA warp fetches
    for (int s = 0; s < C::NST; ++s) {
      mbar_init(&full[s], C::BT_RETILE ? 32 : 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < C::VB; ++a) {
      mbar_init(&vfull[a], 1);
      mbar_init(&vempty[a], 1);
    }
    for (int a = 0; a < C::NACC; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], C::EPI_THREADS);
    }
    fence_mbar_init();
  }
  if (warp == C::MMA_WARP) tmem_alloc(tmem_slot, C::TMEM_COLS);
  if constexpr (R < 16) {
    // r = 8: the Bt stages' K padding chunks stay zero (the producer fills
    // only each row's data chunk)
    for (int i = threadIdx.x; i < C::NST * C::B_SUB / 16; i += C::THREADS)
      reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
    fence_proxy_async_smem();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const int n_tiles = pd.counts[kCntTiles];
  const long long n_items = (long long)n_tiles * args.total_ci;

  if (warp == C::TMA_WARP) {
    // ===================== producer: v tile + Bt sub-tiles =====================
    // (lane 0 alone, except for the r = 128 Bt re-tiling copies of all lanes)
    if (lane == 0 || C::BT_RETILE) {
      const uint64_t pol = (args.tc_flags & 1) ? policy_evict_last() : policy_evict_first();
      int stage = 0, vb = 0;
      uint32_t phase = 0, vphase = 0;
      bool vready = false;
      QueuePos qp;
      for (;;) {
        long long it = -1;
        if (lane == 0) it = wq_push_next(wq, qp, pd.wctr + kWqTcExpand, n_items);
        if constexpr (C::BT_RETILE) it = __shfl_sync(0xffffffffu, it, 0);
        if (it < 0) break;
        const int cig = (int)(it / n_tiles), ti = (int)(it - (long long)cig * n_tiles);
        const SlotTask& t = args.t[find_task_ci(args, cig)];
        const int ci = cig - t.ci_base;
        const int4 tile = pd.tiles[ti];
        if (lane == 0) {
          mbar_wait(&vempty[vb], vphase ^ 1);
          if (!vready) {
            pdl_wait();  // the v tiles come from the v reduction (the Bt rows do not)
            vready = true;
          }
          // one bulk copy per K block: rows [tile.x, tile.x + tile.y) of the slot's v store
          mbar_arrive_expect_tx(&vfull[vb], (uint32_t)tile.y * G::RP * 2);
#pragma unroll
          for (int kb = 0; kb < G::KB; ++kb)
            bulk_g2s(vtile + vb * C::V_TILE + kb * (kTileRows * G::RB),
                     pd.vbf + t.vbf_off + (long long)kb * pd.max_rows * (G::RB / 2) + (long long)tile.x * (G::RB / 2),
                     (uint32_t)tile.y * G::RB, &vfull[vb]);
        }
        if (++vb == C::VB) {
          vb = 0;
          vphase ^= 1;
        }
        const long long unit = store_unit(tile.z, t.E, args.pl, args.cache);
        const uint16_t* bbase = t.Bt + (unit * t.h_out + (long long)ci * t.CI) * R;
        const int n_sub = t.CI / C::MSUB;
        for (int sb = 0; sb < n_sub; ++sb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if constexpr (C::BT_RETILE && R > 64) {
            // 128 columns x 256 bytes: physical chunk p of column c holds k chunk
            // p ^ ((c & 3) << 1) (common.cuh); k chunk ch goes to K block ch / 8,
            // chunk (ch % 8) ^ (c & 7) of the block's row c (SWIZZLE_128B)
            const uint16_t* src = bbase + (long long)sb * C::MSUB * R;
            const uint32_t dst = smem_u32(smem + stage * C::B_SUB);
#pragma unroll 8
            for (int i = 0; i < C::MSUB * 16 / 32; ++i) {
              const int idx = i * 32 + lane, c = idx >> 4, pch = idx & 15;
              const int ch = pch ^ ((c & 3) << 1);
              cp_async16_u32(dst + (ch >> 3) * (C::MSUB * 128) + c * 128 + (((ch & 7) ^ (c & 7)) << 4),
                             src + c * R + pch * 8);
            }
            cp_async_mbar_arrive_noinc(&full[stage]);
          } else if constexpr (C::BT_RETILE) {
            // r = 8: column c's 16 bytes to chunk swz(c, 0) of its 32-byte row
            const uint16_t* src = bbase + (long long)sb * C::MSUB * R;
            const uint32_t dst = smem_u32(smem + stage * C::B_SUB);
#pragma unroll
            for (int i = 0; i < C::MSUB / 32; ++i) {
              const int c = i * 32 + lane;
              cp_async16_u32(dst + c * 32 + (swz_row_chunk(c, 0, 32) << 4), src + c * R);
            }
            cp_async_mbar_arrive_noinc(&full[stage]);
          } else {
            mbar_arrive_expect_tx(&full[stage], C::B_SUB);
            bulk_g2s_hint(smem + stage * C::B_SUB, bbase + (long long)sb * C::MSUB * R, C::B_SUB, &full[stage], pol);
          }
          if (++stage == C::NST) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      if constexpr (C::BT_RETILE) cp_async_wait<0>();
    }
  } else if (warp == C::MMA_WARP) {
    // ===================== MMA issuer =====================
    int stage = 0, vb = 0;
    uint32_t phase = 0, vphase = 0;
    long long k = 0;  // global sub-tile counter -> accumulator k % NACC
    const uint32_t idesc = idesc_bf16(kTileRows, C::MSUB);
    QueuePos qp;
    for (;;) {
      const long long it = wq_pop(wq, qp);
      if (it < 0) break;
      const int cig = (int)(it / n_tiles);
      const SlotTask& t = args.t[find_task_ci(args, cig)];
      const int n_sub = t.CI / C::MSUB;
      mbar_wait(&vfull[vb], vphase);
      // rows >= tile.y of the v tile hold stale data: their D rows are never read
      const uint32_t va = smem_u32(vtile + vb * C::V_TILE);
      for (int sb = 0; sb < n_sub; ++sb, ++k) {
        const int acc = (int)(k % C::NACC);
        mbar_wait(&tempty[acc], (uint32_t)((k / C::NACC) & 1) ^ 1);
        mbar_wait(&full[stage], phase);
        if constexpr (C::BT_RETILE) fence_proxy_async_smem();  // the producer's cp.async writes -> the MMA's async proxy
        tc_fence_after();
        if (lane == 0) {
          const uint32_t ba = smem_u32(smem + stage * C::B_SUB);
          const uint32_t d_tmem = tmem + acc * C::ACC_COLS;
#pragma unroll
          for (int kk = 0; kk < G::RP / 16; ++kk) {
            const int kb = kk / G::KPB, ko = (kk % G::KPB) * 32;
            umma_bf16(d_tmem, kmajor_desc<G::RB>(va + kb * (kTileRows * G::RB) + ko),
                      kmajor_desc<G::RB>(ba + kb * (C::MSUB * G::RB) + ko), idesc, kk > 0 ? 1u : 0u);
          }
          umma_commit(&empty[stage]);
          umma_commit(&tfull[acc]);
          if (sb == n_sub - 1) umma_commit(&vempty[vb]);
        }
        __syncwarp();
        if (++stage == C::NST) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (++vb == C::VB) {
        vb = 0;
        vphase ^= 1;
      }
    }
  } else {
    if constexpr (M == 0 || M == 2 || M == 4) {
    // ===================== epilogue, bf16 output: coalesced y tiles =====================
    // Per sub-tile the 128 x 128 y tile is fetched with coalesced cp.async
    // (16 chunks of 16 bytes per row; YD-1 sub-tiles ahead) into a smem ring;
    // thread (row, 32 columns) adds s_a * D from TMEM in place; the tile
    // leaves with coalesced 16-byte stores.  Two named barriers per sub-tile
    // over the 512 epilogue threads; the ring has one spare slot, so the
    // slot refilled at sub-tile sb was stored out two sub-tiles ago.
    const int q = warp & 3, cb = warp >> 2;
    const int et = threadIdx.x;                  // 0 .. EPI_THREADS-1
    const int n = q * 32 + lane;                 // this thread's tile row (TMEM lane)
    const int cc = et & 15;                      // chunk column of this thread's copies
    const uint32_t ybase = smem_u32(yring);
    const bool ypol_ld = (args.tc_flags & 2) != 0, ypol_st = (args.tc_flags & 4) != 0;
    const uint64_t ypol = policy_evict_first();
    long long k = 0;                             // global sub-tile counter (same as the MMA warp's)
    int kk = 0;                                  // this CTA's sub-tile sequence number (ring slot)
    QueuePos qp;
    for (;;) {
      const long long it = wq_pop(wq, qp);
      if (it < 0) break;
      const int cig = (int)(it / n_tiles), ti = (int)(it - (long long)cig * n_tiles);
      const int task = find_task_ci(args, cig);
      const SlotTask& t = args.t[task];
      const int ci = cig - t.ci_base;
      const int4 tile = pd.tiles[ti];
      const float s_a = args.scale[tile.z / t.E];
      const int n_sub = t.CI / C::MSUB;
      uint16_t* yb = static_cast<uint16_t*>(t.y);
      // this thread's copy rows: r_j = et / 16 + 32 j
      long long coff[4];
      bool cval[4];
      uint16_t* ppush[4];  // push: the origin rows in the sources' y (+ this thread's chunk column)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int r = (et >> 4) + 32 * j;
        cval[j] = r < tile.y;
        const int prow = cval[j] ? __ldg(pd.perm + tile.x + r) : 0;
        coff[j] = (long long)prow * t.h_out + (long long)ci * t.CI + cc * 8;
        if constexpr (M == 4)
          ppush[j] = cval[j] ? reinterpret_cast<uint16_t*>(y_push_row(args, task, prow, 2)) + (long long)ci * t.CI + cc * 8
                             : nullptr;
      }
      auto slot_of = [&](int seq) { return ybase + (uint32_t)(seq % C::YS) * C::Y_TILE; };
      auto chunk_addr = [&](uint32_t sl, int r, int c) { return sl + r * (C::MSUB * 2) + ((c ^ (r & 15)) << 4); };
      auto issue2 = [&](int sb) {
        if (M == 0 && sb < n_sub) {
          const uint32_t sl = slot_of(kk + sb);
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (cval[j]) {
              if (ypol_ld)
                cp_async16_u32_hint(chunk_addr(sl, (et >> 4) + 32 * j, cc), yb + coff[j] + (long long)sb * C::MSUB,
                                    ypol);
              else
                cp_async16_u32(chunk_addr(sl, (et >> 4) + 32 * j, cc), yb + coff[j] + (long long)sb * C::MSUB);
            }
        }
        cp_async_commit();
      };
#pragma unroll 1
      for (int j = 0; j < C::YD - 1; ++j) issue2(j);
      for (int sb = 0; sb < n_sub; ++sb, ++k) {
        issue2(sb + C::YD - 1);
        const uint32_t sl = slot_of(kk + sb);
        const int acc = (int)(k % C::NACC);
        mbar_wait(&tfull[acc], (uint32_t)((k / C::NACC) & 1));
        tc_fence_after();
        if (M == 0) cp_async_wait<C::YD - 1>();
        named_bar_sync(1, C::EPI_THREADS);  // tile sb complete and visible
        const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + acc * C::ACC_COLS + cb * 32;
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          uint32_t d[8];
          tmem_ld8_nowait(ta + h * 8, d);
          const uint32_t a = chunk_addr(sl, n, cb * 4 + h);
          uint4 yv = make_uint4(0, 0, 0, 0);
          if (M == 0) yv = lds128(a);
          tmem_wait_ld();
          const uint32_t y4[4] = {yv.x, yv.y, yv.z, yv.w};
          uint32_t w4[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float e0 = s_a * __uint_as_float(d[2 * i]), e1 = s_a * __uint_as_float(d[2 * i + 1]);
            w4[i] = M == 0 ? pack_bf16x2_rn(bf16lo(y4[i]) + e0, bf16hi(y4[i]) + e1) : pack_bf16x2_rn(e0, e1);
          }
          asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(w4[0]), "r"(w4[1]), "r"(w4[2]),
                       "r"(w4[3])
                       : "memory");
        }
        tc_fence_before();
        mbar_arrive(&tempty[acc]);
        named_bar_sync(1, C::EPI_THREADS);  // results in the tile
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (cval[j]) {
            const uint4 v = lds128(chunk_addr(sl, (et >> 4) + 32 * j, cc));
            if constexpr (M == 4)
              red_add_bf16x8(ppush[j] + (long long)sb * C::MSUB, v);
            else if (ypol_st)
              st_global_v4_hint(yb + coff[j] + (long long)sb * C::MSUB, v, ypol);
            else
              *reinterpret_cast<uint4*>(yb + coff[j] + (long long)sb * C::MSUB) = v;
          }
      }
      cp_async_wait<0>();
      kk += n_sub;
    }
    if constexpr (M == 4) __threadfence_system();  // pushes performed before the owner signals completion
    } else {
    // ===================== epilogue: one row x 32 columns per thread =====================
    // y moves in full 32-byte sectors (256-bit LDG/STG); the segments of the
    // next two sub-tiles of the item are in flight while one is in the
    // epilogue.  (A look-ahead across items, peeking the queue, measured slower:
    // register pressure.)
    const int q = warp & 3, cb = warp >> 2;
    constexpr bool yload = M == 0;
    long long k = 0;                             // global sub-tile counter (same as the MMA warp's)
    QueuePos qp;
    for (;;) {
      const long long it = wq_pop(wq, qp);
      if (it < 0) break;
      const int cig = (int)(it / n_tiles), ti = (int)(it - (long long)cig * n_tiles);
      const int task = find_task_ci(args, cig);
      const SlotTask& t = args.t[task];
      const int ci = cig - t.ci_base;
      const int4 tile = pd.tiles[ti];
      const float s_a = args.scale[tile.z / t.E];
      const int n_sub = t.CI / C::MSUB;
      const int n = q * 32 + lane;
      const bool live = n < tile.y;
      const long long prow = live ? (long long)__ldg(pd.perm + tile.x + n) : 0;
      const long long o0 = prow * t.h_out + (long long)ci * t.CI + cb * 32;  // + sb * MSUB
      uint16_t* yb = static_cast<uint16_t*>(t.y);
      // push (M = 5): this row's columns in the origin row of the source's y
      float* ypush = nullptr;
      if constexpr (M == 5)
        if (live) ypush = reinterpret_cast<float*>(y_push_row(args, task, (int)prow, 4)) + (long long)ci * t.CI + cb * 32;
      // three segment buffers with compile-time roles (a register rotation
      // would wait for the newest load): step sb consumes buf[sb % 3] and
      // starts the load of sub-tile sb + 2 into buf[(sb + 2) % 3]
      auto step = [&](int sb, uint32_t (&ya)[16], uint32_t (&yn)[16]) {
        if (sb >= n_sub) return;
        if (yload && live && sb + 2 < n_sub) ldg256x2(yb + o0 + (long long)(sb + 2) * C::MSUB, yn);
        const int acc = (int)(k % C::NACC);
        mbar_wait(&tfull[acc], (uint32_t)((k / C::NACC) & 1));
        ++k;
        tc_fence_after();
        const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + acc * C::ACC_COLS + cb * 32;
        const long long o = o0 + (long long)sb * C::MSUB;
        if constexpr (M == 0 || M == 2) {
          // four quarters of 8 columns into a separate output w[]: a pending
          // store locks its source registers, so the y buffers stay free for
          // the next loads
          uint32_t w[16];
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            uint32_t d[8];
            tmem_ld8_nowait(ta + h * 8, d);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const float e0 = s_a * __uint_as_float(d[2 * i]), e1 = s_a * __uint_as_float(d[2 * i + 1]);
              const uint32_t yv = ya[h * 4 + i];
              w[h * 4 + i] = yload ? pack_bf16x2_rn(bf16lo(yv) + e0, bf16hi(yv) + e1) : pack_bf16x2_rn(e0, e1);
            }
          }
          tc_fence_before();
          mbar_arrive(&tempty[acc]);
          if (live) stg256x2(yb + o, w);
        } else {
          // fp32 y (accumulate) or fp32 delta store (sharded): 2 halves x 4 x 16 bytes
          float4* yp = M == 5 ? reinterpret_cast<float4*>(ypush + (long long)sb * C::MSUB)
                              : reinterpret_cast<float4*>(static_cast<float*>(t.y) + o);
#pragma unroll 1
          for (int h = 0; h < 2; ++h) {
            uint32_t d[16];
            tmem_ld16_nowait(ta + h * 16, d);
            tmem_wait_ld();
            if (live) {
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const float4 e = make_float4(s_a * __uint_as_float(d[4 * i + 0]), s_a * __uint_as_float(d[4 * i + 1]),
                                             s_a * __uint_as_float(d[4 * i + 2]), s_a * __uint_as_float(d[4 * i + 3]));
                if constexpr (M == 1) {
                  yp[h * 4 + i] = e;
                } else if constexpr (M == 5) {
                  red_add_f32x4(yp + h * 4 + i, e);
                } else {
                  float4 v = yp[h * 4 + i];
                  v.x += e.x; v.y += e.y; v.z += e.z; v.w += e.w;
                  yp[h * 4 + i] = v;
                }
              }
            }
          }
          tc_fence_before();
          mbar_arrive(&tempty[acc]);
        }
      };
      uint32_t b0[16], b1[16], b2[16];
      if (yload && live) {
        ldg256x2(yb + o0, b0);
        if (n_sub > 1) ldg256x2(yb + o0 + C::MSUB, b1);
      }
      for (int sb = 0; sb < n_sub; sb += 3) {
        step(sb, b0, b2);
        step(sb + 1, b1, b0);
        step(sb + 2, b2, b1);
      }
    }
    if constexpr (M == 5) __threadfence_system();  // pushes performed before the owner signals completion
    }
  }
  tc_fence_before();
  __syncthreads();
  wq_finish(pd.wctr + kWqTcExpand, pd.wdone + kWqTcExpand);
  if (warp == C::MMA_WARP) {
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

template <typename K>
cudaError_t set_smem_once(K kernel, int bytes, unsigned long long& mask) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(mask & (1ull << dev))) {
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess) return e;
    mask |= 1ull << dev;
  }
  return cudaSuccess;
}

}  // namespace

bool tc_available() { return true; }

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link)
static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    cudaGetLastError();
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

// x rows by TMA gather4 (opt-in, LORA_TC_GATHER4=1) when every task's x can be
// described by a tensor map (local rows, at most kTcMapTasks tasks).  Measured
// on B200: correct, but one gather4 moves 4 x 128 B and the TMA unit then
// sustains far less than 128 threads of 16-byte cp.async (prefill tc shrink
// 439 us vs 152 us; config 5 438 vs 116 us), so cp.async stays the default.
static void make_x_maps(const MultiArgs& args, int x_rows, TcMaps& m) {
  std::memset(&m, 0, sizeof(m));
  const char* env = getenv("LORA_TC_GATHER4");
  if (!(env && env[0] == '1') || args.push.G > 0 || args.n_tasks > kTcMapTasks || x_rows < 1) return;
  auto enc = tensor_map_encoder();
  if (!enc) return;
  for (int i = 0; i < args.n_tasks; ++i) {
    const SlotTask& t = args.t[i];
    cuuint64_t dims[2] = {(cuuint64_t)t.h_in, (cuuint64_t)x_rows};
    cuuint64_t strides[1] = {(cuuint64_t)t.h_in * 2};
    cuuint32_t box[2] = {64, 1};
    cuuint32_t es[2] = {1, 1};
    if (enc(&m.x[i], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<uint16_t*>(t.x), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return;  // m.use stays 0
  }
  m.use = 1;
}

template <int R>
static cudaError_t launch_tc_shrink_r(const MultiArgs& args, const PlanDev& pd, int x_rows, int grid,
                                      cudaStream_t stream) {
  static unsigned long long mask[4] = {0, 0, 0, 0};
  const bool remote = args.push.G > 0;
  bool pair = false;
  for (int i = 0; i < args.n_tasks; ++i) pair = pair || args.tc_pair[i] >= 0;
  auto kern = remote ? (pair ? tc_shrink_kernel<R, true, true> : tc_shrink_kernel<R, true, false>)
                     : (pair ? tc_shrink_kernel<R, false, true> : tc_shrink_kernel<R, false, false>);
  const int smem = pair ? ShrinkCfgT<R, true>::SMEM : ShrinkCfgT<R, false>::SMEM;
  cudaError_t e = set_smem_once(kern, smem, mask[remote * 2 + pair]);
  if (e != cudaSuccess) return e;
  TcMaps maps;
  make_x_maps(args, x_rows, maps);
  if (pair) maps.use = 0;
  e = launch_pdl(kern, dim3(grid), dim3(ShrinkCfgT<R, false>::THREADS), smem, stream, args, pd, maps);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

template <int R>
static cudaError_t launch_tc_expand_r(const MultiArgs& args, const PlanDev& pd, int grid, cudaStream_t stream) {
  static unsigned long long mask[6] = {0, 0, 0, 0, 0, 0};
  const int m = args.y_store == 3 ? (args.y_fp32 ? 5 : 4)
                                  : args.y_store == 1 ? 1 : args.y_store == 2 ? 2 : args.y_fp32 ? 3 : 0;
  auto kern = m == 0   ? tc_expand_kernel<R, 0>
              : m == 1 ? tc_expand_kernel<R, 1>
              : m == 2 ? tc_expand_kernel<R, 2>
              : m == 3 ? tc_expand_kernel<R, 3>
              : m == 4 ? tc_expand_kernel<R, 4>
                       : tc_expand_kernel<R, 5>;
  using C = ExpandCfg<R>;
  cudaError_t e = set_smem_once(kern, C::SMEM, mask[m]);
  if (e != cudaSuccess) return e;
  e = launch_pdl(kern, dim3(grid), dim3(C::THREADS), C::SMEM, stream, args, pd);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

bool tc_rank_supported(int rank) { return rank == 8 || rank == 16 || rank == 32 || rank == 64 || rank == 128; }

cudaError_t launch_tc_shrink(int rank, const MultiArgs& args, const PlanDev& pd, int x_rows, int grid,
                             cudaStream_t stream) {
  switch (rank) {
    case 8: return launch_tc_shrink_r<8>(args, pd, x_rows, grid, stream);
    case 16: return launch_tc_shrink_r<16>(args, pd, x_rows, grid, stream);
    case 32: return launch_tc_shrink_r<32>(args, pd, x_rows, grid, stream);
    case 64: return launch_tc_shrink_r<64>(args, pd, x_rows, grid, stream);
    case 128: return launch_tc_shrink_r<128>(args, pd, x_rows, grid, stream);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_tc_vreduce(int rank, const MultiArgs& args, const PlanDev& pd, int grid, cudaStream_t stream) {
  cudaError_t e;
  switch (rank) {
    case 8: e = launch_pdl(tc_vreduce_kernel<8>, dim3(grid * 4), dim3(256), 0, stream, args, pd); break;
    case 16: e = launch_pdl(tc_vreduce_kernel<16>, dim3(grid * 4), dim3(256), 0, stream, args, pd); break;
    case 32: e = launch_pdl(tc_vreduce_kernel<32>, dim3(grid * 4), dim3(256), 0, stream, args, pd); break;
    case 64: e = launch_pdl(tc_vreduce_kernel<64>, dim3(grid * 4), dim3(256), 0, stream, args, pd); break;
    case 128: e = launch_pdl(tc_vreduce_kernel<128>, dim3(grid * 4), dim3(256), 0, stream, args, pd); break;
    default: return cudaErrorInvalidValue;
  }
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_tc_expand(int rank, const MultiArgs& args, const PlanDev& pd, int grid, cudaStream_t stream) {
  switch (rank) {
    case 8: return launch_tc_expand_r<8>(args, pd, grid, stream);
    case 16: return launch_tc_expand_r<16>(args, pd, grid, stream);
    case 32: return launch_tc_expand_r<32>(args, pd, grid, stream);
    case 64: return launch_tc_expand_r<64>(args, pd, grid, stream);
    case 128: return launch_tc_expand_r<128>(args, pd, grid, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace lora
