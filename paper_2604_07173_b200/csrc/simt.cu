// simt.cu -- a2 shrink and a3+a4 expand/scatter-accumulate on CUDA cores.
//
// The decode case: most segments hold 1-8 rows,
// so the work is a stream of per-unit weights with 1-8 FMAs per weight
// element -- HBM-bound, far below the tensor-core ridge.  The paper's BGMV
// answer is "thread collaborative execution instead of the heavier wgmma
// pipeline" (Sec. 5.2); the B200 form used here:
//
//   * persistent CTAs, two per SM, each 1 producer warp + 8 consumer warps;
//   * the producer streams each unit's weights with 1-D TMA bulk copies
//     (cp.async.bulk, SASS UBLKCP) into a shared-memory ring (~100 KB per CTA,
//     ~200 KB in flight per SM), together with the group's activation rows
//     (shrink) or its v rows (expand), so consumers never wait on a global
//     load for an operand;
//   * the weight store is pre-swizzled (common.cuh): the consumers' 128-bit
//     shared loads are bank-conflict free;
//   * the consumer code is specialised on the group's row count (1..8), so
//     the inner loops carry no predicates, with two accumulator chains per
//     output;
//   * shrink reduces per-thread partial dot products deterministically
//     through shared memory (no float atomics);
//   * expand applies the per-adapter scale and read-modify-writes y[perm[j]]
//     from registers, consecutive threads on consecutive columns, with the y
//     loads of the next stage in flight one stage ahead.
//
// Work items (device-side counts, no host sync):
//   shrink item = (slot task, row group)            -> vpart[0][row][0:r]  (v = x A_u)
//   expand item = (slot task, c-chunk of CI, group) -> y[perm[row]][c-chunk] += s_a v B_u
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

#ifndef LORA_EXP_PROBE
#define LORA_EXP_PROBE 0  // staged-tile expand timing probes (A/B only; results wrong): bit 0 no consumer work, bit 1 no y loads
#endif
#ifndef LORA_TILE_MAX_R
#define LORA_TILE_MAX_R 64  // staged-tile expand at every rank (measured: r = 64 expand 1302 -> 1254 us on config 5)
#endif

namespace lora {

namespace {

constexpr int kQD = 4;  // work-queue depth (items published ahead of the consumers)

template <int R>
struct SimtCfg {
  static constexpr int NWC = 8;          // consumer warps
  static constexpr int NCT = NWC * 32;   // consumer threads
  static constexpr int THREADS = NCT + 32;
  static constexpr int GR = kGroupRows;  // rows per group
  static constexpr int SMEM_BUDGET = 110 * 1024;  // per CTA, two CTAs per SM
  // shrink.  r = 64: 32 lanes along k, 2 k per lane.  r <= 32: 4 k per lane
  // (an x element widened once feeds 4 products; two k share an FFMA2), the
  // j-groups of a warp pre-reduced with shuffles (SMALL_K).
  static constexpr bool SMALL_K = R <= 32;
  // r <= 32 and r = 128: the shrink on mma.sync (shrink_item_mma); at r = 128
  // the eight 16-row M tiles are one per consumer warp (OWN_M: no cross-warp
  // reduction, no red buffer)
  static constexpr bool MMA = R <= 32 || R >= 128;
  static constexpr bool OWN_M = R >= 128;
  static constexpr int KL = SMALL_K ? R / 4 : 32;  // lanes along k
  static constexpr int KPL = R / KL;               // k per lane
  static constexpr int NJG = NCT / KL;             // j-groups
#ifndef LORA_SMALLR_A_STAGE
#define LORA_SMALLR_A_STAGE 32768
#endif
  // A bytes per stage: 16 KB; r = 16: 32 KB (two 8-j chunks per thread per stage halve the
  // per-stage overhead; measured Llama shrink 233 -> 224 us)
  static constexpr int SJ_MAX = (R == 16 ? LORA_SMALLR_A_STAGE : 16384) / (2 * R);
  static constexpr int A_STAGE = R * SJ_MAX * 2;
  // r <= 32 (MMA consumers): x rows padded by 16 bytes so the ldmatrix row
  // addresses of one 8x8 matrix fall in distinct banks
  static constexpr int X_PITCH = MMA ? SJ_MAX * 2 + 16 : SJ_MAX * 2;
  static constexpr int X_STAGE = GR * X_PITCH;
  static constexpr int S_STAGE = (A_STAGE + X_STAGE + 1023) / 1024 * 1024;
  static constexpr int RED_BYTES = OWN_M ? 0 : (MMA ? NWC : NJG) * GR * R * 4;
  static constexpr int NST_RAW = (SMEM_BUDGET - RED_BYTES) / S_STAGE;
  static constexpr int NST = NST_RAW > 8 ? 8 : (NST_RAW < 2 ? 2 : NST_RAW);
  // + at r <= 32 a resolver warp running kSRQ items ahead of the producer
  // (ShrinkRes ring; measured: Llama r = 16 shrink 253 -> 232 us, but at r = 64
  // the extra warp's register cap costs spills: 178 -> 239 us, so r = 64 keeps
  // the producer resolving its own items)
  static constexpr bool SHRINK_RESOLVER = R <= 32;
#ifndef LORA_RESOLVE_DEPTH
#define LORA_RESOLVE_DEPTH 1  // items resolved ahead (measured on Llama decode: 1 < 2 < 4 < 8 in step time)
#endif
  static constexpr int kSRQ = LORA_RESOLVE_DEPTH;
  static constexpr int SHRINK_THREADS = NCT + (SHRINK_RESOLVER ? 64 : 32);
  static constexpr int SHRINK_SMEM =
      1024 + NST * S_STAGE + RED_BYTES + 2 * NST * 8 + 3 * kQD * 8 + kQD * 16 + kSRQ * (96 + 16);
  // expand: CPT output columns per consumer thread (c = ct + i*NCT); at r <= 32
  // two columns share one FFMA2 (more B and y bytes per stage at small r)
#ifndef LORA_SMALLR_CPT
#define LORA_SMALLR_CPT 2
#endif
  // r <= 16: LORA_SMALLR_CPT columns per thread (4 = 32 KB B stages, staged-tile
  // expand only; measured slower: Llama expand 185 -> 238 us)
  static constexpr int CPT = R >= 64 ? 1 : (R <= 16 ? LORA_SMALLR_CPT : 2);
  // r = 128: two threads per column, one k half each (expand_stage_half), so a
  // stage holds NCT / 2 columns (32 KB of B) and two stages fit the 112 KB share
  static constexpr bool HALF = R >= 128;
  static constexpr bool LOOKAHEAD_OK = CPT <= 2 && !HALF;  // the look-ahead expand's y ring fits
  static constexpr int SC_MAX = HALF ? NCT / 2 : NCT * CPT;
  static constexpr int B_STAGE = SC_MAX * R * 2;
  static constexpr int V_BYTES = GR * R * 4;  // v rows of the group (fp32)
  static constexpr int E_STAGE = B_STAGE + 1024 * ((V_BYTES + 1023) / 1024);
  // bf16 y tiles (cp.async) in a ring of YD slots, fetched YD-1 stages ahead,
  // each with a 64-byte record {item, stage, row indices}
  // At r <= 32 (bf16 y) the stage's results are written back into its tile
  // and leave with coalesced 16-byte stores during the next stage: one extra
  // slot keeps the tile alive until then.
  static constexpr int YD = R >= 32 ? 2 : 4;
  static constexpr int YS = CPT > 1 ? YD + 1 : YD;
  static constexpr int Y_SLOT = GR * SC_MAX * 2;
  static constexpr int META = 128;  // StageRec
  // every byte of the 112 KB two-CTA share not used by the fixed parts goes to B stages
  // + a resolver warp kERQ items ahead of the producer (ExpandRec ring + barriers)
#ifndef LORA_ERQ
#define LORA_ERQ 2
#endif
  static constexpr int kERQ = LORA_ERQ;
  static constexpr int E_THREADS = NCT + 64;
  static constexpr int E_FIXED = 1024 + YS * (Y_SLOT + META) + 3 * kQD * 8 + kQD * 80 + kERQ * (80 + 16);
  static constexpr int NSTE_RAW = (112 * 1024 - E_FIXED) / (E_STAGE + 16);  // a stage + its two barriers
  static constexpr int NSTE = NSTE_RAW > 16 ? 16 : (NSTE_RAW < 2 ? 2 : NSTE_RAW);
  static constexpr int EXPAND_SMEM =
      1024 + NSTE * E_STAGE + YS * (Y_SLOT + META) + 2 * NSTE * 8 + 3 * kQD * 8 + kQD * 80 + kERQ * (80 + 16);
  // the look-ahead pops items the producer has published only if YD - 1 <= NSTE
  // The producer publishes an item after issuing its first stage; at stage s
  // (after releasing it) the consumers' look-ahead takes the item holding
  // stage s+YD, whose first stage needs stage s+YD-NSTE released: YD <= NSTE.
  static_assert(!LOOKAHEAD_OK || YD <= NSTE, "y look-ahead deeper than the B pipeline");
  static_assert(S_STAGE % 1024 == 0 && E_STAGE % 1024 == 0, "stage alignment");
  // staged-tile expand (r <= 16, simt_expand_tile_kernel): the y tile of a
  // stage travels with its B rows and v rows in one stage buffer, loaded by
  // the producer's bulk copies (one per group row), so y is prefetched as
  // deep as B.  Stage = B | v (1 KB aligned) | y tile [GR][SC_MAX] bf16.
  static constexpr int TV_OFF = B_STAGE;
  static constexpr int TY_OFF = B_STAGE + 1024 * ((V_BYTES + 1023) / 1024);
  static constexpr int T_STAGE = TY_OFF + Y_SLOT;
  // + a resolver warp running kRQ items ahead of the producer (ring of
  // resolved ExpandRec records with full/empty barriers)
  static constexpr int TILE_THREADS = NCT + 64;
  static constexpr int kRQ = LORA_RESOLVE_DEPTH;
  static constexpr int T_FIXED = 1024 + 2 * 16 * 8 + 3 * kQD * 8 + kQD * 80 + kRQ * (80 + 16);
  static constexpr int TNST_RAW = (112 * 1024 - T_FIXED) / T_STAGE;
  static constexpr int TNST = TNST_RAW > 8 ? 8 : (TNST_RAW < 2 ? 2 : TNST_RAW);
  static constexpr int TILE_SMEM = 1024 + TNST * T_STAGE + 2 * TNST * 8 + 3 * kQD * 8 + kQD * 80 + kRQ * (80 + 16);
  static_assert(T_STAGE % 1024 == 0 && TILE_SMEM <= 112 * 1024, "tile stage layout");
  static_assert(SHRINK_SMEM <= 112 * 1024 && (!LOOKAHEAD_OK || EXPAND_SMEM <= 112 * 1024), "two CTAs per SM");
  static_assert(R != 64 || NSTE == 3, "r = 64 expand keeps three 34 KB stages");
};

LORA_DEVINL uint8_t* align1024(uint8_t* p) {
  const uint32_t a = smem_u32(p);
  return p + (((a + 1023u) & ~1023u) - a);
}



LORA_DEVINL void unpack8(const uint4& w, float* f) {
  f[0] = bf16lo(w.x); f[1] = bf16hi(w.x);
  f[2] = bf16lo(w.y); f[3] = bf16hi(w.y);
  f[4] = bf16lo(w.z); f[5] = bf16hi(w.z);
  f[6] = bf16lo(w.w); f[7] = bf16hi(w.w);
}

// packed fp32x2 FMA (FFMA2, sm_100): two products per instruction
LORA_DEVINL float2 dot8_acc2(float2 acc, const float* a, const float* b) {
#pragma unroll
  for (int i = 0; i < 8; i += 2) acc = __ffma2_rn(make_float2(a[i], a[i + 1]), make_float2(b[i], b[i + 1]), acc);
  return acc;
}

// ---------------------------------------------------------------------------
// shrink: item = (task, group); v[row][k] = sum_j x[perm[row]][j] A_u[j][k]
// ---------------------------------------------------------------------------
// K-split (small batches, see simt_shrink_kernel): the item covers k-chunk kc
// (KI of h_in, n_st stages) and writes a partial sum into region kc; the last
// of the group's n_kc items to arrive sums the partials in kc order (the same
// order whichever CTA is last, so the result is deterministic) into region 0.
struct SplitCtx {
  int n_st;               // stages of this item
  int kc, n_kc;           // chunk of this item, chunks of the group (n_kc == 1: whole K, no partials)
  long long kc_stride;    // floats between two kc regions (max_rows * R)
  unsigned int* cnt;      // arrivals of the group's items
  int* s_last;            // smem flag
};

template <int NCT>
LORA_DEVINL void split_finish(float* vbase, int n, const SplitCtx& sc) {
  __threadfence();                 // this thread's partial writes, before the arrival
  named_bar_sync(1, NCT);
  if (threadIdx.x == 0) {
    const unsigned int old = atomicAdd(sc.cnt, 1u);
    const int last = old == (unsigned int)(sc.n_kc - 1);
    if (last) {
      *sc.cnt = 0u;                // self-resetting for the next launch
      __threadfence();
    }
    *sc.s_last = last;
  }
  named_bar_sync(1, NCT);
  if (*sc.s_last) {
    for (int idx = threadIdx.x; idx < n; idx += NCT) {
      float s = 0.f;
      for (int kc = 0; kc < sc.n_kc; ++kc) s += __ldcg(vbase + kc * sc.kc_stride + idx);
      vbase[idx] = s;
    }
  }
}

template <int R, int NR>
LORA_DEVINL void shrink_item(uint8_t* smem, uint64_t* full, uint64_t* empty, float* red, int& stage,
                             uint32_t& phase, const SlotTask& t, const int4 g, float* vpart_base,
                             int lane, const SplitCtx& sc) {
  using C = SimtCfg<R>;
  const int ct = threadIdx.x;
  const int kl = ct % C::KL, jg = ct / C::KL;
  const int n_st = sc.n_st;
  const int nchunk = t.SJ >> 3;  // 16-byte chunks along j per stage
  float2 acc[C::KPL][NR];
#pragma unroll
  for (int kk = 0; kk < C::KPL; ++kk)
#pragma unroll
    for (int r = 0; r < NR; ++r) acc[kk][r] = make_float2(0.f, 0.f);

  for (int st = 0; st < n_st; ++st) {
    mbar_wait(&full[stage], phase);
    const uint32_t a_s = smem_u32(smem + stage * C::S_STAGE);
    const uint32_t x_s = a_s + C::A_STAGE;
    for (int c = jg; c < nchunk; c += C::NJG) {
      const int tile = c >> 3, q = c & 7;
      float w[C::KPL][8];
#pragma unroll
      for (int kk = 0; kk < C::KPL; ++kk) {
        const int k = kl + kk * 32;
        unpack8(lds128(a_s + tile * (R * 128) + k * 128 + ((q ^ (k & 7)) << 4)), w[kk]);
      }
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        float xf[8];
        unpack8(lds128(x_s + r * (t.SJ * 2) + (c << 4)), xf);
#pragma unroll
        for (int kk = 0; kk < C::KPL; ++kk) acc[kk][r] = dot8_acc2(acc[kk][r], xf, w[kk]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[stage]);
    if (++stage == C::NST) {
      stage = 0;
      phase ^= 1;
    }
  }

  // deterministic cross-thread reduction over the NJG j-groups
  named_bar_sync(1, C::NCT);
#pragma unroll
  for (int kk = 0; kk < C::KPL; ++kk)
#pragma unroll
    for (int r = 0; r < NR; ++r) red[(jg * NR + r) * R + kl + kk * 32] = acc[kk][r].x + acc[kk][r].y;
  named_bar_sync(1, C::NCT);
  float* vp = vpart_base + (long long)g.x * R;
  for (int idx = ct; idx < NR * R; idx += C::NCT) {
    float s = 0.f;
#pragma unroll 4
    for (int q = 0; q < C::NJG; ++q) s += red[q * NR * R + idx];
    vp[sc.kc * sc.kc_stride + idx] = s;
  }
  if (sc.n_kc > 1) split_finish<C::NCT>(vp, NR * R, sc);
}

// ---------------------------------------------------------------------------
// r <= 32: the shrink on the legacy tensor path (mma.sync m16n8k16 bf16 ->
// fp32, fed by ldmatrix from the pre-swizzled stages).  At small r the
// CUDA-core FMA formulation was instruction-bound (ncu on Llama decode: 60 %
// issue active, math-pipe throttle, bf16 unpacking per weight element); one
// MMA covers 16 rank values x 8 group rows x 16 j with ~3 instructions per
// 512 B of weights (measured: Llama decode shrink 227 -> 195 us).
// ---------------------------------------------------------------------------
LORA_DEVINL void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
LORA_DEVINL void ldsm_x2(uint32_t addr, uint32_t& r0, uint32_t& r1) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];" : "=r"(r0), "=r"(r1) : "r"(addr));
}
// D[16 x 8] += A[16 x 16] . B[16 x 8]  (A row-major, B "col": rows of B^T)
LORA_DEVINL void mma16816(float* d, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
               "{%0,%1,%2,%3};"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
               : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// Shrink item, r <= 32: D[k x n] += A_u^T[k x 16 j] . x^T[16 j x n] per
// 16-j step, M = 16 rank values (r = 32: two M tiles; r = 8: rows 8-15
// duplicate 0-7, ignored), N = the group's 8 rows (rows >= NR hold stale smem:
// their columns are never read), steps dealt round-robin to the 8 consumer
// warps; per-warp partials reduced through shared memory as before.
template <int R>
LORA_DEVINL void shrink_item_mma(uint8_t* smem, uint64_t* full, uint64_t* empty, float* red, int& stage,
                                 uint32_t& phase, const SlotTask& t, const int4 g, float* vpart_base, int lane,
                                 const SplitCtx& sc) {
  using C = SimtCfg<R>;
  constexpr int MT = (R + 15) / 16;
  const int warp = threadIdx.x >> 5;
  const int nsteps = t.SJ >> 4;  // 16-j steps per stage
  float acc[MT][4];
#pragma unroll
  for (int m = 0; m < MT; ++m) acc[m][0] = acc[m][1] = acc[m][2] = acc[m][3] = 0.f;
  // this lane's ldmatrix rows: A (weights) row k of matrix (lane >> 3), x row lane & 7
  const int ka = (lane & 7) + ((lane >> 3) & 1) * 8;  // 0..15
  const int ca = lane >> 4;                           // chunk offset 0 / 1
  const int xn = lane & 7, xc = (lane >> 3) & 1;
  if constexpr (C::OWN_M) {
    // r = 128: warp w computes rank rows 16 w .. 16 w + 15 over every j step
    static_assert(MT == C::NWC, "one M tile per consumer warp");
    float d[4] = {0.f, 0.f, 0.f, 0.f};
    const int k = warp * 16 + ka;
    for (int st = 0; st < sc.n_st; ++st) {
      mbar_wait(&full[stage], phase);
      const uint32_t a_s = smem_u32(smem + stage * C::S_STAGE);
      const uint32_t x_s = a_s + C::A_STAGE;
      for (int q = 0; q < nsteps; ++q) {
        const int j0 = q << 4;
        const int tile = j0 >> 6, ch = ((j0 & 63) >> 3) + ca;
        uint32_t b0, b1, a0, a1, a2, a3;
        ldsm_x2(x_s + xn * C::X_PITCH + ((j0 + xc * 8) << 1), b0, b1);
        ldsm_x4(a_s + tile * (R * 128) + k * 128 + ((ch ^ (k & 7)) << 4), a0, a1, a2, a3);
        mma16816(d, a0, a1, a2, a3, b0, b1);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == C::NST) {
        stage = 0;
        phase ^= 1;
      }
    }
    // D fragment: d[0..1] -> k = 16 w + lane/4, rows 2 (lane % 4) + {0, 1}; d[2..3] -> k + 8
    float* vp = vpart_base + (long long)g.x * R;
    float* vk = vp + sc.kc * sc.kc_stride + warp * 16 + (lane >> 2);
    const int n0 = (lane & 3) * 2;
    if (n0 < g.y) {
      vk[n0 * R] = d[0];
      vk[n0 * R + 8] = d[2];
    }
    if (n0 + 1 < g.y) {
      vk[(n0 + 1) * R] = d[1];
      vk[(n0 + 1) * R + 8] = d[3];
    }
    if (sc.n_kc > 1) split_finish<C::NCT>(vp, g.y * R, sc);
    return;
  }
  for (int st = 0; st < sc.n_st; ++st) {
    mbar_wait(&full[stage], phase);
    const uint32_t a_s = smem_u32(smem + stage * C::S_STAGE);
    const uint32_t x_s = a_s + C::A_STAGE;
    for (int q = warp; q < nsteps; q += C::NWC) {
      const int j0 = q << 4;
      const int tile = j0 >> 6, c0 = (j0 & 63) >> 3;
      uint32_t b0, b1;
      ldsm_x2(x_s + xn * C::X_PITCH + ((j0 + xc * 8) << 1), b0, b1);
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        const int k = R >= 16 ? m * 16 + ka : (ka & 7);
        const int ch = c0 + ca;
        uint32_t a0, a1, a2, a3;
        ldsm_x4(a_s + tile * (R * 128) + k * 128 + ((ch ^ (k & 7)) << 4), a0, a1, a2, a3);
        mma16816(acc[m], a0, a1, a2, a3, b0, b1);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[stage]);
    if (++stage == C::NST) {
      stage = 0;
      phase ^= 1;
    }
  }
  // D fragment: acc[m][0..1] -> k = m*16 + lane/4, rows 2*(lane%4) + {0,1}; [2..3] -> k + 8
  named_bar_sync(1, C::NCT);
  float* rw = red + warp * (C::GR * R);
  const int kq = lane >> 2, nq = (lane & 3) * 2;
#pragma unroll
  for (int m = 0; m < MT; ++m) {
    rw[(nq + 0) * R + m * 16 + kq] = acc[m][0];
    rw[(nq + 1) * R + m * 16 + kq] = acc[m][1];
    if (R >= 16) {
      rw[(nq + 0) * R + m * 16 + kq + 8] = acc[m][2];
      rw[(nq + 1) * R + m * 16 + kq + 8] = acc[m][3];
    }
  }
  named_bar_sync(1, C::NCT);
  float* vp = vpart_base + (long long)g.x * R;
  const int n_out = g.y * R;
  for (int idx = threadIdx.x; idx < n_out; idx += C::NCT) {
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < C::NWC; ++w) s += red[w * (C::GR * R) + idx];
    vp[sc.kc * sc.kc_stride + idx] = s;
  }
  if (sc.n_kc > 1) split_finish<C::NCT>(vp, n_out, sc);
}

template <int R, int NR>
LORA_DEVINL void shrink_dispatch(uint8_t* smem, uint64_t* full, uint64_t* empty, float* red, int& stage,
                                 uint32_t& phase, const SlotTask& t, const int4 g, float* vpart_base, int lane,
                                 const SplitCtx& sc) {
  shrink_item<R, NR>(smem, full, empty, red, stage, phase, t, g, vpart_base, lane, sc);
}

// a shrink item as resolved by the resolver warp: group and x row offsets
struct ShrinkRes {
  long long it;  // -1: end of the stream
  int ti, kc;    // task, k-chunk (K-split; 0 otherwise)
  int4 g;
  long long xrow[kGroupRows];
};
static_assert(sizeof(ShrinkRes) == 96, "resolved record size");

template <int R, bool REMOTE>
__global__ void __launch_bounds__(SimtCfg<R>::SHRINK_THREADS, 2)
    simt_shrink_kernel(const __grid_constant__ MultiArgs args, const PlanDev pd) {
  using C = SimtCfg<R>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  float* red = reinterpret_cast<float*>(smem + C::NST * C::S_STAGE);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::NST * C::S_STAGE + C::RED_BYTES);
  uint64_t* empty = full + C::NST;
  WorkQueue<kQD> wq{reinterpret_cast<long long*>(empty + C::NST), empty + C::NST + kQD, empty + C::NST + 2 * kQD};
  int4* gq = reinterpret_cast<int4*>(empty + C::NST + 3 * kQD);  // [kQD] group of each queued item
  ShrinkRes* rres = reinterpret_cast<ShrinkRes*>(gq + kQD);        // [kSRQ] resolved items
  uint64_t* rfull = reinterpret_cast<uint64_t*>(rres + C::kSRQ);   // [kSRQ]
  uint64_t* rempty = rfull + C::kSRQ;                              // [kSRQ]

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], C::NWC);
    }
    for (int s = 0; s < C::kSRQ; ++s) {
      mbar_init(&rfull[s], 1);
      mbar_init(&rempty[s], 1);
    }
    wq.init(C::NWC);
    fence_mbar_init();
  }
  __syncthreads();
  pdl_wait();               // the plan (segmenter) is complete
  pdl_launch_dependents();  // the expand may launch as SMs free up

  const int n_groups = pd.counts[kCntGroups];
  // Small batches have few (task, group) items, and one item streams a whole
  // unit's A through one CTA (1.8 MB for Mixtral down, ~130 us): with fewer
  // than simt_split_items items the groups' h_in is split into the slots' n_kc
  // chunks of KI (items = groups x sum n_kc), partial sums + last-arriver sum.
  const bool split = (long long)n_groups * args.n_tasks < args.simt_split_items;
  const long long n_items = (long long)n_groups * (split ? args.total_kc : args.n_tasks);
  const int warp = warp_id(), lane = lane_id();
  __shared__ int s_last;
  // item -> (task, k-chunk, group index)
  auto decode = [&](long long it, int& ti, int& kc, int& gi) {
    if (split) {
      const int q = (int)(it / n_groups);
      gi = (int)(it - (long long)q * n_groups);
      ti = find_task_kc(args, q);
      kc = q - args.t[ti].kc_base;
      return;
    }
    // task-major: a slot's groups back to back, so the groups of one unit
    // (segments > 8 rows) stream that unit's A at about the same time (L2
    // hits).  Interleaving the slots that share x group by group measured
    // slower (Llama decode shrink 229 -> 248 us by h_in runs, 286 us by x runs).
    const int q = (int)(it / n_groups);
    gi = (int)(it - (long long)q * n_groups);
    ti = q;
    kc = 0;
  };

  // claim the next item and resolve its group and x rows: x row r of the group
  // is t.x + xrow[r] (REMOTE: xrow[r] is relative to t.x, pointing into a
  // source's registered x)
  auto resolve = [&](long long& it, int& ti, int& kc, int4& g, long long* xrow) {
    it = (long long)atomicAdd(pd.wctr + kWqSimtShrink, 1ull);
    if (it >= n_items) it = -1;
    int gi = 0;
    ti = 0;
    kc = 0;
    if (it >= 0) decode(it, ti, kc, gi);
    g = it < 0 ? make_int4(0, 0, 0, 0) : pd.groups[gi];
    const SlotTask& t = args.t[ti];
#pragma unroll
    for (int r = 0; r < C::GR; ++r) {
      if constexpr (REMOTE)
        xrow[r] = r < g.y ? x_row<true>(args, ti, pd.perm[g.x + r]) - t.x : 0;
      else
        xrow[r] = r < g.y ? (long long)pd.perm[g.x + r] * t.h_in : 0;
    }
  };

  if (C::SHRINK_RESOLVER && warp == C::NWC + 1) {
    // ===================== resolver: up to kSRQ items ahead of the producer =====================
    if (lane == 0) {
      QueuePos rp;
      for (;;) {
        long long it;
        int ti, kc;
        int4 g;
        long long xrow[C::GR];
        resolve(it, ti, kc, g, xrow);
        mbar_wait(&rempty[rp.slot], rp.phase ^ 1);
        ShrinkRes& q = rres[rp.slot];
        q.it = it;
        q.ti = ti;
        q.kc = kc;
        q.g = g;
#pragma unroll
        for (int r = 0; r < C::GR; ++r) q.xrow[r] = xrow[r];
        mbar_arrive(&rfull[rp.slot]);
        rp.advance(C::kSRQ);
        if (it < 0) break;
      }
    }
  } else if (warp == C::NWC) {
    // ===================== producer =====================
    if (lane == 0) {
      const uint64_t pol = (args.tc_flags & 16) ? policy_evict_last() : policy_evict_first();  // A (bit 4)
      int stage = 0;
      uint32_t phase = 0;
      QueuePos qp, rp;
      for (;;) {
        long long it;
        int ti, kc;
        int4 g;
        long long xrow[C::GR];
        if constexpr (C::SHRINK_RESOLVER) {
          mbar_wait(&rfull[rp.slot], rp.phase);
          const ShrinkRes& q = rres[rp.slot];
          it = q.it;
          ti = q.ti;
          kc = q.kc;
          g = q.g;
#pragma unroll
          for (int r = 0; r < C::GR; ++r) xrow[r] = q.xrow[r];
          mbar_arrive(&rempty[rp.slot]);
          rp.advance(C::kSRQ);
        } else {
          resolve(it, ti, kc, g, xrow);
        }
        // the item and its group go to the consumers through the queue
        mbar_wait(&wq.empty[qp.slot], qp.phase ^ 1);
        wq.item[qp.slot] = it;
        gq[qp.slot] = g;
        mbar_arrive(&wq.full[qp.slot]);
        qp.advance(kQD);
        if (it < 0) break;
        const SlotTask& t = args.t[ti];
        const long long unit = store_unit(g.z, t.E, args.pl, args.cache);
        const long long j0 = split ? (long long)kc * t.KI : 0;   // first j of this item
        const uint16_t* abase = t.At + (unit * (long long)t.h_in + j0) * R;
        const int n_st = (split ? t.KI : t.h_in) / t.SJ;
        const uint32_t a_bytes = (uint32_t)R * t.SJ * 2, x_bytes = (uint32_t)t.SJ * 2;
        for (int st = 0; st < n_st; ++st) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sA = smem + stage * C::S_STAGE;
          uint8_t* sX = sA + C::A_STAGE;
          mbar_arrive_expect_tx(&full[stage], a_bytes + x_bytes * g.y);
          bulk_g2s_hint(sA, abase + (long long)st * t.SJ * R, a_bytes, &full[stage], pol);
          const long long jofs = j0 + (long long)st * t.SJ;
#pragma unroll
          for (int r = 0; r < C::GR; ++r)
            if (r < g.y)
              bulk_g2s(sX + r * (C::MMA ? (uint32_t)C::X_PITCH : x_bytes), t.x + xrow[r] + jofs, x_bytes,
                       &full[stage]);
          if (++stage == C::NST) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else {
    // ===================== consumers =====================
    int stage = 0;
    uint32_t phase = 0;
    QueuePos qp;
    for (;;) {
      mbar_wait(&wq.full[qp.slot], qp.phase);
      const long long it = wq.item[qp.slot];
      const int4 g = gq[qp.slot];
      __syncwarp();
      if (lane == 0) mbar_arrive(&wq.empty[qp.slot]);
      qp.advance(kQD);
      if (it < 0) break;
      int ti, kc, gi;
      decode(it, ti, kc, gi);
      const SlotTask& t = args.t[ti];
      float* vb = pd.vpart + t.vpart_off;
      SplitCtx sc;
      sc.n_st = (split ? t.KI : t.h_in) / t.SJ;
      sc.kc = kc;
      sc.n_kc = split ? t.n_kc : 1;
      sc.kc_stride = (long long)pd.max_rows * R;
      sc.cnt = pd.gcnt + (long long)ti * pd.max_rows + gi;
      sc.s_last = &s_last;
      if constexpr (C::MMA) {  // MMA consumers: one code path for any group size
        shrink_item_mma<R>(smem, full, empty, red, stage, phase, t, g, vb, lane, sc);
      } else {
      switch (g.y) {
        case 1: shrink_dispatch<R, 1>(smem, full, empty, red, stage, phase, t, g, vb, lane, sc); break;
        case 2: shrink_dispatch<R, 2>(smem, full, empty, red, stage, phase, t, g, vb, lane, sc); break;
        case 3: shrink_dispatch<R, 3>(smem, full, empty, red, stage, phase, t, g, vb, lane, sc); break;
        case 4: shrink_dispatch<R, 4>(smem, full, empty, red, stage, phase, t, g, vb, lane, sc); break;
        case 5: shrink_dispatch<R, 5>(smem, full, empty, red, stage, phase, t, g, vb, lane, sc); break;
        case 6: shrink_dispatch<R, 6>(smem, full, empty, red, stage, phase, t, g, vb, lane, sc); break;
        case 7: shrink_dispatch<R, 7>(smem, full, empty, red, stage, phase, t, g, vb, lane, sc); break;
        default: shrink_dispatch<R, 8>(smem, full, empty, red, stage, phase, t, g, vb, lane, sc); break;
      }
      }
    }
  }
  __syncthreads();
  wq_finish(pd.wctr + kWqSimtShrink, pd.wdone + kWqSimtShrink);
}

// ---------------------------------------------------------------------------
// expand + scale + scatter-accumulate
// ---------------------------------------------------------------------------
// Consumer-side walk over this CTA's (item, stage) sequence.
struct ExpandPos {
  long long it;
  int st, n_st;
  int sc;             // B rows (columns) in this stage
  int rows;
  int h_out;
  long long c0;       // first column of this stage
  void* y;
  const int32_t* perm_rows;
  float s_a;
  char* prow[kGroupRows];  // push modes: the origin row of each group row in its source's y
};

// y[row][c] for one (row, column) result d (already scaled).  Output mode M
// (compile time): 0 bf16 accumulate with the old value from the stage's smem
// y tile, 1 fp32 store and 2 bf16 store (sharded delta), 3 fp32 accumulate.
// 4 / 5: push -- bf16 / fp32 delta added into the origin row of the source's
// registered y (red.add over NVLink, sharded owner; p.prow).
enum { kOutBf16Acc = 0, kOutF32Store = 1, kOutBf16Store = 2, kOutF32Acc = 3, kOutBf16Push = 4, kOutF32Push = 5 };
constexpr bool out_push(int m) { return m == kOutBf16Push || m == kOutF32Push; }
constexpr bool out_bf16_tile(int m) { return m == kOutBf16Acc || m == kOutBf16Store || m == kOutBf16Push; }
template <int M, bool TILE>
LORA_DEVINL void expand_out(const ExpandPos& p, uint32_t rows, int r, int col, float d, uint32_t ytile, int pitch) {
  if constexpr (TILE) {
    // result back into the stage's smem tile; the tile leaves with bulk stores
    const uint32_t a = ytile + r * pitch + col * 2;
    uint16_t v;
    if constexpr (M == kOutBf16Acc) {
      uint16_t old;
      asm volatile("ld.shared.u16 %0, [%1];" : "=h"(old) : "r"(a));
      v = f32_to_bf16_rne(bf16_to_f32(old) + d);
    } else {
      v = f32_to_bf16_rne(d);
    }
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"(v) : "memory");
    return;
  }
  if constexpr (M == kOutF32Push) {
    red_add_f32(p.prow[r] + (p.c0 + col) * 4, d);
    return;
  }
  int row;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(row) : "r"(rows + r * 4));
  const long long o = (long long)row * p.h_out + p.c0 + col;
  if constexpr (M == kOutF32Store) {
    reinterpret_cast<float*>(p.y)[o] = d;
  } else if constexpr (M == kOutBf16Store) {
    reinterpret_cast<uint16_t*>(p.y)[o] = f32_to_bf16_rne(d);
  } else if constexpr (M == kOutF32Acc) {
    float* yp = reinterpret_cast<float*>(p.y) + o;
    *yp = *yp + d;
  } else {
    uint16_t old;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(old) : "r"(ytile + r * pitch + col * 2));
    reinterpret_cast<uint16_t*>(p.y)[o] = f32_to_bf16_rne(bf16_to_f32(old) + d);
  }
}

// r = 64: one column per thread, FFMA2 over pairs of k (two accumulators for ILP)
template <int R, int NR, int M>
LORA_DEVINL void expand_stage1(uint32_t b_s, uint32_t v_s, int cr, const ExpandPos& p, uint32_t rows,
                               uint32_t ytile, int pitch) {
  float2 acc[NR][2];
#pragma unroll
  for (int r = 0; r < NR; ++r) acc[r][0] = acc[r][1] = make_float2(0.f, 0.f);
#pragma unroll
  for (int ch = 0; ch < R / 8; ++ch) {
    const uint4 w = lds128(b_s + cr * (R * 2) + (swz_row_chunk(cr, ch, R * 2) << 4));
    const float2 b0 = make_float2(bf16lo(w.x), bf16hi(w.x)), b1 = make_float2(bf16lo(w.y), bf16hi(w.y));
    const float2 b2 = make_float2(bf16lo(w.z), bf16hi(w.z)), b3 = make_float2(bf16lo(w.w), bf16hi(w.w));
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const float4 v0 = lds128f(v_s + (r * R + ch * 8) * 4);
      const float4 v1 = lds128f(v_s + (r * R + ch * 8 + 4) * 4);
      float2 a = acc[r][ch & 1];
      a = __ffma2_rn(make_float2(v0.x, v0.y), b0, a);
      a = __ffma2_rn(make_float2(v0.z, v0.w), b1, a);
      a = __ffma2_rn(make_float2(v1.x, v1.y), b2, a);
      a = __ffma2_rn(make_float2(v1.z, v1.w), b3, a);
      acc[r][ch & 1] = a;
    }
  }
  if constexpr (M == kOutBf16Push) {
    // column pairs (cr, cr + 1) meet in the even lane: one 4-byte red per pair
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const float d = p.s_a * ((acc[r][0].x + acc[r][0].y) + (acc[r][1].x + acc[r][1].y));
      const float dn = __shfl_xor_sync(0xffffffffu, d, 1);
      if (!(cr & 1) && cr < p.sc) red_add_bf16x2(p.prow[r] + (p.c0 + cr) * 2, pack_bf16x2_rn(d, dn));
    }
    return;
  }
  if (cr >= p.sc) return;
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    const float d = p.s_a * ((acc[r][0].x + acc[r][0].y) + (acc[r][1].x + acc[r][1].y));
    expand_out<M, false>(p, rows, r, cr, d, ytile, pitch);
  }
}

// r = 128: two threads per column (ct = 2 c + h), thread h taking the
// interleaved 16-byte chunks 2 i + h of the column's Bt row (with the 256-byte
// row swizzle the 8 threads of a quarter warp hit 8 distinct bank groups);
// the two k halves meet in one shuffle before the scale.
template <int R, int NR, int M>
LORA_DEVINL void expand_stage_half(uint32_t b_s, uint32_t v_s, int ct, const ExpandPos& p, uint32_t rows,
                                   uint32_t ytile, int pitch) {
  const int cr = ct >> 1, h = ct & 1;
  float2 acc[NR][2];
#pragma unroll
  for (int r = 0; r < NR; ++r) acc[r][0] = acc[r][1] = make_float2(0.f, 0.f);
#pragma unroll
  for (int i = 0; i < R / 16; ++i) {
    const int ch = 2 * i + h;
    const uint4 w = lds128(b_s + cr * (R * 2) + (swz_row_chunk(cr, ch, R * 2) << 4));
    const float2 b0 = make_float2(bf16lo(w.x), bf16hi(w.x)), b1 = make_float2(bf16lo(w.y), bf16hi(w.y));
    const float2 b2 = make_float2(bf16lo(w.z), bf16hi(w.z)), b3 = make_float2(bf16lo(w.w), bf16hi(w.w));
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const float4 v0 = lds128f(v_s + (r * R + ch * 8) * 4);
      const float4 v1 = lds128f(v_s + (r * R + ch * 8 + 4) * 4);
      float2 a = acc[r][i & 1];
      a = __ffma2_rn(make_float2(v0.x, v0.y), b0, a);
      a = __ffma2_rn(make_float2(v0.z, v0.w), b1, a);
      a = __ffma2_rn(make_float2(v1.x, v1.y), b2, a);
      a = __ffma2_rn(make_float2(v1.z, v1.w), b3, a);
      acc[r][i & 1] = a;
    }
  }
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    float part = (acc[r][0].x + acc[r][0].y) + (acc[r][1].x + acc[r][1].y);
    part += __shfl_xor_sync(0xffffffffu, part, 1);
    const float d = p.s_a * part;
    if constexpr (M == kOutBf16Push) {
      // columns (cr, cr + 1) meet in lane 4 i: one 4-byte red per pair
      const float dn = __shfl_xor_sync(0xffffffffu, d, 2);
      if (!(ct & 3) && cr < p.sc) red_add_bf16x2(p.prow[r] + (p.c0 + cr) * 2, pack_bf16x2_rn(d, dn));
    } else {
      if (h == 0 && cr < p.sc) expand_out<M, false>(p, rows, r, cr, d, ytile, pitch);
    }
  }
}

// r <= 32: CPT columns per thread (c = ct + i*NCT), FFMA2 over pairs of
// columns.  (Adjacent pairs (2 ct, 2 ct + 1) with one 32-bit smem
// read-modify-write of the y tile per row measured equal on Llama decode.)  The B chunk of a column pair is widened to fp32 once and reused
// for every row of the group.
template <int R, int NR, int CPT, int NCT, int M>
LORA_DEVINL void expand_stage_pairs(uint32_t b_s, uint32_t v_s, int ct, const ExpandPos& p, uint32_t rows,
                                    uint32_t ytile, int pitch) {
  constexpr int NP = CPT / 2;
  constexpr bool TILE = out_bf16_tile(M);
  float2 acc[NP][NR];
#pragma unroll
  for (int q = 0; q < NP; ++q)
#pragma unroll
    for (int r = 0; r < NR; ++r) acc[q][r] = make_float2(0.f, 0.f);
#pragma unroll
  for (int ch = 0; ch < R / 8; ++ch) {
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      const int ca = ct + 2 * q * NCT, cb = ca + NCT;
      const uint4 wa = lds128(b_s + ca * (R * 2) + (swz_row_chunk(ca, ch, R * 2) << 4));
      const uint4 wb = lds128(b_s + cb * (R * 2) + (swz_row_chunk(cb, ch, R * 2) << 4));
      const uint32_t a[4] = {wa.x, wa.y, wa.z, wa.w}, b[4] = {wb.x, wb.y, wb.z, wb.w};
      float2 bb[8];  // bb[k] = (B[ca][k], B[cb][k]) for the 8 k of this chunk
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        bb[2 * j] = make_float2(bf16lo(a[j]), bf16lo(b[j]));
        bb[2 * j + 1] = make_float2(bf16hi(a[j]), bf16hi(b[j]));
      }
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        const float4 v0 = lds128f(v_s + (r * R + ch * 8) * 4);
        const float4 v1 = lds128f(v_s + (r * R + ch * 8 + 4) * 4);
        float2 s = acc[q][r];
        s = __ffma2_rn(make_float2(v0.x, v0.x), bb[0], s);
        s = __ffma2_rn(make_float2(v0.y, v0.y), bb[1], s);
        s = __ffma2_rn(make_float2(v0.z, v0.z), bb[2], s);
        s = __ffma2_rn(make_float2(v0.w, v0.w), bb[3], s);
        s = __ffma2_rn(make_float2(v1.x, v1.x), bb[4], s);
        s = __ffma2_rn(make_float2(v1.y, v1.y), bb[5], s);
        s = __ffma2_rn(make_float2(v1.z, v1.z), bb[6], s);
        s = __ffma2_rn(make_float2(v1.w, v1.w), bb[7], s);
        acc[q][r] = s;
      }
    }
  }
#pragma unroll
  for (int q = 0; q < NP; ++q) {
    const int c0 = ct + 2 * q * NCT, c1 = c0 + NCT;
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      if (c0 < p.sc) expand_out<M, TILE>(p, rows, r, c0, p.s_a * acc[q][r].x, ytile, pitch);
      if (c1 < p.sc) expand_out<M, TILE>(p, rows, r, c1, p.s_a * acc[q][r].y, ytile, pitch);
    }
  }
}

template <int R, int NR, int M>
LORA_DEVINL void expand_stage(uint32_t b_s, uint32_t v_s, int ct, const ExpandPos& p, uint32_t rows,
                              uint32_t ytile, int pitch) {
  using C = SimtCfg<R>;
  if constexpr (C::HALF)
    expand_stage_half<R, NR, M>(b_s, v_s, ct, p, rows, ytile, pitch);
  else if constexpr (C::CPT == 1)
    expand_stage1<R, NR, M>(b_s, v_s, ct, p, rows, ytile, pitch);
  else
    expand_stage_pairs<R, NR, C::CPT, C::NCT, M>(b_s, v_s, ct, p, rows, ytile, pitch);
}

// One expand work item as resolved by the producer lane (work-queue entry):
// everything the consumers need, so they never wait on a dependent global
// load for an item.
struct ExpandRec {
  long long it;  // -1: end of the stream
  int task, ci;
  int4 g;        // group {row_begin, nrows, key, seg}
  float s_a;
  int pad;
  int rows[kGroupRows];
};
static_assert(sizeof(ExpandRec) <= 80, "record size");

// One stage of the look-ahead ring (smem), written when its y tile is issued.
struct StageRec {
  long long it;  // item (>= n_items: end)
  long long c0;  // first column
  void* y;
  int st, sc, rows, h_out;
  float s_a;
  int pad;
  int row[kGroupRows];
};
static_assert(sizeof(StageRec) <= 128, "stage record size");

// Expand resolver warp (lane 0): claims items and resolves their group, row
// indices and scale up to nrq items ahead of the copy-issuing producer, so
// the producer never waits on an item's dependent claim -> group -> row loads.
__device__ __forceinline__ void expand_resolver(const MultiArgs& args, const PlanDev& pd, int n_groups,
                                                long long n_items, ExpandRec* rres, uint64_t* rfull,
                                                uint64_t* rempty, int nrq) {
  unsigned long long* ctr = pd.wctr + kWqSimtExpand;
  QueuePos rp;
  for (;;) {
    long long it = (long long)atomicAdd(ctr, 1ull);
    if (it >= n_items) it = -1;
    int ti = 0, ci = 0;
    int4 g = make_int4(0, 0, 0, 0);
    float s_a = 0.f;
    int rows[kGroupRows];
#pragma unroll
    for (int r = 0; r < kGroupRows; ++r) rows[r] = 0;
    if (it >= 0) {
      const int cig = (int)(it / n_groups), gi = (int)(it - (long long)cig * n_groups);
      ti = find_task_ci(args, cig);
      const SlotTask& t = args.t[ti];
      ci = cig - t.ci_base;
      g = pd.groups[gi];
      s_a = args.scale[g.z / t.E];
#pragma unroll
      for (int r = 0; r < kGroupRows; ++r) rows[r] = r < g.y ? __ldg(pd.perm + g.x + r) : 0;
    }
    mbar_wait(&rempty[rp.slot], rp.phase ^ 1);
    ExpandRec& q = rres[rp.slot];
    q.it = it;
    q.task = ti;
    q.ci = ci;
    q.g = g;
    q.s_a = s_a;
#pragma unroll
    for (int r = 0; r < kGroupRows; ++r) q.rows[r] = rows[r];
    mbar_arrive(&rfull[rp.slot]);
    rp.advance(nrq);
    if (it < 0) break;
  }
}

// producer side: the next resolved item (copied out, slot released)
__device__ __forceinline__ void expand_take(ExpandRec* rres, uint64_t* rfull, uint64_t* rempty, QueuePos& rp, int nrq,
                                            long long& it, int& ti, int& ci, int4& g, float& s_a, int* rows) {
  mbar_wait(&rfull[rp.slot], rp.phase);
  const ExpandRec& q = rres[rp.slot];
  it = q.it;
  ti = q.task;
  ci = q.ci;
  g = q.g;
  s_a = q.s_a;
#pragma unroll
  for (int r = 0; r < kGroupRows; ++r) rows[r] = q.rows[r];
  mbar_arrive(&rempty[rp.slot]);
  rp.advance(nrq);
}

template <int R, int M>
__device__ __forceinline__ void simt_expand_consumers(const MultiArgs& args, uint8_t* smem, uint64_t* full,
                                                      uint64_t* empty, WorkQueue<kQD>& wq, const ExpandRec* recs);

template <int R>
__global__ void __launch_bounds__(SimtCfg<R>::E_THREADS, 2)
    simt_expand_kernel(const __grid_constant__ MultiArgs args, const PlanDev pd) {
  using C = SimtCfg<R>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::NSTE * C::E_STAGE + C::YS * (C::Y_SLOT + C::META));
  uint64_t* empty = full + C::NSTE;
  WorkQueue<kQD> wq{reinterpret_cast<long long*>(empty + C::NSTE), empty + C::NSTE + kQD,
                    empty + C::NSTE + 2 * kQD};
  ExpandRec* recs = reinterpret_cast<ExpandRec*>(empty + C::NSTE + 3 * kQD);
  ExpandRec* rres = recs + kQD;                                    // [kERQ] resolved items
  uint64_t* rfull = reinterpret_cast<uint64_t*>(rres + C::kERQ);  // [kERQ]
  uint64_t* rempty = rfull + C::kERQ;                              // [kERQ]

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::NSTE; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], C::NWC);
    }
    for (int s = 0; s < C::kERQ; ++s) {
      mbar_init(&rfull[s], 1);
      mbar_init(&rempty[s], 1);
    }
    wq.init(C::NWC);
    fence_mbar_init();
  }
  __syncthreads();

  const int warp = warp_id(), lane = lane_id();
  const int n_groups = pd.counts[kCntGroups];
  const long long n_items = (long long)n_groups * args.total_ci;

  if (warp == C::NWC + 1) {
    if (lane == 0) expand_resolver(args, pd, n_groups, n_items, rres, rfull, rempty, C::kERQ);
  } else if (warp == C::NWC) {
    // ===================== producer: B rows + the group's v rows of resolved items =====================
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int stage = 0;
      uint32_t phase = 0;
      QueuePos qp, rp;
      bool shrink_done = false;
      for (;;) {
        long long it;
        int ti, ci;
        int4 g;
        float s_a;
        int rows[C::GR];
        expand_take(rres, rfull, rempty, rp, C::kERQ, it, ti, ci, g, s_a, rows);
        mbar_wait(&wq.empty[qp.slot], qp.phase ^ 1);
        ExpandRec& rc = recs[qp.slot];
        if (it < 0) {
          rc.it = -1;
          mbar_arrive(&wq.full[qp.slot]);
          break;
        }
        const SlotTask& t = args.t[ti];
        const long long unit = store_unit(g.z, t.E, args.pl, args.cache);
        const uint16_t* bbase = t.Bt + (unit * t.h_out + (long long)ci * t.CI) * R;
        const float* vsrc = pd.vpart + t.vpart_off + (long long)g.x * R;
        const int n_st = t.CI / t.SC;
        const uint32_t bytes = (uint32_t)t.SC * R * 2, vbytes = (uint32_t)g.y * R * 4;
        for (int st = 0; st < n_st; ++st) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sb = smem + stage * C::E_STAGE;
          mbar_arrive_expect_tx(&full[stage], bytes + vbytes);
          bulk_g2s_hint(sb, bbase + (long long)st * t.SC * R, bytes, &full[stage], pol);
          if (!shrink_done) {
            pdl_wait();  // v rows come from the shrink (the B rows above do not)
            shrink_done = true;
          }
          bulk_g2s(sb + C::B_STAGE, vsrc, vbytes, &full[stage]);
          if (++stage == C::NSTE) {
            stage = 0;
            phase ^= 1;
          }
          if (st == 0) {
            // publish the record after the first copies are in flight (the
            // look-ahead waits for it only YD-1 <= NSTE-1 stages ahead)
            rc.it = it;
            rc.task = ti;
            rc.ci = ci;
            rc.g = g;
            rc.s_a = s_a;
#pragma unroll
            for (int r = 0; r < C::GR; ++r) rc.rows[r] = rows[r];
            mbar_arrive(&wq.full[qp.slot]);
            qp.advance(kQD);
          }
        }
      }
    }
  } else {
    if (args.y_store == 1)
      simt_expand_consumers<R, kOutF32Store>(args, smem, full, empty, wq, recs);
    else if (args.y_store == 2)
      simt_expand_consumers<R, kOutBf16Store>(args, smem, full, empty, wq, recs);
    else if (args.y_fp32)
      simt_expand_consumers<R, kOutF32Acc>(args, smem, full, empty, wq, recs);
    else
      simt_expand_consumers<R, kOutBf16Acc>(args, smem, full, empty, wq, recs);
  }
  __syncthreads();
  wq_finish(pd.wctr + kWqSimtExpand, pd.wdone + kWqSimtExpand);
}

// consumer warps of simt_expand_kernel.  A look-ahead cursor runs YD-1
// stages ahead of the stage being computed: for each position it writes a
// StageRec into a ring slot and (bf16 y) fetches the y tile with cp.async, so
// the y latency hides behind YD-1 stages of B.  Per stage: wait for the
// slot's cp.async group, one named barrier over the consumer warps, issue the
// next look-ahead slot, wait for B + v, compute, write y (r <= 32: back into
// the tile, which all threads store to y with 16-byte stores at the next stage).
template <int R, int M>
__device__ __forceinline__ void simt_expand_consumers(const MultiArgs& args, uint8_t* smem, uint64_t* full,
                                                      uint64_t* empty, WorkQueue<kQD>& wq, const ExpandRec* recs) {
  using C = SimtCfg<R>;
  const int lane = lane_id();
  const int ct = threadIdx.x;
  uint8_t* ysm = smem + C::NSTE * C::E_STAGE;   // [YS][GR][SC_MAX] bf16
  uint8_t* meta = ysm + C::YS * C::Y_SLOT;      // [YS] StageRec
  constexpr bool ytile = M == kOutBf16Acc;
  constexpr bool TILE = C::CPT > 1 && (M == kOutBf16Acc || M == kOutBf16Store);
  constexpr int YS = TILE ? C::YD + 1 : C::YD;
  static_assert(YS <= C::YS, "y ring");
  constexpr int pitch = C::SC_MAX * 2;
  const long long END = 1ll << 62;
  int stage = 0;
  uint32_t phase = 0;

  // look-ahead cursor: the queue record of its item stays held until it moves on
  QueuePos qp;
  int la_slot = -1;
  long long la_it = END;
  int la_st = 0, la_nst = 0;
  auto take = [&]() {  // next item from the queue into the cursor
    mbar_wait(&wq.full[qp.slot], qp.phase);
    la_slot = qp.slot;
    qp.advance(kQD);
    const ExpandRec& rc = recs[la_slot];
    la_it = rc.it < 0 ? END : rc.it;
    la_st = 0;
    if (la_it != END) {
      const SlotTask& t = args.t[rc.task];
      la_nst = t.CI / t.SC;
    }
  };
  auto release = [&]() {
    __syncwarp();
    if (lane == 0 && la_slot >= 0) mbar_arrive(&wq.empty[la_slot]);
  };
  // write the cursor's position into ring slot `slot` and start its y tile
  auto issue = [&](int slot) {
    StageRec* m = reinterpret_cast<StageRec*>(meta + slot * C::META);
    if (la_it == END) {
      if (ct == 0) m->it = END;
      return;
    }
    const ExpandRec& rc = recs[la_slot];
    const SlotTask& t = args.t[rc.task];
    const long long c0 = (long long)rc.ci * t.CI + (long long)la_st * t.SC;
    if (ct == 0) {
      m->it = la_it;
      m->c0 = c0;
      m->y = t.y;
      m->st = la_st;
      m->sc = t.SC;
      m->rows = rc.g.y;
      m->h_out = t.h_out;
      m->s_a = rc.s_a;
    }
    if (ct < C::GR) m->row[ct] = rc.rows[ct];
    if constexpr (!ytile) return;
    const int cpr = t.SC >> 3;  // 16-byte chunks per row
    const int n = rc.g.y * cpr;
    const uint16_t* yb = static_cast<const uint16_t*>(t.y) + c0;
    const uint32_t dst = smem_u32(ysm + slot * C::Y_SLOT);
    for (int q = ct; q < n; q += C::NCT) {
      const int r = q / cpr, ch = q - r * cpr;
      cp_async16_u32(dst + r * pitch + ch * 16, yb + (long long)rc.rows[r] * t.h_out + ch * 8);
    }
  };
  auto advance = [&]() {
    if (la_it == END) return;
    if (la_st + 1 < la_nst) {
      ++la_st;
    } else {
      release();
      take();
    }
  };
  take();
#pragma unroll 1
  for (int k = 0; k < C::YD - 1; ++k) {
    issue(k);
    cp_async_commit();
    advance();
  }

  ExpandPos prev;  // TILE: the stage whose tile is stored next
  prev.it = END;
  int prev_slot = 0;
  // TILE: the finished tile of `prev` goes to y with coalesced 16-byte stores
  // by all consumer threads (the barrier before this made it final; the
  // look-ahead refills its slot only after the next barrier)
  auto store_prev = [&]() {
    if constexpr (TILE) {
      if (prev.it != END) {
        const int* rws = reinterpret_cast<const StageRec*>(meta + prev_slot * C::META)->row;
        const uint32_t src = smem_u32(ysm + prev_slot * C::Y_SLOT);
        const int cpr = prev.sc >> 3;
        const int n = prev.rows * cpr;
        uint16_t* yb = static_cast<uint16_t*>(prev.y) + prev.c0;
        for (int q = ct; q < n; q += C::NCT) {
          const int r = q / cpr, ch = q - r * cpr;
          const uint4 v = lds128(src + r * pitch + ch * 16);
          *reinterpret_cast<uint4*>(yb + (long long)rws[r] * prev.h_out + ch * 8) = v;
        }
      }
    }
  };
  int ys = 0;
  for (;;) {
    cp_async_wait<C::YD - 2>();
    named_bar_sync(1, C::NCT);  // slot ys complete and visible; previous stage's tile final
    store_prev();
    const StageRec* m = reinterpret_cast<const StageRec*>(meta + ys * C::META);
    ExpandPos at;
    at.it = m->it;
    if (at.it == END) break;
    at.c0 = m->c0;
    at.y = m->y;
    at.st = m->st;
    at.sc = m->sc;
    at.rows = m->rows;
    at.h_out = m->h_out;
    at.s_a = m->s_a;
    {
      int ns = ys + C::YD - 1;
      if (ns >= YS) ns -= YS;
      issue(ns);
    }
    cp_async_commit();
    mbar_wait(&full[stage], phase);
    const uint32_t b_s = smem_u32(smem + stage * C::E_STAGE);
    const uint32_t v_s = b_s + C::B_STAGE;
    const uint32_t yt = smem_u32(ysm + ys * C::Y_SLOT);
    const uint32_t rows = smem_u32(m->row);
    switch (at.rows) {
      case 1: expand_stage<R, 1, M>(b_s, v_s, ct, at, rows, yt, pitch); break;
      case 2: expand_stage<R, 2, M>(b_s, v_s, ct, at, rows, yt, pitch); break;
      case 3: expand_stage<R, 3, M>(b_s, v_s, ct, at, rows, yt, pitch); break;
      case 4: expand_stage<R, 4, M>(b_s, v_s, ct, at, rows, yt, pitch); break;
      case 5: expand_stage<R, 5, M>(b_s, v_s, ct, at, rows, yt, pitch); break;
      case 6: expand_stage<R, 6, M>(b_s, v_s, ct, at, rows, yt, pitch); break;
      case 7: expand_stage<R, 7, M>(b_s, v_s, ct, at, rows, yt, pitch); break;
      default: expand_stage<R, 8, M>(b_s, v_s, ct, at, rows, yt, pitch); break;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[stage]);
    if (++stage == C::NSTE) {
      stage = 0;
      phase ^= 1;
    }
    // move the look-ahead on only after releasing this stage: the producer
    // publishes an item after issuing its first stage, which may need this slot
    advance();
    prev = at;
    prev_slot = ys;
    ys = ys + 1 == YS ? 0 : ys + 1;
  }
  cp_async_wait<0>();
}

// ---------------------------------------------------------------------------
// staged-tile expand (r <= 16).  At small r a stage carries few B bytes (16 KB
// at r = 16) against up to 8 KB of y read + 8 KB written, so the y latency
// cannot hide behind a consumer-issued look-ahead of a few short stages.  Here
// the producer lane bulk-copies each group row's y chunk into the stage buffer
// next to the B rows and the v rows (one mbarrier transaction for all), so y
// is in flight exactly as deep as B.  Consumers compute the stage into the
// tile (s_a * v B + y, rounded once), then -- after one named barrier -- store
// the tile with coalesced 16-byte stores and release the stage.
// ---------------------------------------------------------------------------
template <int R, int M>
__device__ __forceinline__ void simt_expand_tile_consumers(const MultiArgs& args, uint8_t* smem, uint64_t* full,
                                                           uint64_t* empty, WorkQueue<kQD>& wq,
                                                           const ExpandRec* recs) {
  using C = SimtCfg<R>;
  // CPT == 1 (r = 64): results go to y straight from registers (expand_stage1)
  constexpr bool TILE = C::CPT > 1 && out_bf16_tile(M);
  constexpr int pitch = C::SC_MAX * 2;
  const int lane = lane_id();
  const int ct = threadIdx.x;
  // store pass mapping: 16-byte chunk sch of rows rsub, rsub + RSTEP, ...
  constexpr int CPRM = C::SC_MAX / 8, RSTEP = C::NCT / CPRM;
  const int rsub = ct / CPRM, sch = ct % CPRM;
  static_assert(C::NCT % CPRM == 0, "store pass mapping");
  int stage = 0;
  uint32_t phase = 0;
  QueuePos qp;
  for (;;) {
    mbar_wait(&wq.full[qp.slot], qp.phase);
    const ExpandRec& rc = recs[qp.slot];
    if (rc.it < 0) break;
    const SlotTask& t = args.t[rc.task];
    const int nr = rc.g.y;
    ExpandPos p;
    p.it = rc.it;
    p.sc = t.SC;
    p.rows = nr;
    p.h_out = t.h_out;
    p.y = t.y;
    p.s_a = rc.s_a;
    if constexpr (out_push(M)) {
#pragma unroll
      for (int r = 0; r < C::GR; ++r)
        p.prow[r] = r < nr ? y_push_row(args, rc.task, rc.rows[r], M == kOutF32Push ? 4 : 2) : nullptr;
    }
    const uint32_t rows = smem_u32(rc.rows);
    const int n_st = t.CI / t.SC;
    for (int st = 0; st < n_st; ++st) {
      p.st = st;
      p.c0 = (long long)rc.ci * t.CI + (long long)st * t.SC;
      mbar_wait(&full[stage], phase);
      const uint32_t b_s = smem_u32(smem + stage * C::T_STAGE);
      const uint32_t v_s = b_s + C::TV_OFF;
      const uint32_t yt = b_s + C::TY_OFF;
      // (an mma.sync formulation of this stage, D[16 c x 8 n] = Bt . v^T with a
      // bf16 hi/lo split of v, measured slower: Llama decode expand 180 ->
      // 223 us -- the stage's cost is the per-element y update, not the dot
      // products -- so the expand keeps the FFMA2 consumers)
      if (!(LORA_EXP_PROBE & 1)) {  // (timing probe bit 0: no consumer arithmetic, no y stores; results wrong)
      switch (nr) {
        case 1: expand_stage<R, 1, M>(b_s, v_s, ct, p, rows, yt, pitch); break;
        case 2: expand_stage<R, 2, M>(b_s, v_s, ct, p, rows, yt, pitch); break;
        case 3: expand_stage<R, 3, M>(b_s, v_s, ct, p, rows, yt, pitch); break;
        case 4: expand_stage<R, 4, M>(b_s, v_s, ct, p, rows, yt, pitch); break;
        case 5: expand_stage<R, 5, M>(b_s, v_s, ct, p, rows, yt, pitch); break;
        case 6: expand_stage<R, 6, M>(b_s, v_s, ct, p, rows, yt, pitch); break;
        case 7: expand_stage<R, 7, M>(b_s, v_s, ct, p, rows, yt, pitch); break;
        default: expand_stage<R, 8, M>(b_s, v_s, ct, p, rows, yt, pitch); break;
      }
      }
      if constexpr (TILE) {
        named_bar_sync(1, C::NCT);  // the whole tile is final
        if (!(LORA_EXP_PROBE & 1) && sch < (p.sc >> 3)) {
          uint16_t* yb = static_cast<uint16_t*>(p.y) + p.c0 + sch * 8;
          for (int r = rsub; r < nr; r += RSTEP) {
            const uint4 v = lds128(yt + r * pitch + sch * 16);
            if constexpr (M == kOutBf16Push)
              red_add_bf16x8(p.prow[r] + (p.c0 + sch * 8) * 2, v);  // r < nr: prow set
            else
              *reinterpret_cast<uint4*>(yb + (long long)rc.rows[r] * p.h_out) = v;
          }
        }
        fence_proxy_async_smem();  // the tile is refilled by bulk copies after the release
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == C::TNST) {
        stage = 0;
        phase ^= 1;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&wq.empty[qp.slot]);
    qp.advance(kQD);
  }
}

template <int R>
__global__ void __launch_bounds__(SimtCfg<R>::TILE_THREADS, 2)
    simt_expand_tile_kernel(const __grid_constant__ MultiArgs args, const PlanDev pd) {
  using C = SimtCfg<R>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::TNST * C::T_STAGE);
  uint64_t* empty = full + C::TNST;
  WorkQueue<kQD> wq{reinterpret_cast<long long*>(empty + C::TNST), empty + C::TNST + kQD,
                    empty + C::TNST + 2 * kQD};
  ExpandRec* recs = reinterpret_cast<ExpandRec*>(empty + C::TNST + 3 * kQD);
  ExpandRec* rres = recs + kQD;                                    // [kRQ] resolved items
  uint64_t* rfull = reinterpret_cast<uint64_t*>(rres + C::kRQ);   // [kRQ]
  uint64_t* rempty = rfull + C::kRQ;                               // [kRQ]

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::TNST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], C::NWC);
    }
    for (int s = 0; s < C::kRQ; ++s) {
      mbar_init(&rfull[s], 1);
      mbar_init(&rempty[s], 1);
    }
    wq.init(C::NWC);
    fence_mbar_init();
  }
  __syncthreads();

  const int warp = warp_id(), lane = lane_id();
  const int n_groups = pd.counts[kCntGroups];
  const long long n_items = (long long)n_groups * args.total_ci;
  if (warp == C::NWC + 1) {
    if (lane == 0) expand_resolver(args, pd, n_groups, n_items, rres, rfull, rempty, C::kRQ);
  } else if (warp == C::NWC) {
    // ===================== producer: B rows, v rows, y chunks of resolved items =====================
    if (lane == 0) {
      const bool load_y = args.y_store == 0 && !args.y_fp32 && !(LORA_EXP_PROBE & 2);  // (probe bit 1: no y loads)
      const uint64_t pol = (args.tc_flags & 8) ? policy_evict_last() : policy_evict_first();  // B (bit 3)
      int stage = 0;
      uint32_t phase = 0;
      QueuePos qp, rp;
      bool shrink_done = false;
      for (;;) {
        long long it;
        int ti, ci;
        int4 g;
        float s_a;
        int rows[C::GR];
        expand_take(rres, rfull, rempty, rp, C::kRQ, it, ti, ci, g, s_a, rows);
        mbar_wait(&wq.empty[qp.slot], qp.phase ^ 1);
        ExpandRec& rc = recs[qp.slot];
        if (it < 0) {
          rc.it = -1;
          mbar_arrive(&wq.full[qp.slot]);
          break;
        }
        const SlotTask& t = args.t[ti];
        const long long unit = store_unit(g.z, t.E, args.pl, args.cache);
        const uint16_t* bbase = t.Bt + (unit * t.h_out + (long long)ci * t.CI) * R;
        const float* vsrc = pd.vpart + t.vpart_off + (long long)g.x * R;
        const int n_st = t.CI / t.SC;
        const uint32_t bytes = (uint32_t)t.SC * R * 2, vbytes = (uint32_t)g.y * R * 4;
        const uint32_t ybytes = load_y ? (uint32_t)t.SC * 2 : 0u;
        const uint16_t* ybase = static_cast<const uint16_t*>(t.y) + (long long)ci * t.CI;
        for (int st = 0; st < n_st; ++st) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sb = smem + stage * C::T_STAGE;
          mbar_arrive_expect_tx(&full[stage], bytes + vbytes + ybytes * g.y);
          bulk_g2s_hint(sb, bbase + (long long)st * t.SC * R, bytes, &full[stage], pol);
          if (!shrink_done) {
            pdl_wait();  // v rows come from the shrink (the B rows above do not)
            shrink_done = true;
          }
          bulk_g2s(sb + C::TV_OFF, vsrc, vbytes, &full[stage]);
          if (ybytes) {
#pragma unroll
            for (int r = 0; r < C::GR; ++r)
              if (r < g.y)
                bulk_g2s(sb + C::TY_OFF + r * (C::SC_MAX * 2),
                         ybase + (long long)rows[r] * t.h_out + (long long)st * t.SC, ybytes, &full[stage]);
          }
          if (++stage == C::TNST) {
            stage = 0;
            phase ^= 1;
          }
          if (st == 0) {
            rc.it = it;
            rc.task = ti;
            rc.ci = ci;
            rc.g = g;
            rc.s_a = s_a;
#pragma unroll
            for (int r = 0; r < C::GR; ++r) rc.rows[r] = rows[r];
            mbar_arrive(&wq.full[qp.slot]);
            qp.advance(kQD);
          }
        }
      }
    }
  } else {
    if (args.y_store == 3) {
      if (args.y_fp32)
        simt_expand_tile_consumers<R, kOutF32Push>(args, smem, full, empty, wq, recs);
      else
        simt_expand_tile_consumers<R, kOutBf16Push>(args, smem, full, empty, wq, recs);
      __threadfence_system();  // this thread's pushes performed before the owner signals completion
    } else if (args.y_store == 1)
      simt_expand_tile_consumers<R, kOutF32Store>(args, smem, full, empty, wq, recs);
    else if (args.y_store == 2)
      simt_expand_tile_consumers<R, kOutBf16Store>(args, smem, full, empty, wq, recs);
    else if (args.y_fp32)
      simt_expand_tile_consumers<R, kOutF32Acc>(args, smem, full, empty, wq, recs);
    else
      simt_expand_tile_consumers<R, kOutBf16Acc>(args, smem, full, empty, wq, recs);
  }
  __syncthreads();
  wq_finish(pd.wctr + kWqSimtExpand, pd.wdone + kWqSimtExpand);
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

template <int R>
cudaError_t launch_shrink_t(const MultiArgs& args, const PlanDev& pd, int grid, cudaStream_t stream) {
  using C = SimtCfg<R>;
  static unsigned long long mask[2] = {0, 0};
  const bool remote = args.push.G > 0;
  auto kern = remote ? simt_shrink_kernel<R, true> : simt_shrink_kernel<R, false>;
  cudaError_t e = set_smem_once(kern, C::SHRINK_SMEM, mask[remote]);
  if (e != cudaSuccess) return e;
  e = launch_pdl(kern, dim3(2 * grid), dim3(C::SHRINK_THREADS), C::SHRINK_SMEM, stream, args, pd);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// staged-tile expand for r <= LORA_TILE_MAX_R (16; LORA_EXPAND_V1=1: the look-ahead kernel at every r)
inline bool use_tile_expand(int r) {
  static const int v1 = [] {
    const char* e = getenv("LORA_EXPAND_V1");
    return e && e[0] == '1' ? 1 : 0;
  }();
  return r <= LORA_TILE_MAX_R && !v1;
}

template <int R>
cudaError_t launch_expand_t(const MultiArgs& args, const PlanDev& pd, int grid, cudaStream_t stream) {
  using C = SimtCfg<R>;
  if constexpr (R <= LORA_TILE_MAX_R || !C::LOOKAHEAD_OK) {
    if (!C::LOOKAHEAD_OK || use_tile_expand(R) || args.y_store == 3) {  // (push: staged-tile kernel only)
      static unsigned long long tmask = 0;
      cudaError_t e = set_smem_once(simt_expand_tile_kernel<R>, C::TILE_SMEM, tmask);
      if (e != cudaSuccess) return e;
      e = launch_pdl(simt_expand_tile_kernel<R>, dim3(2 * grid), dim3(C::TILE_THREADS), C::TILE_SMEM, stream, args,
                     pd);
      if (e != cudaSuccess) return e;
      return cudaGetLastError();
    }
  }
  if constexpr (C::LOOKAHEAD_OK) {
    static unsigned long long mask = 0;
    cudaError_t e = set_smem_once(simt_expand_kernel<R>, C::EXPAND_SMEM, mask);
    if (e != cudaSuccess) return e;
    e = launch_pdl(simt_expand_kernel<R>, dim3(2 * grid), dim3(C::E_THREADS), C::EXPAND_SMEM, stream, args, pd);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
  }
  return cudaErrorInvalidValue;
}

}  // namespace

// `grid` is the SM count; the CUDA-core kernels run two CTAs per SM
cudaError_t launch_simt_shrink(int rank, const MultiArgs& args, const PlanDev& pd, int grid, cudaStream_t stream) {
  switch (rank) {
    case 8: return launch_shrink_t<8>(args, pd, grid, stream);
    case 16: return launch_shrink_t<16>(args, pd, grid, stream);
    case 32: return launch_shrink_t<32>(args, pd, grid, stream);
    case 64: return launch_shrink_t<64>(args, pd, grid, stream);
    case 128: return launch_shrink_t<128>(args, pd, grid, stream);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_simt_expand(int rank, const MultiArgs& args, const PlanDev& pd, int grid, cudaStream_t stream) {
  switch (rank) {
    case 8: return launch_expand_t<8>(args, pd, grid, stream);
    case 16: return launch_expand_t<16>(args, pd, grid, stream);
    case 32: return launch_expand_t<32>(args, pd, grid, stream);
    case 64: return launch_expand_t<64>(args, pd, grid, stream);
    case 128: return launch_expand_t<128>(args, pd, grid, stream);
    default: return cudaErrorInvalidValue;
  }
}

int simt_sj_max(int rank) {
  switch (rank) {
    case 8: return SimtCfg<8>::SJ_MAX;
    case 16: return SimtCfg<16>::SJ_MAX;
    case 32: return SimtCfg<32>::SJ_MAX;
    case 128: return SimtCfg<128>::SJ_MAX;
    default: return SimtCfg<64>::SJ_MAX;
  }
}
int simt_sc_max(int rank) {
  switch (rank) {
    case 8: return SimtCfg<8>::SC_MAX;
    case 16: return SimtCfg<16>::SC_MAX;
    case 32: return SimtCfg<32>::SC_MAX;
    case 128: return SimtCfg<128>::SC_MAX;
    default: return SimtCfg<64>::SC_MAX;
  }
}
int simt_shrink_smem(int rank) {
  switch (rank) {
    case 8: return SimtCfg<8>::SHRINK_SMEM;
    case 16: return SimtCfg<16>::SHRINK_SMEM;
    case 32: return SimtCfg<32>::SHRINK_SMEM;
    case 128: return SimtCfg<128>::SHRINK_SMEM;
    default: return SimtCfg<64>::SHRINK_SMEM;
  }
}
int simt_expand_smem(int rank) {
  // the larger of the two expand kernels' dynamic shared memory
  auto of = [](auto c) {
    using C = decltype(c);
    return C::LOOKAHEAD_OK ? std::max(C::EXPAND_SMEM, C::TILE_SMEM) : C::TILE_SMEM;
  };
  switch (rank) {
    case 8: return of(SimtCfg<8>{});
    case 16: return of(SimtCfg<16>{});
    case 32: return of(SimtCfg<32>{});
    case 128: return of(SimtCfg<128>{});
    default: return of(SimtCfg<64>{});
  }
}

}  // namespace lora
