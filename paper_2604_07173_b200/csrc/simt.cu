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
#include "common.cuh"
#include "kernels.h"

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
  // shrink
  static constexpr int KL = R < 32 ? R : 32;  // lanes along k
  static constexpr int KPL = R / KL;          // k per lane
  static constexpr int NJG = NCT / KL;        // j-groups
  static constexpr int SJ_MAX = 8192 / R;     // 16 KB of A per stage
  static constexpr int A_STAGE = R * SJ_MAX * 2;
  static constexpr int X_STAGE = GR * SJ_MAX * 2;
  static constexpr int S_STAGE = A_STAGE + X_STAGE;
  static constexpr int RED_BYTES = NJG * GR * R * 4;
  static constexpr int NST_RAW = (SMEM_BUDGET - RED_BYTES) / S_STAGE;
  static constexpr int NST = NST_RAW > 8 ? 8 : (NST_RAW < 2 ? 2 : NST_RAW);
  static constexpr int SHRINK_SMEM = 1024 + NST * S_STAGE + RED_BYTES + 2 * NST * 8 + 3 * kQD * 8;
  // expand
  static constexpr int SC_MAX = NCT;        // one B row (output column) per consumer thread per stage
  static constexpr int B_STAGE = SC_MAX * R * 2;
  static constexpr int V_BYTES = GR * R * 4;  // v rows of the group (fp32)
  static constexpr int E_STAGE = B_STAGE + 1024 * ((V_BYTES + 1023) / 1024);
  static constexpr int NSTE_RAW = SMEM_BUDGET / E_STAGE;
  static constexpr int NSTE = NSTE_RAW > 16 ? 16 : NSTE_RAW;
  static constexpr int EXPAND_SMEM = 1024 + NSTE * E_STAGE + 2 * NSTE * 8 + 3 * kQD * 8;
  static_assert(S_STAGE % 1024 == 0 && E_STAGE % 1024 == 0, "stage alignment");
  static_assert(SHRINK_SMEM <= 112 * 1024 && EXPAND_SMEM <= 112 * 1024, "two CTAs per SM");
};

LORA_DEVINL uint8_t* align1024(uint8_t* p) {
  const uint32_t a = smem_u32(p);
  return p + (((a + 1023u) & ~1023u) - a);
}

LORA_DEVINL int find_task_ci(const MultiArgs& args, int g) {
  int t = 0;
  while (t + 1 < args.n_tasks && args.t[t + 1].ci_base <= g) ++t;
  return t;
}

LORA_DEVINL long long unit_of_key(int key, int E, const Placement& pl) {
  const int a = key / E, e = key - a * E;
  return pl.local_index(a) * E + e;
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
template <int R, int NR>
LORA_DEVINL void shrink_item(uint8_t* smem, uint64_t* full, uint64_t* empty, float* red, int& stage,
                             uint32_t& phase, const SlotTask& t, const int4 g, float* vpart_base,
                             int lane) {
  using C = SimtCfg<R>;
  const int ct = threadIdx.x;
  const int kl = ct % C::KL, jg = ct / C::KL;
  const int n_st = t.h_in / t.SJ;
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
    vp[idx] = s;
  }
}

template <int R>
__global__ void __launch_bounds__(SimtCfg<R>::THREADS, 2)
    simt_shrink_kernel(const __grid_constant__ MultiArgs args, const PlanDev pd) {
  using C = SimtCfg<R>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  float* red = reinterpret_cast<float*>(smem + C::NST * C::S_STAGE);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::NST * C::S_STAGE + C::RED_BYTES);
  uint64_t* empty = full + C::NST;
  WorkQueue<kQD> wq{reinterpret_cast<long long*>(empty + C::NST), empty + C::NST + kQD, empty + C::NST + 2 * kQD};

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], C::NWC);
    }
    wq.init(C::NWC);
    fence_mbar_init();
  }
  __syncthreads();

  const int n_groups = pd.counts[kCntGroups];
  const long long n_items = (long long)n_groups * args.n_tasks;
  const int warp = warp_id(), lane = lane_id();

  if (warp == C::NWC) {
    // ===================== producer =====================
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int stage = 0;
      uint32_t phase = 0;
      QueuePos qp;
      for (;;) {
        const long long it = wq_push_next(wq, qp, pd.wctr + kWqSimtShrink, n_items);
        if (it < 0) break;
        const int ti = (int)(it / n_groups), gi = (int)(it - (long long)ti * n_groups);
        const SlotTask& t = args.t[ti];
        const int4 g = pd.groups[gi];
        const long long unit = unit_of_key(g.z, t.E, args.pl);
        const uint16_t* abase = t.At + unit * (long long)t.h_in * R;
        const int n_st = t.h_in / t.SJ;
        const uint32_t a_bytes = (uint32_t)R * t.SJ * 2, x_bytes = (uint32_t)t.SJ * 2;
        long long xrow[C::GR];
#pragma unroll
        for (int r = 0; r < C::GR; ++r) xrow[r] = r < g.y ? (long long)pd.perm[g.x + r] * t.h_in : 0;
        for (int st = 0; st < n_st; ++st) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sA = smem + stage * C::S_STAGE;
          uint8_t* sX = sA + C::A_STAGE;
          mbar_arrive_expect_tx(&full[stage], a_bytes + x_bytes * g.y);
          bulk_g2s_hint(sA, abase + (long long)st * t.SJ * R, a_bytes, &full[stage], pol);
          const long long jofs = (long long)st * t.SJ;
#pragma unroll
          for (int r = 0; r < C::GR; ++r)
            if (r < g.y) bulk_g2s(sX + r * x_bytes, t.x + xrow[r] + jofs, x_bytes, &full[stage]);
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
      const long long it = wq_pop(wq, qp);
      if (it < 0) break;
      const int ti = (int)(it / n_groups), gi = (int)(it - (long long)ti * n_groups);
      const SlotTask& t = args.t[ti];
      const int4 g = pd.groups[gi];
      float* vb = pd.vpart + t.vpart_off;
      switch (g.y) {
        case 1: shrink_item<R, 1>(smem, full, empty, red, stage, phase, t, g, vb, lane); break;
        case 2: shrink_item<R, 2>(smem, full, empty, red, stage, phase, t, g, vb, lane); break;
        case 3: shrink_item<R, 3>(smem, full, empty, red, stage, phase, t, g, vb, lane); break;
        case 4: shrink_item<R, 4>(smem, full, empty, red, stage, phase, t, g, vb, lane); break;
        case 5: shrink_item<R, 5>(smem, full, empty, red, stage, phase, t, g, vb, lane); break;
        case 6: shrink_item<R, 6>(smem, full, empty, red, stage, phase, t, g, vb, lane); break;
        case 7: shrink_item<R, 7>(smem, full, empty, red, stage, phase, t, g, vb, lane); break;
        default: shrink_item<R, 8>(smem, full, empty, red, stage, phase, t, g, vb, lane); break;
      }
    }
  }
  __syncthreads();
  wq_finish(pd.wctr + kWqSimtShrink, pd.wdone + kWqSimtShrink);
}

// ---------------------------------------------------------------------------
// expand + scale + scatter-accumulate
// ---------------------------------------------------------------------------
// Consumer-side walk over this CTA's (item, stage) sequence, so the y loads of
// the next stage can be issued one stage ahead.
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
};

template <int R, int NR>
LORA_DEVINL void expand_stage(uint32_t b_s, uint32_t v_s, int cr, const ExpandPos& p, const uint32_t* yraw,
                              const int* yrow, int y_store, int y_fp32) {
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
  const long long c = p.c0 + cr;
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    const float d = p.s_a * ((acc[r][0].x + acc[r][0].y) + (acc[r][1].x + acc[r][1].y));
    const long long o = (long long)yrow[r] * p.h_out + c;
    if (y_store == 1)
      reinterpret_cast<float*>(p.y)[o] = d;
    else if (y_store == 2)
      reinterpret_cast<uint16_t*>(p.y)[o] = f32_to_bf16_rne(d);
    else if (y_fp32)
      reinterpret_cast<float*>(p.y)[o] = __uint_as_float(yraw[r]) + d;
    else
      reinterpret_cast<uint16_t*>(p.y)[o] = f32_to_bf16_rne(bf16_to_f32((uint16_t)yraw[r]) + d);
  }
}

template <int R>
__device__ __forceinline__ void simt_expand_consumers(const MultiArgs& args, const PlanDev& pd, uint8_t* smem,
                                                      uint64_t* full, uint64_t* empty, WorkQueue<kQD>& wq,
                                                      int n_groups, long long n_items);

template <int R>
__global__ void __launch_bounds__(SimtCfg<R>::THREADS, 2)
    simt_expand_kernel(const __grid_constant__ MultiArgs args, const PlanDev pd) {
  using C = SimtCfg<R>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::NSTE * C::E_STAGE);
  uint64_t* empty = full + C::NSTE;
  WorkQueue<kQD> wq{reinterpret_cast<long long*>(empty + C::NSTE), empty + C::NSTE + kQD,
                    empty + C::NSTE + 2 * kQD};

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::NSTE; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], C::NWC);
    }
    wq.init(C::NWC);
    fence_mbar_init();
  }
  __syncthreads();

  const int n_groups = pd.counts[kCntGroups];
  const long long n_items = (long long)n_groups * args.total_ci;
  const int warp = warp_id(), lane = lane_id();

  if (warp == C::NWC) {
    // ===================== producer: B rows + the group's v rows =====================
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int stage = 0;
      uint32_t phase = 0;
      QueuePos qp;
      for (;;) {
        const long long it = wq_push_next(wq, qp, pd.wctr + kWqSimtExpand, n_items);
        if (it < 0) break;
        const int cig = (int)(it / n_groups), gi = (int)(it - (long long)cig * n_groups);
        const SlotTask& t = args.t[find_task_ci(args, cig)];
        const int ci = cig - t.ci_base;
        const int4 g = pd.groups[gi];
        const long long unit = unit_of_key(g.z, t.E, args.pl);
        const uint16_t* bbase = t.Bt + (unit * t.h_out + (long long)ci * t.CI) * R;
        const float* vsrc = pd.vpart + t.vpart_off + (long long)g.x * R;
        const int n_st = t.CI / t.SC;
        const uint32_t bytes = (uint32_t)t.SC * R * 2, vbytes = (uint32_t)g.y * R * 4;
        for (int st = 0; st < n_st; ++st) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sb = smem + stage * C::E_STAGE;
          mbar_arrive_expect_tx(&full[stage], bytes + vbytes);
          bulk_g2s_hint(sb, bbase + (long long)st * t.SC * R, bytes, &full[stage], pol);
          bulk_g2s(sb + C::B_STAGE, vsrc, vbytes, &full[stage]);
          if (++stage == C::NSTE) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else {
    simt_expand_consumers<R>(args, pd, smem, full, empty, wq, n_groups, n_items);
  }
  __syncthreads();
  wq_finish(pd.wctr + kWqSimtExpand, pd.wdone + kWqSimtExpand);
}

// consumer warps of simt_expand_kernel
template <int R>
__device__ __forceinline__ void simt_expand_consumers(const MultiArgs& args, const PlanDev& pd, uint8_t* smem,
                                                      uint64_t* full, uint64_t* empty, WorkQueue<kQD>& wq,
                                                      int n_groups, long long n_items) {
  using C = SimtCfg<R>;
  const int lane = lane_id();
  const int ct = threadIdx.x;
  int stage = 0;
  uint32_t phase = 0;

  auto locate = [&](long long it, ExpandPos& p) {
    p.it = it;
    p.st = 0;
    if (it >= n_items) return;
    const int cig = (int)(it / n_groups), gi = (int)(it - (long long)cig * n_groups);
    const SlotTask& t = args.t[find_task_ci(args, cig)];
    const int ci = cig - t.ci_base;
    const int4 g = pd.groups[gi];
    p.n_st = t.CI / t.SC;
    p.sc = t.SC;
    p.rows = g.y;
    p.h_out = t.h_out;
    p.c0 = (long long)ci * t.CI;
    p.y = t.y;
    p.perm_rows = pd.perm + g.x;
    p.s_a = args.scale[g.z / t.E];
  };
  // raw y bits of the stage at `p` for this thread's column.  Kept raw (the
  // conversion happens at use), so the loads stay in flight across the next
  // barrier wait and compute.
  uint32_t yv[C::GR];
  int yrow[C::GR];
  auto load_y = [&](const ExpandPos& p) {
    if (args.y_store || ct >= p.sc) return;
    const long long c = p.c0 + ct;
#pragma unroll
    for (int r = 0; r < C::GR; ++r) {
      if (r < p.rows) {
        const long long o = (long long)yrow[r] * p.h_out + c;
        if (args.y_fp32)
          yv[r] = reinterpret_cast<const uint32_t*>(p.y)[o];
        else
          yv[r] = reinterpret_cast<const uint16_t*>(p.y)[o];
      }
    }
  };
  auto load_rows = [&](const ExpandPos& p) {
#pragma unroll
    for (int r = 0; r < C::GR; ++r) yrow[r] = r < p.rows ? p.perm_rows[r] : 0;
  };

  QueuePos qp;
  ExpandPos cur;
  {
    const long long it0 = wq_pop(wq, qp);
    locate(it0 < 0 ? n_items : it0, cur);
  }
  if (cur.it < n_items) {
    load_rows(cur);
    load_y(cur);
  }
  while (cur.it < n_items) {
    mbar_wait(&full[stage], phase);
    const uint32_t b_s = smem_u32(smem + stage * C::E_STAGE);
    const uint32_t v_s = b_s + C::B_STAGE;
    if (ct < cur.sc) {
      switch (cur.rows) {
        case 1: expand_stage<R, 1>(b_s, v_s, ct, cur, yv, yrow, args.y_store, args.y_fp32); break;
        case 2: expand_stage<R, 2>(b_s, v_s, ct, cur, yv, yrow, args.y_store, args.y_fp32); break;
        case 3: expand_stage<R, 3>(b_s, v_s, ct, cur, yv, yrow, args.y_store, args.y_fp32); break;
        case 4: expand_stage<R, 4>(b_s, v_s, ct, cur, yv, yrow, args.y_store, args.y_fp32); break;
        case 5: expand_stage<R, 5>(b_s, v_s, ct, cur, yv, yrow, args.y_store, args.y_fp32); break;
        case 6: expand_stage<R, 6>(b_s, v_s, ct, cur, yv, yrow, args.y_store, args.y_fp32); break;
        case 7: expand_stage<R, 7>(b_s, v_s, ct, cur, yv, yrow, args.y_store, args.y_fp32); break;
        default: expand_stage<R, 8>(b_s, v_s, ct, cur, yv, yrow, args.y_store, args.y_fp32); break;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[stage]);
    if (++stage == C::NSTE) {
      stage = 0;
      phase ^= 1;
    }
    // next stage of this item, or this CTA's next item; issue its y loads now
    if (cur.st + 1 < cur.n_st) {
      cur.st += 1;
      cur.c0 += cur.sc;
    } else {
      const long long nit = wq_pop(wq, qp);
      if (nit < 0) break;
      locate(nit, cur);
      load_rows(cur);
    }
    load_y(cur);
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

template <int R>
cudaError_t launch_shrink_t(const MultiArgs& args, const PlanDev& pd, int grid, cudaStream_t stream) {
  using C = SimtCfg<R>;
  static unsigned long long mask = 0;
  cudaError_t e = set_smem_once(simt_shrink_kernel<R>, C::SHRINK_SMEM, mask);
  if (e != cudaSuccess) return e;
  simt_shrink_kernel<R><<<2 * grid, C::THREADS, C::SHRINK_SMEM, stream>>>(args, pd);
  return cudaGetLastError();
}

template <int R>
cudaError_t launch_expand_t(const MultiArgs& args, const PlanDev& pd, int grid, cudaStream_t stream) {
  using C = SimtCfg<R>;
  static unsigned long long mask = 0;
  cudaError_t e = set_smem_once(simt_expand_kernel<R>, C::EXPAND_SMEM, mask);
  if (e != cudaSuccess) return e;
  simt_expand_kernel<R><<<2 * grid, C::THREADS, C::EXPAND_SMEM, stream>>>(args, pd);
  return cudaGetLastError();
}

}  // namespace

// `grid` is the SM count; the CUDA-core kernels run two CTAs per SM
cudaError_t launch_simt_shrink(int rank, const MultiArgs& args, const PlanDev& pd, int grid, cudaStream_t stream) {
  switch (rank) {
    case 8: return launch_shrink_t<8>(args, pd, grid, stream);
    case 16: return launch_shrink_t<16>(args, pd, grid, stream);
    case 32: return launch_shrink_t<32>(args, pd, grid, stream);
    case 64: return launch_shrink_t<64>(args, pd, grid, stream);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_simt_expand(int rank, const MultiArgs& args, const PlanDev& pd, int grid, cudaStream_t stream) {
  switch (rank) {
    case 8: return launch_expand_t<8>(args, pd, grid, stream);
    case 16: return launch_expand_t<16>(args, pd, grid, stream);
    case 32: return launch_expand_t<32>(args, pd, grid, stream);
    case 64: return launch_expand_t<64>(args, pd, grid, stream);
    default: return cudaErrorInvalidValue;
  }
}

int simt_sj_max(int rank) {
  switch (rank) {
    case 8: return SimtCfg<8>::SJ_MAX;
    case 16: return SimtCfg<16>::SJ_MAX;
    case 32: return SimtCfg<32>::SJ_MAX;
    default: return SimtCfg<64>::SJ_MAX;
  }
}
int simt_sc_max(int rank) { return SimtCfg<64>::SC_MAX + 0 * rank; }
int simt_shrink_smem(int rank) {
  switch (rank) {
    case 8: return SimtCfg<8>::SHRINK_SMEM;
    case 16: return SimtCfg<16>::SHRINK_SMEM;
    case 32: return SimtCfg<32>::SHRINK_SMEM;
    default: return SimtCfg<64>::SHRINK_SMEM;
  }
}
int simt_expand_smem(int rank) {
  switch (rank) {
    case 8: return SimtCfg<8>::EXPAND_SMEM;
    case 16: return SimtCfg<16>::EXPAND_SMEM;
    case 32: return SimtCfg<32>::EXPAND_SMEM;
    default: return SimtCfg<64>::EXPAND_SMEM;
  }
}

}  // namespace lora
