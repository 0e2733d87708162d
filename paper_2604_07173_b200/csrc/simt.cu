// simt.cu -- a2 shrink and a3+a4 expand/scatter-accumulate on CUDA cores.
//
// The decode case: most segments hold 1-8 rows,
// so the work is a stream of per-unit weights with 1-8 FMAs per weight
// element -- HBM-bound, far below the tensor-core ridge.  The paper's BGMV
// answer is "thread collaborative execution instead of the heavier wgmma
// pipeline" (Sec. 5.2); the B200 form used here:
//
//   * persistent CTAs (one per SM), 1 producer warp + 8 consumer warps;
//   * the producer streams each unit's weights with 1-D TMA bulk copies
//     (cp.async.bulk, SASS UBLKCP) into a 4-6 deep shared-memory ring
//     (~150-190 KB in flight per SM), plus the group's activation rows;
//   * the weight store is pre-swizzled (common.cuh), so the consumers' 128-bit
//     shared loads are bank-conflict free;
//   * shrink accumulates per-thread partial dot products and reduces them
//     deterministically through shared memory (no float atomics);
//   * expand applies the per-adapter scale and read-modify-writes y[perm[j]]
//     directly from registers, consecutive threads on consecutive columns.
//
// Work items (device-side counts, no host sync):
//   shrink item = (slot task, k-chunk kc of KI inputs, row group)
//               -> vpart[kc][row][0:r]   (partial v over that k-chunk)
//   expand item = (slot task, c-chunk of CI outputs, row group)
//               -> y[perm[row]][c-chunk] += s_a * (sum_kc vpart) B
#include "common.cuh"
#include "kernels.h"

namespace lora {

namespace {

template <int R>
struct SimtCfg {
  static constexpr int NWC = 8;          // consumer warps
  static constexpr int NCT = NWC * 32;   // consumer threads
  static constexpr int THREADS = NCT + 32;
  static constexpr int GR = kGroupRows;  // rows per group
  // shrink
  static constexpr int KL = R < 32 ? R : 32;  // lanes along k
  static constexpr int KPL = R / KL;          // k per lane
  static constexpr int NJG = NCT / KL;        // j-groups
  static constexpr int SJ_MAX = R == 64 ? 256 : (R == 32 ? 512 : 1024);
  static constexpr int A_STAGE = R * SJ_MAX * 2;
  static constexpr int X_STAGE = GR * SJ_MAX * 2;
  static constexpr int S_STAGE = A_STAGE + X_STAGE;
  static constexpr int RED_BYTES = NJG * GR * R * 4;
  static constexpr int NST_RAW = (200 * 1024 - RED_BYTES) / S_STAGE;
  static constexpr int NST = NST_RAW > 8 ? 8 : (NST_RAW < 2 ? 2 : NST_RAW);
  static constexpr int SHRINK_SMEM = 1024 + NST * S_STAGE + RED_BYTES + 2 * NST * 8;
  // expand
  static constexpr int SC_MAX = 16384 / R;  // 32 KB of B rows per stage
  static constexpr int B_STAGE = SC_MAX * R * 2;
  static constexpr int NSTE = 6;
  static constexpr int VS_BYTES = GR * R * 4;
  static constexpr int EXPAND_SMEM = 1024 + NSTE * B_STAGE + VS_BYTES + 2 * NSTE * 8;
  static_assert(S_STAGE % 1024 == 0 && B_STAGE % 1024 == 0, "stage alignment");
};

LORA_DEVINL uint8_t* align1024(uint8_t* p) {
  const uint32_t a = smem_u32(p);
  return p + (((a + 1023u) & ~1023u) - a);
}

// locate the task owning global chunk index `g` (prefix sums in args)
LORA_DEVINL int find_task_kc(const MultiArgs& args, int g) {
  int t = 0;
  while (t + 1 < args.n_tasks && args.t[t + 1].kc_base <= g) ++t;
  return t;
}
LORA_DEVINL int find_task_ci(const MultiArgs& args, int g) {
  int t = 0;
  while (t + 1 < args.n_tasks && args.t[t + 1].ci_base <= g) ++t;
  return t;
}

LORA_DEVINL long long unit_of_key(int key, int E, int world) {
  const int a = key / E, e = key - a * E;
  return (long long)(a / world) * E + e;
}

LORA_DEVINL void fma8(float& acc, const uint4& w, const float* xf) {
  acc = fmaf(bf16lo(w.x), xf[0], acc);
  acc = fmaf(bf16hi(w.x), xf[1], acc);
  acc = fmaf(bf16lo(w.y), xf[2], acc);
  acc = fmaf(bf16hi(w.y), xf[3], acc);
  acc = fmaf(bf16lo(w.z), xf[4], acc);
  acc = fmaf(bf16hi(w.z), xf[5], acc);
  acc = fmaf(bf16lo(w.w), xf[6], acc);
  acc = fmaf(bf16hi(w.w), xf[7], acc);
}
LORA_DEVINL void unpack8(const uint4& w, float* f) {
  f[0] = bf16lo(w.x); f[1] = bf16hi(w.x);
  f[2] = bf16lo(w.y); f[3] = bf16hi(w.y);
  f[4] = bf16lo(w.z); f[5] = bf16hi(w.z);
  f[6] = bf16lo(w.w); f[7] = bf16hi(w.w);
}

// ---------------------------------------------------------------------------
// shrink
// ---------------------------------------------------------------------------
template <int R>
__global__ void __launch_bounds__(SimtCfg<R>::THREADS, 1)
    simt_shrink_kernel(const __grid_constant__ MultiArgs args, const PlanDev pd) {
  using C = SimtCfg<R>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  float* red = reinterpret_cast<float*>(smem + C::NST * C::S_STAGE);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::NST * C::S_STAGE + C::RED_BYTES);
  uint64_t* empty = full + C::NST;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], C::NWC);
    }
    fence_mbar_init();
  }
  __syncthreads();

  const int n_groups = pd.counts[kCntGroups];
  const long long n_items = (long long)n_groups * args.total_kc;
  const int warp = warp_id(), lane = lane_id();

  if (warp == C::NWC) {
    // ===================== producer =====================
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int stage = 0;
      uint32_t phase = 0;
      for (long long it = blockIdx.x; it < n_items; it += gridDim.x) {
        const int kcg = (int)(it / n_groups), gi = (int)(it - (long long)kcg * n_groups);
        const SlotTask& t = args.t[find_task_kc(args, kcg)];
        const int kc = kcg - t.kc_base;
        const int4 g = pd.groups[gi];
        const long long unit = unit_of_key(g.z, t.E, args.world);
        const int tiles_per_unit = t.h_in >> 6;
        const uint16_t* abase = t.At + ((unit * tiles_per_unit + ((kc * t.KI) >> 6)) * (long long)R * 64);
        const int n_st = t.KI / t.SJ;
        const uint32_t a_bytes = (uint32_t)R * t.SJ * 2, x_bytes = (uint32_t)t.SJ * 2;
        for (int st = 0; st < n_st; ++st) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sA = smem + stage * C::S_STAGE;
          uint8_t* sX = sA + C::A_STAGE;
          mbar_arrive_expect_tx(&full[stage], a_bytes + x_bytes * g.y);
          bulk_g2s_hint(sA, abase + (long long)((st * t.SJ) >> 6) * R * 64, a_bytes, &full[stage], pol);
          const long long jofs = (long long)kc * t.KI + (long long)st * t.SJ;
          for (int r = 0; r < g.y; ++r) {
            const long long row = pd.perm[g.x + r];
            bulk_g2s(sX + r * x_bytes, t.x + row * t.h_in + jofs, x_bytes, &full[stage]);
          }
          if (++stage == C::NST) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
    return;
  }

  // ===================== consumers =====================
  const int ct = threadIdx.x;  // 0..NCT-1
  const int kl = ct % C::KL, jg = ct / C::KL;
  int stage = 0;
  uint32_t phase = 0;
  for (long long it = blockIdx.x; it < n_items; it += gridDim.x) {
    const int kcg = (int)(it / n_groups), gi = (int)(it - (long long)kcg * n_groups);
    const SlotTask& t = args.t[find_task_kc(args, kcg)];
    const int kc = kcg - t.kc_base;
    const int4 g = pd.groups[gi];
    const int rows = g.y;
    const int n_st = t.KI / t.SJ;
    const int nchunk = t.SJ >> 3;  // 16-byte chunks along j per stage

    float acc[C::KPL][C::GR];
#pragma unroll
    for (int kk = 0; kk < C::KPL; ++kk)
#pragma unroll
      for (int r = 0; r < C::GR; ++r) acc[kk][r] = 0.f;

    for (int st = 0; st < n_st; ++st) {
      mbar_wait(&full[stage], phase);
      const uint32_t a_s = smem_u32(smem + stage * C::S_STAGE);
      const uint32_t x_s = a_s + C::A_STAGE;
      for (int c = jg; c < nchunk; c += C::NJG) {
        const int tile = c >> 3, q = c & 7;
        uint4 w[C::KPL];
#pragma unroll
        for (int kk = 0; kk < C::KPL; ++kk) {
          const int k = kl + kk * 32;
          w[kk] = lds128(a_s + tile * (R * 128) + k * 128 + ((q ^ (k & 7)) << 4));
        }
#pragma unroll
        for (int r = 0; r < C::GR; ++r) {
          if (r < rows) {
            float xf[8];
            unpack8(lds128(x_s + r * (t.SJ * 2) + (c << 4)), xf);
#pragma unroll
            for (int kk = 0; kk < C::KPL; ++kk) fma8(acc[kk][r], w[kk], xf);
          }
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
      for (int r = 0; r < C::GR; ++r)
        if (r < rows) red[(jg * C::GR + r) * R + kl + kk * 32] = acc[kk][r];
    named_bar_sync(1, C::NCT);
    float* vp = pd.vpart + t.vpart_off + ((long long)kc * pd.max_rows + g.x) * R;
    for (int idx = ct; idx < rows * R; idx += C::NCT) {
      const int r = idx / R, k = idx - r * R;
      float s = 0.f;
      for (int q = 0; q < C::NJG; ++q) s += red[(q * C::GR + r) * R + k];
      vp[idx] = s;
    }
  }
}

// ---------------------------------------------------------------------------
// expand + scale + scatter-accumulate
// ---------------------------------------------------------------------------
template <int R>
__global__ void __launch_bounds__(SimtCfg<R>::THREADS, 1)
    simt_expand_kernel(const __grid_constant__ MultiArgs args, const PlanDev pd) {
  using C = SimtCfg<R>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  float* vs = reinterpret_cast<float*>(smem + C::NSTE * C::B_STAGE);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::NSTE * C::B_STAGE + C::VS_BYTES);
  uint64_t* empty = full + C::NSTE;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::NSTE; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], C::NWC);
    }
    fence_mbar_init();
  }
  __syncthreads();

  const int n_groups = pd.counts[kCntGroups];
  const long long n_items = (long long)n_groups * args.total_ci;
  const int warp = warp_id(), lane = lane_id();

  if (warp == C::NWC) {
    // ===================== producer =====================
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int stage = 0;
      uint32_t phase = 0;
      for (long long it = blockIdx.x; it < n_items; it += gridDim.x) {
        const int cig = (int)(it / n_groups), gi = (int)(it - (long long)cig * n_groups);
        const SlotTask& t = args.t[find_task_ci(args, cig)];
        const int ci = cig - t.ci_base;
        const int4 g = pd.groups[gi];
        const long long unit = unit_of_key(g.z, t.E, args.world);
        const uint16_t* bbase = t.Bt + (unit * t.h_out + (long long)ci * t.CI) * R;
        const int n_st = t.CI / t.SC;
        const uint32_t bytes = (uint32_t)t.SC * R * 2;
        for (int st = 0; st < n_st; ++st) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], bytes);
          bulk_g2s_hint(smem + stage * C::B_STAGE, bbase + (long long)st * t.SC * R, bytes, &full[stage], pol);
          if (++stage == C::NSTE) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
    return;
  }

  // ===================== consumers =====================
  const int ct = threadIdx.x;
  const uint32_t vs_s = smem_u32(vs);
  int stage = 0;
  uint32_t phase = 0;
  for (long long it = blockIdx.x; it < n_items; it += gridDim.x) {
    const int cig = (int)(it / n_groups), gi = (int)(it - (long long)cig * n_groups);
    const SlotTask& t = args.t[find_task_ci(args, cig)];
    const int ci = cig - t.ci_base;
    const int4 g = pd.groups[gi];
    const int rows = g.y;
    const int a = g.z / t.E;
    const float s_a = args.scale[a];
    long long yrow[C::GR];
#pragma unroll
    for (int r = 0; r < C::GR; ++r) yrow[r] = (r < rows) ? (long long)pd.perm[g.x + r] * t.h_out : 0;

    // v = sum over k-chunks of the shrink partials (fixed order)
    named_bar_sync(1, C::NCT);
    {
      const float* vp = pd.vpart + t.vpart_off + (long long)g.x * R;
      const long long kstride = (long long)pd.max_rows * R;
      for (int idx = ct; idx < rows * R; idx += C::NCT) {
        float v = 0.f;
        for (int kc = 0; kc < t.n_kc; ++kc) v += vp[kc * kstride + idx];
        vs[idx] = v;
      }
    }
    named_bar_sync(1, C::NCT);

    const int n_st = t.CI / t.SC;
    for (int st = 0; st < n_st; ++st) {
      mbar_wait(&full[stage], phase);
      const uint32_t b_s = smem_u32(smem + stage * C::B_STAGE);
      for (int cr = ct; cr < t.SC; cr += C::NCT) {
        float acc[C::GR];
#pragma unroll
        for (int r = 0; r < C::GR; ++r) acc[r] = 0.f;
#pragma unroll
        for (int ch = 0; ch < R / 8; ++ch) {
          float bf[8];
          unpack8(lds128(b_s + cr * (R * 2) + (swz_row_chunk(cr, ch, R * 2) << 4)), bf);
#pragma unroll
          for (int r = 0; r < C::GR; ++r) {
            if (r < rows) {
              const float4 v0 = lds128f(vs_s + (r * R + ch * 8) * 4);
              const float4 v1 = lds128f(vs_s + (r * R + ch * 8 + 4) * 4);
              acc[r] = fmaf(v0.x, bf[0], acc[r]);
              acc[r] = fmaf(v0.y, bf[1], acc[r]);
              acc[r] = fmaf(v0.z, bf[2], acc[r]);
              acc[r] = fmaf(v0.w, bf[3], acc[r]);
              acc[r] = fmaf(v1.x, bf[4], acc[r]);
              acc[r] = fmaf(v1.y, bf[5], acc[r]);
              acc[r] = fmaf(v1.z, bf[6], acc[r]);
              acc[r] = fmaf(v1.w, bf[7], acc[r]);
            }
          }
        }
        const long long c = (long long)ci * t.CI + (long long)st * t.SC + cr;
        if (args.y_store) {
          float* y = reinterpret_cast<float*>(t.y);
#pragma unroll
          for (int r = 0; r < C::GR; ++r)
            if (r < rows) y[yrow[r] + c] = s_a * acc[r];
        } else if (args.y_fp32) {
          float* y = reinterpret_cast<float*>(t.y);
#pragma unroll
          for (int r = 0; r < C::GR; ++r)
            if (r < rows) {
              float* p = y + yrow[r] + c;
              *p = *p + s_a * acc[r];
            }
        } else {
          uint16_t* y = reinterpret_cast<uint16_t*>(t.y);
#pragma unroll
          for (int r = 0; r < C::GR; ++r)
            if (r < rows) {
              uint16_t* p = y + yrow[r] + c;
              *p = f32_to_bf16_rne(bf16_to_f32(*p) + s_a * acc[r]);
            }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == C::NSTE) {
        stage = 0;
        phase ^= 1;
      }
    }
  }
}

template <int R>
cudaError_t launch_shrink_t(const MultiArgs& args, const PlanDev& pd, int grid, cudaStream_t stream) {
  using C = SimtCfg<R>;
  static unsigned long long attr = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(attr & (1ull << dev))) {
    cudaError_t e = cudaFuncSetAttribute(simt_shrink_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         C::SHRINK_SMEM);
    if (e != cudaSuccess) return e;
    attr |= 1ull << dev;
  }
  simt_shrink_kernel<R><<<grid, C::THREADS, C::SHRINK_SMEM, stream>>>(args, pd);
  return cudaGetLastError();
}

template <int R>
cudaError_t launch_expand_t(const MultiArgs& args, const PlanDev& pd, int grid, cudaStream_t stream) {
  using C = SimtCfg<R>;
  static unsigned long long attr = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(attr & (1ull << dev))) {
    cudaError_t e = cudaFuncSetAttribute(simt_expand_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         C::EXPAND_SMEM);
    if (e != cudaSuccess) return e;
    attr |= 1ull << dev;
  }
  simt_expand_kernel<R><<<grid, C::THREADS, C::EXPAND_SMEM, stream>>>(args, pd);
  return cudaGetLastError();
}

}  // namespace

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
int simt_sc_max(int rank) { return 16384 / rank; }
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
