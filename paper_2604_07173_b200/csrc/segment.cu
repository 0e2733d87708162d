// segment.cu -- a1: device-side segmentation (K8 in SURVEY 2b).
//
// Stable sort of the valid rows (a >= 0) by key a*E + e, ties broken by the
// original row index, plus the per-segment work lists the shrink / expand
// kernels consume.  SGMV "aggregat[es] tokens that share the same LoRA
// adapter into a single GEMM" (App. A.2.2); the paper presumes the
// segments, so this kernel is ours (R9 for the ordering contract).
//
// One CTA of 1024 threads.  Each row becomes the 64-bit composite
// (key << 32) | row; composites are unique, so ANY correct sort of them is
// the stable sort by key -- a bitonic network over <= 16384 composites held
// in shared memory (128 KB) is deterministic and bit-exact.
#include "common.cuh"
#include "kernels.h"

namespace lora {

namespace {

constexpr int kSegThreads = 1024;

// Block-wide exclusive scan of one int per thread.  Returns the exclusive
// prefix; *total receives the block sum.  `tmp` holds >= 33 ints.
__device__ int block_exclusive_scan(int v, int* tmp, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) tmp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = (lane < (kSegThreads / 32)) ? tmp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    tmp[lane] = w;  // inclusive prefix of warp sums
  }
  __syncthreads();
  const int warp_excl = (warp == 0) ? 0 : tmp[warp - 1];
  const int tot = tmp[kSegThreads / 32 - 1];
  __syncthreads();
  *total = tot;
  return warp_excl + x - v;
}

__global__ void __launch_bounds__(kSegThreads, 1)
    segment_kernel(const int32_t* __restrict__ adapter_ids, const int32_t* __restrict__ expert_ids, int T,
                   int P, int E, int n_adapters, int world, int shard_rank, SegParams sp, PlanDev pd,
                   int* __restrict__ err_flag) {
  extern __shared__ __align__(16) unsigned long long keys[];  // [P]
  __shared__ int scan_tmp[40];
  const int tid = threadIdx.x;
  const unsigned long long kInvalid = ~0ull;

  // 1. composites
  int bad = 0;
  for (int i = tid; i < P; i += kSegThreads) {
    unsigned long long c = kInvalid;
    if (i < T) {
      const int a = adapter_ids[i];
      const int e = expert_ids ? expert_ids[i] : 0;
      const bool in_range = (a >= -1) && (a < n_adapters) && (a < 0 || (e >= 0 && e < E)) &&
                            (a < 0 || (a % world) == shard_rank);
      if (!in_range) bad = 1;
      if (in_range && a >= 0) {
        const unsigned key = (unsigned)a * (unsigned)E + (unsigned)e;
        c = ((unsigned long long)key << 32) | (unsigned)i;
      }
    }
    keys[i] = c;
  }
  if (bad) atomicOr(err_flag, 1);
  __syncthreads();

  // 2. bitonic sort, ascending
  for (int k = 2; k <= P; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = tid; i < P; i += kSegThreads) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const unsigned long long x = keys[i], y = keys[ixj];
          const bool up = (i & k) == 0;
          if ((x > y) == up) {
            keys[i] = y;
            keys[ixj] = x;
          }
        }
      }
      __syncthreads();
    }
  }

  // 3. n_valid = index of the first invalid composite
  __shared__ int s_nvalid;
  if (tid == 0) s_nvalid = (keys[0] == kInvalid) ? 0 : P;
  __syncthreads();
  for (int i = tid; i + 1 < P; i += kSegThreads)
    if (keys[i] != kInvalid && keys[i + 1] == kInvalid) s_nvalid = i + 1;
  __syncthreads();
  const int n_valid = s_nvalid;

  // 4. perm + segment heads (each thread a contiguous chunk, so the scan is in order)
  const int chunk = (n_valid + kSegThreads - 1) / kSegThreads;
  const int j0 = min(tid * chunk, n_valid), j1 = min(j0 + chunk, n_valid);
  int heads = 0;
  for (int j = j0; j < j1; ++j) {
    const unsigned long long c = keys[j];
    pd.perm[j] = (int32_t)(c & 0xffffffffu);
    if (j == 0 || (keys[j - 1] >> 32) != (c >> 32)) ++heads;
  }
  int S;
  int seg = block_exclusive_scan(heads, scan_tmp, &S);
  for (int j = j0; j < j1; ++j) {
    const unsigned long long c = keys[j];
    if (j == 0 || (keys[j - 1] >> 32) != (c >> 32)) {
      pd.seg_off[seg] = j;
      pd.seg_key[seg] = (int32_t)(c >> 32);
      ++seg;
    }
  }
  if (tid == 0) pd.seg_off[S] = n_valid;
  __syncthreads();  // global writes of this block visible to the block

  // 5. work lists: CUDA-core groups (<= kGroupRows rows) and tcgen05 tiles (<= sp.tile_rows)
  const int schunk = (S + kSegThreads - 1) / kSegThreads;
  const int s0 = min(tid * schunk, S), s1 = min(s0 + schunk, S);
  int ng = 0, nt = 0;
  for (int s = s0; s < s1; ++s) {
    const int size = pd.seg_off[s + 1] - pd.seg_off[s];
    if (sp.tc_enabled && size > sp.small_max)
      nt += (size + sp.tile_rows - 1) / sp.tile_rows;
    else
      ng += (size + kGroupRows - 1) / kGroupRows;
  }
  int NG, NT;
  int g = block_exclusive_scan(ng, scan_tmp, &NG);
  int t = block_exclusive_scan(nt, scan_tmp, &NT);
  for (int s = s0; s < s1; ++s) {
    const int b = pd.seg_off[s], size = pd.seg_off[s + 1] - b, key = pd.seg_key[s];
    const bool tc = sp.tc_enabled && size > sp.small_max;
    const int cap = tc ? sp.tile_rows : kGroupRows;
    const int n = (size + cap - 1) / cap;
    // near-equal split: the first (size % n) pieces get one extra row
    const int base = size / n, extra = size % n;
    int r = b;
    for (int q = 0; q < n; ++q) {
      const int len = base + (q < extra ? 1 : 0);
      const int4 w = make_int4(r, len, key, s);
      if (tc)
        pd.tiles[t++] = w;
      else
        pd.groups[g++] = w;
      r += len;
    }
  }
  if (tid == 0) {
    pd.counts[kCntValid] = n_valid;
    pd.counts[kCntSegs] = S;
    pd.counts[kCntGroups] = NG;
    pd.counts[kCntTiles] = NT;
  }
}

}  // namespace

int segment_smem_bytes(int P) { return P * 8; }

cudaError_t launch_segment(const int32_t* adapter_ids, const int32_t* expert_ids, int T, int E, int n_adapters,
                           int world, int shard_rank, const SegParams& sp, const PlanDev& pd, int* err_flag,
                           cudaStream_t stream) {
  int P = 1;
  while (P < T) P <<= 1;
  if (P < 2) P = 2;
  const int smem = segment_smem_bytes(P);
  static unsigned long long attr_set = 0;  // per-device bitmask
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(attr_set & (1ull << dev))) {
    cudaError_t e = cudaFuncSetAttribute(segment_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         segment_smem_bytes(kMaxPlanRows));
    if (e != cudaSuccess) return e;
    attr_set |= 1ull << dev;
  }
  segment_kernel<<<1, kSegThreads, smem, stream>>>(adapter_ids, expert_ids, T, P, E, n_adapters, world,
                                                   shard_rank, sp, pd, err_flag);
  return cudaGetLastError();
}

}  // namespace lora
