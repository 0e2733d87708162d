// segment.cu -- a1: device-side segmentation (K8 in SURVEY 2b).
//
// Stable sort of the valid rows (a >= 0) by key a*E + e, ties broken by the
// original row index, plus the per-segment work lists the shrink / expand
// kernels consume.  SGMV "aggregat[es] tokens that share the same LoRA
// adapter into a single GEMM" (App. A.2.2); the paper presumes the
// segments, so this kernel is ours (R9 for the ordering contract).
//
// One CTA of 1024 threads, everything in shared memory (T <= 16384); larger
// batches (up to 32768 rows) always take the multi-CTA path below.
//  * Fast path: 32-bit composites (key << ib) | row with an LSD radix sort on
//    the key bits, 8 bits per pass.  Each pass is a stable block-wide counting
//    sort (warp-synchronous multisplit + a block scan over (digit, warp)).
//    Rows enter in index order and every pass is stable, so ties keep the
//    original row order -- bit-exact with the stable-sort definition.
//  * Fallback (key bits + row bits > 32): 64-bit composites sorted with a
//    bitonic network; composites are unique, so any correct sort of them is
//    the stable sort by key.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace lora {

namespace {

constexpr int kSegThreads = 1024;

#ifdef LORA_SEG_PROF
__device__ long long g_seg_t[16];
#define SEG_T(k) do { if (threadIdx.x == 0) g_seg_t[k] = clock64(); } while (0)
#else
#define SEG_T(k) do {} while (0)
#endif

// Block-wide exclusive scan of one int per thread (NT threads).  Returns the
// exclusive prefix; *total receives the block sum.  `tmp` holds >= 33 ints.
template <int NT = kSegThreads>
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
    int w = (lane < (NT / 32)) ? tmp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    tmp[lane] = w;  // inclusive prefix of warp sums
  }
  __syncthreads();
  const int warp_excl = (warp == 0) ? 0 : tmp[warp - 1];
  const int tot = tmp[NT / 32 - 1];
  __syncthreads();
  *total = tot;
  return warp_excl + x - v;
}

// Key of one row (a*E+e), or -1 for "no LoRA" / out of
// range (flagged through *bad).
LORA_DEVINL int key_of(int a, int e, int E, int n_adapters, const Placement& pl, int& bad, const int32_t* cache) {
  const bool in_range = (a >= -1) && (a < n_adapters) && (a < 0 || (e >= 0 && e < E)) &&
                        (a < 0 || pl.owns_unit(a, e)) && (a < 0 || !cache || cache[a] >= 0);
  if (!in_range) bad = 1;
  return (in_range && a >= 0) ? a * E + e : -1;
}
LORA_DEVINL int row_key(const int32_t* __restrict__ adapter_ids, const int32_t* __restrict__ expert_ids, int i, int E,
                        int n_adapters, const Placement& pl, int& bad, const int32_t* cache) {
  return key_of(adapter_ids[i], expert_ids ? expert_ids[i] : 0, E, n_adapters, pl, bad, cache);
}

// ---------------------------------------------------------------------------
// radix path
// ---------------------------------------------------------------------------
// Composite buffers are padded with one word per 32 (index i lives at
// i + i/32): thread t's contiguous run t*EPT.. then falls in 32 distinct banks
// across a warp (EPT in 1..16), so the blocked-layout accesses are conflict-free.
__host__ __device__ __forceinline__ int pad32(int i) { return i + (i >> 5); }

// One stable counting-sort pass on an 8-bit digit (v >> shift) & 255 --
// warp-synchronous multisplit.  Warp w owns the contiguous index range
// [w*32*EPT, (w+1)*32*EPT) and walks it in rounds of 32 consecutive elements
// (lane order = index order); lanes with equal digits find each other (peer
// mask from 8 ballots; match.any's cost grows with the number of distinct
// values) and take ranks in lane order on top of the warp's running count for
// that digit.  A block scan over (digit, warp) in digit-major order then
// gives every (warp, digit) its output base.  cnt: [NT / 32 warps][256] ints.
template <int EPT, int NT = kSegThreads>
__device__ void radix_pass8(const uint32_t* in, uint32_t* out, int shift, int* cnt, int* scan_tmp) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int* wc = cnt + warp * 256;
#pragma unroll
  for (int q = 0; q < 8; ++q) wc[lane + 32 * q] = 0;
  __syncwarp();
  uint32_t lt;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
  uint32_t v[EPT];
  int loc[EPT];
  const int base_idx = warp * 32 * EPT;
#pragma unroll
  for (int r = 0; r < EPT; ++r) {
    v[r] = in[pad32(base_idx + r * 32 + lane)];
    const int d = (v[r] >> shift) & 255;
    // lanes with the same digit: AND over the 8 digit bits of (ballot or its complement)
    uint32_t peers = 0xffffffffu;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const uint32_t m = __ballot_sync(0xffffffffu, (d >> b) & 1);
      peers &= ((d >> b) & 1) ? m : ~m;
    }
    const int before = wc[d];
    loc[r] = before + __popc(peers & lt);
    __syncwarp();
    if ((peers & lt) == 0) wc[d] = before + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // exclusive scan over (digit, warp), digit-major: 256 x NT/32 entries, 8 per
  // thread -- thread t sums digit t / (NT/256), warps 8 (t % (NT/256)) .. +8
  static_assert(NT % 256 == 0, "radix pass thread count");
  constexpr int DPT = NT / 256;
  const int d0 = tid / DPT, w0 = (tid % DPT) * 8;
  int c[8], sum = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    c[q] = cnt[(w0 + q) * 256 + d0];
    sum += c[q];
  }
  int total;
  int run = block_exclusive_scan<NT>(sum, scan_tmp, &total);
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    cnt[(w0 + q) * 256 + d0] = run;
    run += c[q];
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < EPT; ++r) {
    const int d = (v[r] >> shift) & 255;
    out[pad32(wc[d] + loc[r])] = v[r];
  }
  __syncthreads();
}

// builds composites and sorts them; returns the buffer holding the result
template <int EPT, int NT>
__device__ uint32_t* radix_sort(const int32_t* __restrict__ adapter_ids, const int32_t* __restrict__ expert_ids,
                                int T, int E, int n_adapters, const Placement& pl, const int32_t* cache, int K, int kb, int ib,
                                uint32_t* A, uint32_t* B, int* cnt, int* err_flag, int* n_valid_out,
                                int* scan_tmp) {
  const int tid = threadIdx.x;
  int bad = 0, nv = 0;
  // composites in row order; rows read coalesced (row r*1024 + tid) -- the
  // passes below read the array by index, not by thread.  All id loads are
  // issued before any key is formed (one memory latency, not EPT).
  int ad[EPT], ex[EPT];
#pragma unroll
  for (int r = 0; r < EPT; ++r) {
    const int i = r * NT + tid;
    ad[r] = i < T ? __ldg(adapter_ids + i) : -1;
    ex[r] = (i < T && expert_ids) ? __ldg(expert_ids + i) : 0;
  }
#pragma unroll
  for (int r = 0; r < EPT; ++r) {
    const int i = r * NT + tid;
    int key = -1;
    if (i < T) key = key_of(ad[r], ex[r], E, n_adapters, pl, bad, cache);
    nv += key >= 0;
    A[pad32(i)] = ((uint32_t)(key >= 0 ? key : K) << ib) | (uint32_t)i;
  }
  if (bad) atomicOr(err_flag, 1);
  int total;
  SEG_T(1);
  block_exclusive_scan<NT>(nv, scan_tmp, &total);  // its barriers also publish A
  SEG_T(2);
  *n_valid_out = total;
  uint32_t* in = A;
  uint32_t* out = B;
  for (int sh = 0; sh < kb; sh += 8) {
    radix_pass8<EPT, NT>(in, out, ib + sh, cnt, scan_tmp);
    SEG_T(3 + sh / 8);
    uint32_t* t = in;
    in = out;
    out = t;
  }
  return in;
}

// ---------------------------------------------------------------------------
// bitonic fallback on 64-bit composites
// ---------------------------------------------------------------------------
LORA_DEVINL unsigned long long umin64(unsigned long long a, unsigned long long b) { return a < b ? a : b; }
LORA_DEVINL unsigned long long umax64(unsigned long long a, unsigned long long b) { return a < b ? b : a; }

template <int EPT>
__device__ void bitonic_sort(const int32_t* __restrict__ adapter_ids, const int32_t* __restrict__ expert_ids, int T,
                             int E, int n_adapters, const Placement& pl, const int32_t* cache, unsigned long long* sm, int* err_flag,
                             int* n_valid_out, int* scan_tmp) {
  constexpr int P = kSegThreads * EPT;
  const int tid = threadIdx.x;
  unsigned long long v[EPT];
  int bad = 0, nv = 0;
#pragma unroll
  for (int r = 0; r < EPT; ++r) {
    const int i = tid * EPT + r;
    int key = -1;
    if (i < T) key = row_key(adapter_ids, expert_ids, i, E, n_adapters, pl, bad, cache);
    nv += key >= 0;
    v[r] = key >= 0 ? (((unsigned long long)(unsigned)key << 32) | (unsigned)i) : ~0ull;
  }
  if (bad) atomicOr(err_flag, 1);
  int total;
  block_exclusive_scan(nv, scan_tmp, &total);
  *n_valid_out = total;
  for (int k = 2; k <= P; k <<= 1) {
    int j = k >> 1;
    for (; j >= 32 * EPT; j >>= 1) {  // shared memory
      __syncthreads();
#pragma unroll
      for (int r = 0; r < EPT; ++r) sm[tid * EPT + r] = v[r];
      __syncthreads();
#pragma unroll
      for (int r = 0; r < EPT; ++r) {
        const int i = tid * EPT + r;
        const unsigned long long o = sm[i ^ j];
        const bool take_min = ((i & j) == 0) == ((i & k) == 0);
        v[r] = take_min ? umin64(v[r], o) : umax64(v[r], o);
      }
    }
    for (; j >= EPT; j >>= 1) {  // warp shuffles
      const int lj = j / EPT;
#pragma unroll
      for (int r = 0; r < EPT; ++r) {
        const int i = tid * EPT + r;
        const unsigned long long o = __shfl_xor_sync(0xffffffffu, v[r], lj);
        const bool take_min = ((i & j) == 0) == ((i & k) == 0);
        v[r] = take_min ? umin64(v[r], o) : umax64(v[r], o);
      }
    }
#pragma unroll
    for (int jj = EPT / 2; jj > 0; jj >>= 1) {  // registers
      if (jj < k) {
#pragma unroll
        for (int r = 0; r < EPT; ++r) {
          const int p = r ^ jj;
          if (p > r) {
            const bool up = ((tid * EPT + r) & k) == 0;
            const unsigned long long a = v[r], b = v[p];
            if ((a > b) == up) {
              v[r] = b;
              v[p] = a;
            }
          }
        }
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < EPT; ++r) sm[tid * EPT + r] = v[r];
  __syncthreads();
}

// ---------------------------------------------------------------------------
// kernel
// ---------------------------------------------------------------------------
// NT threads: 1024, or 256 / 512 for small batches (radix path only; the
// block-wide barriers and scans of a smaller CTA are cheaper)
template <bool radix, int NT>
__global__ void __launch_bounds__(NT, 1)
    segment_kernel(const int32_t* __restrict__ adapter_ids, const int32_t* __restrict__ expert_ids, int T, int P,
                   int E, int n_adapters, int kb, int ib, SegParams sp, PlanDev pd,
                   int* __restrict__ err_flag, const int* __restrict__ T_dev) {
  extern __shared__ __align__(16) uint8_t seg_smem[];
  pdl_launch_dependents();  // the shrink kernels may launch now; they wait for this grid
  SEG_T(0);
  if (T_dev) {
    // row count known only on the device (the sharded owner's received rows):
    // T and P above are the capacity the shared memory was sized for; sort
    // only the actual rows (P = the padded size of those, fewer radix rounds)
    T = min(T, max(*T_dev, 0));
    int p2 = NT;
    while (p2 < T) p2 <<= 1;
    P = p2;
    int b = 0;
    while ((1 << b) <= P - 1) ++b;
    ib = b;
  }
  const Placement pl = sp.pl;
  const int32_t* cache = sp.cache;
  __shared__ int scan_tmp[40];
  __shared__ int s_nvalid;
  const int tid = threadIdx.x;
  const int EPT = P / NT;

  // 1.+2. composites + sort; afterwards key(j) / row(j) of sorted position j
  const uint32_t* srt32 = nullptr;
  const unsigned long long* srt64 = nullptr;
  int* segoff_s;  // [P+1] segment offsets in shared memory
  if constexpr (radix) {
    uint32_t* A = reinterpret_cast<uint32_t*>(seg_smem);
    uint32_t* B = A + pad32(P) + 4;  // each buffer pad32(P)+4 ints: the free one later holds P+1 segment offsets
    int* cnt = reinterpret_cast<int*>(B + pad32(P) + 4);  // [32 warps][256] digit counts
    const int K = n_adapters * E;
    uint32_t* res = nullptr;
    switch (EPT) {
      case 1: res = radix_sort<1, NT>(adapter_ids, expert_ids, T, E, n_adapters, pl, cache, K, kb, ib, A, B, cnt, err_flag, &s_nvalid, scan_tmp); break;
      case 2: res = radix_sort<2, NT>(adapter_ids, expert_ids, T, E, n_adapters, pl, cache, K, kb, ib, A, B, cnt, err_flag, &s_nvalid, scan_tmp); break;
      case 4: res = radix_sort<4, NT>(adapter_ids, expert_ids, T, E, n_adapters, pl, cache, K, kb, ib, A, B, cnt, err_flag, &s_nvalid, scan_tmp); break;
      case 8: res = radix_sort<8, NT>(adapter_ids, expert_ids, T, E, n_adapters, pl, cache, K, kb, ib, A, B, cnt, err_flag, &s_nvalid, scan_tmp); break;
      default: res = radix_sort<16, NT>(adapter_ids, expert_ids, T, E, n_adapters, pl, cache, K, kb, ib, A, B, cnt, err_flag, &s_nvalid, scan_tmp); break;
    }
    srt32 = res;
    segoff_s = reinterpret_cast<int*>(res == A ? B : A);  // the free buffer (P + 1 ints reserved)
  } else {
    unsigned long long* S64 = reinterpret_cast<unsigned long long*>(seg_smem);
    switch (EPT) {
      case 1: bitonic_sort<1>(adapter_ids, expert_ids, T, E, n_adapters, pl, cache, S64, err_flag, &s_nvalid, scan_tmp); break;
      case 2: bitonic_sort<2>(adapter_ids, expert_ids, T, E, n_adapters, pl, cache, S64, err_flag, &s_nvalid, scan_tmp); break;
      case 4: bitonic_sort<4>(adapter_ids, expert_ids, T, E, n_adapters, pl, cache, S64, err_flag, &s_nvalid, scan_tmp); break;
      case 8: bitonic_sort<8>(adapter_ids, expert_ids, T, E, n_adapters, pl, cache, S64, err_flag, &s_nvalid, scan_tmp); break;
      default: bitonic_sort<16>(adapter_ids, expert_ids, T, E, n_adapters, pl, cache, S64, err_flag, &s_nvalid, scan_tmp); break;
    }
    srt64 = S64;
    segoff_s = reinterpret_cast<int*>(S64 + P);
  }
  __syncthreads();
  const int n_valid = s_nvalid;
  const uint32_t idx_mask = (1u << ib) - 1u;
  auto key_at = [&](int j) -> int {
    if constexpr (radix) return (int)(srt32[pad32(j)] >> ib);
    else return (int)(srt64[j] >> 32);
  };
  auto row_at = [&](int j) -> int {
    if constexpr (radix) return (int)(srt32[pad32(j)] & idx_mask);
    else return (int)(srt64[j] & 0xffffffffu);
  };

  SEG_T(6);
  // 3. perm + segment heads (each thread a contiguous chunk, so the scan is in order)
  const int chunk = (n_valid + NT - 1) / NT;
  const int j0 = min(tid * chunk, n_valid), j1 = min(j0 + chunk, n_valid);
  // perm written coalesced (position tid + 1024 m), heads counted per chunk
  for (int j = tid; j < n_valid; j += NT) pd.perm[j] = row_at(j);
  int heads = 0;
  int prev = j0 > 0 ? key_at(j0 - 1) : -1;
  for (int j = j0; j < j1; ++j) {
    const int k = key_at(j);
    heads += (j == 0 || k != prev);
    prev = k;
  }
  int S;
  int seg = block_exclusive_scan<NT>(heads, scan_tmp, &S);
  prev = j0 > 0 ? key_at(j0 - 1) : -1;
  for (int j = j0; j < j1; ++j) {
    const int k = key_at(j);
    if (j == 0 || k != prev) {
      segoff_s[seg] = j;
      pd.seg_off[seg] = j;
      pd.seg_key[seg] = k;
      ++seg;
    }
    prev = k;
  }
  if (tid == 0) {
    segoff_s[S] = n_valid;
    pd.seg_off[S] = n_valid;
  }
  __syncthreads();

  SEG_T(7);
  // 4. work lists: CUDA-core groups (<= kGroupRows rows) and tcgen05 tiles (<= sp.tile_rows)
  const int schunk = (S + NT - 1) / NT;
  const int s0 = min(tid * schunk, S), s1 = min(s0 + schunk, S);
  // the tcgen05 chain only pays off with enough rows in large segments
  // (a handful of tiles run latency-bound on a few SMs): else all groups
  int big = 0;
  for (int s = s0; s < s1; ++s) {
    const int size = segoff_s[s + 1] - segoff_s[s];
    if (size > sp.small_max) big += size;
  }
  int BIG;
  (void)block_exclusive_scan<NT>(big, scan_tmp, &BIG);
  const bool use_tc = sp.tc_enabled && BIG >= sp.tc_min_rows;
  int ng = 0, nt = 0;
  for (int s = s0; s < s1; ++s) {
    const int size = segoff_s[s + 1] - segoff_s[s];
    if (use_tc && size > sp.small_max)
      nt += (size + sp.tile_rows - 1) / sp.tile_rows;
    else
      ng += (size + sp.group_rows - 1) / sp.group_rows;
  }
  // both list counts in one scan (each < 2^16: T <= 32768)
  int NGT;
  const int gt = block_exclusive_scan<NT>(ng | (nt << 16), scan_tmp, &NGT);
  const int NG = NGT & 0xFFFF, NTL = NGT >> 16;
  int g = gt & 0xFFFF, t = gt >> 16;
  for (int s = s0; s < s1; ++s) {
    const int b = segoff_s[s], size = segoff_s[s + 1] - b, key = key_at(b);
    const bool tc = use_tc && size > sp.small_max;
    const int cap = tc ? sp.tile_rows : sp.group_rows;
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
  SEG_T(8);
#ifdef LORA_SEG_PROF
  if (tid == 0) {
    printf("seg T=%d K=%d EPT=%d cycles: ids %lld scan %lld p0 %lld p1 %lld sorted %lld perm+segs %lld lists %lld\n", T,
           n_adapters * E, EPT, g_seg_t[1] - g_seg_t[0], g_seg_t[2] - g_seg_t[1], g_seg_t[3] - g_seg_t[2],
           kb > 8 ? g_seg_t[4] - g_seg_t[3] : 0ll, g_seg_t[6] - g_seg_t[2], g_seg_t[7] - g_seg_t[6], g_seg_t[8] - g_seg_t[7]);
  }
#endif
  if (tid == 0) {
    pd.counts[kCntValid] = n_valid;
    pd.counts[kCntSegs] = S;
    pd.counts[kCntGroups] = NG;
    pd.counts[kCntTiles] = NTL;
  }
}

// ---------------------------------------------------------------------------
// multi-CTA path (T >= kSegMultiMin): one CTA is instruction-bound on the
// composites and passes, so the rows are split over C CTAs.
//   seg_local_kernel   (C CTAs): CTA c sorts its RPC rows by key (stable, the
//                      radix passes above on composites key << 12 | local row),
//                      stores them with each entry's rank inside its key's
//                      run, and the run lengths into hist[key][c]
//   seg_scan_kernel    (1 CTA):  exclusive prefix of hist in (key, c) order --
//                      offs[key][c] = rows of smaller keys + rows of this key
//                      in CTAs before c (this is what keeps the sort stable)
//                      -- zeroes hist for the next build, and builds the
//                      segments and the work lists from the key totals
//   seg_scatter_kernel (C CTAs): perm[offs[key][c] + rank] = row
// ---------------------------------------------------------------------------
constexpr int kLocBits = 12;        // local row bits (RPC <= 4096)
constexpr int kSegKeysMax = 36864;
constexpr int kSegHistSmall = 16384;  // one scan round of the histogram  // key-space bound (the scan CTA keeps K + 1 key starts in smem)

// first index in the sorted composites [0, n) whose key is >= k
LORA_DEVINL int lower_key(const uint32_t* srt, int n, uint32_t k) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if ((srt[pad32(mid)] >> kLocBits) < k) lo = mid + 1; else hi = mid;
  }
  return lo;
}

template <int EPT>
__global__ void __launch_bounds__(kSegThreads, 1)
    seg_local_kernel(const int32_t* __restrict__ adapter_ids, const int32_t* __restrict__ expert_ids, int T, int E,
                     int n_adapters, int kb, int C, SegParams sp, PlanDev pd, int* __restrict__ err_flag,
                     const int* __restrict__ T_dev) {
  constexpr int RPC = kSegThreads * EPT;
  extern __shared__ __align__(16) uint8_t seg_smem[];
  __shared__ int scan_tmp[40];
  uint32_t* A = reinterpret_cast<uint32_t*>(seg_smem);
  uint32_t* B = A + pad32(RPC) + 4;
  int* cnt = reinterpret_cast<int*>(B + pad32(RPC) + 4);
  const int tid = threadIdx.x, c = blockIdx.x;
  const int row0 = c * RPC;
  const uint32_t K = (uint32_t)n_adapters * E;
  if (T_dev) T = min(T, max(*T_dev, 0));  // device-side row count (T: the capacity the grid was sized for)
  pdl_launch_dependents();  // seg_scan (PDL) may be scheduled; it waits for this grid
  if (blockIdx.x == 0) SEG_T(12);
  int ad[EPT], ex[EPT];
#pragma unroll
  for (int r = 0; r < EPT; ++r) {
    const int i = row0 + r * kSegThreads + tid;
    ad[r] = i < T ? __ldg(adapter_ids + i) : -1;
    ex[r] = (i < T && expert_ids) ? __ldg(expert_ids + i) : 0;
  }
  int bad = 0;
#pragma unroll
  for (int r = 0; r < EPT; ++r) {
    const int l = r * kSegThreads + tid;
    int key = -1;
    if (row0 + l < T) key = key_of(ad[r], ex[r], E, n_adapters, sp.pl, bad, sp.cache);
    A[pad32(l)] = ((key >= 0 ? (uint32_t)key : K) << kLocBits) | (uint32_t)l;
  }
  if (bad) atomicOr(err_flag, 1);
  __syncthreads();
  uint32_t* in = A;
  uint32_t* out = B;
  for (int sh = 0; sh < kb; sh += 8) {
    radix_pass8<EPT>(in, out, kLocBits + sh, cnt, scan_tmp);
    uint32_t* t = in;
    in = out;
    out = t;
  }
  if (blockIdx.x == 0) SEG_T(13);
  // sorted: each entry's rank inside its run; the run head records the length
#pragma unroll
  for (int r = 0; r < EPT; ++r) {
    const int p = r * kSegThreads + tid;
    const uint32_t v = in[pad32(p)];
    const uint32_t k = v >> kLocBits;
    int rank = 0;
    if (k < K) {
      const int start = lower_key(in, RPC, k);
      rank = p - start;
      if (rank == 0) pd.hist[(long long)k * C + c] = lower_key(in, RPC, k + 1) - p;
    }
    pd.lsort[row0 + p] = v;
    pd.lrank[row0 + p] = rank;
  }
#ifdef LORA_SEG_PROF
  if (blockIdx.x == 0 && tid == 0)
    printf("local EPT=%d K=%u cycles: sort %lld runs %lld\n", EPT, K, g_seg_t[13] - g_seg_t[12], clock64() - g_seg_t[13]);
#endif
}

__global__ void __launch_bounds__(kSegThreads, 1)
    seg_scan_kernel(int K, int C, SegParams sp, PlanDev pd) {
  extern __shared__ __align__(16) uint8_t seg_smem[];
  __shared__ int scan_tmp[40];
  constexpr int CH = 16;                  // entries per thread per round
  constexpr int ROUND = kSegThreads * CH;
  int* kstart = reinterpret_cast<int*>(seg_smem);  // [pad32(K + 1)] first sorted position of each key
  int* stage = kstart + pad32(K + 1) + 4;          // [pad32(ROUND)]
  const int tid = threadIdx.x;
  const long long N = (long long)K * C;
  int carry = 0;
  pdl_wait();               // seg_local's histogram is complete
  pdl_launch_dependents();  // seg_scatter (PDL) may be scheduled
  SEG_T(9);
  for (long long base = 0; base < N; base += ROUND) {
    const int n = (int)min((long long)ROUND, N - base);
    {
      // all loads of the round in flight at once, then the zeroing stores
      int h[CH];
#pragma unroll
      for (int q = 0; q < CH; ++q) {
        const int i = q * kSegThreads + tid;
        h[q] = i < n ? __ldcg(pd.hist + base + i) : 0;
      }
#pragma unroll
      for (int q = 0; q < CH; ++q) {
        const int i = q * kSegThreads + tid;
        if (i < n) {
          pd.hist[base + i] = 0;
          stage[pad32(i)] = h[q];
        }
      }
    }
    __syncthreads();
    int v[CH], sum = 0;
#pragma unroll
    for (int q = 0; q < CH; ++q) {
      const int i = tid * CH + q;
      v[q] = i < n ? stage[pad32(i)] : 0;
      sum += v[q];
    }
    int total;
    int run = carry + block_exclusive_scan(sum, scan_tmp, &total);
    // key starts: the entries (k, c = 0) of this thread's run, k = kk, kk + 1, ...
    const int e0 = (int)base + tid * CH;
    int kk = (e0 + C - 1) / C;
    int next = kk * C;
#pragma unroll
    for (int q = 0; q < CH; ++q) {
      const int i = tid * CH + q;
      stage[pad32(i)] = run;
      if (i < n && e0 + q == next) {
        kstart[pad32(kk++)] = run;
        next += C;
      }
      run += v[q];
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < CH; ++q) {
      const int i = q * kSegThreads + tid;
      if (i < n) pd.offs[base + i] = stage[pad32(i)];
    }
    carry += total;
    __syncthreads();
  }
  const int n_valid = carry;
  if (tid == 0) kstart[pad32(K)] = n_valid;
  __syncthreads();
  SEG_T(10);

  // segments = keys with rows, in key order; work lists as in the one-CTA path
  const int kchunk = (K + kSegThreads - 1) / kSegThreads;
  const int k0 = min(tid * kchunk, K), k1 = min(k0 + kchunk, K);
  int big = 0;
  for (int k = k0; k < k1; ++k) {
    const int size = kstart[pad32(k + 1)] - kstart[pad32(k)];
    if (size > sp.small_max) big += size;
  }
  int BIG;
  (void)block_exclusive_scan(big, scan_tmp, &BIG);
  const bool use_tc = sp.tc_enabled && BIG >= sp.tc_min_rows;  // (as in the one-CTA path)
  int heads = 0, ng = 0, nt = 0;
  for (int k = k0; k < k1; ++k) {
    const int size = kstart[pad32(k + 1)] - kstart[pad32(k)];
    if (size == 0) continue;
    ++heads;
    if (use_tc && size > sp.small_max)
      nt += (size + sp.tile_rows - 1) / sp.tile_rows;
    else
      ng += (size + sp.group_rows - 1) / sp.group_rows;
  }
  int S, NGT;
  int seg = block_exclusive_scan(heads, scan_tmp, &S);
  const int gt = block_exclusive_scan(ng | (nt << 16), scan_tmp, &NGT);  // both counts < 2^16
  const int NG = NGT & 0xFFFF, NT = NGT >> 16;
  int g = gt & 0xFFFF, t = gt >> 16;
  for (int k = k0; k < k1; ++k) {
    const int b = kstart[pad32(k)], size = kstart[pad32(k + 1)] - b;
    if (size == 0) continue;
    pd.seg_off[seg] = b;
    pd.seg_key[seg] = k;
    const bool tc = use_tc && size > sp.small_max;
    const int cap = tc ? sp.tile_rows : sp.group_rows;
    const int np = (size + cap - 1) / cap;
    const int base = size / np, extra = size % np;
    int r = b;
    for (int q = 0; q < np; ++q) {
      const int len = base + (q < extra ? 1 : 0);
      const int4 w = make_int4(r, len, k, seg);
      if (tc)
        pd.tiles[t++] = w;
      else
        pd.groups[g++] = w;
      r += len;
    }
    ++seg;
  }
  SEG_T(11);
#ifdef LORA_SEG_PROF
  if (tid == 0) printf("scan K=%d C=%d cycles: flat %lld keys %lld\n", K, C, g_seg_t[10] - g_seg_t[9], g_seg_t[11] - g_seg_t[10]);
#endif
  if (tid == 0) {
    pd.seg_off[S] = n_valid;
    pd.counts[kCntValid] = n_valid;
    pd.counts[kCntSegs] = S;
    pd.counts[kCntGroups] = NG;
    pd.counts[kCntTiles] = NT;
  }
}

template <int EPT>
__global__ void __launch_bounds__(kSegThreads) seg_scatter_kernel(int T, int K, int C, PlanDev pd) {
  constexpr int RPC = kSegThreads * EPT;
  pdl_launch_dependents();  // the shrink kernels may launch now; they wait for this grid
  const int c = blockIdx.x, row0 = c * RPC;
  pdl_wait();  // seg_scan's offsets are complete
#pragma unroll
  for (int r = 0; r < EPT; ++r) {
    const int p = r * kSegThreads + threadIdx.x;
    const uint32_t v = pd.lsort[row0 + p];
    const int k = (int)(v >> kLocBits);
    if (k < K) pd.perm[pd.offs[(long long)k * C + c] + pd.lrank[row0 + p]] = row0 + (int)(v & ((1u << kLocBits) - 1u));
  }
}

// PDL inside the multi-CTA segmenter chain (env LORA_SEG_PDL=0: plain launches)
bool seg_pdl() {
  static const bool on = [] {
    const char* v = std::getenv("LORA_SEG_PDL");
    return !(v && v[0] == '0');
  }();
  return on;
}

int bits_for(long long v) {  // bits needed to represent v (v >= 0)
  int b = 0;
  while ((1LL << b) <= v) ++b;
  return b;
}

}  // namespace

cudaError_t launch_segment(const int32_t* adapter_ids, const int32_t* expert_ids, int T, int E, int n_adapters,
                           const SegParams& sp, const PlanDev& pd, int* err_flag,
                           cudaStream_t stream, const int* T_dev) {
  // multi-CTA path: K * C within the histogram bound, local composites radix-able
  {
    const long long K = (long long)n_adapters * E;
    const int kb = bits_for(K);
    const char* fe = getenv("LORA_SEG_MULTI");  // test hook: 1 forces, 0 disables the multi-CTA path
    const int forced = fe ? atoi(fe) : -1;
    // beyond one CTA's capacity the multi-CTA path is the only one
    const bool big = T > kMaxOneCtaRows;
    // (device-side T: the one-CTA kernel up to its capacity, the multi-CTA
    // kernels -- sized by the capacity, rows past *T_dev masked -- beyond it)
    const bool want = T_dev ? big : (big || (forced < 0 ? T >= kSegMultiMin : forced == 1));
    int ept = 0;
    if (want && pd.hist && T > 0 && kb + kLocBits <= 32 && K > 0 && K <= kSegKeysMax) {
      // rows per CTA: the fewest (1024, 2048) that keep the histogram K x C
      // within one scan round (the one-CTA scan is slow beyond that, measured:
      // T = 8192, K = 16384 is faster on the one-CTA kernel); a forced run
      // (test hook) falls back to 4096 rows per CTA
      const char* ee = getenv("LORA_SEG_EPT");  // tuning hook
      const int pick = ee ? atoi(ee) : 0;
      for (int e : {1, 2, 4}) {
        const long long C = (T + e * kSegThreads - 1) / (e * kSegThreads);
        const bool fits = pick ? e == pick : (K * C <= kSegHistSmall || ((forced == 1 || big) && e == 4));
        if (fits) {
          if (K * C <= kSegHistMax) ept = e;
          break;
        }
      }
    }
    if (ept) {
      const int C = (T + ept * kSegThreads - 1) / (ept * kSegThreads);
      const int rpc = ept * kSegThreads;
      const int lsm = (2 * (rpc + rpc / 32 + 4) + 32 * 256) * 4;
      const int ssm = (int)((pad32((int)K + 1) + 4) * 4 + (16 * kSegThreads + 16 * kSegThreads / 32) * 4);
      static unsigned long long mset = 0;
      int dev = 0;
      cudaGetDevice(&dev);
      if (!(mset & (1ull << dev))) {
        const int lmax = (2 * (4096 + 128 + 4) + 32 * 256) * 4;
        const int smax = (pad32(kSegKeysMax + 1) + 4) * 4 + (16 * kSegThreads + 16 * kSegThreads / 32) * 4;
        cudaError_t e = cudaFuncSetAttribute(seg_local_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, lmax);
        if (e == cudaSuccess)
          e = cudaFuncSetAttribute(seg_local_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, lmax);
        if (e == cudaSuccess)
          e = cudaFuncSetAttribute(seg_local_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, lmax);
        if (e == cudaSuccess)
          e = cudaFuncSetAttribute(seg_scan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smax);
        if (e != cudaSuccess) return e;
        mset |= 1ull << dev;
      }
      {
        auto local = ept == 1 ? seg_local_kernel<1> : ept == 2 ? seg_local_kernel<2> : seg_local_kernel<4>;
        auto scatter = ept == 1 ? seg_scatter_kernel<1> : ept == 2 ? seg_scatter_kernel<2> : seg_scatter_kernel<4>;
        // seg_local waits for everything before it on the stream (the previous
        // applies still read the plan); seg_scan and seg_scatter are launched
        // programmatically dependent (PDL) on their predecessor in the chain
        local<<<C, kSegThreads, lsm, stream>>>(adapter_ids, expert_ids, T, E, n_adapters, kb, C, sp, pd, err_flag,
                                               T_dev);
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = seg_pdl() ? 1 : 0;
        cudaLaunchConfig_t cfg = {};
        cfg.blockDim = dim3(kSegThreads);
        cfg.stream = stream;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cfg.gridDim = dim3(1);
        cfg.dynamicSmemBytes = ssm;
        cudaError_t e = cudaLaunchKernelEx(&cfg, seg_scan_kernel, (int)K, C, sp, pd);
        if (e != cudaSuccess) return e;
        cfg.gridDim = dim3(C);
        cfg.dynamicSmemBytes = 0;
        e = cudaLaunchKernelEx(&cfg, scatter, T, (int)K, C, pd);
        if (e != cudaSuccess) return e;
        return cudaGetLastError();
      }
    }
  }
  const int kb = bits_for((long long)n_adapters * E);  // key K = n_adapters*E marks "no LoRA" (sorts last)
  // CTA size: small batches on 256 / 512 threads (radix path), else 1024
  // one CTA holds at most kMaxOneCtaRows rows; larger batches needed the
  // multi-CTA path (key space within kSegKeysMax / the histogram bound)
  if (T > kMaxOneCtaRows) return cudaErrorInvalidValue;
  // (device T: T is the capacity).  LORA_SEG_NT=1024 (tuning hook): always 1024
  int nt = T <= 256 ? 256 : T <= 512 ? 512 : kSegThreads;
  if (const char* e = getenv("LORA_SEG_NT")) nt = std::max(nt, atoi(e) >= kSegThreads ? kSegThreads : nt);
  int P = nt;  // at least one composite per thread
  while (P < T) P <<= 1;
  const int ib = bits_for(P - 1);
  const int radix = (ib + kb <= 32) ? 1 : 0;
  if (!radix) {  // bitonic fallback: 1024 threads
    nt = kSegThreads;
    P = std::max(P, kSegThreads);
  }
  // radix: two u32 buffers (+1 int for the last segment offset); bitonic: u64 buffer + P+1 ints
  const int smem = radix ? (2 * (P + P / 32) + 8 + (nt / 32) * 256) * 4 : P * 8 + (P + 1) * 4;
  static unsigned long long attr_set = 0;  // per-device bitmask
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(attr_set & (1ull << dev))) {
    const int mx = std::max((2 * (kMaxOneCtaRows + kMaxOneCtaRows / 32) + 8 + 32 * 256) * 4,
                            kMaxOneCtaRows * 8 + (kMaxOneCtaRows + 1) * 4);
    cudaError_t e = cudaFuncSetAttribute(segment_kernel<true, kSegThreads>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(segment_kernel<false, kSegThreads>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    if (e != cudaSuccess) return e;
    attr_set |= 1ull << dev;
  }
  if (radix && nt == 256)
    segment_kernel<true, 256><<<1, 256, smem, stream>>>(adapter_ids, expert_ids, T, P, E, n_adapters, kb, ib, sp, pd,
                                                        err_flag, T_dev);
  else if (radix && nt == 512)
    segment_kernel<true, 512><<<1, 512, smem, stream>>>(adapter_ids, expert_ids, T, P, E, n_adapters, kb, ib, sp, pd,
                                                        err_flag, T_dev);
  else if (radix)
    segment_kernel<true, kSegThreads><<<1, kSegThreads, smem, stream>>>(adapter_ids, expert_ids, T, P, E, n_adapters,
                                                                        kb, ib, sp, pd, err_flag, T_dev);
  else
    segment_kernel<false, kSegThreads><<<1, kSegThreads, smem, stream>>>(adapter_ids, expert_ids, T, P, E, n_adapters,
                                                                         kb, ib, sp, pd, err_flag, T_dev);
  return cudaGetLastError();
}

}  // namespace lora
