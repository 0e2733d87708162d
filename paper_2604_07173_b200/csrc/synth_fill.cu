// synth_fill.cu -- weight-store fill and relayout kernels.
//
// (1) Counter-based synthetic fill.  This is the CUDA side's own
//     implementation of the generator recipe written in DESIGN.md "Input
//     recipe" (the oracle side regenerates the same values with numpy); the
//     two share no code.  For 2048 adapters one MoE layer is 116 GB of
//     weights, so they are generated in HBM instead of crossing PCIe.
//
//         mix64(z) = splitmix64 finaliser
//         base     = mix64(seed*G ^ tag*T ^ major*M)
//         h        = mix64(base + minor*G)
//         value    = ((h >> 56) - 128) * 2^-shift        (exact in bf16)
//
//     A_{a,e}[j,k] uses tag = 1<<16 | slot, major = a*E+e, minor = j*r+k,
//     shift = 7 + ceil(log2(h_in)/2); B_{a,e}[k,c] uses tag = 2<<16 | slot,
//     minor = k*h_out + c, shift = 7 + ceil(log2(r)/2).
//
// (2) Relayout of caller weights in the paper's orientation (A [h_in][r],
//     B [r][h_out]) into the swizzled kernel layout of common.cuh.
#include "common.cuh"
#include "kernels.h"

namespace lora {

namespace {

constexpr unsigned long long kG = 0x9E3779B97F4A7C15ull;
constexpr unsigned long long kT = 0xD1B54A32D192ED03ull;
constexpr unsigned long long kM = 0xC2B2AE3D27D4EB4Full;

LORA_DEVINL unsigned long long mix64(unsigned long long z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

LORA_DEVINL uint16_t hash_bf16(unsigned long long base, unsigned long long minor, float scale) {
  const unsigned long long h = mix64(base + minor * kG);
  const int q = (int)(h >> 56) - 128;
  return (uint16_t)(__float_as_uint((float)q * scale) >> 16);
}

LORA_DEVINL unsigned long long hash_base(unsigned long long seed, unsigned tag, unsigned long long major) {
  return mix64((seed * kG) ^ ((unsigned long long)tag * kT) ^ (major * kM));
}

// map a local unit index of this rank's store to the global unit id a*E+e (-1: padding)
LORA_DEVINL long long global_unit(long long u, int E, const Placement& pl, int n_adapters, long long adapter_base) {
  const long long k = pl.global_key(u, E, n_adapters);
  if (k < 0) return -1;
  const long long gk = k + adapter_base * E;  // resident-cache fill: unsharded, adapters shifted
  return gk < (long long)n_adapters * E ? gk : -1;
}

// one thread = 8 consecutive store elements (one 16-byte chunk)
__global__ void fill_A_kernel(uint16_t* __restrict__ At, long long units, int h_in, int r, unsigned long long seed,
                              unsigned tag, float scale, int E, Placement pl, int n_adapters, long long adapter_base) {
  const long long n_chunks = units * h_in * r / 8;
  const int tiles = h_in >> 6;
  for (long long ch = blockIdx.x * (long long)blockDim.x + threadIdx.x; ch < n_chunks;
       ch += (long long)gridDim.x * blockDim.x) {
    const long long idx = ch * 8;
    const long long tile = idx / (r * 64);
    const int within = (int)(idx - tile * (r * 64));
    const int k = within >> 6, pc = (within & 63) >> 3;
    const int q = pc ^ (k & 7);
    const long long u = tile / tiles;
    const int j0 = (int)(tile - u * tiles) * 64 + q * 8;
    const long long gu = global_unit(u, E, pl, n_adapters, adapter_base);
    uint16_t v[8];
    if (gu < 0) {
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = 0;
    } else {
      const unsigned long long base = hash_base(seed, tag, (unsigned long long)gu);
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = hash_bf16(base, (unsigned long long)(j0 + i) * r + k, scale);
    }
    uint4 w;
    w.x = v[0] | (uint32_t(v[1]) << 16);
    w.y = v[2] | (uint32_t(v[3]) << 16);
    w.z = v[4] | (uint32_t(v[5]) << 16);
    w.w = v[6] | (uint32_t(v[7]) << 16);
    *reinterpret_cast<uint4*>(At + idx) = w;
  }
}

__global__ void fill_B_kernel(uint16_t* __restrict__ Bt, long long units, int h_out, int r, unsigned long long seed,
                              unsigned tag, float scale, int E, Placement pl, int n_adapters, long long adapter_base) {
  const long long n_chunks = units * h_out * r / 8;
  const int cpr = r / 8;  // chunks per row
  for (long long ch = blockIdx.x * (long long)blockDim.x + threadIdx.x; ch < n_chunks;
       ch += (long long)gridDim.x * blockDim.x) {
    const long long row = ch / cpr;
    const int pc = (int)(ch - row * cpr);
    const long long u = row / h_out;
    const int c = (int)(row - u * h_out);
    const int q = swz_row_chunk(c, pc, r * 2);
    const long long gu = global_unit(u, E, pl, n_adapters, adapter_base);
    uint16_t v[8];
    if (gu < 0) {
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = 0;
    } else {
      const unsigned long long base = hash_base(seed, tag, (unsigned long long)gu);
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = hash_bf16(base, (unsigned long long)(q * 8 + i) * h_out + c, scale);
    }
    uint4 w;
    w.x = v[0] | (uint32_t(v[1]) << 16);
    w.y = v[2] | (uint32_t(v[3]) << 16);
    w.z = v[4] | (uint32_t(v[5]) << 16);
    w.w = v[6] | (uint32_t(v[7]) << 16);
    *reinterpret_cast<uint4*>(Bt + ch * 8) = w;
  }
}

__global__ void fill_rows_kernel(uint16_t* __restrict__ dst, long long rows, int width, unsigned long long seed,
                                 unsigned tag, float scale, long long row_base) {
  const long long n = rows * width;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / width;
    const int c = (int)(i - r * width);
    const unsigned long long base = hash_base(seed, tag, (unsigned long long)(row_base + r));
    dst[i] = hash_bf16(base, (unsigned long long)c, scale);
  }
}

// caller A: [U][h_in][r] (paper orientation) -> At store layout
__global__ void relayout_A_kernel(const uint16_t* __restrict__ src, uint16_t* __restrict__ At, long long units,
                                  int h_in, int r) {
  const long long n = units * h_in * r;
  const int tiles = h_in >> 6;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long tile = idx / (r * 64);
    const int within = (int)(idx - tile * (r * 64));
    const int k = within >> 6, pc = (within & 63) >> 3, e8 = within & 7;
    const int q = pc ^ (k & 7);
    const long long u = tile / tiles;
    const int j = (int)(tile - u * tiles) * 64 + q * 8 + e8;
    At[idx] = src[(u * h_in + j) * r + k];
  }
}

// caller B: [U][r][h_out] -> Bt store layout [U][h_out][r] (swizzled rows)
__global__ void relayout_B_kernel(const uint16_t* __restrict__ src, uint16_t* __restrict__ Bt, long long units,
                                  int h_out, int r) {
  const long long n = units * h_out * r;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long row = idx / r;
    const int within = (int)(idx - row * r);
    const int pc = within >> 3, e8 = within & 7;
    const long long u = row / h_out;
    const int c = (int)(row - u * h_out);
    const int k = swz_row_chunk(c, pc, r * 2) * 8 + e8;
    Bt[idx] = src[(u * r + k) * h_out + c];
  }
}

int grid_for(long long n, int threads) {
  long long g = (n + threads - 1) / threads;
  if (g > 148LL * 32) g = 148LL * 32;
  if (g < 1) g = 1;
  return (int)g;
}

}  // namespace

static int shift_of(int width) { return 7 + (int)ceil(log2((double)width) / 2.0); }

cudaError_t launch_fill_store(uint16_t* At, uint16_t* Bt, int h_in, int h_out, int E, int r, long long units,
                              int slot, unsigned long long seed, const Placement& pl, int n_adapters,
                              cudaStream_t stream, long long adapter_base) {
  const float sa = ldexpf(1.0f, -shift_of(h_in));
  const float sb = ldexpf(1.0f, -shift_of(r));
  const unsigned tagA = (1u << 16) | (unsigned)slot, tagB = (2u << 16) | (unsigned)slot;
  const long long na = units * h_in * r / 8, nb = units * h_out * r / 8;
  fill_A_kernel<<<grid_for(na, 256), 256, 0, stream>>>(At, units, h_in, r, seed, tagA, sa, E, pl,
                                                        n_adapters, adapter_base);
  fill_B_kernel<<<grid_for(nb, 256), 256, 0, stream>>>(Bt, units, h_out, r, seed, tagB, sb, E, pl,
                                                        n_adapters, adapter_base);
  return cudaGetLastError();
}

cudaError_t launch_fill_rows(uint16_t* dst, long long rows, int width, unsigned long long seed, unsigned tag,
                             int shift, long long row_base, cudaStream_t stream) {
  const long long n = rows * width;
  if (n == 0) return cudaSuccess;
  fill_rows_kernel<<<grid_for(n, 256), 256, 0, stream>>>(dst, rows, width, seed, tag, ldexpf(1.0f, -shift),
                                                         row_base);
  return cudaGetLastError();
}

cudaError_t launch_relayout_A(const uint16_t* src, uint16_t* At, long long units, int h_in, int r,
                              cudaStream_t stream) {
  const long long n = units * h_in * r;
  if (n == 0) return cudaSuccess;
  relayout_A_kernel<<<grid_for(n, 256), 256, 0, stream>>>(src, At, units, h_in, r);
  return cudaGetLastError();
}

cudaError_t launch_relayout_B(const uint16_t* src, uint16_t* Bt, long long units, int h_out, int r,
                              cudaStream_t stream) {
  const long long n = units * h_out * r;
  if (n == 0) return cudaSuccess;
  relayout_B_kernel<<<grid_for(n, 256), 256, 0, stream>>>(src, Bt, units, h_out, r);
  return cudaGetLastError();
}

}  // namespace lora
