// bw_probe.cu -- microbenchmark of the 1-D TMA bulk-copy streaming pipeline
// used by the CUDA-core kernels (stage size / depth / consumer work), vs a
// plain vectorised LDG read.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Ipaper_2604_07173_b200/csrc
//   -I../paper_2604_07173_b200/csrc bw_probe.cu -o bw_probe
#include <cstdio>
#include <vector>
#include "common.cuh"
using namespace lora;

template <int STAGE, int NST, int WORK>
__global__ void __launch_bounds__(288, 1) stream_kernel(const uint8_t* __restrict__ src, long long n_items,
                                                        int item_bytes, float* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NST * STAGE);
  uint64_t* empty = full + NST;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 8); }
    fence_mbar_init();
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_st = item_bytes / STAGE;
  if (warp == 8) {
    if (lane == 0) {
      uint64_t pol = policy_evict_first();
      int stage = 0; uint32_t ph = 0;
      for (long long it = blockIdx.x; it < n_items; it += gridDim.x)
        for (int st = 0; st < n_st; ++st) {
          mbar_wait(&empty[stage], ph ^ 1);
          mbar_arrive_expect_tx(&full[stage], STAGE);
          bulk_g2s_hint(smem + stage * STAGE, src + it * item_bytes + (long long)st * STAGE, STAGE, &full[stage], pol);
          if (++stage == NST) { stage = 0; ph ^= 1; }
        }
    }
    return;
  }
  float acc = 0.f;
  int stage = 0; uint32_t ph = 0;
  for (long long it = blockIdx.x; it < n_items; it += gridDim.x)
    for (int st = 0; st < n_st; ++st) {
      mbar_wait(&full[stage], ph);
      if (WORK) {
        const uint32_t b = smem_u32(smem + stage * STAGE);
        for (int o = threadIdx.x * 16; o < STAGE; o += 256 * 16) {
          uint4 v = lds128(b + o);
          acc += __uint_as_float(v.x) + __uint_as_float(v.y) + __uint_as_float(v.z) + __uint_as_float(v.w);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == NST) { stage = 0; ph ^= 1; }
    }
  if (acc == 1234.5f) out[0] = acc;
}

__global__ void ldg_kernel(const uint4* __restrict__ src, long long n, float* out) {
  float acc = 0.f;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    uint4 v = __ldg(src + i);
    acc += __uint_as_float(v.x) + __uint_as_float(v.w);
  }
  if (acc == 1234.5f) out[0] = acc;
}

template <int STAGE, int NST, int WORK>
void run(const uint8_t* src, long long bytes, float* out, int item_bytes, int grid) {
  auto k = stream_kernel<STAGE, NST, WORK>;
  int smem = NST * STAGE + 2048;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  long long n_items = bytes / item_bytes;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int w = 0; w < 2; ++w) k<<<grid, 288, smem>>>(src, n_items, item_bytes, out);
  cudaEventRecord(a);
  const int reps = 5;
  for (int w = 0; w < reps; ++w) k<<<grid, 288, smem>>>(src, n_items, item_bytes, out);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("bulk stage=%6d nst=%d work=%d item=%7d grid=%4d : %.1f GB/s  (%s)\n", STAGE, NST, WORK, item_bytes, grid,
         bytes * reps / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const long long bytes = 8LL << 30;
  uint8_t* src; float* out;
  cudaMalloc(&src, bytes); cudaMalloc(&out, 4);
  cudaMemset(src, 1, bytes);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    ldg_kernel<<<sms * 8, 256>>>((const uint4*)src, bytes / 16, out);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) ldg_kernel<<<sms * 8, 256>>>((const uint4*)src, bytes / 16, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("ldg  : %.1f GB/s\n", bytes * 5 / (ms * 1e-3) / 1e9);
  }
  run<32768, 6, 0>(src, bytes, out, 131072, sms);
  run<32768, 6, 1>(src, bytes, out, 131072, sms);
  run<16384, 12, 0>(src, bytes, out, 131072, sms);
  run<16384, 12, 1>(src, bytes, out, 131072, sms);
  run<32768, 4, 1>(src, bytes, out, 131072, sms);
  run<8192, 16, 1>(src, bytes, out, 131072, sms);
  run<65536, 3, 1>(src, bytes, out, 131072, sms);
  run<32768, 6, 1>(src, bytes, out, 1 << 20, sms);
  run<32768, 6, 1>(src, bytes, out, 32768, sms);
  return 0;
}
