// cta_rate_probe.cu -- streaming rate of ONE CTA through a TMA bulk-copy ring
// (the CUDA-core shrink's structure: 1 producer lane, 8 consumer warps that
// wait on `full` and release `empty`), as a function of the number of active
// CTAs, the stage size and the ring depth.  At decode batches a layer has few
// shrink items, each streaming a whole unit's A (up to 1.8 MB for Mixtral
// down) through one CTA, so the per-CTA rate sets the kernel time.
//   nvcc -gencode arch=compute_100a,code=sm_100a -I paper_2604_07173_b200/csrc -o /tmp/ctap tools/cta_rate_probe.cu
#include <cstdio>
#include "common.cuh"
using namespace lora;

__global__ void __launch_bounds__(288, 2) ring_kernel(const uint8_t* __restrict__ src, long long per_cta, int stage,
                                                      int nst, int touch, float* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + nst * stage);
  uint64_t* empty = full + nst;
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 8); }
    fence_mbar_init();
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long n = per_cta / stage;
  const uint8_t* base = src + (long long)blockIdx.x * per_cta;
  float acc = 0.f;
  if (warp == 8) {
    if (lane == 0) {
      for (long long i = 0; i < n; ++i) {
        const int s = (int)(i % nst);
        mbar_wait(&empty[s], (uint32_t)(((i / nst) & 1) ^ 1));
        mbar_arrive_expect_tx(&full[s], stage);
        bulk_g2s(smem + s * stage, base + i * stage, stage, &full[s]);
      }
    }
  } else {
    for (long long i = 0; i < n; ++i) {
      const int s = (int)(i % nst);
      mbar_wait(&full[s], (uint32_t)((i / nst) & 1));
      if (touch) {
        const uint32_t a = smem_u32(smem + s * stage);
        for (int o = threadIdx.x * 16; o < stage; o += 256 * 16) acc += __uint_as_float(lds128(a + o).x);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
  }
  if (acc == 1234.5f) out[0] = acc;
}

int main() {
  const long long total = 1ll << 33;  // 8 GiB source
  uint8_t* src;
  float* out;
  cudaMalloc(&src, total);
  cudaMalloc(&out, 4);
  cudaMemset(src, 1, total);
  cudaFuncSetAttribute(ring_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int grids[] = {1, 16, 64, 148, 296};
  const int stages[][2] = {{16384, 5}, {18432, 5}, {32768, 3}, {8192, 12}};
  for (auto& sn : stages) {
    for (int g : grids) {
      const long long per_cta = 1835008;  // Mixtral down: 14336 x 64 x 2
      for (int touch = 0; touch < 2; ++touch) {
        ring_kernel<<<g, 288, 112 * 1024>>>(src, per_cta, sn[0], sn[1], touch, out);
        cudaEventRecord(e0);
        for (int r = 0; r < 5; ++r) ring_kernel<<<g, 288, 112 * 1024>>>(src, per_cta, sn[0], sn[1], touch, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        ms /= 5;
        printf("stage %6d nst %2d grid %4d touch %d: %8.1f us  per-CTA %6.1f GB/s  total %7.1f GB/s  %s\n", sn[0],
               sn[1], g, touch, ms * 1e3, per_cta / (ms * 1e-3) / 1e9, g * per_cta / (ms * 1e-3) / 1e9,
               cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
  return 0;
}
