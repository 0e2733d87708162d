// mma_sync_probe.cu -- throughput of the legacy tensor path (mma.sync
// m16n8k16 bf16 -> fp32, SASS HMMA) on sm_100a, fed by ldmatrix from shared
// memory, in the shape a small-rank CUDA-core LoRA shrink would use it
// (M = 16 rank values, N = 8 rows, K = 16 j per instruction).
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/mmap tools/mma_sync_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256, 2) probe(int iters, float* out, int use_ld) {
  __shared__ __align__(128) uint16_t sA[8][16 * 64];  // per warp: 16 k rows x 64 j
  __shared__ __align__(128) uint16_t sX[8][8 * 72];   // per warp: 8 rows x 64 j (+8 pad)
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  for (int i = l; i < 16 * 64; i += 32) sA[w][i] = (uint16_t)(0x3f80 + (i & 7));
  for (int i = l; i < 8 * 72; i += 32) sX[w][i] = (uint16_t)(0x3f80 + (i & 3));
  __syncwarp();
  float c[4] = {0, 0, 0, 0};
  uint32_t a0 = 0x3f803f80, a1 = a0, a2 = a0, a3 = a0, b0 = a0, b1 = a0;
  const uint32_t abase = (uint32_t)__cvta_generic_to_shared(&sA[w][0]);
  const uint32_t xbase = (uint32_t)__cvta_generic_to_shared(&sX[w][0]);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {  // 4 k-steps of 16 j = 64 j per iteration
      if (use_ld) {
        // 128B-swizzled [k][64 j] rows (the weight store's At layout): chunk c of row k at c ^ (k & 7)
        const int k = l & 15, c = q * 2 + (l >> 4);
        const uint32_t aa = abase + k * 128 + ((c ^ (k & 7)) << 4);
        asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                     : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3) : "r"(aa));
        const uint32_t xa = xbase + ((l & 7) * 72 + q * 16 + ((l >> 3) & 1) * 8) * 2;
        asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];" : "=r"(b0), "=r"(b1) : "r"(xa));
      }
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                   "{%0,%1,%2,%3};"
                   : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
  }
  if (c[0] + c[1] + c[2] + c[3] == 1.2345f) out[0] = c[0];
}

int main() {
  float* out;
  cudaMalloc(&out, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int use_ld = 0; use_ld < 2; ++use_ld) {
    const int iters = 20000, grid = 296;
    probe<<<grid, 256>>>(100, out, use_ld);
    cudaEventRecord(e0);
    probe<<<grid, 256>>>(iters, out, use_ld);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 16 * 8 * 16 * 4.0 * iters * 8 * grid;
    printf("mma.sync m16n8k16 bf16 %s: %.3f ms, %.1f TFLOP/s (%s)\n", use_ld ? "+ ldmatrix x4/x2" : "regs only", ms,
           flops / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
