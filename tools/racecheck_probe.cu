// racecheck_probe.cu -- is a textbook TMA-bulk-copy / mbarrier ring flagged by
// compute-sanitizer racecheck?  One CTA: lane 0 of warp 0 streams 64 chunks of
// 4 KB through a 2-stage shared-memory ring with cp.async.bulk (completion via
// mbarrier complete_tx on `full`), warp 1 waits on `full`, reads the stage,
// arrives on `empty`; the producer waits on `empty` before refilling.  The
// ordering is exactly the one the library's pipelines use; a racecheck report
// here means racecheck does not model mbarrier-ordered async-proxy writes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/rcp tools/racecheck_probe.cu
//   compute-sanitizer --tool racecheck /tmp/rcp
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mb_expect(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t ph) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                 : "=r"(ok) : "r"(su32(b)), "r"(ph) : "memory");
}

__global__ void probe(const uint4* src, unsigned long long* out) {
  __shared__ __align__(128) uint4 ring[2][256];
  __shared__ uint64_t full[2], empty[2];
  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) { mb_init(&full[s], 1); mb_init(&empty[s], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < 64; ++i) {
      const int s = i & 1;
      mb_wait(&empty[s], ((i >> 1) & 1) ^ 1);
      mb_expect(&full[s], 4096);
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 4096, [%2];"
                   ::"r"(su32(ring[s])), "l"(src + i * 256), "r"(su32(&full[s])) : "memory");
    }
  } else if (warp == 1) {
    unsigned long long acc = 0;
    for (int i = 0; i < 64; ++i) {
      const int s = i & 1;
      mb_wait(&full[s], (i >> 1) & 1);
      for (int j = lane; j < 256; j += 32) acc += ring[s][j].x;
      __syncwarp();
      if (lane == 0) mb_arrive(&empty[s]);
    }
    atomicAdd(out, acc);
  }
}

int main() {
  uint4* src;
  unsigned long long* out;
  cudaMalloc(&src, 64 * 4096);
  cudaMalloc(&out, 8);
  cudaMemset(src, 1, 64 * 4096);
  cudaMemset(out, 0, 8);
  probe<<<1, 64>>>(src, out);
  unsigned long long h = 0;
  cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
  printf("probe sum %llu (expect %llu) %s\n", h, 64ull * 256 * 0x01010101ull,
         h == 64ull * 256 * 0x01010101ull ? "OK" : "WRONG");
  return 0;
}
