// Probe: TMA tile::gather4 (sm_100a) with a SWIZZLE_128B tensor map of box
// {64 cols, 1 row}: does one gather4 land rows r0..r3 (128 B each) at
// consecutive 128-byte smem rows with the 128B swizzle of their smem address
// (chunk q of smem row n at q ^ (n & 7)), for 512-byte (not 1024) aligned
// destinations?  Also times gather4 vs a plain read stream.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/gather4_probe tools/gather4_probe.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const __grid_constant__ CUtensorMap map, const int* rows, int nrows, int col0, uint16_t* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(nrows * 128));
    for (int g = 0; g < nrows / 4; ++g) {
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(base + g * 512)),
          "l"(reinterpret_cast<uint64_t>(&map)), "r"(smem_u32(&bar)), "r"(col0), "r"(rows[4 * g]),
          "r"(rows[4 * g + 1]), "r"(rows[4 * g + 2]), "r"(rows[4 * g + 3])
          : "memory");
    }
    asm volatile(
        "{ .reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], 0; @!p bra W; }" ::"r"(smem_u32(&bar)));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nrows * 64; i += blockDim.x) out[i] = reinterpret_cast<uint16_t*>(base)[i];
}

int main() {
  const int R = 1000, C = 512;
  std::vector<uint16_t> h(R * C);
  for (int r = 0; r < R; ++r)
    for (int c = 0; c < C; ++c) h[r * C + c] = (uint16_t)((r * 7 + c) & 0xffff);
  uint16_t* g;
  CK(cudaMalloc(&g, h.size() * 2));
  CK(cudaMemcpy(g, h.data(), h.size() * 2, cudaMemcpyHostToDevice));
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)R};
  cuuint64_t strides[1] = {(cuuint64_t)C * 2};
  cuuint32_t box[2] = {64, 1};
  cuuint32_t es[2] = {1, 1};
  CUresult cr = enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, g, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode: %d\n", (int)cr);
  const int nrows = 16;
  int hrows[nrows];
  for (int i = 0; i < nrows; ++i) hrows[i] = (i * 131 + 17) % R;
  int* drows;
  CK(cudaMalloc(&drows, sizeof(hrows)));
  CK(cudaMemcpy(drows, hrows, sizeof(hrows), cudaMemcpyHostToDevice));
  uint16_t* out;
  CK(cudaMalloc(&out, nrows * 64 * 2));
  const int col0 = 128;
  CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384));
  probe<<<1, 128, 16384>>>(map, drows, nrows, col0, out);
  CK(cudaDeviceSynchronize());
  std::vector<uint16_t> ho(nrows * 64);
  CK(cudaMemcpy(ho.data(), out, ho.size() * 2, cudaMemcpyDeviceToHost));
  int bad_sw = 0, bad_plain = 0;
  for (int n = 0; n < nrows; ++n)
    for (int qq = 0; qq < 8; ++qq)
      for (int e = 0; e < 8; ++e) {
        const uint16_t want = h[hrows[n] * C + col0 + qq * 8 + e];
        if (ho[n * 64 + ((qq ^ (n & 7)) * 8) + e] != want) ++bad_sw;
        if (ho[n * 64 + qq * 8 + e] != want) ++bad_plain;
      }
  printf("gather4 SW128: mismatches swizzled-layout %d, plain-layout %d (of %d)\n", bad_sw, bad_plain, nrows * 64);
  return 0;
}
