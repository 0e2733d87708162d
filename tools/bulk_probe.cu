// bulk_probe.cu -- throughput of small 1-D TMA bulk operations (row-sized
// pieces, as a row-gathering epilogue would issue them): bulk loads into a
// shared-memory ring, and bulk reduce-add (bf16) from shared memory to global.
#include <cstdio>
#include "common.cuh"
using namespace lora;

__global__ void __launch_bounds__(128, 1) bulk_load_kernel(const uint8_t* __restrict__ src, long long rows, int row_bytes,
                                                           int piece, int iters, float* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  constexpr int NST = 8, STAGE = 32768;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NST * STAGE);
  if (threadIdx.x == 0) { for (int s = 0; s < NST; ++s) mbar_init(&full[s], 1); fence_mbar_init(); }
  __syncthreads();
  const int per_stage = STAGE / piece;
  unsigned long long h = blockIdx.x * 0x9E3779B97F4A7C15ull;
  uint32_t ph = 0;
  float acc = 0;
  if (threadIdx.x < 32) {
    for (int it = 0; it < iters; ++it) {
      const int s = it % NST;
      if (it >= NST) mbar_wait(&full[s], ((it / NST) - 1) & 1);
      if (threadIdx.x == 0) mbar_arrive_expect_tx(&full[s], per_stage * piece);
      __syncwarp();
      for (int k = threadIdx.x; k < per_stage; k += 32) {
        h = h * 6364136223846793005ull + 1442695040888963407ull + k;
        const long long r = (long long)((h >> 17) % (unsigned long long)rows);
        bulk_g2s(smem + s * STAGE + k * piece, src + r * row_bytes, piece, &full[s]);
      }
      __syncwarp();
    }
    // drain
    for (int s = 0; s < NST; ++s) {
      const int last = iters - NST + s;
      if (last >= 0) mbar_wait(&full[last % NST], (last / NST) & 1);
    }
    acc = smem[threadIdx.x];
  }
  if (acc == 1234.5f) out[0] = acc;
}

__global__ void __launch_bounds__(128, 1) bulk_red_kernel(uint8_t* __restrict__ dst, long long rows, int row_bytes,
                                                          int piece, int iters) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  fence_proxy_async_smem();
  __syncthreads();
  unsigned long long h = blockIdx.x * 0x9E3779B97F4A7C15ull + threadIdx.x;
  if (threadIdx.x < 32) {
    const int per = 32768 / piece;
    for (int it = 0; it < iters; ++it) {
      for (int k = threadIdx.x; k < per; k += 32) {
        h = h * 6364136223846793005ull + 1442695040888963407ull;
        const long long r = (long long)((h >> 17) % (unsigned long long)rows);
        asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.noftz.bf16 [%0], [%1], %2;" ::"l"(
                         dst + r * row_bytes),
                     "r"(smem_u32(smem + (it & 1) * 32768 + k * piece)), "r"(piece)
                     : "memory");
      }
      bulk_commit();
      bulk_wait_read<1>();
    }
    bulk_wait<0>();
  }
}

__global__ void __launch_bounds__(128, 1) bulk_store_kernel(uint8_t* __restrict__ dst, long long rows, int row_bytes,
                                                            int piece, int iters) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  unsigned long long h = blockIdx.x * 0x9E3779B97F4A7C15ull + threadIdx.x;
  if (threadIdx.x < 32) {
    const int per = 32768 / piece;
    for (int it = 0; it < iters; ++it) {
      for (int k = threadIdx.x; k < per; k += 32) {
        h = h * 6364136223846793005ull + 1442695040888963407ull;
        const long long r = (long long)((h >> 17) % (unsigned long long)rows);
        bulk_s2g(dst + r * row_bytes, smem + (it & 1) * 32768 + k * piece, piece);
      }
      bulk_commit();
      bulk_wait_read<1>();
    }
    bulk_wait<0>();
  }
}

int main() {
  const long long bytes = 4LL << 30;
  uint8_t* buf; float* out;
  cudaMalloc(&buf, bytes); cudaMalloc(&out, 4); cudaMemset(buf, 0, bytes);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(bulk_load_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 32768 + 2048);
  cudaFuncSetAttribute(bulk_red_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
  cudaFuncSetAttribute(bulk_store_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int row_bytes = 28672;  // a 14336-column bf16 row
  const long long rows = bytes / row_bytes;
  for (int piece : {256, 512, 1024, 2048}) {
    const int iters = 400;
    bulk_load_kernel<<<sms, 128, 8 * 32768 + 2048>>>(buf, rows, row_bytes, piece, 20, out);
    cudaEventRecord(a);
    bulk_load_kernel<<<sms, 128, 8 * 32768 + 2048>>>(buf, rows, row_bytes, piece, iters, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("bulk load   piece %5d: %7.1f GB/s (%s)\n", piece, (double)sms * iters * 32768 / (ms * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
    cudaEventRecord(a);
    bulk_red_kernel<<<sms, 128, 65536 + 1024>>>(buf, rows, row_bytes, piece, iters);
    cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("bulk redadd piece %5d: %7.1f GB/s of smem data (%s)\n", piece,
           (double)sms * iters * 32768 / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    cudaEventRecord(a);
    bulk_store_kernel<<<sms, 128, 65536 + 1024>>>(buf, rows, row_bytes, piece, iters);
    cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("bulk store  piece %5d: %7.1f GB/s (%s)\n", piece, (double)sms * iters * 32768 / (ms * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
