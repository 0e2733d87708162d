// gather_probe.cu -- how much HBM bandwidth does a gathered-row stream keep
// as a function of the contiguous bytes C touched per row per step?
// The tcgen05 expand read-modify-writes y in 128-row x 256-byte pieces (rows
// gathered through the segment permutation), the tcgen05 shrink reads x in
// 128-row x 256-byte pieces; this probe keeps the bytes in flight per CTA fixed
// (32 KB per step: 32768 / C rows x C bytes) and varies C.
//   build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/gather_probe.cu -o tools/gather_probe
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>

template <bool RMW>
__global__ void __launch_bounds__(512) gather_kernel(uint4* __restrict__ y, const int* __restrict__ perm, int n_rows,
                                                      int row16, int C16, float* out) {
  // one step: RT = 2048 / C16 rows x C16 16-byte pieces (32 KB); a CTA walks the
  // row chunks of a tile of RT rows, tiles grid-strided
  const int RT = 2048 / C16;
  constexpr int NPART = 7;  // a row = 7 parts of 4 KB (items = tiles x parts, enough for every CTA)
  const int n_tiles = n_rows / RT, n_sub = row16 / C16 / NPART;
  uint32_t acc = 0;
  for (int it = blockIdx.x; it < n_tiles * NPART; it += gridDim.x) {
    const int t = it / NPART, part = it % NPART;
    int rows[4];
    int col[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int p = threadIdx.x + 512 * u;
      rows[u] = perm[t * RT + p / C16];
      col[u] = p % C16 + part * n_sub * C16;
    }
    for (int sb = 0; sb < n_sub; ++sb) {
      uint4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = y[(long long)rows[u] * row16 + sb * C16 + col[u]];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (RMW) {
          v[u].x += 1u;
          y[(long long)rows[u] * row16 + sb * C16 + col[u]] = v[u];
        } else {
          acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
        }
      }
    }
  }
  if (acc == 0x12345678u) out[0] = 1.f;
}

int main() {
  const int n_rows = 16384, row_bytes = 28672, row16 = row_bytes / 16;
  uint4* y;
  int* perm_d;
  float* out;
  cudaMalloc(&y, (size_t)n_rows * row_bytes);
  cudaMalloc(&perm_d, n_rows * sizeof(int));
  cudaMalloc(&out, 4);
  cudaMemset(y, 0, (size_t)n_rows * row_bytes);
  std::vector<int> perm(n_rows), ident(n_rows);
  for (int i = 0; i < n_rows; ++i) perm[i] = ident[i] = i;
  std::mt19937 rng(1);
  std::shuffle(perm.begin(), perm.end(), rng);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double bytes = (double)n_rows * row_bytes;
  for (int gathered = 1; gathered >= 0; --gathered) {
    cudaMemcpy(perm_d, gathered ? perm.data() : ident.data(), n_rows * sizeof(int), cudaMemcpyHostToDevice);
    for (int rmw = 1; rmw >= 0; --rmw)
      for (int C : {128, 256, 512, 1024, 2048}) {
        const int C16 = C / 16;
        for (int ctas : {2, 3, 4}) {
          auto run = [&]() {
            if (rmw) gather_kernel<true><<<sms * ctas, 512>>>(y, perm_d, n_rows, row16, C16, out);
            else gather_kernel<false><<<sms * ctas, 512>>>(y, perm_d, n_rows, row16, C16, out);
          };
          run();
          cudaDeviceSynchronize();
          cudaEventRecord(e0);
          const int reps = 10;
          for (int i = 0; i < reps; ++i) run();
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms = 0;
          cudaEventElapsedTime(&ms, e0, e1);
          const double gbs = bytes * (rmw ? 2 : 1) * reps / (ms * 1e-3) / 1e9;
          printf("%s %s C=%5d B ctas/SM=%d: %8.1f GB/s (%.1f us per pass)\n", gathered ? "gathered" : "contig  ",
                 rmw ? "rmw " : "read", C, ctas, gbs, ms * 1e3 / reps);
        }
      }
  }
  cudaError_t err = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(err));
  return 0;
}
