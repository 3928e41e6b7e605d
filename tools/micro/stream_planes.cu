// DRAM efficiency of plane-strided (SoA) reads: every warp reads P planes
// (component planes of a field, far apart in memory) at the same site range,
// G bytes per lane per plane, and writes Q planes.  Compares the SoA field
// layout of the solver kernels (8 B per lane: 256 B contiguous per warp and
// plane) with 16 B per lane and with a blocked AoSoA layout (all P planes of
// a 32-site tile contiguous).  Result on a B200 (profiles/r02s5_stream_planes.txt):
// all four layouts stream at the flat-copy rate (5.7-5.8 TB/s) -- the SoA
// component planes cost no DRAM efficiency.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o stream_planes stream_planes.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>

template <typename T, int P, int Q, bool AOSOA>
__global__ void __launch_bounds__(128) planes_kernel(const T *__restrict__ in, T *__restrict__ out, long n) {
  // n elements of T per plane
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    T v[P];
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const long idx = AOSOA ? ((i >> 5) * P + p) * 32 + (i & 31) : (long)p * n + i;
      v[p] = __ldg(in + idx);
    }
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      T s = v[q % P];
      s.x += v[(q + 1) % P].y;
      const long idx = AOSOA ? ((i >> 5) * Q + q) * 32 + (i & 31) : (long)q * n + i;
      __stcs(out + idx, s);
    }
  }
}

template <typename T, int P, int Q, bool AOSOA>
void run(const char *name, long bytes_per_plane) {
  const long n = bytes_per_plane / sizeof(T);
  T *in, *out;
  cudaMalloc(&in, (size_t)P * bytes_per_plane);
  cudaMalloc(&out, (size_t)Q * bytes_per_plane);
  cudaMemset(in, 0, (size_t)P * bytes_per_plane);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, planes_kernel<T, P, Q, AOSOA>, 128, 0);
  const int grid = 148 * per_sm;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 2; ++w) planes_kernel<T, P, Q, AOSOA><<<grid, 128>>>(in, out, n);
  cudaEventRecord(e0);
  const int reps = 5;
  for (int r = 0; r < reps; ++r) planes_kernel<T, P, Q, AOSOA><<<grid, 128>>>(in, out, n);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= reps;
  printf("%-28s P=%2d Q=%2d gran=%2zu B blocks/SM=%2d  %8.3f ms  %7.1f GB/s\n", name, P, Q, sizeof(T), per_sm, ms,
         (double)(P + Q) * bytes_per_plane / ms / 1e6);
  cudaFree(in);
  cudaFree(out);
}

int main() {
  const long plane = 32l << 20;  // 32 MB per plane: 12 planes = 384 MB, far beyond L2
  run<float2, 1, 1, false>("copy 8B", plane * 12);
  run<float4, 1, 1, false>("copy 16B", plane * 12);
  run<float2, 12, 12, false>("SoA 8B", plane);
  run<float4, 12, 12, false>("SoA 16B", plane);
  run<float2, 12, 12, true>("AoSoA 8B", plane);
  run<float4, 12, 12, true>("AoSoA 16B", plane);
  run<double2, 12, 12, false>("SoA fp64 16B", plane);
  return 0;
}
