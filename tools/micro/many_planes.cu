// Does the number of concurrently streamed 2 MB pages matter?  Each thread
// reads its element from P planes (12 loads in flight at a time) and writes
// 12; planes are `stride` bytes apart.  P = 12 .. 384 planes live per pass.
#include <cuda_runtime.h>
#include <cstdio>

template <int P, bool AOSOA, int UNROLL = 1, int LB = 5>
__global__ void __launch_bounds__(128) k(const float2 *__restrict__ in, float2 *__restrict__ out, long n, long pstride) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    float2 acc[12];
#pragma unroll
    for (int j = 0; j < 12; ++j) acc[j] = make_float2(0.f, 0.f);
#pragma unroll UNROLL
    for (int g = 0; g < P / 12; ++g) {
      float2 v[12];
#pragma unroll
      for (int j = 0; j < 12; ++j) v[j] = __ldg(in + (AOSOA ? ((i >> LB) * P + (g * 12 + j)) * (1 << LB) + (i & ((1 << LB) - 1)) : (long)(g * 12 + j) * pstride + i));
#pragma unroll
      for (int j = 0; j < 12; ++j) {
        acc[j].x += v[j].x;
        acc[j].y += v[j].y;
      }
    }
#pragma unroll
    for (int j = 0; j < 12; ++j) __stcs(out + (long)j * pstride + i, acc[j]);
  }
}

template <int P, bool AOSOA, int UNROLL = 1, int LB = 5>
void run(long plane_bytes, long pad_elems = 0) {
  const long n = plane_bytes / sizeof(float2);
  const long ps = n + pad_elems;
  float2 *in, *out;
  cudaMalloc(&in, (size_t)P * ps * sizeof(float2));
  cudaMalloc(&out, (size_t)12 * ps * sizeof(float2));
  cudaMemset(in, 0, (size_t)P * ps * sizeof(float2));
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k<P, AOSOA, UNROLL, LB>, 128, 0);
  if (per_sm > 5) per_sm = 5;  // the occupancy of the stencil kernels
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 2; ++w) k<P, AOSOA, UNROLL, LB><<<148 * per_sm, 128>>>(in, out, n, ps);
  cudaEventRecord(e0);
  for (int r = 0; r < 20; ++r) k<P, AOSOA, UNROLL, LB><<<148 * per_sm, 128>>>(in, out, n, ps);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= 20;
  printf("%s block=%4d unroll=%d pad=%6ld P=%3d planes of %ld MB, %d blocks/SM: %8.3f ms  %7.1f GB/s\n", AOSOA ? "AoSoA" : "SoA  ", AOSOA ? (1 << LB) : 0, UNROLL, pad_elems, P, plane_bytes >> 20, per_sm, ms,
         (double)(P + 12) * plane_bytes / ms / 1e6);
  cudaFree(in);
  cudaFree(out);
}

int main() {
  run<48, false, 1>(16l << 20);
  run<48, true, 1, 5>(16l << 20);
  run<48, true, 1, 6>(16l << 20);
  run<48, true, 1, 7>(16l << 20);
  run<48, true, 1, 9>(16l << 20);
  run<48, true, 1, 11>(16l << 20);
  run<48, true, 1, 13>(16l << 20);
  run<48, true, 1, 16>(16l << 20);
  return 0;
}
