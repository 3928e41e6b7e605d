// FP64 tensor-core (DMMA) issue-rate microbenchmark on sm_100a: independent
// accumulator chains of mma.sync f64 shapes, 8 warps per SM x all SMs.
#include <cstdio>
#include <cuda_runtime.h>

template <int SHAPE>
__global__ void __launch_bounds__(256) k(double *out, int iters, double a0, double b0) {
  double c[8][4];
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 4; ++j) c[i][j] = 0.0;
  double a[4] = {a0, a0 + 1, a0 + 2, a0 + 3}, b[2] = {b0, b0 + 1};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (SHAPE == 0)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a[0]), "d"(b[0]));
      if (SHAPE == 1)
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                     : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
      if (SHAPE == 2)
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
      if (SHAPE == 3) {  // plain DFMA, 4 per "instruction slot" for comparison
        c[i][0] = fma(a[0], b[0], c[i][0]);
        c[i][1] = fma(a[1], b[0], c[i][1]);
        c[i][2] = fma(a[2], b[1], c[i][2]);
        c[i][3] = fma(a[3], b[1], c[i][3]);
      }
    }
  }
  double s = 0;
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 4; ++j) s += c[i][j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int SHAPE>
void run(const char *name, double flops_per_inst, int sms) {
  double *out;
  cudaMalloc(&out, sizeof(double) * sms * 256 * 2);
  const int iters = 20000;
  k<SHAPE><<<sms * 2, 256>>>(out, 10, 1.0, 2.0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<SHAPE><<<sms * 2, 256>>>(out, iters, 1.0, 2.0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double insts = (double)sms * 2 * 8 * iters * 8 * (SHAPE == 3 ? 4 : 1);  // warp instructions
  printf("%-12s %8.3f ms  %.2f TFLOP/s  %.2f warp-inst/us/SM (err %s)\n", name, ms,
         insts * flops_per_inst / ms / 1e9, insts / sms / (ms * 1e3), cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0>("m8n8k4", 512, sms);
  run<1>("m16n8k4", 1024, sms);
  run<2>("m16n8k8", 2048, sms);
  run<3>("dfma", 64, sms);
  return 0;
}
