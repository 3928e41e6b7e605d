// Deterministic complex BLAS-1 on device fields (numpy vdot semantics).
#include "reduce.cuh"

namespace mgt {

// out[2r..2r+1] = sum_i conj(a_i) b_i over field r (len entries each)
__global__ void __launch_bounds__(kRedBlock) cdot_kernel(const double2 *__restrict__ a, const double2 *__restrict__ b,
                                                         int64_t len, double *partials, unsigned *ticket, double *out) {
  double acc[2] = {0.0, 0.0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len; i += (int64_t)gridDim.x * blockDim.x) {
    C<double> x = ldc(a + i), y = ldc(b + i);
    acc[0] += x.re * y.re + x.im * y.im;
    acc[1] += x.re * y.im - x.im * y.re;
  }
  if (reduce_publish<1, 2>(acc, partials, ticket)) {
    double r[2];
    reduce_finish<2>(partials, ticket, r);
    if (threadIdx.x == 0) {
      out[0] = r[0];
      out[1] = r[1];
    }
  }
}

}  // namespace mgt

using namespace mgt;

extern "C" int mgt_cdot(const void *a_dev, const void *b_dev, int64_t len, int n_rhs, double *out_dev, void *stream) {
  if (!a_dev || !b_dev || !out_dev || len < 0 || n_rhs < 1) return fail(MGT_ERR_INVALID, "mgt_cdot: bad argument");
  cudaStream_t st = as_stream(stream);
  const int grid = grid_for(len, kRedBlock, 4);
  void *tmp = nullptr;
  const size_t bytes = (size_t)grid * 2 * sizeof(double) + 256;
  MGT_CUDA(scratch_alloc(&tmp, bytes, st));
  double *partials = (double *)((char *)tmp + 256);
  unsigned *ticket = (unsigned *)tmp;
  MGT_CUDA(cudaMemsetAsync(ticket, 0, sizeof(unsigned), st));
  for (int r = 0; r < n_rhs; ++r) {
    cdot_kernel<<<grid, kRedBlock, 0, st>>>((const double2 *)a_dev + r * len, (const double2 *)b_dev + r * len, len,
                                            partials, ticket, out_dev + 2 * r);
    MGT_LAUNCH_CHECK("cdot_kernel");
  }
  MGT_CUDA(cudaFreeAsync(tmp, st));
  return MGT_OK;
}
