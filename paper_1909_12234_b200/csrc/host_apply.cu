// Host-buffer apply (the reference-facing LatticeOperator.apply with numpy
// inputs, lattice.py:214-217): y_host = A x_host for reference-layout host
// vectors, with the PCIe transfers, the layout permutation and the stencil
// pipelined over x0-chunks on three streams.
//
// In the reference layout x0 is the slowest index, so chunk c = sites with
// x0 in [x0_c, x0_{c+1}) is one contiguous host range.  Chunk c's output
// needs input chunks c-1, c, c+1 (x0 hops, periodic), so the input is sent
// in the order n-1, 0, 1, ..., n-2 and output chunk c is computed as soon as
// its +1 neighbour has arrived; its device->host copy then overlaps the next
// chunks' host->device copies (PCIe is full duplex) and stencils.
#include <algorithm>
#include <vector>

#include "handle.cuh"

namespace mgt {

// ref chunk (sites x0 in [xb, xe), reference order) -> native field
template <typename R>
__global__ void from_ref_range_kernel(Geom g, int xb, int xe, const double2 *__restrict__ ref_chunk,
                                      cplx<R> *__restrict__ nat) {
  const int64_t per = (int64_t)g.L[1] * g.L[2] * g.L[3];
  const int64_t n = (int64_t)(xe - xb) * per;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i;
    int x[4];
    x[3] = (int)(r % g.L[3]);
    r /= g.L[3];
    x[2] = (int)(r % g.L[2]);
    r /= g.L[2];
    x[1] = (int)(r % g.L[1]);
    x[0] = xb + (int)(r / g.L[1]);
    const int64_t s = native_site(g, x);
    const double2 *src = ref_chunk + i * 12;
#pragma unroll
    for (int c = 0; c < 12; ++c) {
      double2 v = src[c];
      cplx<R> o;
      o.x = (R)v.x;
      o.y = (R)v.y;
      nat[(int64_t)c * g.V + s] = o;
    }
  }
}

template <typename R>
__global__ void to_ref_range_kernel(Geom g, int xb, int xe, const cplx<R> *__restrict__ nat,
                                    double2 *__restrict__ ref_chunk) {
  const int64_t per = (int64_t)g.L[1] * g.L[2] * g.L[3];
  const int64_t n = (int64_t)(xe - xb) * per;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i;
    int x[4];
    x[3] = (int)(r % g.L[3]);
    r /= g.L[3];
    x[2] = (int)(r % g.L[2]);
    r /= g.L[2];
    x[1] = (int)(r % g.L[1]);
    x[0] = xb + (int)(r / g.L[1]);
    const int64_t s = native_site(g, x);
    double2 *dst = ref_chunk + i * 12;
#pragma unroll
    for (int c = 0; c < 12; ++c) {
      cplx<R> v = nat[(int64_t)c * g.V + s];
      dst[c] = make_double2((double)v.x, (double)v.y);
    }
  }
}

// stencil on the sites with x0 in [xb, xe)
template <typename R, int RECON>
__global__ void __launch_bounds__(128, (sizeof(R) == 8 ? 3 : 4))
    wilson_range_kernel(WilsonParams P, int xb, int xe, const cplx<R> *__restrict__ in, cplx<R> *__restrict__ out,
                        LinkField<R, RECON> links) {
  const int64_t row = (int64_t)P.g.L[1] * P.g.L[2];
  const int64_t w = (int64_t)(xe - xb) * row;
  const int64_t n = w * P.g.L[3];
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < n; o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = o / w;
    const int64_t site = t * P.g.stride[3] + (int64_t)xb * row + (o - t * w);
    C<R> y[4][3], xc[4][3];
    wilson_eval<R, RECON>(P, in, links, site, y, xc);
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int c = 0; c < 3; ++c) stc_cs(out + (a * 3 + c) * P.g.V + site, y[a][c]);
  }
}

template <typename R, int RECON>
static int host_apply_t(mgt_wilson_s *h, const double2 *xh, double2 *yh, int flags, double tau, int nchunks,
                        cudaStream_t user) {
  const Geom &g = h->g;
  const int L0 = g.L[0];
  nchunks = std::max(1, std::min(nchunks, L0));
  std::vector<int> xb(nchunks + 1);
  for (int c = 0; c <= nchunks; ++c) xb[c] = (int)((int64_t)L0 * c / nchunks);
  const int64_t per = (int64_t)g.L[1] * g.L[2] * g.L[3];  // sites per x0 plane
  const size_t field_ref = (size_t)g.V * 12 * sizeof(double2);
  const size_t field_nat = (size_t)g.V * 12 * sizeof(cplx<R>);
  double2 *din = nullptr, *dout = nullptr;
  cplx<R> *nin = nullptr, *nout = nullptr;
  MGT_CUDA(scratch_alloc((void **)&din, field_ref, user));
  MGT_CUDA(scratch_alloc((void **)&dout, field_ref, user));
  MGT_CUDA(scratch_alloc((void **)&nin, field_nat, user));
  MGT_CUDA(scratch_alloc((void **)&nout, field_nat, user));
  cudaStream_t s_in, s_cmp, s_out;
  MGT_CUDA(cudaStreamCreateWithFlags(&s_in, cudaStreamNonBlocking));
  MGT_CUDA(cudaStreamCreateWithFlags(&s_cmp, cudaStreamNonBlocking));
  MGT_CUDA(cudaStreamCreateWithFlags(&s_out, cudaStreamNonBlocking));
  cudaEvent_t start, done_out;
  std::vector<cudaEvent_t> ev_in(nchunks), ev_cmp(nchunks);
  MGT_CUDA(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
  MGT_CUDA(cudaEventCreateWithFlags(&done_out, cudaEventDisableTiming));
  for (int c = 0; c < nchunks; ++c) {
    MGT_CUDA(cudaEventCreateWithFlags(&ev_in[c], cudaEventDisableTiming));
    MGT_CUDA(cudaEventCreateWithFlags(&ev_cmp[c], cudaEventDisableTiming));
  }
  // everything starts after the scratch allocations on the user stream
  MGT_CUDA(cudaEventRecord(start, user));
  MGT_CUDA(cudaStreamWaitEvent(s_in, start, 0));
  MGT_CUDA(cudaStreamWaitEvent(s_cmp, start, 0));
  MGT_CUDA(cudaStreamWaitEvent(s_out, start, 0));
  WilsonParams P = make_params(h, flags, tau);
  LinkField<R, RECON> lf{reinterpret_cast<const cplx<R> *>(h->links), g.V};
  auto send = [&](int c) -> int {
    const int64_t off = (int64_t)xb[c] * per * 12;
    const size_t bytes = (size_t)(xb[c + 1] - xb[c]) * per * 12 * sizeof(double2);
    MGT_CUDA(cudaMemcpyAsync(din + off, xh + off, bytes, cudaMemcpyHostToDevice, s_in));
    const int64_t n = (int64_t)(xb[c + 1] - xb[c]) * per;
    from_ref_range_kernel<R><<<grid_for(n, 256, 8), 256, 0, s_in>>>(g, xb[c], xb[c + 1], din + off, nin);
    MGT_LAUNCH_CHECK("from_ref_range_kernel");
    MGT_CUDA(cudaEventRecord(ev_in[c], s_in));
    return MGT_OK;
  };
  auto compute = [&](int c) -> int {
    // needs chunks c-1, c, c+1 (periodic in x0)
    for (int d : {c - 1, c, c + 1}) MGT_CUDA(cudaStreamWaitEvent(s_cmp, ev_in[(d + nchunks) % nchunks], 0));
    const int64_t n = (int64_t)(xb[c + 1] - xb[c]) * per;
    wilson_range_kernel<R, RECON><<<grid_for(n, 128, 3), 128, 0, s_cmp>>>(P, xb[c], xb[c + 1], nin, nout, lf);
    MGT_LAUNCH_CHECK("wilson_range_kernel");
    const int64_t off = (int64_t)xb[c] * per * 12;
    to_ref_range_kernel<R><<<grid_for(n, 256, 8), 256, 0, s_cmp>>>(g, xb[c], xb[c + 1], nout, dout + off);
    MGT_LAUNCH_CHECK("to_ref_range_kernel");
    MGT_CUDA(cudaEventRecord(ev_cmp[c], s_cmp));
    MGT_CUDA(cudaStreamWaitEvent(s_out, ev_cmp[c], 0));
    MGT_CUDA(cudaMemcpyAsync(yh + off, dout + off, (size_t)n * 12 * sizeof(double2), cudaMemcpyDeviceToHost, s_out));
    return MGT_OK;
  };
  int rc = MGT_OK;
  // input order n-1, 0, 1, ..., n-2; output c once c+1 is in
  if (nchunks == 1) {
    rc = send(0);
    if (!rc) rc = compute(0);
  } else {
    rc = send(nchunks - 1);
    for (int c = 0; c < nchunks - 1 && !rc; ++c) {
      rc = send(c);
      if (!rc && c >= 1) rc = compute(c - 1);
    }
    if (!rc) rc = compute(nchunks - 2);
    if (!rc) rc = compute(nchunks - 1);
  }
  cudaEventRecord(done_out, s_out);
  cudaStreamWaitEvent(user, done_out, 0);
  cudaFreeAsync(din, user);
  cudaFreeAsync(dout, user);
  cudaFreeAsync(nin, user);
  cudaFreeAsync(nout, user);
  cudaStreamSynchronize(user);  // host output is complete when the call returns
  for (int c = 0; c < nchunks; ++c) {
    cudaEventDestroy(ev_in[c]);
    cudaEventDestroy(ev_cmp[c]);
  }
  cudaEventDestroy(start);
  cudaEventDestroy(done_out);
  cudaStreamDestroy(s_in);
  cudaStreamDestroy(s_cmp);
  cudaStreamDestroy(s_out);
  return rc;
}

}  // namespace mgt

using namespace mgt;

extern "C" int mgt_wilson_apply_host(mgt_wilson_t h, const void *x_host, void *y_host, int n_rhs, int flags,
                                     double tau, int nchunks, void *stream) {
  if (!h || !x_host || !y_host || n_rhs < 1) return fail(MGT_ERR_INVALID, "mgt_wilson_apply_host: bad argument");
  if (h->slab) return fail(MGT_ERR_INVALID, "mgt_wilson_apply_host: slab handles are not supported");
  cudaStream_t st = as_stream(stream);
  const size_t field = (size_t)h->g.V * 12;
  for (int r = 0; r < n_rhs; ++r) {
    const double2 *x = (const double2 *)x_host + r * field;
    double2 *y = (double2 *)y_host + r * field;
    int rc;
    if (h->prec == 64)
      rc = h->recon == 18 ? host_apply_t<double, 18>(h, x, y, flags, tau, nchunks, st)
                          : host_apply_t<double, 12>(h, x, y, flags, tau, nchunks, st);
    else
      rc = h->recon == 18 ? host_apply_t<float, 18>(h, x, y, flags, tau, nchunks, st)
                          : host_apply_t<float, 12>(h, x, y, flags, tau, nchunks, st);
    if (rc) return rc;
  }
  return MGT_OK;
}
