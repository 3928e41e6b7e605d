// Reference <-> native layout permutation and the SU(3) link exponential.
#include "common.cuh"

namespace mgt {

// native (n_rhs, 12, V)  <->  rhs-interleaved (12, V, n_rhs)
template <typename R>
__global__ void rhs_interleave_kernel(int64_t n12v, int n_rhs, int inverse, const cplx<R> *__restrict__ a,
                                      cplx<R> *__restrict__ b) {
  const int64_t n = n12v * n_rhs;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n; idx += (int64_t)gridDim.x * blockDim.x) {
    // idx walks the interleaved order: e = idx / n_rhs, rhs = idx % n_rhs
    const int64_t e = idx / n_rhs;
    const int rhs = (int)(idx - e * n_rhs);
    const int64_t nat = (int64_t)rhs * n12v + e;
    if (inverse)
      b[nat] = a[idx];
    else
      b[idx] = a[nat];
  }
}

// ref (n_rhs, V_ref, 12) complex128  ->  native (n_rhs, 12, V_native)
template <typename R>
__global__ void spinor_from_ref_kernel(Geom g, int n_rhs, const double2 *__restrict__ ref, cplx<R> *__restrict__ nat) {
  const int64_t n = g.V * n_rhs;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n; idx += (int64_t)gridDim.x * blockDim.x) {
    const int rhs = (int)(idx / g.V);
    const int64_t s = idx - (int64_t)rhs * g.V;
    int x[4];
    native_coords(g, s, x);
    const int64_t r = ref_site(g, x);
    const double2 *src = ref + ((int64_t)rhs * g.V + r) * 12;
    cplx<R> *dst = nat + (int64_t)rhs * 12 * g.V + s;
#pragma unroll
    for (int c = 0; c < 12; ++c) {
      double2 v = src[c];
      cplx<R> o;
      o.x = (R)v.x;
      o.y = (R)v.y;
      dst[(int64_t)c * g.V] = o;
    }
  }
}

template <typename R>
__global__ void spinor_to_ref_kernel(Geom g, int n_rhs, const cplx<R> *__restrict__ nat, double2 *__restrict__ ref) {
  const int64_t n = g.V * n_rhs;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n; idx += (int64_t)gridDim.x * blockDim.x) {
    const int rhs = (int)(idx / g.V);
    const int64_t s = idx - (int64_t)rhs * g.V;
    int x[4];
    native_coords(g, s, x);
    const int64_t r = ref_site(g, x);
    double2 *dst = ref + ((int64_t)rhs * g.V + r) * 12;
    const cplx<R> *src = nat + (int64_t)rhs * 12 * g.V + s;
#pragma unroll
    for (int c = 0; c < 12; ++c) {
      cplx<R> v = src[(int64_t)c * g.V];
      dst[c] = make_double2((double)v.x, (double)v.y);
    }
  }
}

// ---------------------------------------------------------------------------
// U = expm(i eps H), H traceless Hermitian from 8 normals (draw order and the
// normals -> H map are documented in paper_1909_12234_b200/gauge.py).
// Scaling and squaring with a degree-18 Taylor polynomial on ||Q|| <= 1/2.
struct M3 {
  C<double> a[3][3];
};

__device__ __forceinline__ M3 m3_mul(const M3 &x, const M3 &y) {
  M3 z;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      C<double> s(0.0, 0.0);
#pragma unroll
      for (int k = 0; k < 3; ++k) s = cfma(x.a[i][k], y.a[k][j], s);
      z.a[i][j] = s;
    }
  return z;
}

__global__ void su3_expm_kernel(double eps, const double *__restrict__ normals, int64_t site_begin, int64_t nsites,
                                double2 *__restrict__ links) {
  const int64_t n = nsites * 4;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n; idx += (int64_t)gridDim.x * blockDim.x) {
    const double *nv = normals + idx * 8;
    const double r2 = 1.4142135623730951, r6 = 2.449489742783178;
    C<double> H[3][3];
    H[0][1] = C<double>(nv[0] / r2, nv[1] / r2);
    H[0][2] = C<double>(nv[2] / r2, nv[3] / r2);
    H[1][2] = C<double>(nv[4] / r2, nv[5] / r2);
    H[1][0] = conj(H[0][1]);
    H[2][0] = conj(H[0][2]);
    H[2][1] = conj(H[1][2]);
    H[0][0] = C<double>(nv[6] / r2 + nv[7] / r6, 0.0);
    H[1][1] = C<double>(-nv[6] / r2 + nv[7] / r6, 0.0);
    H[2][2] = C<double>(-2.0 * nv[7] / r6, 0.0);
    // Q = i eps H
    M3 Q;
    double nrm2 = 0.0;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        Q.a[i][j] = times_i(eps * H[i][j]);
        nrm2 += Q.a[i][j].re * Q.a[i][j].re + Q.a[i][j].im * Q.a[i][j].im;
      }
    double nrm = sqrt(nrm2);
    int sq = 0;
    double scale = 1.0;
    while (nrm * scale > 0.5) {
      scale *= 0.5;
      ++sq;
    }
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) Q.a[i][j] = scale * Q.a[i][j];
    // Horner: E = I + Q/1 (I + Q/2 (I + ... (I + Q/18)))
    M3 E;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) E.a[i][j] = C<double>(i == j ? 1.0 : 0.0, 0.0);
    for (int k = 18; k >= 1; --k) {
      M3 T = m3_mul(Q, E);
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) E.a[i][j] = (1.0 / k) * T.a[i][j] + C<double>(i == j ? 1.0 : 0.0, 0.0);
    }
    for (int k = 0; k < sq; ++k) E = m3_mul(E, E);
    double2 *out = links + (site_begin * 4 + idx) * 9;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) out[i * 3 + j] = make_double2(E.a[i][j].re, E.a[i][j].im);
  }
}

}  // namespace mgt

using namespace mgt;

extern "C" {

int mgt_spinor_from_ref(const int dims[4], int prec, const void *ref_dev, void *native_dev, int n_rhs, void *stream) {
  if (!dims || !ref_dev || !native_dev || n_rhs < 1) return fail(MGT_ERR_INVALID, "mgt_spinor_from_ref: bad argument");
  Geom g = make_geom(dims);
  const int block = 256, grid = grid_for(g.V * n_rhs, block, 8);
  if (prec == 64)
    spinor_from_ref_kernel<double><<<grid, block, 0, as_stream(stream)>>>(g, n_rhs, (const double2 *)ref_dev,
                                                                           (double2 *)native_dev);
  else if (prec == 32)
    spinor_from_ref_kernel<float><<<grid, block, 0, as_stream(stream)>>>(g, n_rhs, (const double2 *)ref_dev,
                                                                          (float2 *)native_dev);
  else
    return fail(MGT_ERR_INVALID, "prec must be 64 or 32");
  MGT_LAUNCH_CHECK("spinor_from_ref_kernel");
  return MGT_OK;
}

int mgt_spinor_to_ref(const int dims[4], int prec, const void *native_dev, void *ref_dev, int n_rhs, void *stream) {
  if (!dims || !ref_dev || !native_dev || n_rhs < 1) return fail(MGT_ERR_INVALID, "mgt_spinor_to_ref: bad argument");
  Geom g = make_geom(dims);
  const int block = 256, grid = grid_for(g.V * n_rhs, block, 8);
  if (prec == 64)
    spinor_to_ref_kernel<double><<<grid, block, 0, as_stream(stream)>>>(g, n_rhs, (const double2 *)native_dev,
                                                                         (double2 *)ref_dev);
  else if (prec == 32)
    spinor_to_ref_kernel<float><<<grid, block, 0, as_stream(stream)>>>(g, n_rhs, (const float2 *)native_dev,
                                                                        (double2 *)ref_dev);
  else
    return fail(MGT_ERR_INVALID, "prec must be 64 or 32");
  MGT_LAUNCH_CHECK("spinor_to_ref_kernel");
  return MGT_OK;
}

int mgt_su3_expm(double eps, const double *normals_dev, int64_t site_begin, int64_t nsites, void *links_ref_dev,
                 void *stream) {
  if (!normals_dev || !links_ref_dev || nsites < 0 || site_begin < 0)
    return fail(MGT_ERR_INVALID, "mgt_su3_expm: bad argument");
  if (nsites == 0) return MGT_OK;
  const int block = 128, grid = grid_for(nsites * 4, block, 16);
  su3_expm_kernel<<<grid, block, 0, as_stream(stream)>>>(eps, normals_dev, site_begin, nsites,
                                                          (double2 *)links_ref_dev);
  MGT_LAUNCH_CHECK("su3_expm_kernel");
  return MGT_OK;
}

int mgt_rhs_interleave(int64_t V, int prec, int n_rhs, int inverse, const void *in_dev, void *out_dev,
                       void *stream) {
  if (!in_dev || !out_dev || n_rhs < 1 || V < 1 || in_dev == out_dev)
    return fail(MGT_ERR_INVALID, "mgt_rhs_interleave: bad argument");
  const int64_t n12v = 12 * V;
  const int block = 256, grid = grid_for(n12v * n_rhs, block, 8);
  if (prec == 64)
    rhs_interleave_kernel<double><<<grid, block, 0, as_stream(stream)>>>(
        n12v, n_rhs, inverse, (const cplx<double> *)in_dev, (cplx<double> *)out_dev);
  else if (prec == 32)
    rhs_interleave_kernel<float><<<grid, block, 0, as_stream(stream)>>>(
        n12v, n_rhs, inverse, (const cplx<float> *)in_dev, (cplx<float> *)out_dev);
  else
    return fail(MGT_ERR_INVALID, "prec must be 64 or 32");
  MGT_LAUNCH_CHECK("rhs_interleave_kernel");
  return MGT_OK;
}

}  // extern "C"
