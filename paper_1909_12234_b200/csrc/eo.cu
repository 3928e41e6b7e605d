// Even-odd (checkerboard) support: per-parity links, parity split/merge of
// native fields and the Schur-complement operator S (eo_core.cuh).  The
// BiCGStab solver (bicgstab.cu) runs on S; these entry points expose the
// same pieces to callers and tests.
#include <string>

#include "eo_core.cuh"
#include "handle.cuh"

namespace mgt {

template <typename R, int NL>
__global__ void eo_links_kernel(EoGeom E, const cplx<R> *__restrict__ full, cplx<R> *__restrict__ cb) {
  const int64_t n = E.g.V;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n; idx += (int64_t)gridDim.x * blockDim.x) {
    const int p = (int)(idx / E.Vh);
    const int64_t c = idx - (int64_t)p * E.Vh;
    int x[4];
    const int64_t f = eo_coords(E, p, c, x);
    cplx<R> *dst = cb + (int64_t)p * 4 * NL * E.Vh;
    constexpr int RECON = 2 * NL;
#pragma unroll
    for (int mu = 0; mu < 4; ++mu)
#pragma unroll
      for (int e = 0; e < NL; ++e) dst[link_index<RECON>(mu, e, c, E.Vh)] = full[link_index<RECON>(mu, e, f, E.g.V)];
  }
}

// full native (n, 12, V) <-> parity halves (n, 12, Vh); dir 0 split, 1 merge
template <typename R>
__global__ void eo_split_kernel(EoGeom E, int n_rhs, int dir, cplx<R> *__restrict__ full, cplx<R> *__restrict__ ev,
                                cplx<R> *__restrict__ od) {
  const int64_t n = E.Vh * n_rhs;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n; idx += (int64_t)gridDim.x * blockDim.x) {
    const int rhs = (int)(idx / E.Vh);
    const int64_t c = idx - (int64_t)rhs * E.Vh;
    int x[4];
    const int64_t fe = eo_coords(E, 0, c, x);
    const int64_t fo = eo_coords(E, 1, c, x);
    cplx<R> *F = full + (int64_t)rhs * 12 * E.g.V;
    cplx<R> *Ev = ev + (int64_t)rhs * 12 * E.Vh + c;
    cplx<R> *Od = od + (int64_t)rhs * 12 * E.Vh + c;
#pragma unroll
    for (int k = 0; k < 12; ++k) {
      if (dir == 0) {
        Ev[(int64_t)k * E.Vh] = F[(int64_t)k * E.g.V + fe];
        Od[(int64_t)k * E.Vh] = F[(int64_t)k * E.g.V + fo];
      } else {
        F[(int64_t)k * E.g.V + fe] = Ev[(int64_t)k * E.Vh];
        F[(int64_t)k * E.g.V + fo] = Od[(int64_t)k * E.Vh];
      }
    }
  }
}

// one half-lattice role over n_rhs fields (blockIdx.y = rhs)
template <typename R, int RECON>
__global__ void __launch_bounds__(128, (sizeof(R) == 8 ? 3 : 4))
    eo_role_kernel(EoGeom E, int pout, EoCoef K, const cplx<R> *__restrict__ in, const cplx<R> *__restrict__ ctr,
                   cplx<R> *__restrict__ out, LinkField<R, RECON> lout, LinkField<R, RECON> lin) {
  const int rhs = blockIdx.y;
  const int64_t off = (int64_t)rhs * 12 * E.Vh;
  const cplx<R> *ctr_r = ctr ? ctr + off : nullptr;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < E.Vh; c += (int64_t)gridDim.x * blockDim.x) {
    C<R> y[4][3], cc[4][3];
    eo_eval<R, RECON>(E, pout, K, in + off, ctr_r, lout, lin, c, y, cc);
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int k = 0; k < 3; ++k) stc(out + off + (int64_t)(a * 3 + k) * E.Vh + c, y[a][k]);
  }
}

bool eo_available(const mgt_wilson_s *h) {
  if (h->slab) return false;
  for (int i = 0; i < 4; ++i)
    if (h->g.L[i] % 2) return false;
  return true;
}

template <typename R>
static void launch_eo_links(const mgt_wilson_s *h, const EoGeom &E, cudaStream_t st) {
  const int grid = grid_for(h->g.V, 256, 8);
  if (h->recon == 12)
    eo_links_kernel<R, 6><<<grid, 256, 0, st>>>(E, (const cplx<R> *)h->links, (cplx<R> *)h->links_cb);
  else
    eo_links_kernel<R, 9><<<grid, 256, 0, st>>>(E, (const cplx<R> *)h->links, (cplx<R> *)h->links_cb);
}

int eo_prepare(mgt_wilson_s *h, cudaStream_t st) {
  if (!eo_available(h)) return fail(MGT_ERR_INVALID, "even-odd form needs every lattice extent even");
  std::lock_guard<std::mutex> lk(h->eo_mu);
  if (h->links_cb) return MGT_OK;
  void *p = nullptr;
  MGT_CUDA(cudaMalloc(&p, h->link_bytes));
  h->links_cb = p;
  EoGeom E = make_eo_geom(h->g, h->antiperiodic);
  if (h->prec == 64)
    launch_eo_links<double>(h, E, st);
  else
    launch_eo_links<float>(h, E, st);
  MGT_LAUNCH_CHECK("eo_links_kernel");
  // other threads' streams may use the copy as soon as this returns
  MGT_CUDA(cudaStreamSynchronize(st));
  return MGT_OK;
}

__global__ void narrow_kernel(const double2 *__restrict__ in, float2 *__restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double2 v = in[i];
    out[i] = make_float2((float)v.x, (float)v.y);
  }
}

// fp32 per-parity links of the mixed solver, full 3x3 (18 reals): built from
// the fp64 per-parity links (either storage), third row reconstructed once
// here in fp64 instead of in every fp32 hop.  Layout ((mu*9 + e)*Vh + c) per
// parity, parities back to back.
template <int RECON>
__global__ void narrow_full_kernel(const double2 *__restrict__ cb, float2 *__restrict__ out, int64_t Vh,
                                   size_t parity_bytes) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < 2 * 4 * Vh;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int par = (int)(i / (4 * Vh));
    const int64_t j = i - (int64_t)par * 4 * Vh;
    const int mu = (int)(j / Vh);
    const int64_t c = j - (int64_t)mu * Vh;
    LinkField<double, RECON> L{reinterpret_cast<const double2 *>((const char *)cb + par * parity_bytes), Vh};
    C<double> u[3][3];
    L.load(mu, c, u);
    float2 *o = out + (int64_t)par * 4 * 9 * Vh;
#pragma unroll
    for (int e = 0; e < 9; ++e)
      o[((int64_t)mu * 9 + e) * Vh + c] = make_float2((float)u[e / 3][e % 3].re, (float)u[e / 3][e % 3].im);
  }
}

int eo_prepare_mixed(mgt_wilson_s *h, cudaStream_t st) {
  if (h->prec != 64) return fail(MGT_ERR_INVALID, "mixed-precision solve needs a complex128 operator");
  int rc = eo_prepare(h, st);
  if (rc) return rc;
  std::lock_guard<std::mutex> lk(h->eo_mu);
  if (h->links_cb32) return MGT_OK;
  void *p = nullptr;
#if MGT_MIXED_L18
  const int64_t Vh = h->g.V / 2;
  MGT_CUDA(cudaMalloc(&p, (size_t)2 * 4 * 9 * Vh * sizeof(float2)));
  h->links_cb32 = p;
  if (h->recon == 12)
    narrow_full_kernel<12><<<grid_for(8 * Vh, 256, 8), 256, 0, st>>>((const double2 *)h->links_cb, (float2 *)p, Vh,
                                                                     h->link_bytes / 2);
  else
    narrow_full_kernel<18><<<grid_for(8 * Vh, 256, 8), 256, 0, st>>>((const double2 *)h->links_cb, (float2 *)p, Vh,
                                                                     h->link_bytes / 2);
  MGT_LAUNCH_CHECK("narrow_full_kernel (fp32 links)");
#else
  MGT_CUDA(cudaMalloc(&p, h->link_bytes / 2));
  h->links_cb32 = p;
  const int64_t n = (int64_t)(h->link_bytes / sizeof(double2));
  narrow_kernel<<<grid_for(n, 256, 8), 256, 0, st>>>((const double2 *)h->links_cb, (float2 *)p, n);
  MGT_LAUNCH_CHECK("narrow_kernel (fp32 links)");
#endif
  MGT_CUDA(cudaStreamSynchronize(st));
  return MGT_OK;
}

template <typename R, int RECON>
static int schur_t(mgt_wilson_s *h, const WilsonParams &P, const void *x, void *y, int n_rhs, cudaStream_t st) {
  EoGeom E = make_eo_geom(h->g, h->antiperiodic);
  EoRoles Ro = make_eo_roles(P);
  const size_t lb = h->link_bytes / 2;  // one parity's links
  LinkField<R, RECON> le{(const cplx<R> *)h->links_cb, E.Vh};
  LinkField<R, RECON> lo{(const cplx<R> *)((const char *)h->links_cb + lb), E.Vh};
  void *tmp = nullptr;
  MGT_CUDA(scratch_alloc(&tmp, (size_t)n_rhs * 12 * E.Vh * sizeof(cplx<R>), st));
  dim3 grid(grid_for(E.Vh, 128, 4), n_rhs);
  eo_role_kernel<R, RECON><<<grid, 128, 0, st>>>(E, 1, Ro.first, (const cplx<R> *)x, nullptr, (cplx<R> *)tmp, lo, le);
  eo_role_kernel<R, RECON><<<grid, 128, 0, st>>>(E, 0, Ro.second, (const cplx<R> *)tmp, (const cplx<R> *)x,
                                                 (cplx<R> *)y, le, lo);
  MGT_LAUNCH_CHECK("eo_role_kernel");
  cudaFreeAsync(tmp, st);
  return MGT_OK;
}

}  // namespace mgt

using namespace mgt;

extern "C" {

int mgt_wilson_eo_split(mgt_wilson_t h, const void *x_full_dev, void *x_even_dev, void *x_odd_dev, int n_rhs,
                        void *stream) {
  if (!h || !x_full_dev || !x_even_dev || !x_odd_dev || n_rhs < 1)
    return fail(MGT_ERR_INVALID, "mgt_wilson_eo_split: bad argument");
  if (!eo_available(h)) return fail(MGT_ERR_INVALID, "even-odd form needs every lattice extent even");
  EoGeom E = make_eo_geom(h->g, h->antiperiodic);
  const int grid = grid_for(E.Vh * n_rhs, 256, 8);
  if (h->prec == 64)
    eo_split_kernel<double><<<grid, 256, 0, as_stream(stream)>>>(E, n_rhs, 0, (cplx<double> *)x_full_dev,
                                                                  (cplx<double> *)x_even_dev, (cplx<double> *)x_odd_dev);
  else
    eo_split_kernel<float><<<grid, 256, 0, as_stream(stream)>>>(E, n_rhs, 0, (cplx<float> *)x_full_dev,
                                                                 (cplx<float> *)x_even_dev, (cplx<float> *)x_odd_dev);
  MGT_LAUNCH_CHECK("eo_split_kernel");
  return MGT_OK;
}

int mgt_wilson_eo_merge(mgt_wilson_t h, const void *x_even_dev, const void *x_odd_dev, void *x_full_dev, int n_rhs,
                        void *stream) {
  if (!h || !x_full_dev || !x_even_dev || !x_odd_dev || n_rhs < 1)
    return fail(MGT_ERR_INVALID, "mgt_wilson_eo_merge: bad argument");
  if (!eo_available(h)) return fail(MGT_ERR_INVALID, "even-odd form needs every lattice extent even");
  EoGeom E = make_eo_geom(h->g, h->antiperiodic);
  const int grid = grid_for(E.Vh * n_rhs, 256, 8);
  if (h->prec == 64)
    eo_split_kernel<double><<<grid, 256, 0, as_stream(stream)>>>(
        E, n_rhs, 1, (cplx<double> *)x_full_dev, (cplx<double> *)x_even_dev, (cplx<double> *)x_odd_dev);
  else
    eo_split_kernel<float><<<grid, 256, 0, as_stream(stream)>>>(
        E, n_rhs, 1, (cplx<float> *)x_full_dev, (cplx<float> *)x_even_dev, (cplx<float> *)x_odd_dev);
  MGT_LAUNCH_CHECK("eo_split_kernel");
  return MGT_OK;
}

int mgt_wilson_schur_apply(mgt_wilson_t h, const void *x_even_dev, void *y_even_dev, int n_rhs, int flags, double tau,
                           void *stream) {
  if (!h || !x_even_dev || !y_even_dev || n_rhs < 1) return fail(MGT_ERR_INVALID, "mgt_wilson_schur_apply: bad argument");
  if (x_even_dev == y_even_dev) return fail(MGT_ERR_INVALID, "mgt_wilson_schur_apply: in-place apply is not supported");
  cudaStream_t st = as_stream(stream);
  int rc = eo_prepare(h, st);
  if (rc) return rc;
  WilsonParams P = make_params(h, flags, tau);
  if (h->prec == 64)
    return h->recon == 18 ? schur_t<double, 18>(h, P, x_even_dev, y_even_dev, n_rhs, st)
                          : schur_t<double, 12>(h, P, x_even_dev, y_even_dev, n_rhs, st);
  return h->recon == 18 ? schur_t<float, 18>(h, P, x_even_dev, y_even_dev, n_rhs, st)
                        : schur_t<float, 12>(h, P, x_even_dev, y_even_dev, n_rhs, st);
}

}  // extern "C"
