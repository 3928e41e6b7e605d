// Restarted GCR(m) and GMRES(m) on the GPU.
//
// GCR(m) (reference: gcr_solve, krylov.py:52-118) -- the
// relaxation used by generate_null_vectors (multigrid.py:87-95, with
// restart = max_iter) and the GCR smoother (krylov.py:236-252).
//
// The control flow, breakdown test (||q|| <= 1e-14 ||q0||), restart by
// explicit residual and explicit-residual convergence confirmation follow the
// reference line by line; the vector algebra runs in fp64 device kernels and
// the handful of scalars per iteration are read back to the host (setup
// path, not the per-probe hot loop).  Modified Gram-Schmidt against the
// stored (z_j, q_j) pairs, in the reference's order.
#include <cmath>
#include <complex>
#include <vector>

#include "handle.cuh"
#include "reduce.cuh"

namespace mgt {

// y += a x ; w += a u   (a complex), n complex entries
__global__ void axpy2_kernel(int64_t n, double ar, double ai, const double2 *__restrict__ x, double2 *__restrict__ y,
                             const double2 *__restrict__ u, double2 *__restrict__ w) {
  const C<double> a(ar, ai);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    stc(y + i, ldc(y + i) + a * ldc(x + i));
    if (w) stc(w + i, ldc(w + i) + a * ldc(u + i));
  }
}

__global__ void scale2_kernel(int64_t n, double s, double2 *__restrict__ a, double2 *__restrict__ b) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double2 v = a[i];
    a[i] = make_double2(v.x * s, v.y * s);
    v = b[i];
    b[i] = make_double2(v.x * s, v.y * s);
  }
}

// r = b - y
__global__ void sub_kernel(int64_t n, const double2 *__restrict__ b, const double2 *__restrict__ y,
                           double2 *__restrict__ r) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    r[i] = make_double2(b[i].x - y[i].x, b[i].y - y[i].y);
}

// Device-scalar variants for the GCR loop: the coefficient (complex, from a
// dot product left in device memory) is applied as sgn * c; a set breakdown
// flag (device double) turns the update into a no-op, exactly as the host
// loop's `break` skips it.
__global__ void axpy2_dev_kernel(int64_t n, const double *__restrict__ c, double sgn, const double2 *__restrict__ x,
                                 double2 *__restrict__ y, const double2 *__restrict__ u, double2 *__restrict__ w,
                                 const double *__restrict__ flag) {
  if (flag && *flag != 0.0) return;
  const C<double> a(sgn * c[0], sgn * c[1]);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    stc(y + i, ldc(y + i) + a * ldc(x + i));
    if (w) stc(w + i, ldc(w + i) + a * ldc(u + i));
  }
}

// a, b *= 1 / sqrt(nrm2[0])   (the host loop's 1.0 / std::sqrt(|q|^2))
__global__ void scale2_dev_kernel(int64_t n, const double *__restrict__ nrm2, double2 *__restrict__ a,
                                  double2 *__restrict__ b, const double *__restrict__ flag) {
  if (*flag != 0.0) return;
  const double s = 1.0 / sqrt(nrm2[0]);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double2 v = a[i];
    a[i] = make_double2(v.x * s, v.y * s);
    v = b[i];
    b[i] = make_double2(v.x * s, v.y * s);
  }
}

// breakdown test of gcr_solve (krylov.py:95-97): ||q|| <= 1e-14 ||q0||
__global__ void gcr_flag_kernel(const double *__restrict__ q0sq, const double *__restrict__ qnsq, double *flag) {
  const double q0 = sqrt(q0sq[0]), qn = sqrt(qnsq[0]);
  *flag = (qn <= 1e-14 * fmax(q0, 1e-300)) ? 1.0 : 0.0;
}

struct Gcr {
  mgt_wilson_s *h;
  cudaStream_t st;
  int64_t n;
  double *dbuf;  // device scalar scratch (2 doubles)
  double *hbuf;  // pinned host copy

  int dot(const double2 *a, const double2 *b, C<double> &out) {
    int rc = mgt_cdot(a, b, n, 1, dbuf, st);
    if (rc) return rc;
    MGT_CUDA(cudaMemcpyAsync(hbuf, dbuf, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
    MGT_CUDA(cudaStreamSynchronize(st));
    out = C<double>(hbuf[0], hbuf[1]);
    return MGT_OK;
  }
  int norm(const double2 *a, double &out) {
    C<double> d;
    int rc = dot(a, a, d);
    out = std::sqrt(d.re);
    return rc;
  }
  int axpy2(C<double> a, const double2 *x, double2 *y, const double2 *u = nullptr, double2 *w = nullptr) {
    axpy2_kernel<<<grid_for(n, 256, 8), 256, 0, st>>>(n, a.re, a.im, x, y, u, w);
    MGT_LAUNCH_CHECK("axpy2_kernel");
    return MGT_OK;
  }
  int residual(const double2 *b, const double2 *x, double2 *tmp, double2 *r) {
    int rc = wilson_apply_native(h, x, tmp, 1, 0, 0.0, st);
    if (rc) return rc;
    sub_kernel<<<grid_for(n, 256, 8), 256, 0, st>>>(n, b, tmp, r);
    MGT_LAUNCH_CHECK("sub_kernel");
    return MGT_OK;
  }
};

}  // namespace mgt

using namespace mgt;

extern "C" {

size_t mgt_gcr_workspace_bytes(mgt_wilson_t h, int m) {
  if (!h || m < 1) return 0;
  return (size_t)(2 * m + 3) * 12 * h->g.V * sizeof(double2) + 256 + (size_t)(10 + 2 * m) * sizeof(double);
}

int mgt_gcr_solve(mgt_wilson_t h, const void *b_dev, void *x_dev, int m, int max_iter, double tol,
                  void *workspace_dev, int64_t *report_out, double *relres_out, void *stream) {
  if (!h || !b_dev || !x_dev || !workspace_dev || !report_out || !relres_out)
    return fail(MGT_ERR_INVALID, "mgt_gcr_solve: null argument");
  if (h->prec != 64) return fail(MGT_ERR_INVALID, "mgt_gcr_solve: needs a complex128 operator");
  if (m < 1 || max_iter < 1) return fail(MGT_ERR_INVALID, "mgt_gcr_solve: restart and max_iter must be >= 1");
  Gcr g;
  g.h = h;
  g.st = as_stream(stream);
  g.n = 12 * h->g.V;
  const double2 *b = (const double2 *)b_dev;
  double2 *x = (double2 *)x_dev;
  double2 *base = (double2 *)workspace_dev;
  double2 *r = base, *z = base + g.n, *q = base + 2 * g.n;
  double2 *Z = base + 3 * g.n, *Q = Z + (size_t)m * g.n;
  // scratch: reuse z as the apply temporary where safe; scalars after the fields
  g.dbuf = (double *)(Q + (size_t)m * g.n);
  static thread_local double *hb = nullptr;
  if (!hb) MGT_CUDA(cudaMallocHost((void **)&hb, 16 * sizeof(double)));
  g.hbuf = hb;
  const int64_t nb = g.n * sizeof(double2);
  int rc;
  int64_t matvecs = 0;
  double bn;
  if ((rc = g.norm(b, bn))) return rc;
  MGT_CUDA(cudaMemsetAsync(x, 0, nb, g.st));
  if (bn == 0.0) {
    report_out[0] = 0, report_out[1] = 0, report_out[2] = 1, report_out[3] = 0;
    relres_out[0] = 0.0;
    return MGT_OK;
  }
  MGT_CUDA(cudaMemcpyAsync(r, b, nb, cudaMemcpyDeviceToDevice, g.st));
  int stored = 0, it = 0, reason = 1;  // 1 max_iter, 2 breakdown
  double rn;
  if ((rc = g.norm(r, rn))) return rc;
  double rel = rn / bn;
  while (it < max_iter) {
    if (rel <= tol) {
      if ((rc = g.residual(b, x, z, r))) return rc;
      ++matvecs;
      if ((rc = g.norm(r, rn))) return rc;
      rel = rn / bn;
      if (rel <= tol) {
        report_out[0] = it, report_out[1] = matvecs, report_out[2] = 1, report_out[3] = 0;
        relres_out[0] = rel;
        return MGT_OK;
      }
      stored = 0;
    }
    MGT_CUDA(cudaMemcpyAsync(z, r, nb, cudaMemcpyDeviceToDevice, g.st));
    if ((rc = wilson_apply_native(h, z, q, 1, 0, 0.0, g.st))) return rc;
    ++matvecs;
    // the iteration's scalars stay on the device (sc[]): one host round trip
    // per iteration instead of one per dot product; the same arithmetic and
    // order as the host-scalar loop (modified Gram-Schmidt, krylov.py:86-111)
    double *sc = g.dbuf;  // [0] |q0|^2, [2] |q|^2, [4] alpha, [6] |r|^2, [8] flag, [10 + 2j] beta_j
    if ((rc = mgt_cdot(q, q, g.n, 1, sc + 0, g.st))) return rc;
    for (int j = 0; j < stored; ++j) {
      double2 *qj = Q + (size_t)j * g.n, *zj = Z + (size_t)j * g.n;
      if ((rc = mgt_cdot(qj, q, g.n, 1, sc + 10 + 2 * j, g.st))) return rc;
      axpy2_dev_kernel<<<grid_for(g.n, 256, 8), 256, 0, g.st>>>(g.n, sc + 10 + 2 * j, -1.0, qj, q, zj, z, nullptr);
      MGT_LAUNCH_CHECK("axpy2_dev_kernel");
    }
    if ((rc = mgt_cdot(q, q, g.n, 1, sc + 2, g.st))) return rc;
    gcr_flag_kernel<<<1, 1, 0, g.st>>>(sc + 0, sc + 2, sc + 8);
    scale2_dev_kernel<<<grid_for(g.n, 256, 8), 256, 0, g.st>>>(g.n, sc + 2, q, z, sc + 8);
    MGT_LAUNCH_CHECK("scale2_dev_kernel");
    if ((rc = mgt_cdot(q, r, g.n, 1, sc + 4, g.st))) return rc;
    axpy2_dev_kernel<<<grid_for(g.n, 256, 8), 256, 0, g.st>>>(g.n, sc + 4, 1.0, z, x, nullptr, nullptr, sc + 8);
    axpy2_dev_kernel<<<grid_for(g.n, 256, 8), 256, 0, g.st>>>(g.n, sc + 4, -1.0, q, r, nullptr, nullptr, sc + 8);
    MGT_LAUNCH_CHECK("axpy2_dev_kernel");
    if ((rc = mgt_cdot(r, r, g.n, 1, sc + 6, g.st))) return rc;
    MGT_CUDA(cudaMemcpyAsync(g.hbuf, sc, 10 * sizeof(double), cudaMemcpyDeviceToHost, g.st));
    MGT_CUDA(cudaStreamSynchronize(g.st));
    if (g.hbuf[8] != 0.0) {  // breakdown: x and r were left untouched
      reason = 2;
      break;
    }
    MGT_CUDA(cudaMemcpyAsync(Z + (size_t)stored * g.n, z, nb, cudaMemcpyDeviceToDevice, g.st));
    MGT_CUDA(cudaMemcpyAsync(Q + (size_t)stored * g.n, q, nb, cudaMemcpyDeviceToDevice, g.st));
    ++stored;
    ++it;
    rn = std::sqrt(g.hbuf[6]);
    rel = rn / bn;
    if (stored >= m) {
      stored = 0;
      if ((rc = g.residual(b, x, z, r))) return rc;
      ++matvecs;
      if ((rc = g.norm(r, rn))) return rc;
      rel = rn / bn;
    }
  }
  if ((rc = g.residual(b, x, z, r))) return rc;
  ++matvecs;
  if ((rc = g.norm(r, rn))) return rc;
  rel = rn / bn;
  const bool ok = rel <= tol;
  report_out[0] = it, report_out[1] = matvecs, report_out[2] = ok ? 1 : 0, report_out[3] = ok ? 0 : reason;
  relres_out[0] = rel;
  return MGT_OK;
}

// ---------------------------------------------------------------------------
// Restarted GMRES(m) (the north star's "BiCGStab/GMRES"; SURVEY 8(b)
// solve_gmres): Arnoldi with modified Gram-Schmidt on the device (fp64
// dot/axpy kernels), Givens rotations and the (m+1) x m least-squares
// problem on the host, x += V y at the end of each cycle, then the
// explicit residual b - A x restarts the next cycle -- the same
// explicit-residual contract (||b - A x|| <= tol ||b||) as gcr_solve.
// Operator variant by flags / tau as mgt_wilson_apply.  Breakdown: the
// Arnoldi vector vanishes (||w|| <= 1e-14 ||A v_j||) before convergence.
size_t mgt_gmres_workspace_bytes(mgt_wilson_t h, int m) {
  if (!h || m < 1) return 0;
  return (size_t)(m + 3) * 12 * h->g.V * sizeof(double2) + 256;
}

int mgt_gmres_solve(mgt_wilson_t h, const void *b_dev, void *x_dev, int m, int max_iter, double tol, int flags,
                    double tau, void *workspace_dev, int64_t *report_out, double *relres_out, void *stream) {
  if (!h || !b_dev || !x_dev || !workspace_dev || !report_out || !relres_out)
    return fail(MGT_ERR_INVALID, "mgt_gmres_solve: null argument");
  if (h->prec != 64) return fail(MGT_ERR_INVALID, "mgt_gmres_solve: needs a complex128 operator");
  if (m < 1 || max_iter < 1) return fail(MGT_ERR_INVALID, "mgt_gmres_solve: restart and max_iter must be >= 1");
  Gcr g;
  g.h = h;
  g.st = as_stream(stream);
  g.n = 12 * h->g.V;
  const double2 *b = (const double2 *)b_dev;
  double2 *x = (double2 *)x_dev;
  double2 *base = (double2 *)workspace_dev;
  double2 *r = base, *w = base + g.n, *Vb = base + 2 * g.n;  // Vb: m + 1 basis vectors
  g.dbuf = (double *)(Vb + (size_t)(m + 1) * g.n);
  static thread_local double *hb = nullptr;
  if (!hb) MGT_CUDA(cudaMallocHost((void **)&hb, 4 * sizeof(double)));
  g.hbuf = hb;
  const int64_t nb = g.n * sizeof(double2);
  auto apply = [&](const double2 *in, double2 *out) { return wilson_apply_native(h, in, out, 1, flags, tau, g.st); };
  auto resid = [&]() -> int {  // r = b - A x
    int rc = apply(x, w);
    if (rc) return rc;
    sub_kernel<<<grid_for(g.n, 256, 8), 256, 0, g.st>>>(g.n, b, w, r);
    MGT_LAUNCH_CHECK("sub_kernel");
    return MGT_OK;
  };
  using cd = std::complex<double>;
  int rc;
  int64_t matvecs = 0;
  double bn;
  if ((rc = g.norm(b, bn))) return rc;
  MGT_CUDA(cudaMemsetAsync(x, 0, nb, g.st));
  if (bn == 0.0) {
    report_out[0] = 0, report_out[1] = 0, report_out[2] = 1, report_out[3] = 0;
    relres_out[0] = 0.0;
    return MGT_OK;
  }
  MGT_CUDA(cudaMemcpyAsync(r, b, nb, cudaMemcpyDeviceToDevice, g.st));
  double beta = bn, rel = 1.0;
  int it = 0, reason = 1;  // 1 max_iter, 2 breakdown
  std::vector<cd> H((size_t)(m + 1) * m), gv(m + 1), cs(m), sn(m), y(m);
  auto Hij = [&](int i, int j) -> cd & { return H[(size_t)j * (m + 1) + i]; };
  bool broke = false;
  while (it < max_iter && !broke) {
    // v_0 = r / beta
    MGT_CUDA(cudaMemcpyAsync(Vb, r, nb, cudaMemcpyDeviceToDevice, g.st));
    scale2_kernel<<<grid_for(g.n, 256, 8), 256, 0, g.st>>>(g.n, 1.0 / beta, Vb, r);  // (r scaled too; rebuilt below)
    MGT_LAUNCH_CHECK("scale2_kernel");
    std::fill(gv.begin(), gv.end(), cd(0.0));
    gv[0] = cd(beta);
    int k = 0;
    for (int j = 0; j < m && it < max_iter; ++j) {
      double2 *vj = Vb + (size_t)j * g.n;
      if ((rc = apply(vj, w))) return rc;
      ++matvecs;
      double w0;
      if ((rc = g.norm(w, w0))) return rc;
      for (int i = 0; i <= j; ++i) {  // modified Gram-Schmidt
        C<double> hij;
        const double2 *vi = Vb + (size_t)i * g.n;
        if ((rc = g.dot(vi, w, hij))) return rc;
        Hij(i, j) = cd(hij.re, hij.im);
        if ((rc = g.axpy2(C<double>(-hij.re, -hij.im), vi, w))) return rc;
      }
      double hn;
      if ((rc = g.norm(w, hn))) return rc;
      Hij(j + 1, j) = cd(hn);
      for (int i = 0; i < j; ++i) {  // previous rotations
        const cd a = Hij(i, j), c2 = Hij(i + 1, j);
        Hij(i, j) = std::conj(cs[i]) * a + std::conj(sn[i]) * c2;
        Hij(i + 1, j) = -sn[i] * a + cs[i] * c2;
      }
      const cd a = Hij(j, j), c2 = Hij(j + 1, j);
      const double den = std::sqrt(std::norm(a) + std::norm(c2));
      if (den == 0.0) {
        cs[j] = cd(1.0), sn[j] = cd(0.0);
      } else {
        cs[j] = a / den;
        sn[j] = c2 / den;
      }
      Hij(j, j) = std::conj(cs[j]) * a + std::conj(sn[j]) * c2;
      Hij(j + 1, j) = cd(0.0);
      gv[j + 1] = -sn[j] * gv[j];
      gv[j] = std::conj(cs[j]) * gv[j];
      ++it;
      k = j + 1;
      rel = std::abs(gv[j + 1]) / bn;
      if (hn <= 1e-14 * std::max(w0, 1e-300)) {  // invariant subspace / breakdown
        broke = rel > tol;
        break;
      }
      if (rel <= tol) break;
      if (j + 1 < m) {
        double2 *vn = Vb + (size_t)(j + 1) * g.n;
        MGT_CUDA(cudaMemcpyAsync(vn, w, nb, cudaMemcpyDeviceToDevice, g.st));
        scale2_kernel<<<grid_for(g.n, 256, 8), 256, 0, g.st>>>(g.n, 1.0 / hn, vn, w);
        MGT_LAUNCH_CHECK("scale2_kernel");
      }
    }
    // y = R^-1 g ; x += V y
    for (int i = k - 1; i >= 0; --i) {
      cd t = gv[i];
      for (int l = i + 1; l < k; ++l) t -= Hij(i, l) * y[l];
      y[i] = Hij(i, i) == cd(0.0) ? cd(0.0) : t / Hij(i, i);
    }
    for (int i = 0; i < k; ++i)
      if ((rc = g.axpy2(C<double>(y[i].real(), y[i].imag()), Vb + (size_t)i * g.n, x))) return rc;
    if ((rc = resid())) return rc;
    ++matvecs;
    double rn;
    if ((rc = g.norm(r, rn))) return rc;
    rel = rn / bn;
    beta = rn;
    if (rel <= tol) {
      report_out[0] = it, report_out[1] = matvecs, report_out[2] = 1, report_out[3] = 0;
      relres_out[0] = rel;
      return MGT_OK;
    }
    if (broke) reason = 2;
  }
  report_out[0] = it, report_out[1] = matvecs, report_out[2] = 0, report_out[3] = reason;
  relres_out[0] = rel;
  return MGT_OK;
}

}  // extern "C"
