// Multigrid prolongator P (block-orthonormal, chirality split) and its
// adjoint on the GPU (reference: multigrid.py:116-225, Prolongator.restrict /
// prolong :153-157).
//
// Storage ("native P"): aggregate b in native coarse order (t slowest),
// chirality c (0: gamma5 = +1 -> spins 0,1; 1: spins 2,3), vector k < nv,
// entry j < bs = 6*S of the (b, c) support:
//     P[((b*2 + c)*nv + k)*bs + j],   j = q*S + s,
// q = (spin - 2c)*3 + colour, s = local site in the aggregate (x2 fastest,
// t slowest).  The reference orders the support rows by global fine index;
// the MGS result does not depend on the row order (only the reduction
// order of the dots, i.e. rounding).  Coarse vectors: (b, 2*nv) complex,
// column c*nv + k (multigrid.py:189-216).
#include <vector>

#include "reduce.cuh"

namespace mgt {

struct Agg {
  Geom g;
  int B[4];       // block extents (reference dims order)
  int Cd[4];      // coarse extents
  int S;          // sites per aggregate
  int bs;         // 6*S entries per (b, c)
  int nv;
  int64_t nb;     // number of aggregates
};

static int make_agg(const int dims[4], const int block[4], int nv, Agg &a) {
  a.g = make_geom(dims);
  a.S = 1;
  a.nb = 1;
  for (int i = 0; i < 4; ++i) {
    if (block[i] < 1 || dims[i] % block[i] != 0)
      return fail(MGT_ERR_BLOCKING, "block extent does not divide lattice extent");
    a.B[i] = block[i];
    a.Cd[i] = dims[i] / block[i];
    a.S *= block[i];
    a.nb *= a.Cd[i];
  }
  if (nv < 1 || nv > 64) return fail(MGT_ERR_INVALID, "nv must be in [1, 64]");
  a.bs = 6 * a.S;
  a.nv = nv;
  return MGT_OK;
}

// (b, s) -> native fine site
__device__ __forceinline__ int64_t agg_site(const Agg &a, int64_t b, int s) {
  int c[4], l[4];
  int64_t r = b;
  c[2] = (int)(r % a.Cd[2]);
  r /= a.Cd[2];
  c[1] = (int)(r % a.Cd[1]);
  r /= a.Cd[1];
  c[0] = (int)(r % a.Cd[0]);
  c[3] = (int)(r / a.Cd[0]);
  int q = s;
  l[2] = q % a.B[2];
  q /= a.B[2];
  l[1] = q % a.B[1];
  q /= a.B[1];
  l[0] = q % a.B[0];
  l[3] = q / a.B[0];
  int x[4];
  for (int i = 0; i < 4; ++i) x[i] = c[i] * a.B[i] + l[i];
  return native_site(a.g, x);
}

// gather nv native null-vector fields into the (unorthogonalised) P layout
__global__ void prolong_gather_kernel(Agg a, const double2 *__restrict__ nulls, double2 *__restrict__ P) {
  const int64_t n = a.nb * 2 * a.nv * (int64_t)a.bs;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n; idx += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(idx % a.bs);
    int64_t r = idx / a.bs;
    const int k = (int)(r % a.nv);
    r /= a.nv;
    const int c = (int)(r % 2);
    const int64_t b = r / 2;
    const int q = j / a.S, s = j % a.S;
    const int comp = (2 * c + q / 3) * 3 + q % 3;
    const int64_t site = agg_site(a, b, s);
    P[idx] = nulls[((int64_t)k * 12 + comp) * a.g.V + site];
  }
}

// block-wide sum of (re, im) with a fixed tree; all threads get the result
__device__ __forceinline__ C<double> block_sum(C<double> v, double *sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    v.re += __shfl_xor_sync(0xffffffffu, v.re, off);
    v.im += __shfl_xor_sync(0xffffffffu, v.im, off);
  }
  __syncthreads();
  if (lane == 0) {
    sm[2 * warp] = v.re;
    sm[2 * warp + 1] = v.im;
  }
  __syncthreads();
  C<double> t(0.0, 0.0);
  for (int w = 0; w < nw; ++w) {
    t.re += sm[2 * w];
    t.im += sm[2 * w + 1];
  }
  return t;
}

// Per-(b, c) modified Gram-Schmidt, two passes, drop < 1e-8 (multigrid.py:195-205).
// keep[(b*2+c)*nv + k] = 1 if column k survives.
__global__ void __launch_bounds__(256) prolong_mgs_kernel(Agg a, double2 *__restrict__ P, int *__restrict__ keep) {
  __shared__ double sm[64];
  const int64_t grp = blockIdx.x;  // b*2 + c
  double2 *G = P + grp * a.nv * (int64_t)a.bs;
  int *kp = keep + grp * a.nv;
  for (int i = 0; i < a.nv; ++i) {
    double2 *v = G + (int64_t)i * a.bs;
    for (int pass = 0; pass < 2; ++pass) {
      for (int u = 0; u < i; ++u) {
        if (!kp[u]) continue;
        const double2 *w = G + (int64_t)u * a.bs;
        C<double> d(0.0, 0.0);
        for (int j = threadIdx.x; j < a.bs; j += blockDim.x) d = cfma_conj(ldc(w + j), C<double>(v[j].x, v[j].y), d);
        d = block_sum(d, sm);
        for (int j = threadIdx.x; j < a.bs; j += blockDim.x) {
          C<double> x = C<double>(v[j].x, v[j].y) - d * ldc(w + j);
          v[j] = make_double2(x.re, x.im);
        }
        __syncthreads();
      }
    }
    double s2 = 0.0;
    for (int j = threadIdx.x; j < a.bs; j += blockDim.x) s2 += v[j].x * v[j].x + v[j].y * v[j].y;
    const double nrm = sqrt(block_sum(C<double>(s2, 0.0), sm).re);
    const bool ok = nrm >= 1e-8;
    if (threadIdx.x == 0) kp[i] = ok ? 1 : 0;
    const double inv = ok ? 1.0 / nrm : 0.0;
    for (int j = threadIdx.x; j < a.bs; j += blockDim.x) v[j] = make_double2(v[j].x * inv, v[j].y * inv);
    __syncthreads();
  }
}

// x (native fine) = P xc ; one CTA per (b, c, rhs)
__global__ void __launch_bounds__(256) prolong_kernel(Agg a, int n_rhs, const double2 *__restrict__ P,
                                                     const double2 *__restrict__ xc, double2 *__restrict__ x) {
  // rhs fastest in the grid: the CTAs that read one P block run together (L2 reuse)
  __shared__ double2 sx[64];
  const int64_t grp = blockIdx.x / n_rhs;
  const int rhs = (int)(blockIdx.x - grp * n_rhs);
  const int64_t b = grp >> 1;
  const int c = (int)(grp & 1);
  const int nc = 2 * a.nv;
  const double2 *xcr = xc + (int64_t)rhs * a.nb * nc;
  double2 *xr = x + (int64_t)rhs * 12 * a.g.V;
  if (threadIdx.x < a.nv) sx[threadIdx.x] = xcr[b * nc + c * a.nv + threadIdx.x];
  __syncthreads();
  const double2 *G = P + grp * a.nv * (int64_t)a.bs;
  for (int j = threadIdx.x; j < a.bs; j += blockDim.x) {
    C<double> acc(0.0, 0.0);
    for (int k = 0; k < a.nv; ++k) acc = cfma(ldc(G + (int64_t)k * a.bs + j), C<double>(sx[k].x, sx[k].y), acc);
    const int q = j / a.S, s = j % a.S;
    const int comp = (2 * c + q / 3) * 3 + q % 3;
    xr[(int64_t)comp * a.g.V + agg_site(a, b, s)] = make_double2(acc.re, acc.im);
  }
}

// xc = P^H (g5? x) for NR rhs at once; one CTA per (b, c).  The CTA stages
// the x block of its aggregate/chirality (all NR rhs, tiles of JT entries)
// in shared memory; warp w owns columns k = w, w+8, .., so every P entry is
// read from HBM once for all rhs and every staged x entry feeds CPW columns.
// The gather offsets of the support entries (comp * V + site offset inside
// the aggregate, the same for every aggregate since the native index is
// linear in the coordinates) are tabulated once per CTA in shared memory,
// so the staging loop does no index arithmetic.
// Fixed reduction order: per-lane partial sums, then a shuffle-xor tree.
constexpr int kRestrictJT = 1024;

// native offset of local site s inside an aggregate, relative to its origin
__device__ __forceinline__ int64_t agg_local_offset(const Agg &a, int s) {
  const int l2 = s % a.B[2];
  int q = s / a.B[2];
  const int l1 = q % a.B[1];
  q /= a.B[1];
  const int l0 = q % a.B[0];
  const int l3 = q / a.B[0];
  return (int64_t)l3 * a.g.stride[3] + (int64_t)l0 * a.g.stride[0] + (int64_t)l1 * a.g.stride[1] + l2;
}

template <int CPW, int NR>
__global__ void __launch_bounds__(256) restrict_mrhs_kernel(Agg a, const double2 *__restrict__ P,
                                                           const double2 *__restrict__ x,
                                                           double2 *__restrict__ xc, int gamma5_in) {
  extern __shared__ double2 sx[];  // [NR][kRestrictJT], then the bs gather offsets
  int64_t *joff = reinterpret_cast<int64_t *>(sx + NR * kRestrictJT);
  const int64_t grp = blockIdx.x;
  const int64_t b = grp >> 1;
  const int c = (int)(grp & 1);
  const int nc = 2 * a.nv;
  const double sign = (gamma5_in && c == 1) ? -1.0 : 1.0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double2 *G = P + grp * a.nv * (int64_t)a.bs;
  const double2 *xb = x + agg_site(a, b, 0);
  for (int j = threadIdx.x; j < a.bs; j += blockDim.x) {
    const int q = j / a.S, s = j - (j / a.S) * a.S;
    const int comp = (2 * c + q / 3) * 3 + q % 3;
    joff[j] = (int64_t)comp * a.g.V + agg_local_offset(a, s);
  }
  C<double> acc[CPW][NR];
#pragma unroll
  for (int i = 0; i < CPW; ++i)
#pragma unroll
    for (int r = 0; r < NR; ++r) acc[i][r] = C<double>(0.0, 0.0);
  for (int j0 = 0; j0 < a.bs; j0 += kRestrictJT) {
    const int jn = min(kRestrictJT, a.bs - j0);
    __syncthreads();
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const double2 *xr = xb + (int64_t)r * 12 * a.g.V;
#pragma unroll 4
      for (int jj = threadIdx.x; jj < jn; jj += blockDim.x) {
        const double2 v = xr[joff[j0 + jj]];
        sx[r * kRestrictJT + jj] = make_double2(sign * v.x, sign * v.y);
      }
    }
    __syncthreads();
#pragma unroll 4
    for (int jj = lane; jj < jn; jj += 32) {
      C<double> xv[NR];
#pragma unroll
      for (int r = 0; r < NR; ++r) xv[r] = C<double>(sx[r * kRestrictJT + jj].x, sx[r * kRestrictJT + jj].y);
#pragma unroll
      for (int i = 0; i < CPW; ++i) {
        const int k = warp + 8 * i;
        if (k < a.nv) {
          const C<double> pk = ldc(G + (int64_t)k * a.bs + j0 + jj);
#pragma unroll
          for (int r = 0; r < NR; ++r) acc[i][r] = cfma_conj(pk, xv[r], acc[i][r]);
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < CPW; ++i) {
    const int k = warp + 8 * i;
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      C<double> v = acc[i][r];
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) {
        v.re += __shfl_xor_sync(0xffffffffu, v.re, off);
        v.im += __shfl_xor_sync(0xffffffffu, v.im, off);
      }
      if (lane == 0 && k < a.nv) xc[(int64_t)r * a.nb * nc + b * nc + c * a.nv + k] = make_double2(v.re, v.im);
    }
  }
}

template <int CPW, int NR>
static int launch_restrict_mrhs(const Agg &a, const double2 *P, const double2 *x, double2 *xc, int g5,
                                cudaStream_t st) {
  const size_t smem = (size_t)NR * kRestrictJT * sizeof(double2) + (size_t)a.bs * sizeof(int64_t);
  if (smem > 200 * 1024) return fail(MGT_ERR_INVALID, "mgt_restrict: aggregate too large");
  static bool attr = false;
  if (!attr) {
    MGT_CUDA(cudaFuncSetAttribute(restrict_mrhs_kernel<CPW, NR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  200 * 1024));
    attr = true;
  }
  restrict_mrhs_kernel<CPW, NR><<<(unsigned)(a.nb * 2), 256, smem, st>>>(a, P, x, xc, g5);
  MGT_LAUNCH_CHECK("restrict_mrhs_kernel");
  return MGT_OK;
}

template <int CPW>
static int restrict_groups(const Agg &a, const double2 *P, const double2 *x, double2 *xc, int n_rhs, int g5,
                           cudaStream_t st) {
  const int64_t fstride = (int64_t)12 * a.g.V, cstride = a.nb * 2 * a.nv;
  int r = 0;
  while (r < n_rhs) {
    const int left = n_rhs - r;
    int rc;
    if (left >= 4) {
      rc = launch_restrict_mrhs<CPW, 4>(a, P, x + r * fstride, xc + r * cstride, g5, st);
      r += 4;
    } else if (left >= 2) {
      rc = launch_restrict_mrhs<CPW, 2>(a, P, x + r * fstride, xc + r * cstride, g5, st);
      r += 2;
    } else {
      rc = launch_restrict_mrhs<CPW, 1>(a, P, x + r * fstride, xc + r * cstride, g5, st);
      r += 1;
    }
    if (rc) return rc;
  }
  return MGT_OK;
}

// coarse vectors: reference order (b_ref lexicographic, last coarse dim
// fastest) <-> native order (t slowest)
__global__ void coarse_perm_kernel(Agg a, int nc, int n_rhs, const double2 *__restrict__ in,
                                   double2 *__restrict__ out, int to_ref) {
  const int64_t n = a.nb * nc * (int64_t)n_rhs;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n; idx += (int64_t)gridDim.x * blockDim.x) {
    const int col = (int)(idx % nc);
    int64_t r = idx / nc;
    const int64_t bn = r % a.nb;
    const int64_t rhs = r / a.nb;
    int64_t q = bn;
    int c[4];
    c[2] = (int)(q % a.Cd[2]);
    q /= a.Cd[2];
    c[1] = (int)(q % a.Cd[1]);
    q /= a.Cd[1];
    c[0] = (int)(q % a.Cd[0]);
    c[3] = (int)(q / a.Cd[0]);
    const int64_t br = (((int64_t)c[0] * a.Cd[1] + c[1]) * a.Cd[2] + c[2]) * a.Cd[3] + c[3];
    const int64_t nat = (rhs * a.nb + bn) * nc + col;
    const int64_t ref = (rhs * a.nb + br) * nc + col;
    if (to_ref)
      out[ref] = in[nat];
    else
      out[nat] = in[ref];
  }
}

}  // namespace mgt

using namespace mgt;

extern "C" {

int mgt_prolong_build(const int dims[4], const int block[4], int nv, const void *null_native_dev, void *P_dev,
                      int *keep_host, void *stream) {
  if (!dims || !block || !null_native_dev || !P_dev) return fail(MGT_ERR_INVALID, "mgt_prolong_build: null argument");
  Agg a;
  int rc = make_agg(dims, block, nv, a);
  if (rc) return rc;
  cudaStream_t st = as_stream(stream);
  const int64_t n = a.nb * 2 * a.nv * (int64_t)a.bs;
  prolong_gather_kernel<<<grid_for(n, 256, 8), 256, 0, st>>>(a, (const double2 *)null_native_dev, (double2 *)P_dev);
  MGT_LAUNCH_CHECK("prolong_gather_kernel");
  int *keep = nullptr;
  const size_t kb = (size_t)a.nb * 2 * nv * sizeof(int);
  MGT_CUDA(scratch_alloc((void **)&keep, kb, st));
  prolong_mgs_kernel<<<(unsigned)(a.nb * 2), 256, 0, st>>>(a, (double2 *)P_dev, keep);
  MGT_LAUNCH_CHECK("prolong_mgs_kernel");
  if (keep_host) MGT_CUDA(cudaMemcpyAsync(keep_host, keep, kb, cudaMemcpyDeviceToHost, st));
  MGT_CUDA(cudaFreeAsync(keep, st));
  MGT_CUDA(cudaStreamSynchronize(st));
  return MGT_OK;
}

int mgt_prolong(const int dims[4], const int block[4], int nv, const void *P_dev, const void *xc_dev,
                void *x_native_dev, int n_rhs, void *stream) {
  if (!dims || !block || !P_dev || !xc_dev || !x_native_dev || n_rhs < 1)
    return fail(MGT_ERR_INVALID, "mgt_prolong: bad argument");
  Agg a;
  int rc = make_agg(dims, block, nv, a);
  if (rc) return rc;
  prolong_kernel<<<(unsigned)(a.nb * 2 * n_rhs), 256, 0, as_stream(stream)>>>(
      a, n_rhs, (const double2 *)P_dev, (const double2 *)xc_dev, (double2 *)x_native_dev);
  MGT_LAUNCH_CHECK("prolong_kernel");
  return MGT_OK;
}

int mgt_restrict(const int dims[4], const int block[4], int nv, const void *P_dev, const void *x_native_dev,
                 void *xc_dev, int n_rhs, int gamma5_in, void *stream) {
  if (!dims || !block || !P_dev || !xc_dev || !x_native_dev || n_rhs < 1)
    return fail(MGT_ERR_INVALID, "mgt_restrict: bad argument");
  Agg a;
  int rc = make_agg(dims, block, nv, a);
  if (rc) return rc;
  cudaStream_t st = as_stream(stream);
  const double2 *Pp = (const double2 *)P_dev, *xp = (const double2 *)x_native_dev;
  double2 *cp = (double2 *)xc_dev;
  if (nv <= 8) return restrict_groups<1>(a, Pp, xp, cp, n_rhs, gamma5_in, st);
  if (nv <= 24) return restrict_groups<3>(a, Pp, xp, cp, n_rhs, gamma5_in, st);
  if (nv <= 32) return restrict_groups<4>(a, Pp, xp, cp, n_rhs, gamma5_in, st);
  return restrict_groups<8>(a, Pp, xp, cp, n_rhs, gamma5_in, st);
}

int mgt_coarse_perm(const int dims[4], const int block[4], int nc, int n_rhs, const void *in_dev, void *out_dev,
                    int to_ref, void *stream) {
  if (!dims || !block || !in_dev || !out_dev || nc < 1 || n_rhs < 1)
    return fail(MGT_ERR_INVALID, "mgt_coarse_perm: bad argument");
  Agg a;
  int rc = make_agg(dims, block, 1, a);
  if (rc) return rc;
  const int64_t n = a.nb * nc * (int64_t)n_rhs;
  coarse_perm_kernel<<<grid_for(n, 256, 8), 256, 0, as_stream(stream)>>>(a, nc, n_rhs, (const double2 *)in_dev,
                                                                          (double2 *)out_dev, to_ref);
  MGT_LAUNCH_CHECK("coarse_perm_kernel");
  return MGT_OK;
}

}  // extern "C"
