// Galerkin coarse operator C = P^H A P and the coarse block-stencil matvec
// (reference: build_coarse_operator multigrid.py:246-259 via a scipy SpGEMM,
// CoarseOperator :228-243).
//
// C couples each aggregate to itself and its 8 neighbours.  It is built
// column by column without any sparse-sparse product: for coarse column
// (c', k') the fine field v = P e_(c',k') (the unit vector placed in every
// aggregate at once) is pushed through a "split" Wilson apply that routes
// the diagonal term and every hop that stays inside its aggregate into
// output 0 and each hop that crosses into the neighbouring aggregate in
// direction (mu, +/-) into output 1 + 2 mu + (0: +, 1: -).  Restricting the 9
// outputs with P^H gives column (c', k') of the 9 coarse blocks of every
// aggregate simultaneously: 2 nv split-applies + 18 nv restrictions in all.
//
// Storage: C[((b*9 + dir)*nc + col)*nc + row] (column-major 2nv x 2nv
// blocks, nc = 2 nv), b in native coarse order; block dir couples b to
// nbr(b, dir) (dir 0: b itself).  The antiperiodic phase lives in the hops.
#include <algorithm>

#include "handle.cuh"
#include "reduce.cuh"

namespace mgt {

struct CoarseGeom {
  int Cd[4];
  int B[4];
  int64_t nb;
  int nc;
};

__device__ __forceinline__ int64_t coarse_nbr(const CoarseGeom &cg, int64_t b, int dir) {
  if (dir == 0) return b;
  const int mu = (dir - 1) >> 1;
  const int sgn = ((dir - 1) & 1) ? -1 : 1;
  int c[4];
  int64_t r = b;
  c[2] = (int)(r % cg.Cd[2]);
  r /= cg.Cd[2];
  c[1] = (int)(r % cg.Cd[1]);
  r /= cg.Cd[1];
  c[0] = (int)(r % cg.Cd[0]);
  c[3] = (int)(r / cg.Cd[0]);
  c[mu] = (c[mu] + sgn + cg.Cd[mu]) % cg.Cd[mu];
  return (((int64_t)c[3] * cg.Cd[0] + c[0]) * cg.Cd[1] + c[1]) * cg.Cd[2] + c[2];
}

// 9-way split apply (fp64).  out: 9 native fields back to back.
template <int RECON>
__global__ void __launch_bounds__(128, 3) wilson_split_kernel(WilsonParams P, CoarseGeom cg, const double2 *__restrict__ in,
                                                              double2 *__restrict__ out, LinkField<double, RECON> links) {
  const int64_t V = P.g.V;
  for (int64_t site = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; site < V;
       site += (int64_t)gridDim.x * blockDim.x) {
    int x[4];
    native_coords(P.g, site, x);
    const bool ap = P.antiperiodic != 0;
    C<double> self[4][3];
    // diagonal term
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        C<double> v = ldc(in + (a * 3 + c) * V + site);
        self[a][c] = (a < 2 ? C<double>(P.diag_up_re, P.diag_up_im) : C<double>(P.diag_dn_re, P.diag_dn_im)) * v;
      }
    auto route = [&](int dir, bool cross, C<double>(&h)[4][3]) {
      double2 *o = out + (int64_t)dir * 12 * V + site;
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          C<double> v = -0.5 * h[a][c];
          if (cross) {
            stc(o + (a * 3 + c) * V, v);
          } else {
            self[a][c] = self[a][c] + v;
            stc(o + (a * 3 + c) * V, C<double>(0.0, 0.0));
          }
        }
    };
#define MGT_SPLIT_HOP(MU)                                                                            \
  {                                                                                                  \
    C<double> h[4][3];                                                                               \
    for (int a = 0; a < 4; ++a)                                                                      \
      for (int c = 0; c < 3; ++c) h[a][c] = C<double>(0.0, 0.0);                                     \
    wilson_hop<MU, true>(P.g, in, links, site, x, 1.0, ap, h);                                       \
    route(1 + 2 * MU, (x[MU] % cg.B[MU]) == cg.B[MU] - 1, h);                                        \
    for (int a = 0; a < 4; ++a)                                                                      \
      for (int c = 0; c < 3; ++c) h[a][c] = C<double>(0.0, 0.0);                                     \
    wilson_hop<MU, false>(P.g, in, links, site, x, 1.0, ap, h);                                      \
    route(2 + 2 * MU, (x[MU] % cg.B[MU]) == 0, h);                                                   \
  }
    MGT_SPLIT_HOP(0)
    MGT_SPLIT_HOP(1)
    MGT_SPLIT_HOP(2)
    MGT_SPLIT_HOP(3)
#undef MGT_SPLIT_HOP
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int c = 0; c < 3; ++c) stc(out + (a * 3 + c) * V + site, self[a][c]);
  }
}

__global__ void unit_coarse_kernel(int64_t nb, int nc, int col, double2 *__restrict__ xc) {
  const int64_t n = nb * nc;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    xc[i] = make_double2((i % nc) == col ? 1.0 : 0.0, 0.0);
}

// xc9[dir][b][row] -> C[b][dir][col][row]
__global__ void scatter_column_kernel(int64_t nb, int nc, int col, const double2 *__restrict__ xc9,
                                      double2 *__restrict__ C) {
  const int64_t n = 9 * nb * nc;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int row = (int)(i % nc);
    const int64_t r = i / nc;
    const int64_t b = r % nb;
    const int dir = (int)(r / nb);
    C[((b * 9 + dir) * nc + col) * (int64_t)nc + row] = xc9[i];
  }
}

// y[b] = sum_dir C[b][dir] x[nbr(b, dir)] for NR rhs at once; CTA per b.
// Thread (row, group g) accumulates the dirs g, g+G, .. of its row for every
// rhs, so each C entry is read once for all rhs (coalesced: a column of a
// block is contiguous in rows); the neighbour vectors are staged in shared
// memory and read as broadcasts.  The G group partials are summed in group
// order (fixed, deterministic).
// CT: double2 (the Galerkin operator) or float2 (its fp32 copy for loose
// inner solves: half the bytes, fp64 vectors and accumulation)
template <int NR, typename CT = double2>
__global__ void __launch_bounds__(256) coarse_apply_kernel(CoarseGeom cg, int G, const CT *__restrict__ Cm,
                                                           const double2 *__restrict__ x, double2 *__restrict__ y) {
  extern __shared__ double2 sm[];
  const int nc = cg.nc;
  double2 *sx = sm;                    // [9][nc][NR]
  double2 *part = sm + 9 * nc * NR;    // [G][NR][nc]
  const int64_t b = blockIdx.x;
  for (int i = threadIdx.x; i < 9 * nc * NR; i += blockDim.x) {
    const int r = i % NR, q = i / NR;
    const int dir = q / nc, col = q % nc;
    sx[i] = x[((int64_t)r * cg.nb + coarse_nbr(cg, b, dir)) * nc + col];
  }
  __syncthreads();
  const int row = threadIdx.x % nc, grp = threadIdx.x / nc;
  if (grp < G) {
    C<double> acc[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) acc[r] = C<double>(0.0, 0.0);
    for (int dir = grp; dir < 9; dir += G) {
      const CT *Cb = Cm + (b * 9 + dir) * (int64_t)nc * nc + row;
      const double2 *xs = sx + dir * nc * NR;
#pragma unroll 4
      for (int col = 0; col < nc; ++col) {
        const auto cl = ldc(Cb + (int64_t)col * nc);
        const C<double> cv((double)cl.re, (double)cl.im);
#pragma unroll
        for (int r = 0; r < NR; ++r) acc[r] = cfma(cv, C<double>(xs[col * NR + r].x, xs[col * NR + r].y), acc[r]);
      }
    }
#pragma unroll
    for (int r = 0; r < NR; ++r) part[(grp * NR + r) * nc + row] = make_double2(acc[r].re, acc[r].im);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < NR * nc; i += blockDim.x) {
    const int r = i / nc, rw = i % nc;
    C<double> t(0.0, 0.0);
    for (int g = 0; g < G; ++g) {
      const double2 v = part[(g * NR + r) * nc + rw];
      t = t + C<double>(v.x, v.y);
    }
    y[((int64_t)r * cg.nb + b) * nc + rw] = make_double2(t.re, t.im);
  }
}

template <int NR, typename CT = double2>
static int launch_coarse_apply(const CoarseGeom &cg, const CT *C, const double2 *x, double2 *y,
                               cudaStream_t st) {
  const int G = std::max(1, std::min(9, 256 / cg.nc));
  const int block = ((G * cg.nc + 31) / 32) * 32;
  const size_t smem = (size_t)(9 * cg.nc * NR + G * NR * cg.nc) * sizeof(double2);
  if (smem > 48 * 1024) {
    static size_t set = 0;
    if (smem > set) {
      MGT_CUDA(cudaFuncSetAttribute(coarse_apply_kernel<NR, CT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem));
      set = smem;
    }
  }
  coarse_apply_kernel<NR, CT><<<(unsigned)cg.nb, block, smem, st>>>(cg, G, C, x, y);
  MGT_LAUNCH_CHECK("coarse_apply_kernel");
  return MGT_OK;
}

static int make_cg(const int dims[4], const int block[4], int nv, CoarseGeom &cg) {
  cg.nb = 1;
  for (int i = 0; i < 4; ++i) {
    if (block[i] < 1 || dims[i] % block[i]) return fail(MGT_ERR_BLOCKING, "block extent does not divide lattice extent");
    cg.B[i] = block[i];
    cg.Cd[i] = dims[i] / block[i];
    cg.nb *= cg.Cd[i];
  }
  cg.nc = 2 * nv;
  return MGT_OK;
}

}  // namespace mgt

using namespace mgt;

extern "C" {

int mgt_coarse_build(mgt_wilson_t h, const int block[4], int nv, const void *P_dev, void *C_dev, void *stream) {
  if (!h || !block || !P_dev || !C_dev) return fail(MGT_ERR_INVALID, "mgt_coarse_build: null argument");
  if (h->prec != 64) return fail(MGT_ERR_INVALID, "mgt_coarse_build: needs a complex128 operator");
  CoarseGeom cg;
  int rc = make_cg(h->g.L, block, nv, cg);
  if (rc) return rc;
  cudaStream_t st = as_stream(stream);
  const int64_t V = h->g.V;
  const int nc = cg.nc;
  double2 *v = nullptr, *split = nullptr, *xc = nullptr, *xc9 = nullptr;
  MGT_CUDA(scratch_alloc((void **)&v, (size_t)12 * V * sizeof(double2), st));
  MGT_CUDA(scratch_alloc((void **)&split, (size_t)9 * 12 * V * sizeof(double2), st));
  MGT_CUDA(scratch_alloc((void **)&xc, (size_t)cg.nb * nc * sizeof(double2), st));
  MGT_CUDA(scratch_alloc((void **)&xc9, (size_t)9 * cg.nb * nc * sizeof(double2), st));
  WilsonParams P = make_params(h, 0, 0.0);
  const int grid = grid_for(V, 128, 3);
  for (int col = 0; col < nc && rc == MGT_OK; ++col) {
    unit_coarse_kernel<<<grid_for(cg.nb * nc, 256, 4), 256, 0, st>>>(cg.nb, nc, col, xc);
    note_launch();
    rc = mgt_prolong(h->g.L, block, nv, P_dev, xc, v, 1, stream);
    if (rc) break;
    if (h->recon == 18)
      wilson_split_kernel<18><<<grid, 128, 0, st>>>(P, cg, v, split,
                                                    LinkField<double, 18>{(const double2 *)h->links, V});
    else
      wilson_split_kernel<12><<<grid, 128, 0, st>>>(P, cg, v, split,
                                                    LinkField<double, 12>{(const double2 *)h->links, V});
    note_launch();
    rc = mgt_restrict(h->g.L, block, nv, P_dev, split, xc9, 9, 0, stream);
    if (rc) break;
    scatter_column_kernel<<<grid_for(9 * cg.nb * nc, 256, 4), 256, 0, st>>>(cg.nb, nc, col, xc9,
                                                                             (double2 *)C_dev);
    note_launch();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) rc = cuda_fail(e, "coarse build");
  }
  cudaFreeAsync(v, st);
  cudaFreeAsync(split, st);
  cudaFreeAsync(xc, st);
  cudaFreeAsync(xc9, st);
  return rc;
}

}  // extern "C"

namespace mgt {
template <typename CT>
static int coarse_apply_impl(const int dims[4], const int block[4], int nv, const void *C_dev, const void *xc_dev,
                             void *yc_dev, int n_rhs, void *stream) {
  if (!dims || !block || !C_dev || !xc_dev || !yc_dev || n_rhs < 1)
    return fail(MGT_ERR_INVALID, "mgt_coarse_apply: bad argument");
  if (xc_dev == yc_dev) return fail(MGT_ERR_INVALID, "mgt_coarse_apply: in-place apply is not supported");
  CoarseGeom cg;
  int rc = make_cg(dims, block, nv, cg);
  if (rc) return rc;
  cudaStream_t st = as_stream(stream);
  const CT *Cp = (const CT *)C_dev;
  const double2 *xp = (const double2 *)xc_dev;
  double2 *yp = (double2 *)yc_dev;
  const int64_t stride = cg.nb * cg.nc;
  int r = 0;
  while (r < n_rhs) {
    const int left = n_rhs - r;
    const int nr = left >= 4 ? 4 : (left >= 2 ? 2 : 1);
    rc = nr == 4 ? launch_coarse_apply<4, CT>(cg, Cp, xp + r * stride, yp + r * stride, st)
                 : (nr == 2 ? launch_coarse_apply<2, CT>(cg, Cp, xp + r * stride, yp + r * stride, st)
                            : launch_coarse_apply<1, CT>(cg, Cp, xp + r * stride, yp + r * stride, st));
    if (rc) return rc;
    r += nr;
  }
  return MGT_OK;
}
}  // namespace mgt

extern "C" {

int mgt_coarse_apply(const int dims[4], const int block[4], int nv, const void *C_dev, const void *xc_dev,
                     void *yc_dev, int n_rhs, void *stream) {
  return coarse_apply_impl<double2>(dims, block, nv, C_dev, xc_dev, yc_dev, n_rhs, stream);
}

int mgt_coarse_apply_c32(const int dims[4], const int block[4], int nv, const void *C32_dev, const void *xc_dev,
                         void *yc_dev, int n_rhs, void *stream) {
  return coarse_apply_impl<float2>(dims, block, nv, C32_dev, xc_dev, yc_dev, n_rhs, stream);
}

}  // extern "C"
