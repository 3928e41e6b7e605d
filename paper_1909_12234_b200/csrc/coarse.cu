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
#include <type_traits>

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
  // scalar coordinates (no local array: keeps the kernels off the stack)
  int64_t r = b;
  int c2 = (int)(r % cg.Cd[2]);
  r /= cg.Cd[2];
  int c1 = (int)(r % cg.Cd[1]);
  r /= cg.Cd[1];
  int c0 = (int)(r % cg.Cd[0]);
  int c3 = (int)(r / cg.Cd[0]);
  if (mu == 0)
    c0 = (c0 + sgn + cg.Cd[0]) % cg.Cd[0];
  else if (mu == 1)
    c1 = (c1 + sgn + cg.Cd[1]) % cg.Cd[1];
  else if (mu == 2)
    c2 = (c2 + sgn + cg.Cd[2]) % cg.Cd[2];
  else
    c3 = (c3 + sgn + cg.Cd[3]) % cg.Cd[3];
  return (((int64_t)c3 * cg.Cd[0] + c0) * cg.Cd[1] + c1) * cg.Cd[2] + c2;
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
  __shared__ int64_t nbr[9];
  if (threadIdx.x < 9) nbr[threadIdx.x] = coarse_nbr(cg, b, threadIdx.x);
  __syncthreads();
  for (int i = threadIdx.x; i < 9 * nc * NR; i += blockDim.x) {
    const int r = i % NR, q = i / NR;
    const int dir = q / nc, col = q % nc;
    sx[i] = x[((int64_t)r * cg.nb + nbr[dir]) * nc + col];
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

// The same product with one thread per (dir, row): 9 nc threads per
// aggregate, each streaming one block row-slice of C (48 columns, loads
// issued 8 at a time so ~8 x 16 B per thread are in flight) against the
// staged neighbour vectors; the 9 direction partials are then summed in
// direction order through shared memory (the staging buffer, reused).
// Every rhs sees the same arithmetic whatever NR is (bitwise-stable across
// batchings).  For nc <= 49 (9 nc <= 448 threads, two CTAs per SM).
constexpr int kCoarseDirThreads = 448;
template <int NR, typename CT = double2>
__global__ void __launch_bounds__(kCoarseDirThreads, 2)
    coarse_apply_dir_kernel(CoarseGeom cg, const CT *__restrict__ Cm, const double2 *__restrict__ x,
                            double2 *__restrict__ y) {
  extern __shared__ double2 sm[];  // [9][nc][NR], then [9][NR][nc]
  __shared__ int64_t nbr[9];
  const int nc = cg.nc;
  const int64_t b = blockIdx.x;
  // the 9 neighbour aggregates once per CTA (64-bit div/mod is not cheap)
  if (threadIdx.x < 9) nbr[threadIdx.x] = coarse_nbr(cg, b, threadIdx.x);
  __syncthreads();
  // arithmetic type: fp64 with the fp64 C; fp32 with its fp32 copy (loose
  // inner solves only: ~1e-7 relative per product, well inside tol >= 1e-5)
  using AT = std::conditional_t<sizeof(CT) == 8, float, double>;
  using A2 = std::conditional_t<sizeof(CT) == 8, float2, double2>;
  A2 *sx = reinterpret_cast<A2 *>(sm);
  for (int i = threadIdx.x; i < 9 * nc * NR; i += blockDim.x) {
    const int col = i % nc, q = i / nc;
    const int r = q % NR, dir = q / NR;
    const double2 xv = x[((int64_t)r * cg.nb + nbr[dir]) * nc + col];
    A2 a;
    a.x = (AT)xv.x;
    a.y = (AT)xv.y;
    sx[(dir * nc + col) * NR + r] = a;
  }
  __syncthreads();
  const int dir = threadIdx.x / nc, row = threadIdx.x - dir * nc;
  const bool on = dir < 9;
  C<AT> acc[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) acc[r] = C<AT>(AT(0), AT(0));
  if (on) {
    const CT *Cb = Cm + (b * 9 + dir) * (int64_t)nc * nc + row;
    const A2 *xs = sx + dir * nc * NR;
    // loads in flight per thread: 8 (4 for 8 fp64 rhs, register budget)
    constexpr int U = (sizeof(CT) == 16 && NR >= 2) ? 4 : 8;
    for (int c0 = 0; c0 < nc; c0 += U) {
      CT cl[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (c0 + u < nc) cl[u] = Cb[(int64_t)(c0 + u) * nc];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (c0 + u < nc) {
          const C<AT> cv(cl[u].x, cl[u].y);
#pragma unroll
          for (int r = 0; r < NR; ++r) {
            const A2 xv = xs[(c0 + u) * NR + r];
            acc[r] = cfma(cv, C<AT>(xv.x, xv.y), acc[r]);
          }
        }
      }
    }
  }
  __syncthreads();
  if (on) {
#pragma unroll
    for (int r = 0; r < NR; ++r) sm[(dir * NR + r) * nc + row] = make_double2((double)acc[r].re, (double)acc[r].im);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < NR * nc; i += blockDim.x) {
    const int r = i / nc, rw = i % nc;
    C<double> t(0.0, 0.0);
#pragma unroll
    for (int d = 0; d < 9; ++d) {
      const double2 v = sm[(d * NR + r) * nc + rw];
      t = t + C<double>(v.x, v.y);
    }
    y[((int64_t)r * cg.nb + b) * nc + rw] = make_double2(t.re, t.im);
  }
}

template <int NR, typename CT = double2>
static int launch_coarse_apply(const CoarseGeom &cg, const CT *C, const double2 *x, double2 *y,
                               cudaStream_t st) {
  if (9 * cg.nc <= kCoarseDirThreads) {
    const int block = ((9 * cg.nc + 31) / 32) * 32;
    const size_t smem = (size_t)9 * cg.nc * NR * sizeof(double2);
    if (smem > 40 * 1024) {  // (static shared memory counts toward the 48 KB default as well)
      static size_t set = 0;
      if (smem > set) {
        MGT_CUDA(cudaFuncSetAttribute(coarse_apply_dir_kernel<NR, CT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
        set = smem;
      }
    }
    coarse_apply_dir_kernel<NR, CT><<<(unsigned)cg.nb, block, smem, st>>>(cg, C, x, y);
    MGT_LAUNCH_CHECK("coarse_apply_dir_kernel");
    return MGT_OK;
  }
  const int G = std::max(1, std::min(9, 256 / cg.nc));
  const int block = ((G * cg.nc + 31) / 32) * 32;
  const size_t smem = (size_t)(9 * cg.nc * NR + G * NR * cg.nc) * sizeof(double2);
  if (smem > 40 * 1024) {  // (static shared memory counts toward the 48 KB default as well)
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
    // up to 8 rhs per launch where the per-(dir, row) kernel applies (its
    // staging buffer is 9 nc NR complex; the older group kernel stops at 4)
    const bool dirk = 9 * cg.nc <= kCoarseDirThreads;
    const int nr = (left >= 8 && dirk) ? 8 : (left >= 4 ? 4 : (left >= 2 ? 2 : 1));
    rc = nr == 8   ? launch_coarse_apply<8, CT>(cg, Cp, xp + r * stride, yp + r * stride, st)
         : nr == 4 ? launch_coarse_apply<4, CT>(cg, Cp, xp + r * stride, yp + r * stride, st)
         : nr == 2 ? launch_coarse_apply<2, CT>(cg, Cp, xp + r * stride, yp + r * stride, st)
                   : launch_coarse_apply<1, CT>(cg, Cp, xp + r * stride, yp + r * stride, st);
    if (rc) return rc;
    r += nr;
  }
  return MGT_OK;
}
}  // namespace mgt

namespace mgt {

// ---------------------------------------------------------------------------
// One BiCGStab iteration on the coarse operator (C + i tau g5_c) for n
// independent rhs, every vector op fused and every scalar kept on the
// device (multigrid.coarse_bicgstab drives the loop and the explicit-residual
// confirmations).  Per-rhs state row (doubles):
//   [rho re, im, alpha re, im, omega re, im, beta re, im, r2, active, tol2, conv]
//   [12] iterations taken, [13] freeze: a converged rhs deactivates itself
//   (multi-iteration calls), [14..15] reserved
// Reductions: per-block partials in a fixed grid, summed in block order by a
// one-warp finisher per rhs (deterministic).
enum { CK_RHO = 0, CK_ALPHA = 2, CK_OMEGA = 4, CK_BETA = 6, CK_R2 = 8, CK_ACT = 9, CK_TOL2 = 10, CK_CONV = 11,
       CK_ITS = 12, CK_FREEZE = 13, CK_W = 16 };
constexpr int kCkBlock = 256;

__device__ __forceinline__ C<double> cdiv(C<double> a, C<double> b) {
  const double d = b.re * b.re + b.im * b.im;
  return C<double>((a.re * b.re + a.im * b.im) / d, (a.im * b.re - a.re * b.im) / d);
}

// sum v[NV] over the block; thread 0 writes part[(rhs * nblk + blk) * NV ..]
template <int NV>
__device__ __forceinline__ void ck_publish(double (&v)[NV], double *part) {
  __shared__ double sm[kCkBlock / 32][NV];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double x = v[k];
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
    if (lane == 0) sm[warp][k] = x;
  }
  __syncthreads();
  if (threadIdx.x < NV) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < kCkBlock / 32; ++w) t += sm[w][threadIdx.x];
    part[((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * NV + threadIdx.x] = t;
  }
}

// g5_c of element e of a (nb, nc) field: -1 on the second nv columns
__device__ __forceinline__ double ck_g5(int64_t e, int nc, int nv) { return (int)(e % nc) >= nv ? -1.0 : 1.0; }

// KIND 1: v += i tau g5 p ; sigma = <rhat, v>
// KIND 3: t += i tau g5 s ; <t, t>, <t, s>
template <int KIND>
__global__ void __launch_bounds__(kCkBlock) ck_dots(int64_t L, int nc, int nv, double tau, double2 *__restrict__ a,
                                                    const double2 *__restrict__ b, const double2 *__restrict__ c,
                                                    double *part) {
  const int64_t off = (int64_t)blockIdx.y * L;
  double acc[3] = {0.0, 0.0, 0.0};
  for (int64_t e = blockIdx.x * (int64_t)kCkBlock + threadIdx.x; e < L; e += (int64_t)gridDim.x * kCkBlock) {
    C<double> y = ldc(a + off + e);
    const C<double> q = ldc(b + off + e);  // the applied vector (p or s)
    if (tau != 0.0) {
      const double g = tau * ck_g5(e, nc, nv);
      y = C<double>(y.re - g * q.im, y.im + g * q.re);
      stc(a + off + e, y);
    }
    if (KIND == 1) {
      const C<double> rh = ldc(c + off + e);
      acc[0] += rh.re * y.re + rh.im * y.im;
      acc[1] += rh.re * y.im - rh.im * y.re;
    } else {
      acc[0] += y.re * y.re + y.im * y.im;
      acc[1] += y.re * q.re + y.im * q.im;
      acc[2] += y.re * q.im - y.im * q.re;
    }
  }
  ck_publish<3>(acc, part);
}

// s = r - alpha v
__global__ void __launch_bounds__(kCkBlock) ck_sub(int64_t L, const double *__restrict__ st,
                                                   const double2 *__restrict__ r, const double2 *__restrict__ v,
                                                   double2 *__restrict__ s) {
  const int64_t off = (int64_t)blockIdx.y * L;
  const double *S = st + blockIdx.y * CK_W;
  const C<double> al(S[CK_ALPHA], S[CK_ALPHA + 1]);
  for (int64_t e = blockIdx.x * (int64_t)kCkBlock + threadIdx.x; e < L; e += (int64_t)gridDim.x * kCkBlock)
    stc(s + off + e, ldc(r + off + e) - al * ldc(v + off + e));
}

// x += alpha p + omega s ; r = s - omega t ; <rhat, r>, <r, r>
__global__ void __launch_bounds__(kCkBlock) ck_update(int64_t L, const double *__restrict__ st,
                                                      double2 *__restrict__ x, double2 *__restrict__ r,
                                                      const double2 *__restrict__ rhat, const double2 *__restrict__ p,
                                                      const double2 *__restrict__ s, const double2 *__restrict__ t,
                                                      double *part) {
  const int64_t off = (int64_t)blockIdx.y * L;
  const double *S = st + blockIdx.y * CK_W;
  const C<double> al(S[CK_ALPHA], S[CK_ALPHA + 1]), om(S[CK_OMEGA], S[CK_OMEGA + 1]);
  double acc[3] = {0.0, 0.0, 0.0};
  for (int64_t e = blockIdx.x * (int64_t)kCkBlock + threadIdx.x; e < L; e += (int64_t)gridDim.x * kCkBlock) {
    const C<double> ss = ldc(s + off + e);
    stc(x + off + e, ldc(x + off + e) + al * ldc(p + off + e) + om * ss);
    const C<double> rr = ss - om * ldc(t + off + e);
    stc(r + off + e, rr);
    const C<double> rh = ldc(rhat + off + e);
    acc[0] += rh.re * rr.re + rh.im * rr.im;
    acc[1] += rh.re * rr.im - rh.im * rr.re;
    acc[2] += rr.re * rr.re + rr.im * rr.im;
  }
  ck_publish<3>(acc, part);
}

// p = r + beta (p - omega v)
__global__ void __launch_bounds__(kCkBlock) ck_dir(int64_t L, const double *__restrict__ st,
                                                   const double2 *__restrict__ r, double2 *__restrict__ p,
                                                   const double2 *__restrict__ v) {
  const int64_t off = (int64_t)blockIdx.y * L;
  const double *S = st + blockIdx.y * CK_W;
  const C<double> be(S[CK_BETA], S[CK_BETA + 1]), om(S[CK_OMEGA], S[CK_OMEGA + 1]);
  for (int64_t e = blockIdx.x * (int64_t)kCkBlock + threadIdx.x; e < L; e += (int64_t)gridDim.x * kCkBlock)
    stc(p + off + e, ldc(r + off + e) + be * (ldc(p + off + e) - om * ldc(v + off + e)));
}

// scalar recurrences, one warp per rhs (blockIdx.x = rhs); same guards as the
// torch formulation (zero denominators freeze the rhs' step)
template <int KIND>
__global__ void ck_finish(int nblk, const double *__restrict__ part, double *__restrict__ st) {
  const int rhs = blockIdx.x, lane = threadIdx.x;
  double v[3] = {0.0, 0.0, 0.0};
  for (int b = lane; b < nblk; b += 32)
#pragma unroll
    for (int k = 0; k < 3; ++k) v[k] += part[((int64_t)rhs * nblk + b) * 3 + k];
#pragma unroll
  for (int k = 0; k < 3; ++k)
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], off);
  if (lane) return;
  double *S = st + rhs * CK_W;
  const bool act = S[CK_ACT] != 0.0;
  const C<double> rho(S[CK_RHO], S[CK_RHO + 1]);
  if (KIND == 1) {
    const C<double> sig(v[0], v[1]);
    const bool ok = act && (sig.re != 0.0 || sig.im != 0.0);
    const C<double> al = ok ? cdiv(rho, sig) : C<double>(0.0, 0.0);
    S[CK_ALPHA] = al.re, S[CK_ALPHA + 1] = al.im;
  } else if (KIND == 3) {
    const double tt = v[0];
    const C<double> om = (act && tt > 0.0) ? C<double>(v[1] / tt, v[2] / tt) : C<double>(0.0, 0.0);
    S[CK_OMEGA] = om.re, S[CK_OMEGA + 1] = om.im;
  } else {
    const C<double> rn(v[0], v[1]);
    const C<double> om(S[CK_OMEGA], S[CK_OMEGA + 1]), al(S[CK_ALPHA], S[CK_ALPHA + 1]);
    const bool rz = rho.re == 0.0 && rho.im == 0.0, oz = om.re == 0.0 && om.im == 0.0;
    const C<double> be = (act && !rz && !oz) ? cdiv(rn, rho) * cdiv(al, om) : C<double>(0.0, 0.0);
    S[CK_BETA] = be.re, S[CK_BETA + 1] = be.im;
    S[CK_RHO] = rn.re, S[CK_RHO + 1] = rn.im;
    S[CK_R2] = v[2];
    const bool nz = rn.re == 0.0 && rn.im == 0.0;
    const bool conv = act && (v[2] <= S[CK_TOL2] || oz || nz);
    if (act) {  // an inactive (frozen) rhs keeps its converged flag for the caller
      S[CK_CONV] = conv ? 1.0 : 0.0;
      S[CK_ITS] += 1.0;
    }
    if (conv && S[CK_FREEZE] != 0.0) S[CK_ACT] = 0.0;
  }
}

template <typename CT>
static int coarse_bicg_iter_impl(const int dims[4], const int block[4], int nv, const void *C_dev, double tau,
                                 int n, double2 *x, double2 *r, const double2 *rhat, double2 *p, double2 *v,
                                 double2 *s, double2 *t, double *st_dev, cudaStream_t st) {
  CoarseGeom cg;
  int rc = make_cg(dims, block, nv, cg);
  if (rc) return rc;
  const int64_t L = cg.nb * cg.nc;
  const int nblk = (int)std::max<int64_t>(1, std::min<int64_t>((L + 4 * kCkBlock - 1) / (4 * kCkBlock),
                                                               std::max(1, 4 * num_sms() / n)));
  double *part = nullptr;
  MGT_CUDA(scratch_alloc((void **)&part, (size_t)n * nblk * 3 * sizeof(double), st));
  const dim3 grid(nblk, n);
  rc = coarse_apply_impl<CT>(dims, block, nv, C_dev, p, v, n, st);
  if (rc) return rc;
  ck_dots<1><<<grid, kCkBlock, 0, st>>>(L, cg.nc, nv, tau, v, p, rhat, part);
  ck_finish<1><<<n, 32, 0, st>>>(nblk, part, st_dev);
  ck_sub<<<grid, kCkBlock, 0, st>>>(L, st_dev, r, v, s);
  rc = coarse_apply_impl<CT>(dims, block, nv, C_dev, s, t, n, st);
  if (rc) return rc;
  ck_dots<3><<<grid, kCkBlock, 0, st>>>(L, cg.nc, nv, tau, t, s, nullptr, part);
  ck_finish<3><<<n, 32, 0, st>>>(nblk, part, st_dev);
  ck_update<<<grid, kCkBlock, 0, st>>>(L, st_dev, x, r, rhat, p, s, t, part);
  ck_finish<4><<<n, 32, 0, st>>>(nblk, part, st_dev);
  ck_dir<<<grid, kCkBlock, 0, st>>>(L, st_dev, r, p, v);
  note_launch(8);
  MGT_LAUNCH_CHECK("coarse bicgstab iteration");
  MGT_CUDA(cudaFreeAsync(part, st));
  return MGT_OK;
}

// ---------------------------------------------------------------------------
// Coarse even-odd (checkerboard) form.  With every coarse extent even the
// 9-point coarse stencil couples only opposite-parity aggregates, so with
// the shift in the self blocks, C_tau = [[C_ee, C_eo], [C_oe, C_oo]] has
// block-diagonal C_ee, C_oo and its Schur complement on the even aggregates
//   S = C_ee - C_eo C_oo^-1 C_oe
// is applied as two half stencils: t_o = sum_dir D[o, dir] x_e[nbr] with
// D = C_oo^-1 C_o,dir (8 hops), then y_e = E[e, 0] x_e + sum_dir E[e, dir]
// t_o[nbr] with E[e, 0] = C_ee, E[e, dir] = -C_e,dir.  Both read 8-9 blocks
// per aggregate of one parity: an S apply streams as many bytes as one full
// C apply on half the unknowns, and BiCGStab on S needs about half the
// iterations (the reference solves the full coarse system with GCR,
// multigrid.py:228-243 via krylov.py:52-118; the stopping test is the same
// full residual, the odd rows being solved exactly).
// Compact parity fields: aggregate b has cb index b >> 1 (the fastest coarse
// extent is even, so every pair b = 2c, 2c + 1 holds one of each parity);
// vectors (n_rhs, nb / 2, nc), blocks M[((c * ND + d) * nc + col) * nc + row].
__device__ __forceinline__ int64_t coarse_cb_full(const CoarseGeom &cg, int64_t c, int par) {
  const int64_t b0 = 2 * c;
  int64_t r = b0;
  const int c2 = (int)(r % cg.Cd[2]);
  r /= cg.Cd[2];
  const int c1 = (int)(r % cg.Cd[1]);
  r /= cg.Cd[1];
  const int c0 = (int)(r % cg.Cd[0]);
  const int c3 = (int)(r / cg.Cd[0]);
  return b0 + ((((c0 + c1 + c2 + c3) & 1) != par) ? 1 : 0);
}

// y[c] = sum_{d < ND} M[c][d] src_d, output parity `par`; ND = 8: hops
// 1..8 from x_other; ND = 9: dir 0 (self, from x_self; dropped when
// skip_self) and hops 1..8 from x_other.  Thread per (d, row), the ND
// source vectors staged in shared memory, direction partials summed in
// direction order (deterministic, the same for every NR).
template <int NR, typename CT, int ND>
__global__ void __launch_bounds__(kCoarseDirThreads, 2)
    coarse_half_kernel(CoarseGeom cg, int par, const CT *__restrict__ Mb, const double2 *__restrict__ xs,
                       const double2 *__restrict__ xo, double2 *__restrict__ y, int skip_self) {
  extern __shared__ double2 sm[];
  __shared__ int64_t nbr[ND];
  const int nc = cg.nc;
  const int64_t nbh = cg.nb / 2;
  const int64_t c = blockIdx.x;
  if (threadIdx.x < ND) {
    const int dir = ND == 8 ? threadIdx.x + 1 : threadIdx.x;
    nbr[threadIdx.x] = coarse_nbr(cg, coarse_cb_full(cg, c, par), dir) >> 1;
  }
  __syncthreads();
  using AT = std::conditional_t<sizeof(CT) == 8, float, double>;
  using A2 = std::conditional_t<sizeof(CT) == 8, float2, double2>;
  A2 *sx = reinterpret_cast<A2 *>(sm);
  for (int i = threadIdx.x; i < ND * nc * NR; i += blockDim.x) {
    const int col = i % nc, q = i / nc;
    const int r = q % NR, d = q / NR;
    const bool self = ND == 9 && d == 0;
    const double2 xv = (self && skip_self) ? make_double2(0.0, 0.0) : (self ? xs : xo)[((int64_t)r * nbh + nbr[d]) * nc + col];
    A2 a;
    a.x = (AT)xv.x;
    a.y = (AT)xv.y;
    sx[(d * nc + col) * NR + r] = a;
  }
  __syncthreads();
  const int d = threadIdx.x / nc, row = threadIdx.x - d * nc;
  const bool on = d < ND && !(ND == 9 && d == 0 && skip_self);
  C<AT> acc[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) acc[r] = C<AT>(AT(0), AT(0));
  if (on) {
    const CT *Cb = Mb + (c * ND + d) * (int64_t)nc * nc + row;
    const A2 *xsd = sx + d * nc * NR;
    constexpr int U = (sizeof(CT) == 16 && NR >= 2) ? 4 : 8;
    for (int c0 = 0; c0 < nc; c0 += U) {
      CT cl[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (c0 + u < nc) cl[u] = Cb[(int64_t)(c0 + u) * nc];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (c0 + u < nc) {
          const C<AT> cv(cl[u].x, cl[u].y);
#pragma unroll
          for (int r = 0; r < NR; ++r) {
            const A2 xv = xsd[(c0 + u) * NR + r];
            acc[r] = cfma(cv, C<AT>(xv.x, xv.y), acc[r]);
          }
        }
      }
    }
  }
  __syncthreads();
  if (d < ND) {
#pragma unroll
    for (int r = 0; r < NR; ++r) sm[(d * NR + r) * nc + row] = make_double2((double)acc[r].re, (double)acc[r].im);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < NR * nc; i += blockDim.x) {
    const int r = i / nc, rw = i % nc;
    C<double> t(0.0, 0.0);
#pragma unroll
    for (int dd = 0; dd < ND; ++dd) {
      const double2 v = sm[(dd * NR + r) * nc + rw];
      t = t + C<double>(v.x, v.y);
    }
    y[((int64_t)r * nbh + c) * nc + rw] = make_double2(t.re, t.im);
  }
}

template <int NR, typename CT, int ND>
static int launch_coarse_half(const CoarseGeom &cg, int par, const CT *M, const double2 *xs, const double2 *xo,
                              double2 *y, int skip_self, cudaStream_t st) {
  const int block = ((ND * cg.nc + 31) / 32) * 32;
  if (block > kCoarseDirThreads) return fail(MGT_ERR_INVALID, "coarse even-odd form: 2 nv > 49 is not supported");
  const size_t smem = (size_t)ND * cg.nc * NR * sizeof(double2);
  // (opt in whenever the dynamic part grows: the static nbr table counts
  // toward the 48 KB default too, e.g. 8 x 48 x 8 x 16 B = exactly 48 KB)
  static size_t set = 0;
  if (smem > set) {
    MGT_CUDA(cudaFuncSetAttribute(coarse_half_kernel<NR, CT, ND>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
    set = smem;
  }
  coarse_half_kernel<NR, CT, ND><<<(unsigned)(cg.nb / 2), block, smem, st>>>(cg, par, M, xs, xo, y, skip_self);
  MGT_LAUNCH_CHECK("coarse_half_kernel");
  return MGT_OK;
}

// n_rhs fields, up to 8 per launch
template <typename CT, int ND>
static int coarse_half_impl(const CoarseGeom &cg, int par, const CT *M, const double2 *xs, const double2 *xo,
                            double2 *y, int skip_self, int n_rhs, cudaStream_t st) {
  const int64_t stride = (cg.nb / 2) * cg.nc;
  for (int r = 0; r < n_rhs;) {
    const int left = n_rhs - r;
    const int nr = left >= 8 ? 8 : (left >= 4 ? 4 : (left >= 2 ? 2 : 1));
    const double2 *s0 = xs ? xs + r * stride : nullptr;
    const double2 *o0 = xo + r * stride;
    double2 *y0 = y + r * stride;
    int rc = nr == 8   ? launch_coarse_half<8, CT, ND>(cg, par, M, s0, o0, y0, skip_self, st)
             : nr == 4 ? launch_coarse_half<4, CT, ND>(cg, par, M, s0, o0, y0, skip_self, st)
             : nr == 2 ? launch_coarse_half<2, CT, ND>(cg, par, M, s0, o0, y0, skip_self, st)
                       : launch_coarse_half<1, CT, ND>(cg, par, M, s0, o0, y0, skip_self, st);
    if (rc) return rc;
    r += nr;
  }
  return MGT_OK;
}

static int make_cg_eo(const int dims[4], const int block[4], int nv, CoarseGeom &cg) {
  int rc = make_cg(dims, block, nv, cg);
  if (rc) return rc;
  for (int i = 0; i < 4; ++i)
    if (cg.Cd[i] % 2) return fail(MGT_ERR_INVALID, "coarse even-odd form needs every coarse extent even");
  return MGT_OK;
}

// y_e = S x_e through t_o (scratch, n_rhs odd fields)
template <typename CT>
static int schur_apply(const CoarseGeom &cg, const CT *D, const CT *E, const double2 *x, double2 *y, double2 *t_o,
                       int n, cudaStream_t st) {
  int rc = coarse_half_impl<CT, 8>(cg, 1, D, nullptr, x, t_o, 0, n, st);
  if (rc) return rc;
  return coarse_half_impl<CT, 9>(cg, 0, E, x, t_o, y, 0, n, st);
}

// n_iters BiCGStab iterations on S for n independent rhs, scalars on the
// device; rhs with freeze set stop themselves once converged
template <typename CT>
static int schur_bicg_iters(const CoarseGeom &cg, const CT *D, const CT *E, int n, int n_iters, double2 *x,
                            double2 *r, const double2 *rhat, double2 *p, double2 *v, double2 *s, double2 *t,
                            double2 *t_o, double *st_dev, cudaStream_t st) {
  const int64_t L = (cg.nb / 2) * cg.nc;
  const int nblk = (int)std::max<int64_t>(1, std::min<int64_t>((L + 4 * kCkBlock - 1) / (4 * kCkBlock),
                                                               std::max(1, 4 * num_sms() / n)));
  double *part = nullptr;
  MGT_CUDA(scratch_alloc((void **)&part, (size_t)n * nblk * 3 * sizeof(double), st));
  const dim3 grid(nblk, n);
  int rc = MGT_OK;
  for (int it = 0; it < n_iters && rc == MGT_OK; ++it) {
    rc = schur_apply<CT>(cg, D, E, p, v, t_o, n, st);
    if (rc) break;
    ck_dots<1><<<grid, kCkBlock, 0, st>>>(L, cg.nc, cg.nc / 2, 0.0, v, p, rhat, part);
    ck_finish<1><<<n, 32, 0, st>>>(nblk, part, st_dev);
    ck_sub<<<grid, kCkBlock, 0, st>>>(L, st_dev, r, v, s);
    rc = schur_apply<CT>(cg, D, E, s, t, t_o, n, st);
    if (rc) break;
    ck_dots<3><<<grid, kCkBlock, 0, st>>>(L, cg.nc, cg.nc / 2, 0.0, t, s, nullptr, part);
    ck_finish<3><<<n, 32, 0, st>>>(nblk, part, st_dev);
    ck_update<<<grid, kCkBlock, 0, st>>>(L, st_dev, x, r, rhat, p, s, t, part);
    ck_finish<4><<<n, 32, 0, st>>>(nblk, part, st_dev);
    ck_dir<<<grid, kCkBlock, 0, st>>>(L, st_dev, r, p, v);
    note_launch(8);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) rc = cuda_fail(e, "coarse Schur bicgstab iteration");
  }
  cudaFreeAsync(part, st);
  return rc;
}

}  // namespace mgt

extern "C" {

int mgt_coarse_half_apply(const int dims[4], const int block[4], int nv, const void *M_dev, int nd, int par,
                          int m_fp32, int skip_self, const void *x_self, const void *x_other, void *y, int n_rhs,
                          void *stream) {
  if (!dims || !block || !M_dev || !x_other || !y || n_rhs < 1 || (nd != 8 && nd != 9) || (par != 0 && par != 1) ||
      (nd == 9 && !skip_self && !x_self))
    return fail(MGT_ERR_INVALID, "mgt_coarse_half_apply: bad argument");
  CoarseGeom cg;
  int rc = make_cg_eo(dims, block, nv, cg);
  if (rc) return rc;
  cudaStream_t st = as_stream(stream);
  auto D = [](const void *q) { return (const double2 *)q; };
  if (m_fp32)
    return nd == 8 ? coarse_half_impl<float2, 8>(cg, par, (const float2 *)M_dev, D(x_self), D(x_other), (double2 *)y,
                                                 skip_self, n_rhs, st)
                   : coarse_half_impl<float2, 9>(cg, par, (const float2 *)M_dev, D(x_self), D(x_other), (double2 *)y,
                                                 skip_self, n_rhs, st);
  return nd == 8 ? coarse_half_impl<double2, 8>(cg, par, (const double2 *)M_dev, D(x_self), D(x_other), (double2 *)y,
                                                skip_self, n_rhs, st)
                 : coarse_half_impl<double2, 9>(cg, par, (const double2 *)M_dev, D(x_self), D(x_other), (double2 *)y,
                                                skip_self, n_rhs, st);
}

int mgt_coarse_schur_apply(const int dims[4], const int block[4], int nv, const void *D_dev, const void *E_dev,
                           int m_fp32, const void *x_e, void *y_e, void *t_o, int n_rhs, void *stream) {
  if (!dims || !block || !D_dev || !E_dev || !x_e || !y_e || !t_o || n_rhs < 1)
    return fail(MGT_ERR_INVALID, "mgt_coarse_schur_apply: bad argument");
  CoarseGeom cg;
  int rc = make_cg_eo(dims, block, nv, cg);
  if (rc) return rc;
  cudaStream_t st = as_stream(stream);
  if (m_fp32)
    return schur_apply<float2>(cg, (const float2 *)D_dev, (const float2 *)E_dev, (const double2 *)x_e, (double2 *)y_e,
                               (double2 *)t_o, n_rhs, st);
  return schur_apply<double2>(cg, (const double2 *)D_dev, (const double2 *)E_dev, (const double2 *)x_e,
                              (double2 *)y_e, (double2 *)t_o, n_rhs, st);
}

int mgt_coarse_schur_bicgstab(const int dims[4], const int block[4], int nv, const void *D_dev, const void *E_dev,
                              int m_fp32, int n_rhs, int n_iters, void *x, void *r, const void *rhat, void *p,
                              void *v, void *s, void *t, void *t_o, double *state, void *stream) {
  if (!dims || !block || !D_dev || !E_dev || !x || !r || !rhat || !p || !v || !s || !t || !t_o || !state ||
      n_rhs < 1 || n_iters < 1)
    return fail(MGT_ERR_INVALID, "mgt_coarse_schur_bicgstab: bad argument");
  CoarseGeom cg;
  int rc = make_cg_eo(dims, block, nv, cg);
  if (rc) return rc;
  cudaStream_t st = as_stream(stream);
  auto Q = [](const void *q) { return (double2 *)q; };
  if (m_fp32)
    return schur_bicg_iters<float2>(cg, (const float2 *)D_dev, (const float2 *)E_dev, n_rhs, n_iters, Q(x), Q(r),
                                    Q(rhat), Q(p), Q(v), Q(s), Q(t), Q(t_o), state, st);
  return schur_bicg_iters<double2>(cg, (const double2 *)D_dev, (const double2 *)E_dev, n_rhs, n_iters, Q(x), Q(r),
                                   Q(rhat), Q(p), Q(v), Q(s), Q(t), Q(t_o), state, st);
}

int mgt_coarse_bicgstab_iter(const int dims[4], const int block[4], int nv, const void *C_dev, int c_fp32,
                             double tau, int n_rhs, void *x, void *r, const void *rhat, void *p, void *v, void *s,
                             void *t, double *state, void *stream) {
  if (!dims || !block || !C_dev || !x || !r || !rhat || !p || !v || !s || !t || !state || n_rhs < 1)
    return fail(MGT_ERR_INVALID, "mgt_coarse_bicgstab_iter: bad argument");
  cudaStream_t st = as_stream(stream);
  auto D = [](const void *q) { return (double2 *)q; };
  return c_fp32 ? coarse_bicg_iter_impl<float2>(dims, block, nv, C_dev, tau, n_rhs, D(x), D(r), D(rhat), D(p), D(v), D(s),
                                                D(t), state, st)
                : coarse_bicg_iter_impl<double2>(dims, block, nv, C_dev, tau, n_rhs, D(x), D(r), D(rhat), D(p), D(v),
                                                 D(s), D(t), state, st);
}

int mgt_coarse_apply(const int dims[4], const int block[4], int nv, const void *C_dev, const void *xc_dev,
                     void *yc_dev, int n_rhs, void *stream) {
  return coarse_apply_impl<double2>(dims, block, nv, C_dev, xc_dev, yc_dev, n_rhs, stream);
}

int mgt_coarse_apply_c32(const int dims[4], const int block[4], int nv, const void *C32_dev, const void *xc_dev,
                         void *yc_dev, int n_rhs, void *stream) {
  return coarse_apply_impl<float2>(dims, block, nv, C32_dev, xc_dev, yc_dev, n_rhs, stream);
}

}  // extern "C"
