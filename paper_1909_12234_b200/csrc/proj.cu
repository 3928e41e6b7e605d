// Tall-skinny deflation projections (reference: trace.py:179-183, :266-267;
// eigen.py:79-86 CGS2 `v - Q (Q^H v)`):
//   H = V^H X            (k x s),   V: k vectors, X: s vectors, length len
//   X <- X - V H         (the projected probes X - V (V^H X) when H = V^H X)
// fp64 complex on the FP64 pipe (B200 has no fp64 tensor-core advantage).
// V^H X is split over the long dimension: every block produces a k x s
// partial in a fixed order and a final kernel sums the partials in block
// order, so results are bitwise reproducible.
//  * s <= 8 ("GEMV-like", HBM-bound on V): thread per element, each warp
//    owns 2-8 vectors, a block 8 warps; X comes from L1 to the 8 warps.
//  * k <= 8 < s (a few vectors against many, e.g. a Davidson block against
//    the search space): the same kernel with the roles swapped, H = (X^H V)^H
//    conjugate-transposed by the final reduction.
//  * k, s > 8  ("GEMM-like", FP64-bound): 64x64 output tiles staged through
//    shared memory with 4x4 complex register micro-tiles.
#include <algorithm>

#include "reduce.cuh"

namespace mgt {

// WV vectors per warp (8 warps per block): WV * S complex accumulators per
// thread; fewer vectors per warp for more rhs keeps the register count (and
// so the loads in flight per SM) up.
template <int S>
constexpr int warp_vecs() {
  return S <= 2 ? 8 : (S <= 4 ? 4 : 2);
}

// e-elements per lane per loop trip: their V and X loads are issued together
// ahead of the FMAs (more bytes in flight per SM for the HBM-bound few-column
// shapes; 1 at S = 8 where the accumulators already fill the registers).
template <int S>
constexpr int vhx_unroll() {
#ifdef MGT_VHX_NO_UNROLL
  return 1;
#else
  return S <= 2 ? 4 : (S <= 4 ? 2 : 1);
#endif
}

// S: compile-time column capacity, s <= S the actual column count
template <int S>
__global__ void __launch_bounds__(256, 2) vhx_small_kernel(const double2 *__restrict__ V, const double2 *__restrict__ X,
                                                           int64_t len, int k, int s, double2 *__restrict__ part) {
  constexpr int kWarpVecs = warp_vecs<S>();
  constexpr int kBlockVecs = 8 * kWarpVecs;
  constexpr int U = vhx_unroll<S>();
  __shared__ double2 red[8][kWarpVecs * S];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int i0 = blockIdx.y * kBlockVecs + warp * kWarpVecs;
  C<double> acc[kWarpVecs][S];
#pragma unroll
  for (int a = 0; a < kWarpVecs; ++a)
#pragma unroll
    for (int j = 0; j < S; ++j) acc[a][j] = C<double>(0.0, 0.0);
  const int64_t stride = (int64_t)gridDim.x * 32;
  for (int64_t e = blockIdx.x * 32 + lane; e < len; e += stride * U) {
    // element u of this trip: e + u * stride (absent ones load zeros)
    C<double> xv[U][S], v[U][kWarpVecs];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t eu = e + u * stride;
      const bool in = eu < len;
#pragma unroll
      for (int j = 0; j < S; ++j) xv[u][j] = (j < s && in) ? ldc(X + (int64_t)j * len + eu) : C<double>(0.0, 0.0);
#pragma unroll
      for (int a = 0; a < kWarpVecs; ++a)
        v[u][a] = (i0 + a < k && in) ? ldc(V + (int64_t)(i0 + a) * len + eu) : C<double>(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int a = 0; a < kWarpVecs; ++a)
#pragma unroll
        for (int j = 0; j < S; ++j) acc[a][j] = cfma_conj(v[u][a], xv[u][j], acc[a][j]);
  }
  // warp reduce, then each warp writes its own 8 x S values (distinct i)
#pragma unroll
  for (int a = 0; a < kWarpVecs; ++a)
#pragma unroll
    for (int j = 0; j < S; ++j) {
      C<double> v = acc[a][j];
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) {
        v.re += __shfl_xor_sync(0xffffffffu, v.re, off);
        v.im += __shfl_xor_sync(0xffffffffu, v.im, off);
      }
      if (lane == 0) red[warp][a * S + j] = make_double2(v.re, v.im);
    }
  __syncwarp();
  for (int q = lane; q < kWarpVecs * S; q += 32) {
    const int a = q / S, j = q % S;
    if (i0 + a < k && j < s) part[((int64_t)blockIdx.x * k + (i0 + a)) * s + j] = red[warp][q];
  }
}

// 64 x TJ tile of V^H X over an e-chunk range; part: [block.x][k][s].
// 16 x (TJ/4) threads, a 4 x 4 complex register micro-tile each; TJ follows
// s (16, 32 or 64) so skinny column counts do not run mostly-empty tiles.
template <int TJ>
__global__ void __launch_bounds__(16 * (TJ / 4)) vhx_tile_kernel(const double2 *__restrict__ V,
                                                                const double2 *__restrict__ X, int64_t len, int k,
                                                                int s, double2 *__restrict__ part) {
  constexpr int T = 64, E = 8, NT = 16 * (TJ / 4);
  __shared__ double2 sV[E][T + 1];
  __shared__ double2 sX[E][TJ + 1];
  const int ti = threadIdx.x / (TJ / 4), tj = threadIdx.x % (TJ / 4);
  const int i0 = blockIdx.y * T, j0 = blockIdx.z * TJ;
  C<double> acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = C<double>(0.0, 0.0);
  for (int64_t e0 = (int64_t)blockIdx.x * E; e0 < len; e0 += (int64_t)gridDim.x * E) {
    // one staging loop for both tiles (their loads in flight together)
    for (int q = threadIdx.x; q < T * E; q += NT) {
      const int r = q / E, c = q % E;
      const int64_t e = e0 + c;
      const double2 vv = (i0 + r < k && e < len) ? V[(int64_t)(i0 + r) * len + e] : make_double2(0.0, 0.0);
      if (r < TJ) sX[c][r] = (j0 + r < s && e < len) ? X[(int64_t)(j0 + r) * len + e] : make_double2(0.0, 0.0);
      sV[c][r] = vv;
    }
    __syncthreads();
#pragma unroll
    for (int c = 0; c < E; ++c) {
      C<double> va[4], xb[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) va[a] = C<double>(sV[c][ti * 4 + a].x, sV[c][ti * 4 + a].y);
#pragma unroll
      for (int b = 0; b < 4; ++b) xb[b] = C<double>(sX[c][tj * 4 + b].x, sX[c][tj * 4 + b].y);
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = cfma_conj(va[a], xb[b], acc[a][b]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int i = i0 + ti * 4 + a, j = j0 + tj * 4 + b;
      if (i < k && j < s) part[((int64_t)blockIdx.x * k + i) * s + j] = make_double2(acc[a][b].re, acc[a][b].im);
    }
}

// H[j*k + i] (column major k x s) = sum over blocks of part[b][i][j]
// one warp per output: lanes stride over the block partials, then a fixed
// shuffle tree (deterministic).  swapped: part holds (X^H V) as [b][j][i]
// (k = its column count), so H[q] = conj(sum part[b][q]).
__global__ void vhx_reduce_kernel(const double2 *__restrict__ part, int nblk, int k, int s, double2 *__restrict__ H,
                                  int swapped) {
  const int64_t n = (int64_t)k * s;
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t q = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); q < n; q += warps) {
    const int i = (int)(q / s), j = (int)(q % s);
    C<double> t(0.0, 0.0);
    for (int b = lane; b < nblk; b += 32) t = t + ldc(part + (int64_t)b * n + q);
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
      t.re += __shfl_xor_sync(0xffffffffu, t.re, off);
      t.im += __shfl_xor_sync(0xffffffffu, t.im, off);
    }
    if (lane == 0) {
      if (swapped)
        H[q] = make_double2(t.re, -t.im);
      else
        H[(int64_t)j * k + i] = make_double2(t.re, t.im);
    }
  }
}

// X[j] -= sum_i V[i] H[i, j] for j in a TJ-wide tile (grid.y); TJ follows s
// (1, 2, 4, 8) so no accumulator or H load is wasted on absent columns, and
// the V loads are issued 8 vectors at a time (independent, in flight
// together) ahead of their FMAs.
template <int TJ>
__global__ void __launch_bounds__(256) proj_sub_kernel(const double2 *__restrict__ V, const double2 *__restrict__ H,
                                                       double2 *__restrict__ X, int64_t len, int k, int s) {
  extern __shared__ double2 sH[];  // k x TJ
  const int j0 = blockIdx.y * TJ;
  for (int q = threadIdx.x; q < k * TJ; q += blockDim.x) {
    const int i = q / TJ, j = q % TJ;
    sH[q] = (j0 + j < s) ? H[(int64_t)(j0 + j) * k + i] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  constexpr int U = 8;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < len; e += (int64_t)gridDim.x * blockDim.x) {
    C<double> acc[TJ];
#pragma unroll
    for (int j = 0; j < TJ; ++j) acc[j] = C<double>(0.0, 0.0);
    for (int i0 = 0; i0 < k; i0 += U) {
      C<double> v[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (i0 + u < k) v[u] = ldc(V + (int64_t)(i0 + u) * len + e);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (i0 + u < k) {
#pragma unroll
          for (int j = 0; j < TJ; ++j) {
            const double2 hv = sH[(i0 + u) * TJ + j];
            acc[j] = cfma(v[u], C<double>(hv.x, hv.y), acc[j]);
          }
        }
      }
    }
#pragma unroll
    for (int j = 0; j < TJ; ++j) {
      if (j0 + j < s) {
        double2 *p = X + (int64_t)(j0 + j) * len + e;
        const double2 x = *p;
        *p = make_double2(x.x - acc[j].re, x.y - acc[j].im);
      }
    }
  }
}

}  // namespace mgt

using namespace mgt;

extern "C" {

int mgt_proj_vhx(const void *V_dev, const void *X_dev, int64_t len, int k, int s, void *H_dev, void *stream) {
  if (!V_dev || !X_dev || !H_dev || len < 0 || k < 1 || s < 1) return fail(MGT_ERR_INVALID, "mgt_proj_vhx: bad argument");
  cudaStream_t st = as_stream(stream);
  const double2 *V = (const double2 *)V_dev, *X = (const double2 *)X_dev;
  int nblk;
  double2 *part = nullptr;
  // few columns (or, swapped, few vectors): the GEMV-like kernel
  const bool swapped = s > 8 && k <= 8;
  if (s <= 8 || swapped) {
    const double2 *Vv = swapped ? X : V, *Xv = swapped ? V : X;
    const int kk = swapped ? s : k, ss = swapped ? k : s;
    const int bv = 8 * (ss <= 2 ? warp_vecs<1>() : (ss <= 4 ? warp_vecs<4>() : warp_vecs<8>()));
    const int gy = (kk + bv - 1) / bv;
#ifdef MGT_VHX_OLD_GRID
    nblk = (int)std::max<int64_t>(1, std::min<int64_t>((len + 31) / 32, (int64_t)num_sms() * 6 / gy + 1));
#else
    // one full wave of the 2 resident blocks per SM (grid-stride over len):
    // no partial tail wave, and fewer partials for the final reduction
    nblk = (int)std::max<int64_t>(1, std::min<int64_t>((len + 31) / 32, std::max(1, num_sms() * 2 / gy)));
#endif
    MGT_CUDA(scratch_alloc((void **)&part, (size_t)nblk * k * s * sizeof(double2), st));
    dim3 grid(nblk, gy);
#define MGT_VHX(SS) vhx_small_kernel<SS><<<grid, 256, 0, st>>>(Vv, Xv, len, kk, ss, part)
    if (ss == 1)
      MGT_VHX(1);
    else if (ss == 2)
      MGT_VHX(2);
    else if (ss == 3)
      MGT_VHX(3);
    else if (ss == 4)
      MGT_VHX(4);
    else
      MGT_VHX(8);
#undef MGT_VHX
    MGT_LAUNCH_CHECK("vhx_small_kernel");
  } else {
    const int tj = s <= 16 ? 16 : (s <= 32 ? 32 : 64);
    const int gy = (k + 63) / 64, gz = (s + tj - 1) / tj;
    // ~16 resident 64-thread tiles (4 of 256 threads) per SM
#ifdef MGT_VHX_OLD_GRID
    const int per_sm = 4 * 64 / tj;
    nblk = (int)std::max<int64_t>(1, std::min<int64_t>((len + 7) / 8, (int64_t)num_sms() * per_sm / (gy * gz) + 1));
#else
    // one full wave of resident tiles (occupancy-queried), no partial tail
    const int per_sm = tj == 16 ? blocks_per_sm((const void *)vhx_tile_kernel<16>, 64)
                       : tj == 32 ? blocks_per_sm((const void *)vhx_tile_kernel<32>, 128)
                                  : blocks_per_sm((const void *)vhx_tile_kernel<64>, 256);
    if (per_sm < 1) return per_sm < 0 ? MGT_ERR_CUDA : fail(MGT_ERR_CUDA, "vhx_tile_kernel cannot be resident");
    nblk = (int)std::max<int64_t>(1, std::min<int64_t>((len + 7) / 8, std::max(1, num_sms() * per_sm / (gy * gz))));
#endif
    MGT_CUDA(scratch_alloc((void **)&part, (size_t)nblk * k * s * sizeof(double2), st));
    dim3 grid(nblk, gy, gz);
    if (tj == 16)
      vhx_tile_kernel<16><<<grid, 64, 0, st>>>(V, X, len, k, s, part);
    else if (tj == 32)
      vhx_tile_kernel<32><<<grid, 128, 0, st>>>(V, X, len, k, s, part);
    else
      vhx_tile_kernel<64><<<grid, 256, 0, st>>>(V, X, len, k, s, part);
    MGT_LAUNCH_CHECK("vhx_tile_kernel");
  }
  // the reduction reads part as [blk][rows][cols]: swapped, rows = s and cols = k
  vhx_reduce_kernel<<<grid_for((int64_t)k * s * 32, 128, 8), 128, 0, st>>>(
      part, nblk, swapped ? s : k, swapped ? k : s, (double2 *)H_dev, swapped ? 1 : 0);
  MGT_LAUNCH_CHECK("vhx_reduce_kernel");
  MGT_CUDA(cudaFreeAsync(part, st));
  return MGT_OK;
}

int mgt_proj_sub(const void *V_dev, const void *H_dev, void *X_dev, int64_t len, int k, int s, void *stream) {
  if (!V_dev || !X_dev || !H_dev || len < 0 || k < 1 || s < 1) return fail(MGT_ERR_INVALID, "mgt_proj_sub: bad argument");
  cudaStream_t st = as_stream(stream);
  const int TJ = s >= 8 ? 8 : (s >= 4 ? 4 : (s >= 2 ? 2 : 1));
  const int gy = (s + TJ - 1) / TJ;
  dim3 grid(grid_for(len, 256, 4), gy);
  const size_t smem = (size_t)k * TJ * sizeof(double2);
  if (smem > 200 * 1024) return fail(MGT_ERR_INVALID, "mgt_proj_sub: k too large");
  // MGT_PSUB: one full wave of resident blocks over (len, column tiles)
#ifdef MGT_VHX_OLD_GRID
#define MGT_PSUB_GRID(T)
#else
#define MGT_PSUB_GRID(T)                                                                                 \
  do {                                                                                                   \
    const int per_sm = blocks_per_sm((const void *)proj_sub_kernel<T>, 256, smem);                     \
    if (per_sm < 1) return per_sm < 0 ? MGT_ERR_CUDA : fail(MGT_ERR_CUDA, "proj_sub_kernel cannot be resident"); \
    grid.x = (unsigned)std::max<int64_t>(                                                                \
        1, std::min<int64_t>((len + 255) / 256, std::max(1, num_sms() * per_sm / gy)));                 \
  } while (0)
#endif
#define MGT_PSUB(T)                                                                                                \
  do {                                                                                                             \
    if (smem > 48 * 1024)                                                                                          \
      MGT_CUDA(cudaFuncSetAttribute(proj_sub_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    MGT_PSUB_GRID(T);                                                                                              \
    proj_sub_kernel<T><<<grid, 256, smem, st>>>((const double2 *)V_dev, (const double2 *)H_dev, (double2 *)X_dev, \
                                                len, k, s);                                                        \
  } while (0)
  if (TJ == 8)
    MGT_PSUB(8);
  else if (TJ == 4)
    MGT_PSUB(4);
  else if (TJ == 2)
    MGT_PSUB(2);
  else
    MGT_PSUB(1);
#undef MGT_PSUB
#undef MGT_PSUB_GRID
  MGT_LAUNCH_CHECK("proj_sub_kernel");
  return MGT_OK;
}

}  // extern "C"
