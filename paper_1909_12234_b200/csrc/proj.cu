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
#include <cstdlib>

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

// V^H X for 4 < s <= 16 on the FP64 tensor cores (DMMA, mma.sync m8n8k4:
// fp64 products and fp64 accumulation, so the 1e-12 parity bar holds).  The
// thread-per-element kernel above re-reads the s columns of X from L1 for
// every pair of vectors a warp owns (at s = 8 four fifths of its L1 request
// bytes are X), and the 64 x TJ tile kernel is issue-bound on shared-memory
// operands; here a warp owns 64 vectors x all s columns of an e-range, the
// X fragment is loaded once per 64 vectors and the complex product is four
// real m8n8k4 MMAs per (8 vectors x 8 columns x 4 elements):
//   Re += vr xr + vi xi,   Im += vr xi + vi (-xr)     (conj(v) x)
// Fragment maps (lane = 4 r + c): A[m = r][k = c] = V_{i0 + r}[e + c'],
// B[k = c][n = r] = X_{j0 + r}[e + c'], C[m = r][n = 2 c + {0, 1}].  A lane
// loads 32 contiguous bytes (elements e0 + 2c, e0 + 2c + 1) of its vector, so
// a warp load covers 8 vectors x one 128-byte line; the two elements feed two
// k-steps (elements {0,2,4,6} and {1,3,5,7}: A and B use the same map, so
// the products pair up; the e-sum is order-fixed, hence deterministic).
// Every warp writes its own k x s partial (part[warp][k][s]); the final
// kernel sums them in warp order.
struct alignas(32) d4 {
  double x0, y0, x1, y1;
};
__device__ __forceinline__ void dmma884(double &c0, double &c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int NT>  // column tiles of 8: s <= 8 * NT
__global__ void __launch_bounds__(128, 2) vhx_dmma_kernel(const double2 *__restrict__ V, const double2 *__restrict__ X,
                                                          int64_t len, int k, int s, double2 *__restrict__ part) {
  constexpr int MT = 8;  // 64 vectors per warp
  const int lane = threadIdx.x & 31, r = lane >> 2, c = lane & 3;
  const int64_t gw = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5), GW = (int64_t)gridDim.x * 4;
  const int i0 = blockIdx.y * (8 * MT);
  double cre[MT][NT][2], cim[MT][NT][2];
#pragma unroll
  for (int m = 0; m < MT; ++m)
#pragma unroll
    for (int n = 0; n < NT; ++n) cre[m][n][0] = cre[m][n][1] = cim[m][n][0] = cim[m][n][1] = 0.0;
  const d4 zero{0.0, 0.0, 0.0, 0.0};
  const d4 *vp[MT];
  const d4 *xp[NT];
  bool vok[MT], xok[NT];
#pragma unroll
  for (int m = 0; m < MT; ++m) {
    const int i = i0 + m * 8 + r;
    vok[m] = i < k;
    vp[m] = reinterpret_cast<const d4 *>(V + (int64_t)(vok[m] ? i : 0) * len) + c;
  }
#pragma unroll
  for (int n = 0; n < NT; ++n) {
    const int j = n * 8 + r;
    xok[n] = j < s;
    xp[n] = reinterpret_cast<const d4 *>(X + (int64_t)(xok[n] ? j : 0) * len) + c;
  }
  const int64_t nsteps = (len + 7) / 8;  // 8 elements (4 d4 per vector) per step
  d4 va[MT], xa[NT];
  auto load = [&](int64_t st, d4 (&v)[MT], d4 (&x)[NT]) {
    const bool in = st < nsteps && st * 8 + 2 * c < len;  // len even: both elements of the d4 are inside
#pragma unroll
    for (int n = 0; n < NT; ++n) x[n] = (in && xok[n]) ? xp[n][st * 4] : zero;
#pragma unroll
    for (int m = 0; m < MT; ++m) v[m] = (in && vok[m]) ? vp[m][st * 4] : zero;
  };
  load(gw, va, xa);
#pragma unroll 1
  for (int64_t st = gw; st < nsteps; st += GW) {
    d4 vb[MT], xb[NT];
    load(st + GW, vb, xb);  // next step's loads in flight during this step's MMAs
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      const double nx0 = -xa[n].x0, nx1 = -xa[n].x1;
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        dmma884(cre[m][n][0], cre[m][n][1], va[m].x0, xa[n].x0);
        dmma884(cim[m][n][0], cim[m][n][1], va[m].x0, xa[n].y0);
        dmma884(cre[m][n][0], cre[m][n][1], va[m].y0, xa[n].y0);
        dmma884(cim[m][n][0], cim[m][n][1], va[m].y0, nx0);
        dmma884(cre[m][n][0], cre[m][n][1], va[m].x1, xa[n].x1);
        dmma884(cim[m][n][0], cim[m][n][1], va[m].x1, xa[n].y1);
        dmma884(cre[m][n][0], cre[m][n][1], va[m].y1, xa[n].y1);
        dmma884(cim[m][n][0], cim[m][n][1], va[m].y1, nx1);
      }
    }
#pragma unroll
    for (int m = 0; m < MT; ++m) va[m] = vb[m];
#pragma unroll
    for (int n = 0; n < NT; ++n) xa[n] = xb[n];
  }
  double2 *out = part + gw * (int64_t)k * s;
#pragma unroll
  for (int m = 0; m < MT; ++m) {
    const int i = i0 + m * 8 + r;
#pragma unroll
    for (int n = 0; n < NT; ++n)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = n * 8 + 2 * c + h;
        if (i < k && j < s) out[(int64_t)i * s + j] = make_double2(cre[m][n][h], cim[m][n][h]);
      }
  }
}

// The same DMMA contraction fed by an asynchronous bulk-copy pipeline (the
// Blackwell idiom for a streaming operand: cp.async.bulk global -> shared
// completing on an mbarrier, consumers released by a second mbarrier), for
// lengths that are a multiple of the 32-element stage tile.  One CTA per SM:
// a producer warp keeps kVhxStages tiles of (64 vectors + s columns) x 32
// elements in flight (up to 184 KB of loads per SM, no registers held by
// them), 8 consumer warps each own one 4-element k-step of every tile and
// all 64 x s outputs of it.  Rows are padded to 576 B (= 64 mod 128) so the
// 16-byte fragment reads of a quarter warp (2 rows x 64 B) hit 32 distinct
// banks.  s <= 8: HBM-bound (36 B/clk/SM of operands against 4 cycles per
// DMMA); s = 16: FP64-pipe-bound.
constexpr int kVhxTE = 32;                       // elements per stage tile
constexpr int kVhxRow = kVhxTE * 16 + 64;        // padded row stride in bytes
constexpr int kVhxStages = 4;

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

template <int MT, int NT, bool BULK>
__global__ void __launch_bounds__(288, 1) vhx_bulk_kernel(const double2 *__restrict__ V, const double2 *__restrict__ X,
                                                          int64_t len, int k, int s, double2 *__restrict__ part) {
  constexpr int ROWS = 8 * MT + 8 * NT, STAGE = ROWS * kVhxRow;
  extern __shared__ __align__(128) unsigned char vsm[];
  __shared__ __align__(8) unsigned long long bars[2 * kVhxStages];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i0 = blockIdx.y * (8 * MT);
  const int nrow = min(8 * MT, k - i0);
  const int64_t ntiles = len / kVhxTE;
  const int64_t mine = blockIdx.x < ntiles ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  if (threadIdx.x == 0) {
    for (int st = 0; st < kVhxStages; ++st) {
      mbar_init(smem_u32(&bars[st]), BULK ? 1 : 32);   // full: the expect_tx arrival / one per producer lane
      mbar_init(smem_u32(&bars[kVhxStages + st]), 8);  // empty: one arrival per consumer warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 8) {
    // ---- producer warp ----
    if (BULK) {
      // one 512-byte bulk copy per (row, tile), completing on the stage's
      // transaction count
      const uint32_t tx = (uint32_t)(nrow + s) * kVhxTE * 16;
      for (int64_t it = 0; it < mine; ++it) {
        const int st = (int)(it % kVhxStages);
        const uint32_t full = smem_u32(&bars[st]), empty = smem_u32(&bars[kVhxStages + st]);
        if (it >= kVhxStages) mbar_wait(empty, (uint32_t)((it / kVhxStages - 1) & 1));
        if (lane == 0) mbar_expect_tx(full, tx);
        __syncwarp();
        const int64_t e0 = (blockIdx.x + it * gridDim.x) * kVhxTE;
        const uint32_t base = smem_u32(vsm) + st * STAGE;
        for (int row = lane; row < ROWS; row += 32) {
          if (row < 8 * MT) {
            if (row < nrow) bulk_g2s(base + row * kVhxRow, V + (int64_t)(i0 + row) * len + e0, kVhxTE * 16, full);
          } else if (row - 8 * MT < s) {
            bulk_g2s(base + row * kVhxRow, X + (int64_t)(row - 8 * MT) * len + e0, kVhxTE * 16, full);
          }
        }
      }
    } else {
      // 16-byte cp.async per lane: one instruction moves a row's 512-byte
      // tile slice; each lane's arrival on the stage barrier fires when its
      // copies have landed
      for (int64_t it = 0; it < mine; ++it) {
        const int st = (int)(it % kVhxStages);
        const uint32_t full = smem_u32(&bars[st]), empty = smem_u32(&bars[kVhxStages + st]);
        if (it >= kVhxStages) mbar_wait(empty, (uint32_t)((it / kVhxStages - 1) & 1));
        const int64_t e0 = (blockIdx.x + it * gridDim.x) * kVhxTE + lane;
        const uint32_t dst = smem_u32(vsm) + st * STAGE + lane * 16;
#pragma unroll 8
        for (int row = 0; row < nrow; ++row)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + row * kVhxRow),
                       "l"(V + (int64_t)(i0 + row) * len + e0)
                       : "memory");
        for (int j = 0; j < s; ++j)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + (8 * MT + j) * kVhxRow),
                       "l"(X + (int64_t)j * len + e0)
                       : "memory");
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(full) : "memory");
      }
    }
    return;
  }
  // ---- consumer warps: warp w owns elements 4w .. 4w + 3 of every tile ----
  const int r = lane >> 2, c = lane & 3;
  double cre[MT][NT][2], cim[MT][NT][2];
#pragma unroll
  for (int m = 0; m < MT; ++m)
#pragma unroll
    for (int n = 0; n < NT; ++n) cre[m][n][0] = cre[m][n][1] = cim[m][n][0] = cim[m][n][1] = 0.0;
  const int eoff = (4 * warp + c) * 16;
#pragma unroll 1
  for (int64_t it = 0; it < mine; ++it) {
    const int st = (int)(it % kVhxStages);
    mbar_wait(smem_u32(&bars[st]), (uint32_t)((it / kVhxStages) & 1));
    const unsigned char *base = vsm + st * STAGE + eoff;
    double2 xa[NT], va[MT];
#pragma unroll
    for (int n = 0; n < NT; ++n) xa[n] = *reinterpret_cast<const double2 *>(base + (8 * MT + n * 8 + r) * kVhxRow);
#pragma unroll
    for (int m = 0; m < MT; ++m) va[m] = *reinterpret_cast<const double2 *>(base + (m * 8 + r) * kVhxRow);
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      const double nx = -xa[n].x;
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        dmma884(cre[m][n][0], cre[m][n][1], va[m].x, xa[n].x);
        dmma884(cim[m][n][0], cim[m][n][1], va[m].x, xa[n].y);
      }
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        dmma884(cre[m][n][0], cre[m][n][1], va[m].y, xa[n].y);
        dmma884(cim[m][n][0], cim[m][n][1], va[m].y, nx);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(smem_u32(&bars[kVhxStages + st]));
  }
  double2 *out = part + ((int64_t)blockIdx.x * 8 + warp) * (int64_t)k * s;
#pragma unroll
  for (int m = 0; m < MT; ++m) {
    const int i = i0 + m * 8 + r;
#pragma unroll
    for (int n = 0; n < NT; ++n)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = n * 8 + 2 * c + h;
        if (i < k && j < s) out[(int64_t)i * s + j] = make_double2(cre[m][n][h], cim[m][n][h]);
      }
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

// X <- X - V H for 4 < s <= 16 on the FP64 tensor cores with the same
// cp.async + mbarrier pipeline: C[m = element][n = column] += A[m][k = vector]
// B[k][n], A[e][i] = V_i[e], B[i][j] = H[i][j] (from shared memory).  A CTA
// walks tiles of 256 elements; for each it streams the k vectors in stages of
// 8 rows x 256 elements (33 KB, kVhxStages in flight); consumer warp w owns
// elements 32 w .. 32 w + 31 of the tile (four 8-element MMA row tiles x all s
// columns) and, after the last vector, subtracts its accumulators from X.
// Rows are padded to 4,128 B (= 32 mod 128): a quarter warp's fragment read
// (4 vectors x 2 consecutive elements) is conflict-free; H rows to s*16 + 32.
// The i-sum of every element runs in vector order whatever the grid, so the
// result is deterministic.  Absent vectors of the last stage are zero-filled
// (cp.async src-size 0).
constexpr int kSubTE = 256, kSubKI = 8;
constexpr int kSubRow = kSubTE * 16 + 32;
constexpr int kSubStage = kSubKI * kSubRow;

template <int NT>
__global__ void __launch_bounds__(288, 1) proj_sub_pipe_kernel(const double2 *__restrict__ V,
                                                               const double2 *__restrict__ H,
                                                               double2 *__restrict__ X, int64_t len, int k, int s) {
  constexpr int HROW = NT * 128 + 32;  // bytes per H row (8 NT columns + pad)
  extern __shared__ __align__(128) unsigned char psm[];
  __shared__ __align__(8) unsigned long long bars[2 * kVhxStages];
  unsigned char *hs = psm + kVhxStages * kSubStage;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nst = (k + kSubKI - 1) / kSubKI;  // vector stages per tile
  const int64_t ntiles = len / kSubTE;
  const int64_t mine = blockIdx.x < ntiles ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const int64_t total = mine * nst;
  // H -> shared, zero-padded to 8 nst rows x 8 NT columns
  for (int q = threadIdx.x; q < nst * kSubKI * 8 * NT; q += blockDim.x) {
    const int i = q / (8 * NT), j = q % (8 * NT);
    *reinterpret_cast<double2 *>(hs + i * HROW + j * 16) =
        (i < k && j < s) ? H[(int64_t)j * k + i] : make_double2(0.0, 0.0);
  }
  if (threadIdx.x == 0) {
    for (int st = 0; st < kVhxStages; ++st) {
      mbar_init(smem_u32(&bars[st]), 32);
      mbar_init(smem_u32(&bars[kVhxStages + st]), 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 8) {
    for (int64_t it = 0; it < total; ++it) {
      const int st = (int)(it % kVhxStages);
      const uint32_t full = smem_u32(&bars[st]), empty = smem_u32(&bars[kVhxStages + st]);
      if (it >= kVhxStages) mbar_wait(empty, (uint32_t)((it / kVhxStages - 1) & 1));
      const int64_t tile = blockIdx.x + (it / nst) * gridDim.x;
      const int ib = (int)(it % nst) * kSubKI;
      const uint32_t dst = smem_u32(psm) + st * kSubStage + lane * 16;
      const int64_t e0 = tile * kSubTE + lane;
#pragma unroll
      for (int row = 0; row < kSubKI; ++row) {
        const bool ok = ib + row < k;
        const double2 *src = V + (int64_t)(ok ? ib + row : 0) * len + e0;
        const uint32_t sz = ok ? 16u : 0u;
#pragma unroll
        for (int ch = 0; ch < kSubTE / 32; ++ch)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst + row * kSubRow + ch * 512),
                       "l"(src + ch * 32), "r"(sz)
                       : "memory");
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(full) : "memory");
    }
    return;
  }
  const int r = lane >> 2, c = lane & 3;
  int64_t it = 0;
#pragma unroll 1
  for (int64_t tl = 0; tl < mine; ++tl) {
    double cre[4][NT][2], cim[4][NT][2];
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
      for (int n = 0; n < NT; ++n) cre[t][n][0] = cre[t][n][1] = cim[t][n][0] = cim[t][n][1] = 0.0;
#pragma unroll 1
    for (int is = 0; is < nst; ++is, ++it) {
      const int st = (int)(it % kVhxStages);
      mbar_wait(smem_u32(&bars[st]), (uint32_t)((it / kVhxStages) & 1));
      const unsigned char *base = psm + st * kSubStage + (32 * warp + r) * 16;
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        double2 hb[NT], va[4];
#pragma unroll
        for (int n = 0; n < NT; ++n)
          hb[n] = *reinterpret_cast<const double2 *>(hs + (is * kSubKI + half * 4 + c) * HROW + (n * 8 + r) * 16);
#pragma unroll
        for (int t = 0; t < 4; ++t)
          va[t] = *reinterpret_cast<const double2 *>(base + (half * 4 + c) * kSubRow + t * 128);
#pragma unroll
        for (int n = 0; n < NT; ++n) {
          const double nhi = -hb[n].y;
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            dmma884(cre[t][n][0], cre[t][n][1], va[t].x, hb[n].x);
            dmma884(cim[t][n][0], cim[t][n][1], va[t].x, hb[n].y);
          }
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            dmma884(cre[t][n][0], cre[t][n][1], va[t].y, nhi);
            dmma884(cim[t][n][0], cim[t][n][1], va[t].y, hb[n].x);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&bars[kVhxStages + st]));
    }
    // X_j[e] -= acc: lane holds rows e = e0 + 8 t + r, columns 8 n + 2 c + {0, 1}
    const int64_t e0 = (blockIdx.x + tl * gridDim.x) * kSubTE + 32 * warp + r;
#pragma unroll
    for (int n = 0; n < NT; ++n)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = n * 8 + 2 * c + h;
        if (j < s) {
          double2 *xp = X + (int64_t)j * len + e0;
          double2 xv[4];
#pragma unroll
          for (int t = 0; t < 4; ++t) xv[t] = xp[8 * t];
#pragma unroll
          for (int t = 0; t < 4; ++t) xp[8 * t] = make_double2(xv[t].x - cre[t][n][h], xv[t].y - cim[t][n][h]);
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
  // 4 < s <= 16 against more than 8 vectors: the FP64 tensor-core kernel
  // (32-byte loads: even length, 32-byte aligned fields)
  static const bool dmma_on = [] {
    const char *e = getenv("MGT_VHX_DMMA");
    return !e || atoi(e) != 0;
  }();
  // MGT_VHX_BULK: 0 = register-fed DMMA kernel, 1 = shared-memory pipeline fed
  // by cp.async (default), 2 = fed by cp.async.bulk row copies
  static const int bulk_mode = [] {
    const char *e = getenv("MGT_VHX_BULK");
    return e ? atoi(e) : 1;
  }();
  const bool bulk_on = bulk_mode != 0;
  const bool dmma_shape = dmma_on && s > 4 && s <= 16 && k > 8;
  // bulk-copy pipeline: whole 32-element tiles (16-byte alignment is a double2's)
  const bool bulk = dmma_shape && bulk_on && len % kVhxTE == 0 && len >= kVhxTE;
  // register-fed variant: 32-byte loads need an even length and 32-byte aligned fields
  const bool dmma = dmma_shape && !bulk && len % 2 == 0 && ((uintptr_t)V_dev % 32) == 0 && ((uintptr_t)X_dev % 32) == 0;
  if (!dmma && !bulk && (s <= 8 || swapped)) {
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
  } else if (bulk) {
    // shared-memory pipeline: one 288-thread CTA per SM owning 8 * MT vectors
    // (k split evenly over the fewest blocks of at most 80 vectors, so no
    // block multiplies mostly-absent rows); partials per consumer warp
    const int nt = s <= 8 ? 1 : 2;
    const int cap = nt == 1 ? 80 : 72;  // vectors per CTA (accumulator registers)
    const int gy = (k + cap - 1) / cap;
    const int mt = ((k + gy - 1) / gy + 7) / 8;  // 2 .. 10
    const size_t smem = (size_t)kVhxStages * (8 * mt + 8 * nt) * kVhxRow;
    const int nb = (int)std::max<int64_t>(1, std::min<int64_t>(len / kVhxTE, std::max(1, num_sms() / gy)));
    nblk = nb * 8;
    MGT_CUDA(scratch_alloc((void **)&part, (size_t)nblk * k * s * sizeof(double2), st));
    dim3 grid(nb, gy);
#define MGT_VHX_PIPE(MTV, NTV, BK)                                                                                  \
  do {                                                                                                               \
    MGT_CUDA(cudaFuncSetAttribute(vhx_bulk_kernel<MTV, NTV, BK>, cudaFuncAttributeMaxDynamicSharedMemorySize,      \
                                  (int)smem));                                                                       \
    vhx_bulk_kernel<MTV, NTV, BK><<<grid, 288, smem, st>>>(V, X, len, k, s, part);                                  \
  } while (0)
#define MGT_VHX_PIPE_NT(MTV)                  \
  do {                                        \
    if (nt == 1 && bulk_mode == 2)            \
      MGT_VHX_PIPE(MTV, 1, true);             \
    else if (nt == 1)                         \
      MGT_VHX_PIPE(MTV, 1, false);            \
    else if (bulk_mode == 2)                  \
      MGT_VHX_PIPE(MTV, 2, true);             \
    else                                      \
      MGT_VHX_PIPE(MTV, 2, false);            \
  } while (0)
    switch (mt) {
      case 2: MGT_VHX_PIPE_NT(2); break;
      case 3: MGT_VHX_PIPE_NT(3); break;
      case 4: MGT_VHX_PIPE_NT(4); break;
      case 5: MGT_VHX_PIPE_NT(5); break;
      case 6: MGT_VHX_PIPE_NT(6); break;
      case 7: MGT_VHX_PIPE_NT(7); break;
      case 8: MGT_VHX_PIPE_NT(8); break;
      case 9: MGT_VHX_PIPE_NT(9); break;
      default: MGT_VHX_PIPE_NT(10); break;
    }
#undef MGT_VHX_PIPE_NT
#undef MGT_VHX_PIPE
    MGT_LAUNCH_CHECK("vhx_bulk_kernel");
  } else if (dmma) {
    // a warp per (e-range, 64 vectors): one wave of 2 x 128-thread blocks per SM
    const int gy = (k + 63) / 64;
    const int per_sm = s <= 8 ? blocks_per_sm((const void *)vhx_dmma_kernel<1>, 128)
                              : blocks_per_sm((const void *)vhx_dmma_kernel<2>, 128);
    if (per_sm < 1) return per_sm < 0 ? MGT_ERR_CUDA : fail(MGT_ERR_CUDA, "vhx_dmma_kernel cannot be resident");
    const int nb = (int)std::max<int64_t>(1, std::min<int64_t>((len + 31) / 32, std::max(1, num_sms() * per_sm / gy)));
    nblk = nb * 4;  // partials per warp
    MGT_CUDA(scratch_alloc((void **)&part, (size_t)nblk * k * s * sizeof(double2), st));
    dim3 grid(nb, gy);
    if (s <= 8)
      vhx_dmma_kernel<1><<<grid, 128, 0, st>>>(V, X, len, k, s, part);
    else
      vhx_dmma_kernel<2><<<grid, 128, 0, st>>>(V, X, len, k, s, part);
    MGT_LAUNCH_CHECK("vhx_dmma_kernel");
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
  // 4 < s <= 16, whole 256-element tiles (at least two per SM) and H in
  // shared memory next to the stages: the FP64 tensor-core pipeline
  {
    static const bool pipe_on = [] {
      const char *e = getenv("MGT_SUB_PIPE");
      return !e || atoi(e) != 0;
    }();
    const int nt = s <= 8 ? 1 : 2;
    const int nst = (k + kSubKI - 1) / kSubKI;
    const size_t smem_p = (size_t)kVhxStages * kSubStage + (size_t)nst * kSubKI * (nt * 128 + 32);
    if (pipe_on && s > 4 && s <= 16 && k > 8 && len % kSubTE == 0 && len / kSubTE >= 2 * (int64_t)num_sms() &&
        smem_p <= 220 * 1024) {
      const int nb = (int)std::min<int64_t>(len / kSubTE, num_sms());
      if (nt == 1) {
        MGT_CUDA(cudaFuncSetAttribute(proj_sub_pipe_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_p));
        proj_sub_pipe_kernel<1><<<nb, 288, smem_p, st>>>((const double2 *)V_dev, (const double2 *)H_dev,
                                                         (double2 *)X_dev, len, k, s);
      } else {
        MGT_CUDA(cudaFuncSetAttribute(proj_sub_pipe_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_p));
        proj_sub_pipe_kernel<2><<<nb, 288, smem_p, st>>>((const double2 *)V_dev, (const double2 *)H_dev,
                                                         (double2 *)X_dev, len, k, s);
      }
      MGT_LAUNCH_CHECK("proj_sub_pipe_kernel");
      return MGT_OK;
    }
  }
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
