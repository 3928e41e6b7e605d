// Deterministic fixed-order reductions fused into streaming kernels.
//
// Each kernel runs a fixed grid (grid-stride loops), so the assignment of
// sites to threads, the in-thread summation order, the warp-shuffle trees
// and the final cross-block sum are all fixed: results are bitwise
// reproducible run to run (the reference promises byte-identical reruns,
// trace.py:95-97).  The last block to finish (atomic ticket)
// sums the per-block partials and runs a scalar "finisher" callback, so a
// reduction costs no extra launch.
#pragma once
#include "common.cuh"

namespace mgt {

constexpr int kRedBlock = 128;  // threads per block in reducing kernels
constexpr int kRedWarps = kRedBlock / 32;

// Multi-rhs kernels map warp w of a block to rhs w % NR (see RhsMap), so a
// warp's threads all belong to one rhs.  Sum `v[NV]` over each warp, combine
// the warps of the same rhs in fixed order and publish NR*NV partials for
// this block.  Returns true in every thread of the LAST block to arrive,
// after which `partials` holds all blocks' values.
template <int NR, int NV>
__device__ __forceinline__ bool reduce_publish(double (&v)[NV], double *partials, unsigned *ticket) {
  __shared__ double sm[kRedWarps][NV];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double x = v[k];
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
    v[k] = x;
  }
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) sm[warp][k] = v[k];
  }
  __syncthreads();
  if (threadIdx.x < NR * NV) {
    const int r = threadIdx.x / NV, k = threadIdx.x % NV;
    double s = 0.0;
#pragma unroll
    for (int w = r; w < kRedWarps; w += NR) s += sm[w][k];
    partials[(size_t)blockIdx.x * NR * NV + threadIdx.x] = s;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned t = atomicAdd(ticket, 1u);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  return last;
}

// Per-chunk variant for dynamically scheduled kernels (next_chunk): the
// block reduces its chunk's values and writes them to dst[NR*NV] (the
// chunk's own slot), so the final sum over chunks in chunk order does not
// depend on which block processed which chunk.  All threads must call it.
template <int NR, int NV>
__device__ __forceinline__ void chunk_publish(const double (&v)[NV], double *dst) {
  __shared__ double sm[kRedWarps][NV];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double x = v[k];
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
    if (lane == 0) sm[warp][k] = x;
  }
  __syncthreads();
  if (threadIdx.x < NR * NV) {
    const int r = threadIdx.x / NV, k = threadIdx.x % NV;
    double s = 0.0;
#pragma unroll
    for (int w = r; w < kRedWarps; w += NR) s += sm[w][k];
    dst[threadIdx.x] = s;
  }
  __syncthreads();
}

// Arrival ticket: true in every thread of the last block to arrive.
__device__ __forceinline__ bool last_block(unsigned *ticket) {
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = (atomicAdd(ticket, 1u) == gridDim.x - 1);
  __syncthreads();
  return last;
}

// In the last block: out[j] = sum_c partials[c*M + j] over n chunks (fixed order).
template <int M>
__device__ __forceinline__ void reduce_finish_n(const double *partials, int64_t n, unsigned *ticket, double (&out)[M]) {
  __shared__ double res[M > 0 ? M : 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int j = warp; j < M; j += kRedWarps) {
    double s = 0.0;
    for (int64_t b = lane; b < n; b += 32) s += __ldcg(partials + (size_t)b * M + j);
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) res[j] = s;
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < M; ++j) out[j] = res[j];
  if (threadIdx.x == 0) *ticket = 0u;
}

// Thread -> (rhs, ordered site) map of the multi-rhs kernels: each block
// iteration covers SPB = 128 / NR consecutive ordered sites; warp w serves
// rhs w % NR on 32 of them.  Every load instruction streams one field.
template <int NR>
struct RhsMap {
  static constexpr int SPB = kRedBlock / NR;
  int rhs, local;
  __device__ __forceinline__ RhsMap() {
    const int w = threadIdx.x >> 5;
    rhs = w % NR;
    local = (w / NR) * 32 + (threadIdx.x & 31);
  }
  // tile (32 consecutive ordered sites) of ordered site o of this thread
  __device__ __forceinline__ static int64_t tile(int64_t o) { return o >> 5; }
  __device__ __forceinline__ int64_t first() const { return blockIdx.x * (int64_t)SPB + local; }
  __device__ __forceinline__ int64_t stride() const { return (int64_t)gridDim.x * SPB; }
};

// ---------------------------------------------------------------------------
// Tile-ordered reductions (the solver kernels, bicgstab.cu).  A sum over
// ordered sites is defined by the site index alone, so a right-hand side's
// reductions -- and with them its whole BiCGStab iterate sequence -- do not
// depend on how many rhs share a launch (NR), on the number of batched
// groups, or on the grid size:
//   1. tile  = 32 consecutive ordered sites: xor-shuffle tree over the warp
//              serving them (lane = site in the tile), stored by lane 0;
//   2. final = lane l sums tiles l, l + 32, l + 64, ... in order, then an
//              xor tree over the lanes (the kernel's last block).
// Tile partials are laid out [tile][rhs][value] (M = NR * NV doubles per
// tile); the order of the sum of one (rhs, value) is the same for every NR.
// (Folding 32-tile supers inside the kernel by the last-arriving warp needs
// a fence and an atomic round trip per tile: measured 3-8 % slower per
// solver iteration.)
struct TileRed {
  double *tiles;  // [ntiles][M]
};

__host__ __device__ __forceinline__ int64_t n_tiles(int64_t sites) { return (sites + 31) / 32; }

// Publish this warp's tile partial v[NV] (rhs r of NR; `tile` warp-uniform;
// every lane must call it).
template <int NR, int NV>
__device__ __forceinline__ void tile_publish(double (&v)[NV], const TileRed &T, int64_t tile, int64_t ntiles, int r) {
  constexpr int M = NR * NV;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double x = v[k];
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
    v[k] = x;
  }
  if ((threadIdx.x & 31) == 0 && tile < ntiles) {
#pragma unroll
    for (int k = 0; k < NV; ++k) T.tiles[tile * M + r * NV + k] = v[k];
  }
}

// Variant for kernels that stream two adjacent sites per thread (16-byte
// fp32 accesses): lanes 0-15 hold tile A, lanes 16-31 tile B (`tile` per
// lane); the tile tree is over the 16 lanes of a half-warp.  Each such
// kernel uses this shape for every NR, so its sums stay batch-invariant.
template <int NR, int NV>
__device__ __forceinline__ void tile_publish_pairs(double (&v)[NV], const TileRed &T, int64_t tile, int64_t ntiles,
                                                   int r) {
  constexpr int M = NR * NV;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double x = v[k];
#pragma unroll
    for (int off = 8; off >= 1; off >>= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
    v[k] = x;
  }
  if ((threadIdx.x & 15) == 0 && tile < ntiles) {
#pragma unroll
    for (int k = 0; k < NV; ++k) T.tiles[tile * M + r * NV + k] = v[k];
  }
}

// In the last block (after last_block()): out[j] = the ordered sum above for
// j < M, then reset the ticket.  Warp w takes values w, w + 4, ...; each
// lane keeps 8 tile loads in flight and adds them in tile order.  Result
// visible to the whole block.
template <int M>
__device__ __forceinline__ void tiles_final(const TileRed &T, int64_t sites, unsigned *ticket, double (&out)[M]) {
  __shared__ double res[M > 0 ? M : 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nt = n_tiles(sites);
  for (int j = warp; j < M; j += kRedWarps) {
    double s = 0.0;
    int64_t b = lane;
    for (; b + 7 * 32 < nt; b += 8 * 32) {
      double x[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) x[u] = __ldcg(T.tiles + (b + u * 32) * M + j);
#pragma unroll
      for (int u = 0; u < 8; ++u) s += x[u];
    }
    for (; b < nt; b += 32) s += __ldcg(T.tiles + b * M + j);
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) res[j] = s;
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < M; ++j) out[j] = res[j];
  if (threadIdx.x == 0) *ticket = 0u;
}

// In the last block: out[j] = sum_b partials[b*M + j] for j < M (fixed
// order), then reset the ticket.  Result visible to the whole block.
template <int M>
__device__ __forceinline__ void reduce_finish(const double *partials, unsigned *ticket, double (&out)[M]) {
  __shared__ double res[M > 0 ? M : 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nb = gridDim.x;
  for (int j = warp; j < M; j += kRedWarps) {
    double s = 0.0;
    for (int b = lane; b < nb; b += 32) s += __ldcg(partials + (size_t)b * M + j);
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) res[j] = s;
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < M; ++j) out[j] = res[j];
  if (threadIdx.x == 0) *ticket = 0u;
}

}  // namespace mgt
