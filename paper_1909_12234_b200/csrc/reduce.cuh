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
  __device__ __forceinline__ int64_t first() const { return blockIdx.x * (int64_t)SPB + local; }
  __device__ __forceinline__ int64_t stride() const { return (int64_t)gridDim.x * SPB; }
};

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
