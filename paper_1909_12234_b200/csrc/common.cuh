// Shared helpers for the mgtrace-b200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "../../include/mgtrace_b200.h"

namespace mgt {

// ---- error plumbing (thread-local message, int codes across the ABI) -----
void set_error(const std::string &msg);
int fail(int code, const std::string &msg);
int cuda_fail(cudaError_t e, const char *what);
void note_launch(uint64_t n = 1);

#define MGT_CUDA(call)                                  \
  do {                                                  \
    cudaError_t _e = (call);                            \
    if (_e != cudaSuccess) return ::mgt::cuda_fail(_e, #call); \
  } while (0)

#define MGT_LAUNCH_CHECK(what)                          \
  do {                                                  \
    ::mgt::note_launch();                               \
    cudaError_t _e = cudaGetLastError();                \
    if (_e != cudaSuccess) return ::mgt::cuda_fail(_e, what); \
  } while (0)

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// Stream-ordered scratch allocation from the device's default memory pool,
// with the pool's release threshold raised once so freed scratch stays
// cached instead of being unmapped at every synchronisation.
cudaError_t scratch_alloc(void **p, size_t bytes, cudaStream_t st);

// SM count of the current device (cudaDevAttrMultiProcessorCount), queried
// once per device: grids sized in multiples of it follow the device (148 on
// a B200, fewer on a MIG slice) instead of a hard-coded constant.
int num_sms();
// Resident blocks per SM of `kernel` at (block, dynamic smem) from the
// occupancy calculator, cached per (device, kernel, block, smem); -1 if the
// query fails (the error message is recorded).
int blocks_per_sm(const void *kernel, int block, size_t smem = 0);

// ---- complex arithmetic on double2 / float2 ------------------------------
template <typename R> struct cplx_t;
template <> struct cplx_t<double> { using type = double2; };
template <> struct cplx_t<float> { using type = float2; };
template <typename R> using cplx = typename cplx_t<R>::type;

template <typename R> struct C {
  R re, im;
  __host__ __device__ C() = default;
  __host__ __device__ constexpr C(R r, R i) : re(r), im(i) {}
};

template <typename R> __device__ __forceinline__ C<R> operator+(C<R> a, C<R> b) { return {a.re + b.re, a.im + b.im}; }
template <typename R> __device__ __forceinline__ C<R> operator-(C<R> a, C<R> b) { return {a.re - b.re, a.im - b.im}; }
template <typename R> __device__ __forceinline__ C<R> operator-(C<R> a) { return {-a.re, -a.im}; }
template <typename R> __device__ __forceinline__ C<R> operator*(C<R> a, C<R> b) {
  return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
}
template <typename R> __device__ __forceinline__ C<R> operator*(R s, C<R> a) { return {s * a.re, s * a.im}; }
template <typename R> __device__ __forceinline__ C<R> conj(C<R> a) { return {a.re, -a.im}; }
// i * a
template <typename R> __device__ __forceinline__ C<R> times_i(C<R> a) { return {-a.im, a.re}; }
// conj(a) * b
template <typename R> __device__ __forceinline__ C<R> cmul_conj(C<R> a, C<R> b) {
  return {a.re * b.re + a.im * b.im, a.re * b.im - a.im * b.re};
}
// acc + a*b
template <typename R> __device__ __forceinline__ C<R> cfma(C<R> a, C<R> b, C<R> acc) {
  acc.re = fma(a.re, b.re, acc.re);
  acc.re = fma(-a.im, b.im, acc.re);
  acc.im = fma(a.re, b.im, acc.im);
  acc.im = fma(a.im, b.re, acc.im);
  return acc;
}
// acc + conj(a)*b
template <typename R> __device__ __forceinline__ C<R> cfma_conj(C<R> a, C<R> b, C<R> acc) {
  acc.re = fma(a.re, b.re, acc.re);
  acc.re = fma(a.im, b.im, acc.re);
  acc.im = fma(a.re, b.im, acc.im);
  acc.im = fma(-a.im, b.re, acc.im);
  return acc;
}

// streaming 128-bit / 64-bit loads through the read-only path
__device__ __forceinline__ C<double> ldc(const double2 *p) {
  double2 v = __ldg(p);
  return {v.x, v.y};
}
__device__ __forceinline__ C<float> ldc(const float2 *p) {
  float2 v = __ldg(p);
  return {v.x, v.y};
}
// L2-only (L1-bypassing) loads
__device__ __forceinline__ C<double> ldc_cg(const double2 *p) {
  double2 v = __ldcg(p);
  return {v.x, v.y};
}
__device__ __forceinline__ C<float> ldc_cg(const float2 *p) {
  float2 v = __ldcg(p);
  return {v.x, v.y};
}
__device__ __forceinline__ void stc(double2 *p, C<double> v) { *p = make_double2(v.re, v.im); }
__device__ __forceinline__ void stc(float2 *p, C<float> v) { *p = make_float2(v.re, v.im); }
// streaming store (evict-first): output fields are not re-read by this kernel
__device__ __forceinline__ void stc_cs(double2 *p, C<double> v) { __stcs(p, make_double2(v.re, v.im)); }
__device__ __forceinline__ void stc_cs(float2 *p, C<float> v) { __stcs(p, make_float2(v.re, v.im)); }

// ---- constant-divisor division ---------------------------------------------
// n / d for 0 <= n < 2^31 as a multiply-high, add and shift (Granlund-
// Montgomery round-up method; exhaustively spot-checked over divisors
// 1..2^26 and every power of two +-1).  The site -> coordinate decodes run
// per site in every stencil kernel; the compiler's generic 32/64-bit
// division sequence (I2F + MUFU.RCP + Newton steps, a slow-path CALL for
// 64-bit operands) is ~5x longer and sits on the latency chain in front of
// the site's first load.
struct FastDiv {
  uint32_t d, m, l;
};
inline FastDiv make_fastdiv(uint32_t d) {
  FastDiv f;
  f.d = d;
  f.l = 0;
  while ((1ull << f.l) < d) ++f.l;
  f.m = (uint32_t)((((1ull << 32) * ((1ull << f.l) - d)) / d) + 1);
  return f;
}
__host__ __device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv &f) {
#ifdef __CUDA_ARCH__
  return (__umulhi(n, f.m) + n) >> f.l;
#else
  return (uint32_t)((((uint64_t)n * f.m >> 32) + n) >> f.l);
#endif
}

// ---- lattice geometry -----------------------------------------------------
// dims in reference order (L0, L1, L2, L3 = t).  Native site order:
//   s = ((x3*L0 + x0)*L1 + x1)*L2 + x2   (x2 fastest, t slowest)
// Every handle keeps V < 2^31 (mgt_wilson_create), so site indices decode in
// 32-bit arithmetic.
struct Geom {
  int L[4];
  int64_t V;
  // native strides for directions mu = 0..3
  int64_t stride[4];
  FastDiv fd[3];  // by L[0], L[1], L[2]
};

inline Geom make_geom(const int dims[4]) {
  Geom g;
  for (int i = 0; i < 4; ++i) g.L[i] = dims[i];
  g.V = (int64_t)dims[0] * dims[1] * dims[2] * dims[3];
  g.stride[2] = 1;
  g.stride[1] = dims[2];
  g.stride[0] = (int64_t)dims[1] * dims[2];
  g.stride[3] = (int64_t)dims[0] * dims[1] * dims[2];
  for (int i = 0; i < 3; ++i) g.fd[i] = make_fastdiv((uint32_t)dims[i]);
  return g;
}

// native site -> coords (x0..x3)
__host__ __device__ __forceinline__ void native_coords(const Geom &g, int64_t s, int x[4]) {
  uint32_t r = (uint32_t)s;
  uint32_t q = fdiv(r, g.fd[2]);
  x[2] = (int)(r - q * (uint32_t)g.L[2]);
  r = q;
  q = fdiv(r, g.fd[1]);
  x[1] = (int)(r - q * (uint32_t)g.L[1]);
  r = q;
  q = fdiv(r, g.fd[0]);
  x[0] = (int)(r - q * (uint32_t)g.L[0]);
  x[3] = (int)q;
}

__host__ __device__ __forceinline__ int64_t ref_site(const Geom &g, const int x[4]) {
  return (((int64_t)x[0] * g.L[1] + x[1]) * g.L[2] + x[2]) * g.L[3] + x[3];
}

__host__ __device__ __forceinline__ int64_t native_site(const Geom &g, const int x[4]) {
  return (((int64_t)x[3] * g.L[0] + x[0]) * g.L[1] + x[1]) * g.L[2] + x[2];
}

// L2-friendly traversal order.  Blocks walk the lattice slab by slab
// (slabs of w consecutive x0 planes), and inside a slab t-plane by t-plane,
// so the largest neighbour reuse distance is the slab's t-stride
// (w*L1*L2 sites, chosen to fit comfortably in L2) instead of the full
// spatial volume L0*L1*L2.  Ordered index o -> native site.
struct Sched {
  int64_t slab_sites;  // w * L1 * L2
  int64_t plane;       // L0 * L1 * L2 (native t stride)
  int L3;
  FastDiv f_slab, f_L3;
};

inline Sched make_sched(const Geom &g, int64_t bytes_per_site, int64_t budget = (int64_t)24 << 20) {
  const int64_t row = (int64_t)g.L[1] * g.L[2];
  int w = 1;
  for (int d = 1; d <= g.L[0]; ++d)
    if (g.L[0] % d == 0 && d * row * bytes_per_site <= budget) w = d;
  Sched s;
  s.slab_sites = w * row;
  s.plane = (int64_t)g.L[0] * row;
  s.L3 = g.L[3];
  s.f_slab = make_fastdiv((uint32_t)s.slab_sites);
  s.f_L3 = make_fastdiv((uint32_t)s.L3);
  return s;
}

__host__ __device__ __forceinline__ int64_t sched_site(const Sched &s, int64_t o) {
  const uint32_t ou = (uint32_t)o;
  const uint32_t q = fdiv(ou, s.f_slab);
  const uint32_t r = ou - q * (uint32_t)s.slab_sites;
  const uint32_t k = fdiv(q, s.f_L3);
  const uint32_t t = q - k * (uint32_t)s.L3;
  return (int64_t)t * s.plane + (int64_t)k * s.slab_sites + r;
}

// Dynamic in-order chunk scheduler for persistent grids: CTAs take
// consecutive chunks from a global counter, so the chunks in flight always
// form one contiguous window of the schedule (a static grid-stride split
// lets CTAs drift apart over hundreds of steps and the neighbour reuse
// window no longer fits in L2).  Every thread of the block must call it.
__device__ __forceinline__ int64_t next_chunk(unsigned long long *ctr) {
  __shared__ long long c;
  __syncthreads();
  if (threadIdx.x == 0) c = (long long)atomicAdd(ctr, 1ull);
  __syncthreads();
  return c;
}

// Resident-grid size for a kernel (blocks per SM from the occupancy
// calculator): grid-stride loops then march one contiguous window through the
// schedule instead of scattering a block's iterations across the lattice.
template <typename K>
inline int resident_grid(K kernel, int block, int64_t work_items) {
  int per_sm = blocks_per_sm(reinterpret_cast<const void *>(kernel), block, 0);
  if (per_sm < 1) per_sm = 1;  // a kernel that cannot launch fails at its launch check
  int64_t need = (work_items + block - 1) / block;
  int64_t g = (int64_t)num_sms() * per_sm;
  if (g > need) g = need;
  return (int)(g < 1 ? 1 : g);
}

inline int grid_for(int64_t n, int block, int max_blocks_per_sm = 16) {
  int64_t b = (n + block - 1) / block;
  int64_t cap = (int64_t)num_sms() * max_blocks_per_sm;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (int)b;
}

}  // namespace mgt
