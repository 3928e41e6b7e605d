// Bit-exact numpy PCG64 probe noise on the GPU (reference: probing.py:94-107,
// make_noise -> numpy default_rng(seed).integers(0, 2 | 4, size=N)).
//
// numpy's bounded 32-bit path draws buffered 32-bit words (low half of each
// PCG64 64-bit output first) and applies Lemire's multiply-shift; for the
// ranges 2 and 4 there is never a rejection, so entry i is the top bit (top
// two bits) of word i.  Site r of the reference order owns entries
// 12r .. 12r+11, i.e. 64-bit outputs 6r .. 6r+5: every thread jumps its
// stream ahead by 6r steps (affine 128-bit power table from the host) and
// produces its site's 12 entries, written directly in the native layout.
#include <algorithm>
#include <vector>

#include "common.cuh"

namespace mgt {

struct U128 {
  uint64_t hi, lo;
};

__host__ __device__ __forceinline__ U128 mul128(U128 a, U128 b) {
  U128 r;
#ifdef __CUDA_ARCH__
  r.lo = a.lo * b.lo;
  r.hi = __umul64hi(a.lo, b.lo) + a.hi * b.lo + a.lo * b.hi;
#else
  unsigned __int128 p = (unsigned __int128)a.lo * b.lo;
  r.lo = (uint64_t)p;
  r.hi = (uint64_t)(p >> 64) + a.hi * b.lo + a.lo * b.hi;
#endif
  return r;
}

__host__ __device__ __forceinline__ U128 add128(U128 a, U128 b) {
  U128 r;
  r.lo = a.lo + b.lo;
  r.hi = a.hi + b.hi + (r.lo < a.lo ? 1 : 0);
  return r;
}

constexpr int kJumpBits = 40;
constexpr int kFieldsPerLaunch = 16;
static const U128 kMult = {0x2360ED051FC65DA4ULL, 0x4385DF649FCCF645ULL};

__constant__ U128 c_mult_pow[kJumpBits];  // M^(2^b)

struct NoiseBatch {
  U128 state[kFieldsPerLaunch];
  U128 inc[kFieldsPerLaunch];
  U128 cpow[kFieldsPerLaunch][kJumpBits];  // additive part of 2^b steps
};

__device__ __forceinline__ uint64_t xsl_rr(U128 s) {
  const uint64_t x = s.hi ^ s.lo;
  const unsigned rot = (unsigned)(s.hi >> 58);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

template <int KIND>
__device__ __forceinline__ void emit(uint32_t w, double2 *dst) {
  if (KIND == 0) {
    *dst = make_double2((w >> 31) ? 1.0 : -1.0, 0.0);
  } else {
    const uint32_t k = w >> 30;
    double2 v;
    if (k == 0) v = make_double2(1.0, 0.0);
    else if (k == 1) v = make_double2(0.0, 1.0);
    else if (k == 2) v = make_double2(-1.0, 0.0);
    else v = make_double2(-0.0, -1.0);
    *dst = v;
  }
}

// Thread = (field, spatial site, run of kSeg consecutive t): reference order
// has t fastest, so the run's 6 * kSeg outputs are consecutive steps of the
// stream -- one jump ahead per run instead of one per site (the jump's
// 128-bit multiplies were the kernel's cost).  A warp covers 32 consecutive
// native spatial sites, so every store is coalesced.
constexpr int kSeg = 8;

template <int KIND, bool NATIVE>
__global__ void noise_kernel(Geom g, Geom gref, int t_begin, const __grid_constant__ NoiseBatch nb, int nf, int field0,
                             double2 *__restrict__ out) {
  const int64_t plane = g.stride[3];
  const int nseg = (g.L[3] + kSeg - 1) / kSeg;
  const int64_t per_field = plane * nseg;
  const int64_t n = per_field * nf;
  const U128 M = {0x2360ED051FC65DA4ULL, 0x4385DF649FCCF645ULL};
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n; idx += (int64_t)gridDim.x * blockDim.x) {
    const int f = (int)(idx / per_field);
    const int64_t rem = idx - (int64_t)f * per_field;
    const int seg = (int)(rem / plane);
    const int64_t sp = rem - (int64_t)seg * plane;  // native spatial index (t = 0)
    const int tl0 = seg * kSeg, tl1 = min(g.L[3], tl0 + kSeg);
    int x[4];
    native_coords(g, sp, x);
    x[3] = t_begin + tl0;  // t-slab: the probe is the global one restricted to this slab
    const int64_t r0 = ref_site(gref, x);
    // jump 6 r0 steps: st <- A_k st + C_k
    U128 st = nb.state[f];
    const U128 inc = nb.inc[f];
    uint64_t k = (uint64_t)r0 * 6u;
    for (int b = 0; k; ++b, k >>= 1) {
      if (k & 1) st = add128(mul128(st, c_mult_pow[b]), nb.cpow[f][b]);
    }
    const int fg = field0 + f;
    for (int tl = tl0; tl < tl1; ++tl) {
      const int64_t s = (int64_t)tl * plane + sp;
      const int64_t r = r0 + (tl - tl0);
#pragma unroll
      for (int m = 0; m < 6; ++m) {
        st = add128(mul128(st, M), inc);
        const uint64_t o = xsl_rr(st);
        const int c0 = 2 * m, c1 = 2 * m + 1;
        double2 *d0, *d1;
        if (NATIVE) {
          d0 = out + ((int64_t)fg * 12 + c0) * g.V + s;
          d1 = out + ((int64_t)fg * 12 + c1) * g.V + s;
        } else {
          d0 = out + (int64_t)fg * 12 * g.V + r * 12 + c0;
          d1 = d0 + 1;
        }
        emit<KIND>((uint32_t)(o & 0xFFFFFFFFu), d0);
        emit<KIND>((uint32_t)(o >> 32), d1);
      }
    }
  }
}

static bool g_pow_ready = false;

static int ensure_pow_table() {
  if (g_pow_ready) return MGT_OK;
  U128 t[kJumpBits];
  U128 a = kMult;
  for (int b = 0; b < kJumpBits; ++b) {
    t[b] = a;
    a = mul128(a, a);
  }
  MGT_CUDA(cudaMemcpyToSymbol(c_mult_pow, t, sizeof(t)));
  g_pow_ready = true;
  return MGT_OK;
}

}  // namespace mgt

using namespace mgt;

static int noise_impl(const int dims[4], const int dims_ref[4], int t_begin, int kind, const uint64_t *seeds_host,
                      int n_fields, int native_layout, void *out_dev, void *stream) {
  if (!dims || !seeds_host || !out_dev || n_fields < 0) return fail(MGT_ERR_INVALID, "mgt_noise: bad argument");
  if (kind != 0 && kind != 1) return fail(MGT_ERR_INVALID, "mgt_noise: kind must be 0 (rademacher) or 1 (z4)");
  Geom g = make_geom(dims), gref = make_geom(dims_ref);
  if ((uint64_t)gref.V * 6u >= (1ull << kJumpBits)) return fail(MGT_ERR_INVALID, "mgt_noise: lattice too large");
  int rc = ensure_pow_table();
  if (rc) return rc;
  cudaStream_t st = as_stream(stream);
  for (int f0 = 0; f0 < n_fields; f0 += kFieldsPerLaunch) {
    const int nf = std::min(kFieldsPerLaunch, n_fields - f0);
    NoiseBatch nb;
    for (int f = 0; f < nf; ++f) {
      const uint64_t *q = seeds_host + 4 * (f0 + f);
      nb.state[f] = U128{q[0], q[1]};
      nb.inc[f] = U128{q[2], q[3]};
      // C_0 = inc, C_{b+1} = C_b (A_b + 1)
      U128 c = nb.inc[f], a = kMult;
      for (int b = 0; b < kJumpBits; ++b) {
        nb.cpow[f][b] = c;
        c = mul128(c, add128(a, U128{0, 1}));
        a = mul128(a, a);
      }
    }
    const int block = 128;
    const int grid = grid_for(g.stride[3] * ((g.L[3] + kSeg - 1) / kSeg) * nf, block, 8);
    double2 *o = (double2 *)out_dev;
    if (kind == 0 && native_layout)
      noise_kernel<0, true><<<grid, block, 0, st>>>(g, gref, t_begin, nb, nf, f0, o);
    else if (kind == 0)
      noise_kernel<0, false><<<grid, block, 0, st>>>(g, gref, t_begin, nb, nf, f0, o);
    else if (native_layout)
      noise_kernel<1, true><<<grid, block, 0, st>>>(g, gref, t_begin, nb, nf, f0, o);
    else
      noise_kernel<1, false><<<grid, block, 0, st>>>(g, gref, t_begin, nb, nf, f0, o);
    MGT_LAUNCH_CHECK("noise_kernel");
  }
  return MGT_OK;
}

extern "C" int mgt_noise(const int dims[4], int kind, const uint64_t *seeds_host, int n_fields, int native_layout,
                         void *out_dev, void *stream) {
  if (!dims) return fail(MGT_ERR_INVALID, "mgt_noise: bad argument");
  return noise_impl(dims, dims, 0, kind, seeds_host, n_fields, native_layout, out_dev, stream);
}

extern "C" int mgt_noise_slab(const int dims_global[4], int t_begin, int t_local, int kind, const uint64_t *seeds_host,
                              int n_fields, void *out_native_dev, void *stream) {
  if (!dims_global || t_begin < 0 || t_local < 1 || t_begin + t_local > dims_global[3])
    return fail(MGT_ERR_INVALID, "mgt_noise_slab: slab outside the global t range");
  const int dl[4] = {dims_global[0], dims_global[1], dims_global[2], t_local};
  return noise_impl(dl, dims_global, t_begin, kind, seeds_host, n_fields, 1, out_native_dev, stream);
}
