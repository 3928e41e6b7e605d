// fp32 even-odd stencil with two adjacent checkerboard sites per thread, sm_100a.
//
// The fp32 inner solves of the mixed-precision BiCGStab (bicgstab.cu) stream
// 8-byte complex<float> elements: at one site per thread every load moves half
// the bytes of the fp64 kernel's for the same address arithmetic, and the
// kernels end up issue/latency-bound instead of HBM-bound (ncu
// profiles/r01e_k1eo_f32_ncu.txt).  Here a thread owns the cb sites c0 (even)
// and c0 + 1 of one lattice row (L2/2 even): in the t, x0 and x1 hops their
// neighbours are again the aligned pair (cn, cn + 1) of the other parity, so a
// spinor component of both sites is one 16-byte load and the two sites' links
// one 32-byte load -- the access widths of the fp64 kernel -- with the site
// decode, neighbour index and boundary phase computed once per pair.  Only
// the x2 hop towards the pair's unaligned side (x2 + 1 for rows that start at
// x2 = 1, x2 - 1 for rows that start at 0) loads per site.
//
// Same operator, coefficients and per-site arithmetic as eo_eval (eo_core.cuh;
// reference operator: lattice.py:274-318).
#pragma once
#include "eo_core.cuh"

namespace mgt {

struct alignas(16) f4 {
  float x, y, z, w;
};
struct alignas(32) f8 {
  float v[8];
};

__device__ __forceinline__ void ld2(const float2 *p, C<float> &a, C<float> &b) {
  const float4 v = __ldg(reinterpret_cast<const float4 *>(p));
  a = C<float>(v.x, v.y);
  b = C<float>(v.z, v.w);
}
__device__ __forceinline__ void st2(float2 *p, C<float> a, C<float> b) {
  *reinterpret_cast<float4 *>(p) = make_float4(a.re, a.im, b.re, b.im);
}

// third row of an SU(3) link from its first two
__device__ __forceinline__ void su3_row2(C<float> (&u)[3][3]) {
  u[2][0] = conj(u[0][1] * u[1][2] - u[0][2] * u[1][1]);
  u[2][1] = conj(u[0][2] * u[1][0] - u[0][0] * u[1][2]);
  u[2][2] = conj(u[0][0] * u[1][1] - u[0][1] * u[1][0]);
}

// links (mu, site) and (mu, site + 1), site even
template <int RECON>
__device__ __forceinline__ void load_link_pair(const LinkField<float, RECON> &lf, int mu, int64_t site,
                                               C<float> (&u0)[3][3], C<float> (&u1)[3][3]) {
  if constexpr (RECON == 12 && MGT_LINK_PAIRS) {
    // element pairs (e, e + 1) of one site are 16 bytes: two sites = 32 bytes
    const f8 *q = reinterpret_cast<const f8 *>(reinterpret_cast<const cpair<float> *>(lf.p) +
                                               (int64_t)mu * 3 * lf.V + site);
    const int64_t st = lf.V >> 1;
#pragma unroll
    for (int pp = 0; pp < 3; ++pp) {
      const f8 v = q[pp * st];
      u0[(2 * pp) / 3][(2 * pp) % 3] = C<float>(v.v[0], v.v[1]);
      u0[(2 * pp + 1) / 3][(2 * pp + 1) % 3] = C<float>(v.v[2], v.v[3]);
      u1[(2 * pp) / 3][(2 * pp) % 3] = C<float>(v.v[4], v.v[5]);
      u1[(2 * pp + 1) / 3][(2 * pp + 1) % 3] = C<float>(v.v[6], v.v[7]);
    }
  } else {
    constexpr int NL = RECON / 2;
    const float2 *q = lf.p + (int64_t)mu * NL * lf.V + site;
#pragma unroll
    for (int e = 0; e < NL; ++e) ld2(q + e * lf.V, u0[e / 3][e % 3], u1[e / 3][e % 3]);
  }
  if constexpr (RECON == 12) {
    su3_row2(u0);
    su3_row2(u1);
  }
}

// spin projection of one neighbour (p2, p3 already carry the G_in sign)
template <int MU, bool FWD>
__device__ __forceinline__ void hop_project(C<float> p0, C<float> p1, C<float> p2, C<float> p3, C<float> &h0,
                                            C<float> &h1) {
  C<float> b0, b1;
  b_mul<MU>(p2, p3, b0, b1);
  if constexpr (FWD) {
    h0 = p0 - b0;
    h1 = p1 - b1;
  } else {
    h0 = p0 + b0;
    h1 = p1 + b1;
  }
}

// colour multiply (U h forward, U^dag h backward), phase, reconstruction
template <int MU, bool FWD>
__device__ __forceinline__ void hop_accumulate(const C<float> (&u)[3][3], const C<float> (&h)[2][3], float ph,
                                               C<float> (&acc)[4][3]) {
  C<float> w[2][3];
#pragma unroll
  for (int a = 0; a < 2; ++a) {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      C<float> s(0.f, 0.f);
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        if constexpr (FWD)
          s = cfma(u[i][j], h[a][j], s);
        else
          s = cfma_conj(u[j][i], h[a][j], s);
      }
      w[a][i] = ph * s;
    }
  }
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    acc[0][i] = acc[0][i] + w[0][i];
    acc[1][i] = acc[1][i] + w[1][i];
    C<float> o2, o3;
    bdag_mul<MU>(w[0][i], w[1][i], o2, o3);
    if constexpr (FWD) {
      acc[2][i] = acc[2][i] - o2;
      acc[3][i] = acc[3][i] - o3;
    } else {
      acc[2][i] = acc[2][i] + o2;
      acc[3][i] = acc[3][i] + o3;
    }
  }
}

// t, x0, x1 hops of the pair (site, site + 2): neighbours (nb, nb + 2) are the
// aligned cb pair (cn, cn + 1).
template <int MU, bool FWD, int RECON>
__device__ __forceinline__ void eo_hop_pair(const EoGeom &E, const float2 *__restrict__ in,
                                            const LinkField<float, RECON> &lout,
                                            const LinkField<float, RECON> &lin, int64_t site, int64_t c,
                                            const int (&x)[4], float gin, C<float> (&acc)[2][4][3]) {
  static_assert(MU != 2, "x2 hops: eo_hop_pair_x2");
  const int L = E.g.L[MU];
  const int64_t st = E.g.stride[MU];
  int64_t nb;
  float ph = 1.f;
  if constexpr (FWD) {
    nb = (x[MU] == L - 1) ? site - (int64_t)(L - 1) * st : site + st;
    if (MU == 3 && E.antiperiodic && x[3] == L - 1) ph = -1.f;
  } else {
    nb = (x[MU] == 0) ? site + (int64_t)(L - 1) * st : site - st;
    if (MU == 3 && E.antiperiodic && x[3] == 0) ph = -1.f;
  }
  const int64_t cn = nb >> 1;
  const int64_t Vh = E.Vh;
  C<float> h[2][2][3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    C<float> p0[2], p1[2], p2[2], p3[2];
    ld2(in + (0 * 3 + k) * Vh + cn, p0[0], p0[1]);
    ld2(in + (1 * 3 + k) * Vh + cn, p1[0], p1[1]);
    ld2(in + (2 * 3 + k) * Vh + cn, p2[0], p2[1]);
    ld2(in + (3 * 3 + k) * Vh + cn, p3[0], p3[1]);
#pragma unroll
    for (int s = 0; s < 2; ++s)
      hop_project<MU, FWD>(p0[s], p1[s], gin * p2[s], gin * p3[s], h[s][0][k], h[s][1][k]);
  }
  C<float> u0[3][3], u1[3][3];
  if constexpr (FWD)
    load_link_pair<RECON>(lout, MU, c, u0, u1);
  else
    load_link_pair<RECON>(lin, MU, cn, u0, u1);
  hop_accumulate<MU, FWD>(u0, h[0], ph, acc[0]);
  hop_accumulate<MU, FWD>(u1, h[1], ph, acc[1]);
}

// x2 hops: the neighbours of the pair's sites x2 and x2 + 2 are the cb sites
// (ca, cb) computed per site (consecutive but not always 16-byte aligned; the
// row wraps at x2 = 0 / L2 - 1).
template <bool FWD, int RECON>
__device__ __forceinline__ void eo_hop_pair_x2(const EoGeom &E, const float2 *__restrict__ in,
                                               const LinkField<float, RECON> &lout,
                                               const LinkField<float, RECON> &lin, int64_t site, int64_t c,
                                               const int (&x)[4], float gin, C<float> (&acc)[2][4][3]) {
  const int L2 = E.g.L[2];
  int64_t ca, cb;
  if constexpr (FWD) {
    // x2 + 1 never wraps (x2 <= L2 - 3); x2 + 3 wraps when it reaches L2
    ca = (site + 1) >> 1;
    cb = (x[2] + 3 == L2) ? (site - x[2]) >> 1 : (site + 3) >> 1;
  } else {
    ca = (x[2] == 0) ? (site + L2 - 1) >> 1 : (site - 1) >> 1;
    cb = (site + 1) >> 1;
  }
  const int64_t Vh = E.Vh;
  C<float> h[2][2][3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    C<float> p0[2], p1[2], p2[2], p3[2];
    p0[0] = ldc(in + (0 * 3 + k) * Vh + ca);
    p0[1] = ldc(in + (0 * 3 + k) * Vh + cb);
    p1[0] = ldc(in + (1 * 3 + k) * Vh + ca);
    p1[1] = ldc(in + (1 * 3 + k) * Vh + cb);
    p2[0] = ldc(in + (2 * 3 + k) * Vh + ca);
    p2[1] = ldc(in + (2 * 3 + k) * Vh + cb);
    p3[0] = ldc(in + (3 * 3 + k) * Vh + ca);
    p3[1] = ldc(in + (3 * 3 + k) * Vh + cb);
#pragma unroll
    for (int s = 0; s < 2; ++s)
      hop_project<2, FWD>(p0[s], p1[s], gin * p2[s], gin * p3[s], h[s][0][k], h[s][1][k]);
  }
  C<float> u0[3][3], u1[3][3];
  if constexpr (FWD) {
    load_link_pair<RECON>(lout, 2, c, u0, u1);
  } else {
    lin.load(2, ca, u0);
    lin.load(2, cb, u1);
  }
  hop_accumulate<2, FWD>(u0, h[0], 1.f, acc[0]);
  hop_accumulate<2, FWD>(u1, h[1], 1.f, acc[1]);
}

// eo_eval for the cb sites c and c + 1 (c even, L2/2 even): y[s], cc[s] are
// site c + s's result and raw centre value.
template <int RECON>
__device__ __forceinline__ void eo_eval_pair(const EoGeom &E, int pout, const EoCoef &K,
                                             const float2 *__restrict__ in, const float2 *__restrict__ ctr,
                                             const LinkField<float, RECON> &lout,
                                             const LinkField<float, RECON> &lin, int64_t c,
                                             C<float> (&y)[2][4][3], C<float> (&cc)[2][4][3]) {
  int x[4];
  const int64_t site = eo_coords(E, pout, c, x);
  const float gin = (float)K.gin;
  C<float> acc[2][4][3];
#pragma unroll
  for (int s = 0; s < 2; ++s)
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int k = 0; k < 3; ++k) acc[s][a][k] = C<float>(0.f, 0.f);
#define MGT_HOP_FENCE asm volatile("" ::: "memory")
  eo_hop_pair<3, true>(E, in, lout, lin, site, c, x, gin, acc);
  MGT_HOP_FENCE;
  eo_hop_pair<3, false>(E, in, lout, lin, site, c, x, gin, acc);
  MGT_HOP_FENCE;
  eo_hop_pair<0, true>(E, in, lout, lin, site, c, x, gin, acc);
  MGT_HOP_FENCE;
  eo_hop_pair<0, false>(E, in, lout, lin, site, c, x, gin, acc);
  MGT_HOP_FENCE;
  eo_hop_pair<1, true>(E, in, lout, lin, site, c, x, gin, acc);
  MGT_HOP_FENCE;
  eo_hop_pair<1, false>(E, in, lout, lin, site, c, x, gin, acc);
  MGT_HOP_FENCE;
  eo_hop_pair_x2<true>(E, in, lout, lin, site, c, x, gin, acc);
  MGT_HOP_FENCE;
  eo_hop_pair_x2<false>(E, in, lout, lin, site, c, x, gin, acc);
  MGT_HOP_FENCE;
#undef MGT_HOP_FENCE
  const float ch = (float)K.ch, gc = (float)K.gc, go = (float)K.go;
  const C<float> dcu((float)K.dcu_re, (float)K.dcu_im), dcd((float)K.dcd_re, (float)K.dcd_im);
  const C<float> eu((float)K.eu_re, (float)K.eu_im), ed((float)K.ed_re, (float)K.ed_im);
#pragma unroll
  for (int a = 0; a < 4; ++a) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      C<float> z[2];
      if (ctr) {
        ld2(ctr + (a * 3 + k) * E.Vh + c, z[0], z[1]);
      } else {
        z[0] = z[1] = C<float>(0.f, 0.f);
      }
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        C<float> v = ch * acc[s][a][k];
        cc[s][a][k] = z[s];
        if (ctr) {
          C<float> zz = a >= 2 ? gc * z[s] : z[s];
          v = v + (a < 2 ? dcu : dcd) * zz;
        }
        v = (a < 2 ? eu : ed) * v;
        y[s][a][k] = a >= 2 ? go * v : v;
      }
    }
  }
}

}  // namespace mgt
