// Wilson-Dirac stencil core (4D, SU(3), DeGrand-Rossi gammas), sm_100a.
//
// Operator (restated from the reference's 2D assembly, lattice.py:274-318,
// generalised to 4D SU(3)):
//   (A z)(x) = (4 + m0) z(x)
//            - 1/2 sum_mu [ (1 - g_mu) U_mu(x)        z(x+mu) ph_f
//                         + (1 + g_mu) U_mu(x-mu)^dag z(x-mu) ph_b ]
// ph = -1 on the hops that wrap in t when the boundary is antiperiodic
// (lattice.py:91-102).  In the chiral DeGrand-Rossi basis every gamma_mu is
// [[0, B_mu], [B_mu^dag, 0]] with B_mu unitary and monomial, so
//   (1 -/+ g_mu) psi = ( h, -/+ B^dag h ),   h = psi_up -/+ B psi_dn,
// i.e. each hop is a spin projection to a half spinor (6 complex), one
// SU(3) multiply per half-spinor row, and a free reconstruction.  That is
// 1320 flop/site for the 8 hops; the data each site streams is its 8
// neighbour spinors (mostly cache hits) and its 4 forward links.
#pragma once
#include "common.cuh"

namespace mgt {

// (B_mu psi_dn): returns (o0, o1) from (psi2, psi3)
template <int MU, typename R>
__device__ __forceinline__ void b_mul(C<R> p2, C<R> p3, C<R> &o0, C<R> &o1) {
  if constexpr (MU == 0) {  // B = [[0, i], [i, 0]]
    o0 = times_i(p3);
    o1 = times_i(p2);
  } else if constexpr (MU == 1) {  // B = [[0, -1], [1, 0]]
    o0 = -p3;
    o1 = p2;
  } else if constexpr (MU == 2) {  // B = [[i, 0], [0, -i]]
    o0 = times_i(p2);
    o1 = -times_i(p3);
  } else {  // B = I
    o0 = p2;
    o1 = p3;
  }
}

// (B_mu^dag w): returns (o2, o3) from (w0, w1)
template <int MU, typename R>
__device__ __forceinline__ void bdag_mul(C<R> w0, C<R> w1, C<R> &o2, C<R> &o3) {
  if constexpr (MU == 0) {  // B^dag = [[0, -i], [-i, 0]]
    o2 = -times_i(w1);
    o3 = -times_i(w0);
  } else if constexpr (MU == 1) {  // B^dag = [[0, 1], [-1, 0]]
    o2 = w1;
    o3 = -w0;
  } else if constexpr (MU == 2) {  // B^dag = [[-i, 0], [0, i]]
    o2 = -times_i(w0);
    o3 = times_i(w1);
  } else {
    o2 = w0;
    o3 = w1;
  }
}

// Native link storage: element e of link (mu, site) at ((mu*NL + e)*V + site),
// NL = 9 (full 3x3, row-major) or 6 (rows 0 and 1; row 2 = conj(r0 x r1)).
#ifndef MGT_LINK_PAIRS
#define MGT_LINK_PAIRS 1
#endif
// Mixed-precision solves: fp32 per-parity links stored as full 3x3 (no
// third-row reconstruction in the fp32 hops) when 1.
#ifndef MGT_MIXED_L18
#define MGT_MIXED_L18 0
#endif
// With MGT_LINK_PAIRS the 12-real links are stored as 3 element pairs per
// (mu, site), ((mu*3 + e/2)*V + site)*2 + (e & 1): one 256-bit (fp64) /
// 128-bit (fp32) load per pair.
template <typename R> struct alignas(2 * sizeof(cplx<R>)) cpair {
  cplx<R> a, b;
};
template <int RECON>
__host__ __device__ __forceinline__ int64_t link_index(int mu, int e, int64_t site, int64_t V) {
  if constexpr (RECON == 12 && MGT_LINK_PAIRS)
    return (((int64_t)mu * 3 + e / 2) * V + site) * 2 + (e & 1);
  else
    return ((int64_t)mu * (RECON / 2) + e) * V + site;
}

template <typename R, int RECON>
struct LinkField {
  static constexpr int NL = RECON / 2;
  const cplx<R> *__restrict__ p;
  int64_t V;
  __device__ __forceinline__ void load(int mu, int64_t site, C<R> (&u)[3][3]) const {
    if constexpr (RECON == 12 && MGT_LINK_PAIRS) {
      const cpair<R> *q = reinterpret_cast<const cpair<R> *>(p) + (int64_t)mu * 3 * V + site;
#pragma unroll
      for (int pp = 0; pp < 3; ++pp) {
        const cpair<R> v = q[pp * V];
        u[(2 * pp) / 3][(2 * pp) % 3] = C<R>(v.a.x, v.a.y);
        u[(2 * pp + 1) / 3][(2 * pp + 1) % 3] = C<R>(v.b.x, v.b.y);
      }
    } else {
      const cplx<R> *q = p + (int64_t)mu * NL * V + site;
#pragma unroll
      for (int e = 0; e < NL; ++e) u[e / 3][e % 3] = ldc(q + e * V);
    }
    if constexpr (RECON == 12) {
      // u2 = conj(u0 x u1)  (exact for SU(3): det = 1, unitary)
      u[2][0] = conj(u[0][1] * u[1][2] - u[0][2] * u[1][1]);
      u[2][1] = conj(u[0][2] * u[1][0] - u[0][0] * u[1][2]);
      u[2][2] = conj(u[0][0] * u[1][1] - u[0][1] * u[1][0]);
    }
  }
};

// neighbour-spinor load of the hops (experiment hook: ldc_cg bypasses L1)
#ifndef MGT_SPINOR_LD
#define MGT_SPINOR_LD ldc
#endif

// Accumulate one hop into acc[spin][colour] (without the -1/2).
// SS: site stride of the spinor field (1: native SoA; NR: rhs-interleaved
// ((comp*V + site)*NR + rhs), `in` pre-offset by rhs).
template <int MU, bool FWD, typename R, int RECON, int SS = 1>
__device__ __forceinline__ void wilson_hop(const Geom &g, const cplx<R> *__restrict__ in,
                                           const LinkField<R, RECON> &links, int64_t site,
                                           const int (&x)[4], R g5in, bool antiperiodic,
                                           C<R> (&acc)[4][3]) {
  const int L = g.L[MU];
  const int64_t st = g.stride[MU];
  int64_t nb;
  R ph = R(1);
  if constexpr (FWD) {
    nb = (x[MU] == L - 1) ? site - (int64_t)(L - 1) * st : site + st;
    if (MU == 3 && antiperiodic && x[3] == L - 1) ph = R(-1);
  } else {
    nb = (x[MU] == 0) ? site + (int64_t)(L - 1) * st : site - st;
    if (MU == 3 && antiperiodic && x[3] == 0) ph = R(-1);
  }
  const int64_t V = g.V;
  // spin projection
  C<R> h[2][3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    C<R> p0 = MGT_SPINOR_LD(in + ((0 * 3 + c) * V + nb) * SS);
    C<R> p1 = MGT_SPINOR_LD(in + ((1 * 3 + c) * V + nb) * SS);
    C<R> p2 = g5in * MGT_SPINOR_LD(in + ((2 * 3 + c) * V + nb) * SS);
    C<R> p3 = g5in * MGT_SPINOR_LD(in + ((3 * 3 + c) * V + nb) * SS);
    C<R> b0, b1;
    b_mul<MU>(p2, p3, b0, b1);
    if constexpr (FWD) {
      h[0][c] = p0 - b0;
      h[1][c] = p1 - b1;
    } else {
      h[0][c] = p0 + b0;
      h[1][c] = p1 + b1;
    }
  }
  // colour multiply: U h (forward) or U^dag h (backward, link of x - mu)
  C<R> u[3][3];
  links.load(MU, FWD ? site : nb, u);
  C<R> w[2][3];
#pragma unroll
  for (int a = 0; a < 2; ++a) {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      C<R> s(R(0), R(0));
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
  // reconstruction
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    acc[0][i] = acc[0][i] + w[0][i];
    acc[1][i] = acc[1][i] + w[1][i];
    C<R> o2, o3;
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

struct WilsonParams {
  Geom g;
  Sched sched;
  int antiperiodic;
  // t-slab decomposition: this operator owns global t in [t_begin, t_begin + L3)
  // of T_global; with slab != 0 the t hops that leave the slab read the
  // neighbours' pre-projected faces (6 complex per spatial site and rhs):
  //   halo_next: (1 - g_4) projection of rank+1's first slice,
  //   halo_prev: U_4^dag (1 + g_4) projection of rank-1's last slice.
  int slab, t_begin, T_global;
  const void *halo_next, *halo_prev;
  double diag_up_re, diag_up_im;  // (4 + m0) + i tau   acting on spins 0,1
  double diag_dn_re, diag_dn_im;  // (4 + m0) - i tau   acting on spins 2,3
  double g5in, g5out;             // +1 or -1
};

// t hops across a slab boundary, from the received faces (gamma_4: B = I).
template <bool FWD, typename R, int RECON>
__device__ __forceinline__ void wilson_thop_halo(const WilsonParams &P, const LinkField<R, RECON> &links,
                                                 int64_t site, const int (&x)[4], int rhs, C<R> (&acc)[4][3]) {
  const int64_t S3 = P.g.stride[3];
  const int64_t s = site - (int64_t)x[3] * S3;
  const cplx<R> *hb = reinterpret_cast<const cplx<R> *>(FWD ? P.halo_next : P.halo_prev) + (int64_t)rhs * 6 * S3 + s;
  const int tg = P.t_begin + x[3];
  const R ph = (P.antiperiodic && (FWD ? tg == P.T_global - 1 : tg == 0)) ? R(-1) : R(1);
  C<R> w[2][3];
  if constexpr (FWD) {
    C<R> h[2][3];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int c = 0; c < 3; ++c) h[a][c] = ldc(hb + (a * 3 + c) * S3);
    C<R> u[3][3];
    links.load(3, site, u);
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        C<R> t(R(0), R(0));
#pragma unroll
        for (int j = 0; j < 3; ++j) t = cfma(u[i][j], h[a][j], t);
        w[a][i] = ph * t;
      }
  } else {
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int c = 0; c < 3; ++c) w[a][c] = ph * ldc(hb + (a * 3 + c) * S3);
  }
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    acc[0][i] = acc[0][i] + w[0][i];
    acc[1][i] = acc[1][i] + w[1][i];
    if constexpr (FWD) {
      acc[2][i] = acc[2][i] - w[0][i];
      acc[3][i] = acc[3][i] - w[1][i];
    } else {
      acc[2][i] = acc[2][i] + w[0][i];
      acc[3][i] = acc[3][i] + w[1][i];
    }
  }
}

// y = G_out [ diag z - 1/2 hop(z) ],  z = G_in x.  Also returns the raw input
// x at the site (xc, before G_in) for fused epilogues.
// EARLY (callers that do not need xc): the centre value is loaded together
// with the first hop's neighbours and folded into the accumulators at once,
// acc = -2 diag z, so the site has 8 dependent memory phases instead of 9
// (the centre's registers are free again before the accumulators of the
// second hop are live); y = G_out (-1/2 acc).  Same terms, summed in a
// different order than the default (differences at rounding level).
template <typename R, int RECON, int SS = 1, bool EARLY = false>
__device__ __forceinline__ void wilson_eval(const WilsonParams &P, const cplx<R> *__restrict__ in,
                                            const LinkField<R, RECON> &links, int64_t site,
                                            C<R> (&y)[4][3], C<R> (&xc)[4][3], int rhs = 0) {
  int x[4];
  native_coords(P.g, site, x);
  const R g5in = (R)P.g5in;
  const bool ap = P.antiperiodic != 0;
  C<R> acc[4][3];
  if constexpr (EARLY) {
    const C<R> dup2((R)(-2.0 * P.diag_up_re), (R)(-2.0 * P.diag_up_im));
    const C<R> ddn2((R)(-2.0 * P.diag_dn_re), (R)(-2.0 * P.diag_dn_im));
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        C<R> v = ldc(in + ((a * 3 + c) * P.g.V + site) * SS);
        acc[a][c] = a >= 2 ? ddn2 * (g5in * v) : dup2 * v;
      }
  } else {
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int c = 0; c < 3; ++c) acc[a][c] = C<R>(R(0), R(0));
  }
  // The compiler would otherwise hoist the loads of all 8 hops (168 loads per
  // thread) and spill; one hop's 21 independent 16-byte loads in flight per
  // thread is already ~4x the bytes-in-flight HBM needs at this occupancy.
#define MGT_HOP_FENCE asm volatile("" ::: "memory")
  if (P.slab && x[3] == P.g.L[3] - 1)
    wilson_thop_halo<true>(P, links, site, x, rhs, acc);
  else
    wilson_hop<3, true, R, RECON, SS>(P.g, in, links, site, x, g5in, ap, acc);
  MGT_HOP_FENCE;
  if (P.slab && x[3] == 0)
    wilson_thop_halo<false>(P, links, site, x, rhs, acc);
  else
    wilson_hop<3, false, R, RECON, SS>(P.g, in, links, site, x, g5in, ap, acc);
  MGT_HOP_FENCE;
  wilson_hop<0, true, R, RECON, SS>(P.g, in, links, site, x, g5in, ap, acc);
  MGT_HOP_FENCE;
  wilson_hop<0, false, R, RECON, SS>(P.g, in, links, site, x, g5in, ap, acc);
  MGT_HOP_FENCE;
  wilson_hop<1, true, R, RECON, SS>(P.g, in, links, site, x, g5in, ap, acc);
  MGT_HOP_FENCE;
  wilson_hop<1, false, R, RECON, SS>(P.g, in, links, site, x, g5in, ap, acc);
  MGT_HOP_FENCE;
  wilson_hop<2, true, R, RECON, SS>(P.g, in, links, site, x, g5in, ap, acc);
  MGT_HOP_FENCE;
  wilson_hop<2, false, R, RECON, SS>(P.g, in, links, site, x, g5in, ap, acc);
  MGT_HOP_FENCE;
#undef MGT_HOP_FENCE
  const C<R> dup((R)P.diag_up_re, (R)P.diag_up_im);
  const C<R> ddn((R)P.diag_dn_re, (R)P.diag_dn_im);
  const R half = R(0.5);
  const R g5out = (R)P.g5out;
  if constexpr (EARLY) {
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        xc[a][c] = C<R>(R(0), R(0));
        const C<R> r = (-half) * acc[a][c];
        y[a][c] = a >= 2 ? g5out * r : r;
      }
    return;
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      C<R> v = ldc(in + ((a * 3 + c) * P.g.V + site) * SS);
      xc[a][c] = v;
      if (a >= 2) {
        v = g5in * v;
        C<R> r = ddn * v - half * acc[a][c];
        y[a][c] = g5out * r;
      } else {
        y[a][c] = dup * v - half * acc[a][c];
      }
    }
  }
}

// Two threads per site: lane parity h = 0 applies the t and x0 hops, h = 1 the
// x1 and x2 hops; the partial sums are exchanged with one shuffle round and
// thread h finalises spins 2h, 2h+1 (comps 6h .. 6h+5).  Halves the serial
// hop chain per thread and doubles the loads in flight per site.
// y6/xc6: this thread's 6 output comps and raw input comps.
template <typename R, int RECON>
__device__ __forceinline__ void wilson_eval_split2(const WilsonParams &P, const cplx<R> *__restrict__ in,
                                                   const LinkField<R, RECON> &links, int64_t site, int h,
                                                   C<R> (&y6)[2][3], C<R> (&xc6)[2][3]) {
  int x[4];
  native_coords(P.g, site, x);
  const R g5in = (R)P.g5in;
  const bool ap = P.antiperiodic != 0;
  C<R> acc[4][3];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int c = 0; c < 3; ++c) acc[a][c] = C<R>(R(0), R(0));
#define MGT_HOP_FENCE asm volatile("" ::: "memory")
  if (h == 0) {
    wilson_hop<3, true>(P.g, in, links, site, x, g5in, ap, acc);
    MGT_HOP_FENCE;
    wilson_hop<3, false>(P.g, in, links, site, x, g5in, ap, acc);
    MGT_HOP_FENCE;
    wilson_hop<0, true>(P.g, in, links, site, x, g5in, ap, acc);
    MGT_HOP_FENCE;
    wilson_hop<0, false>(P.g, in, links, site, x, g5in, ap, acc);
  } else {
    wilson_hop<1, true>(P.g, in, links, site, x, g5in, ap, acc);
    MGT_HOP_FENCE;
    wilson_hop<1, false>(P.g, in, links, site, x, g5in, ap, acc);
    MGT_HOP_FENCE;
    wilson_hop<2, true>(P.g, in, links, site, x, g5in, ap, acc);
    MGT_HOP_FENCE;
    wilson_hop<2, false>(P.g, in, links, site, x, g5in, ap, acc);
  }
#undef MGT_HOP_FENCE
  // exchange: h = 0 keeps spins 0,1 and ships 2,3; h = 1 the reverse
  C<R> mine[2][3];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      C<R> send = h ? acc[a][c] : acc[2 + a][c];
      C<R> keep = h ? acc[2 + a][c] : acc[a][c];
      C<R> got;
      got.re = __shfl_xor_sync(0xffffffffu, send.re, 1);
      got.im = __shfl_xor_sync(0xffffffffu, send.im, 1);
      mine[a][c] = keep + got;
    }
  const C<R> dup((R)P.diag_up_re, (R)P.diag_up_im);
  const C<R> ddn((R)P.diag_dn_re, (R)P.diag_dn_im);
  const R half = R(0.5);
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      C<R> v = ldc(in + ((2 * h + a) * 3 + c) * P.g.V + site);
      xc6[a][c] = v;
      if (h) {
        C<R> r = ddn * (g5in * v) - half * mine[a][c];
        y6[a][c] = (R)P.g5out * r;
      } else {
        y6[a][c] = dup * v - half * mine[a][c];
      }
    }
}

}  // namespace mgt
