// GPU-resident BiCGStab for the Wilson operator -- the TruncatedInverse solver
// plugin (reference: krylov.py:200-229; the reference's own solver is GCR,
// krylov.py:52-118, BASELINE.json names BiCGStab).
//
// Per iteration (complex BiCGStab, x0 = 0), NR right-hand sides at once:
//   K1  v = A p                       sigma = (rhat, v)      alpha = rho/sigma
//   K2  s = r - alpha v               |s|^2  (early exit when s is converged)
//   K3  t = A s                       (t, s), |t|^2          omega = (t,s)/|t|^2
//   K4  x += alpha p + omega s; r = s - omega t;  rho' = (rhat, r), |r|^2, beta
//   K5  p = r + beta (p - omega v)
// Every reduction is fused into the producing kernel (reduce.cuh) and the
// scalar recurrences run in that kernel's last block, so the host only
// launches: chunks of iterations are replayed from a cached CUDA graph and
// the host reads the per-rhs status words once per chunk.  Kernels of a
// converged rhs return immediately.  Convergence is confirmed on the
// explicitly recomputed residual b - A x (krylov.py:78-85, :113-118); a
// recursion / true-residual mismatch restarts with rhat = r.
#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <type_traits>
#include <vector>

#include "comm.cuh"
#include "eo_core.cuh"
// two-sites-per-thread fp32 stencils (eo_pair.cuh): compiled in with
// -DMGT_F32_STENCIL_PAIRS=1, then on by default (env MGT_F32_STENCIL_PAIRS=0
// switches back).  Measured equal or slower than the one-site kernels
// (profiles/r02s4_pair_stencil_ab.txt), so the default build leaves them out.
#ifndef MGT_F32_STENCIL_PAIRS
#define MGT_F32_STENCIL_PAIRS 0
#endif
#if MGT_F32_STENCIL_PAIRS
#include "eo_pair.cuh"
#endif
#include "handle.cuh"
#include "reduce.cuh"

namespace mgt {

enum : int { ST_RUN = 0, ST_CONV = 1, ST_BREAK = 2, ST_MAXIT = 3, ST_RESTART = 4, ST_DONE = 5 };

struct BiState {
  C<double> rho, alpha, omega, beta, dotq;
  double b2, r2, s2, true_r2, tol2, bfull2;
  int status, half, iters, maxit, matvecs, reason, pad0, pad1;
};

// Workspace: fields of NR rhs each (native layout) + reduction scratch.
// R: the field precision (double; float for the inner solves of the mixed-
// precision solver).  Scalars, reductions and states are always double.
template <typename R>
struct BiWST {
  using F = cplx<R>;
  F *r, *rhat, *p, *v, *s, *t, *x, *b;
  F *be, *bo, *tmp;    // even-odd solve: b_e, b_o, odd-parity scratch
  TileRed tr;       // tile-ordered reduction scratch (reduce.cuh)
  unsigned *ticket;
  unsigned long long *ctr;   // dynamic chunk counter (dslash kernels), reset by their last block
  unsigned long long *ctr2;  // counter of the eo first-half kernels, reset by the following kernel
  double *red;               // distributed solve: rank-local sums handed to the all-reduce
  BiState *st;
  // batched solves: group g of kMaxGroup rhs (blockIdx.y) owns field slice
  // g*gfield, tile partials g*gpart, ticket area g*256 B and states
  // g*kMaxGroup
  int64_t gfield, gpart;
  __host__ __device__ __forceinline__ BiWST at(int g) const {
    BiWST o = *this;
    const int64_t f = (int64_t)g * gfield;
    F *BiWST::*fs[11] = {&BiWST::r, &BiWST::rhat, &BiWST::p, &BiWST::v, &BiWST::s, &BiWST::t,
                         &BiWST::x, &BiWST::b, &BiWST::be, &BiWST::bo, &BiWST::tmp};
#pragma unroll
    for (int i = 0; i < 11; ++i)
      if (o.*fs[i]) o.*fs[i] += f;
    o.tr.tiles += (int64_t)g * gpart;
    o.ticket = (unsigned *)((char *)ticket + 256 * (int64_t)g);
    o.ctr = (unsigned long long *)((char *)ctr + 256 * (int64_t)g);
    o.ctr2 = (unsigned long long *)((char *)ctr2 + 256 * (int64_t)g);
    o.red = (double *)((char *)red + 256 * (int64_t)g);
    o.st += (int64_t)g * 4;
    return o;
  }
};
using BiWS = BiWST<double>;

// double-precision dot-product pieces of fields of either precision
template <typename R>
__device__ __forceinline__ double dre(C<R> a, C<R> b) {  // Re conj(a) b
  return (double)a.re * (double)b.re + (double)a.im * (double)b.im;
}
template <typename R>
__device__ __forceinline__ double dim(C<R> a, C<R> b) {  // Im conj(a) b
  return (double)a.re * (double)b.im - (double)a.im * (double)b.re;
}
template <typename R>
__device__ __forceinline__ double dnorm2(C<R> a) {
  return (double)a.re * (double)a.re + (double)a.im * (double)a.im;
}
template <typename R>
__device__ __forceinline__ C<R> cvt(C<double> a) {
  return C<R>((R)a.re, (R)a.im);
}
template <int NR>
__device__ __forceinline__ bool any_status(const BiState *st, int want) {
  bool any = false;
#pragma unroll
  for (int r = 0; r < NR; ++r) any |= (st[r].status == want);
  return any;
}

__device__ __forceinline__ C<double> cdiv(C<double> a, C<double> b) {
  double d = b.re * b.re + b.im * b.im;
  return C<double>((a.re * b.re + a.im * b.im) / d, (a.im * b.re - a.re * b.im) / d);
}
__device__ __forceinline__ bool czero(C<double> a) { return a.re == 0.0 && a.im == 0.0; }
__device__ __forceinline__ double cabs2(C<double> a) { return a.re * a.re + a.im * a.im; }
__device__ __forceinline__ bool cfinite(C<double> a) { return isfinite(a.re) && isfinite(a.im); }

// fp32 streaming kernels with two sites per thread (bi_k2v / k4v / k5v)
#ifndef MGT_F32_PAIRS
#define MGT_F32_PAIRS 1
#endif

// resident blocks per SM of the even-odd stencil kernels: fp64 at 3 (168
// registers, no spills); the fp32 inner kernels need fewer registers
#ifndef MGT_F32_MINB
#define MGT_F32_MINB 3
#endif
template <typename R>
constexpr int eo_minb() {
  return sizeof(R) == 4 ? MGT_F32_MINB : 3;
}

// Experiment (off by default, -DMGT_F32_BLOCKED=1): the mixed solver's fp32
// fields (its own workspace: r, rhat, p, v, s, t, x, tmp) in the row-blocked
// layout of eo_core.cuh (EoGeom::Bh): the stencil kernels address them
// through eo_base / eo_cstride, mx_begin / mx_accum translate from / to the
// fp64 component planes, and the streaming kernels (bi_k2v / k4v / k5v) are
// position-wise, so they do not care.  Motivation: a microbenchmark
// (tools/micro/many_planes.cu) streams 48 component planes at 2.2 TB/s and
// the same bytes in a blocked layout at 5.7-6.0 TB/s, and a 4-rhs stencil
// pass touches ~200 distinct 2 MB pages per SM at a time.  Result
// (profiles/r02s5_blocked_f32_fields_ab_rejected.txt): correct (same
// iteration counts, solver tests pass) and SLOWER -- bi_eo_first 150 -> 154
// us, bi_k1_eo 242 -> 262, bi_k3_eo 251 -> 353 (32^4, 4 rhs), solver -8 %:
// the stencils are not limited by the number of pages they stream.
#ifndef MGT_F32_BLOCKED
#define MGT_F32_BLOCKED 0
#endif
#if MGT_F32_BLOCKED && MGT_F32_STENCIL_PAIRS
#error "the two-sites-per-thread fp32 stencils (eo_pair.cuh) address SoA planes: build them with -DMGT_F32_BLOCKED=0"
#endif
template <typename R>
constexpr bool eo_blk() {
  return sizeof(R) == 4 && MGT_F32_BLOCKED;
}
// 1: fp32 K1 / K3 load the centre field (and K1's rhat) before the hops
// instead of after them (two latency phases fewer).  Measured 3 % SLOWER
// (32^4: 425 -> 440 us per iteration and rhs): off.
#ifndef MGT_F32_PRELOAD
#define MGT_F32_PRELOAD 0
#endif
template <typename R>
constexpr bool eo_pre() {
  return sizeof(R) == 4 && MGT_F32_PRELOAD;
}

#define MGT_SITE_LOOP(M, V) for (int64_t o = (M).first(); o < (V); o += (M).stride())

// Dynamically scheduled loop over chunks of RhsMap<NR>::SPB ordered sites
// (next_chunk): every thread of the block iterates (the body must not
// return/break early); `o` is the thread's ordered site (may be >= V in the
// last chunk), `chunk` the chunk index; NCH receives the number of chunks.
#define MGT_DYN_LOOP(M, V, CTR, NCH)                                                  \
  NCH = ((V) + (M).SPB - 1) / (M).SPB;                                                \
  for (int64_t chunk = next_chunk(CTR), o = chunk * (M).SPB + (M).local; chunk < NCH; \
       chunk = next_chunk(CTR), o = chunk * (M).SPB + (M).local)

// Static chunk loop of the streaming kernels: block b takes chunks b, b +
// grid, ... of SPB ordered sites (every thread iterates; `o` may be >= V in
// the last chunk).  Their reductions are tile-ordered (reduce.cuh), so the
// grid size does not enter the result.
#define MGT_CHUNK_LOOP(M, V)                                                                              \
  _Pragma("unroll 1") for (int64_t chunk = blockIdx.x, nch_ = ((V) + (M).SPB - 1) / (M).SPB, o = chunk * (M).SPB + (M).local; \
       chunk < nch_; chunk += gridDim.x, o = chunk * (M).SPB + (M).local)

// Last-block scalar recurrences of the stencil kernels (shared by the full
// and the even-odd kernels).  They also reset the chunk counters.
template <int M, class W>
__device__ __forceinline__ void store_red(const W &w, const double (&out)[M]) {
  if (threadIdx.x == 0) {
#pragma unroll
    for (int j = 0; j < M; ++j) w.red[j] = out[j];
  }
}

template <int NR, class W>
__device__ __forceinline__ void k1_logic(const W &w, const double (&out)[NR * 2]) {
  const int r = threadIdx.x;
  if (r < NR && w.st[r].status == ST_RUN) {
    BiState &s = w.st[r];
    C<double> sigma(out[2 * r], out[2 * r + 1]);
    s.matvecs += 1;
    if (czero(sigma) || !cfinite(sigma)) {
      s.status = ST_BREAK;
      s.reason = 2;
    } else {
      s.alpha = cdiv(s.rho, sigma);
    }
  }
}

template <int NR, int DIST = 0, class W>
__device__ __forceinline__ void k1_finish(const W &w, int64_t sites) {
  double out[NR * 2];
  tiles_final<NR * 2>(w.tr, sites, w.ticket, out);
  if (threadIdx.x == 0) {
    *w.ctr = 0ull;
    *w.ctr2 = 0ull;
  }
  if (DIST)
    store_red<NR * 2>(w, out);
  else
    k1_logic<NR>(w, out);
}

template <int NR, class W>
__device__ __forceinline__ void k3_logic(const W &w, const double (&out)[NR * 3]) {
  const int r = threadIdx.x;
  if (r < NR && w.st[r].status == ST_RUN) {
    BiState &s = w.st[r];
    C<double> ts(out[3 * r], out[3 * r + 1]);
    const double tt = out[3 * r + 2];
    s.matvecs += 1;
    if (s.half) {
      s.omega = C<double>(0.0, 0.0);
    } else if (tt == 0.0 || !isfinite(tt)) {
      s.status = ST_BREAK;
      s.reason = 2;
    } else {
      s.omega = C<double>(ts.re / tt, ts.im / tt);
    }
  }
}

template <int NR, int DIST = 0, class W>
__device__ __forceinline__ void k3_finish(const W &w, int64_t sites) {
  double out[NR * 3];
  tiles_final<NR * 3>(w.tr, sites, w.ticket, out);
  if (threadIdx.x == 0) {
    *w.ctr = 0ull;
    *w.ctr2 = 0ull;
  }
  if (DIST)
    store_red<NR * 3>(w, out);
  else
    k3_logic<NR>(w, out);
}

template <int NR, class W>
__device__ __forceinline__ void resid_logic(const W &w, const double (&out)[NR]) {
  const int r = threadIdx.x;
  if (r < NR) {
    BiState &s = w.st[r];
    const int st = s.status;
    if (st == ST_CONV || st == ST_MAXIT || st == ST_BREAK) {
      s.true_r2 = out[r];
      s.matvecs += 1;
      if (s.true_r2 <= s.tol2) {
        s.status = ST_DONE;
        s.reason = 0;
      } else if (st == ST_CONV && s.iters < s.maxit) {
        s.status = ST_RESTART;  // recursion drifted from the true residual
      } else {
        s.status = ST_DONE;
        if (s.reason == 0) s.reason = 1;
      }
    }
  }
}

template <int NR, int DIST = 0, class W>
__device__ __forceinline__ void resid_finish(const W &w, int64_t sites) {
  double out[NR];
  tiles_final<NR>(w.tr, sites, w.ticket, out);
  if (threadIdx.x == 0) {
    *w.ctr = 0ull;
    *w.ctr2 = 0ull;
  }
  if (DIST)
    store_red<NR>(w, out);
  else
    resid_logic<NR>(w, out);
}

template <int NR>
__device__ __forceinline__ bool resid_active(int st) {
  return st == ST_CONV || st == ST_MAXIT || st == ST_BREAK;
}

// ---------------------------------------------------------------------------
// init: b -> workspace, r = rhat = p = b, x = 0, |b|^2
template <int NR, class W>
__device__ __forceinline__ void init_logic(const W &w, const double (&out)[NR], double tol, int maxit,
                                           int use_bfull) {
  const int r = threadIdx.x;
  if (r < NR) {
    BiState &s = w.st[r];
    const double b2 = out[r];
    // even-odd: the stopping norm is the FULL right-hand side's (the Schur
    // residual is the full residual), set by bi_eo_split
    s.b2 = use_bfull ? s.bfull2 : b2;
    s.r2 = b2;
    s.s2 = b2;
    s.true_r2 = b2;
    s.tol2 = tol * tol * s.b2;
    s.rho = C<double>(b2, 0.0);
    s.alpha = C<double>(1.0, 0.0);
    s.omega = C<double>(1.0, 0.0);
    s.beta = C<double>(0.0, 0.0);
    s.dotq = C<double>(0.0, 0.0);
    s.half = 0;
    s.iters = 0;
    s.maxit = maxit;
    s.matvecs = 0;
    s.reason = 0;
    s.status = (b2 == 0.0) ? ST_DONE : ST_RUN;
  }
}

template <int NR, int DIST = 0>
__global__ void __launch_bounds__(kRedBlock) bi_init(int64_t V, const double2 *__restrict__ b, BiWS w_, double tol,
                                                     int maxit, int use_bfull) {
  const BiWS w = w_.at(blockIdx.y);
  RhsMap<NR> m;
  b += (int64_t)blockIdx.y * NR * 12 * V;
  MGT_CHUNK_LOOP(m, V) {
    double acc[1] = {0.0};
    if (o < V) {
      const int64_t base = (int64_t)m.rhs * 12 * V + o;
#pragma unroll
      for (int c = 0; c < 12; ++c) {
        const int64_t q = base + (int64_t)c * V;
        double2 bb = b[q];
        w.b[q] = bb;
        w.r[q] = bb;
        w.rhat[q] = bb;
        w.p[q] = bb;
        w.x[q] = make_double2(0.0, 0.0);
        acc[0] += bb.x * bb.x + bb.y * bb.y;
      }
    }
    tile_publish<NR, 1>(acc, w.tr, m.tile(o), n_tiles(V), m.rhs);
  }
  if (last_block(w.ticket)) {
    double out[NR];
    tiles_final<NR>(w.tr, V, w.ticket, out);
    if (DIST)
      store_red<NR>(w, out);
    else
      init_logic<NR>(w, out, tol, maxit, use_bfull);
  }
}

// K1: v = A p ; sigma = (rhat, v)
template <int NR, int RECON, int DIST = 0>
__global__ void __launch_bounds__(kRedBlock, 3) bi_k1(WilsonParams P, LinkField<double, RECON> L, BiWS w_) {
  const BiWS w = w_.at(blockIdx.y);
  if (!any_status<NR>(w.st, ST_RUN)) return;
  RhsMap<NR> m;
  const bool run_me = w.st[m.rhs].status == ST_RUN;
  const int64_t V = P.g.V;
  const int64_t off = (int64_t)m.rhs * 12 * V;
  int64_t nchunks = 0;
  MGT_DYN_LOOP(m, V, w.ctr, nchunks) {
    double acc[2] = {0.0, 0.0};
    if (run_me && o < V) {
      const int64_t site = sched_site(P.sched, o);
      C<double> y[4][3], xc[4][3];
      wilson_eval<double, RECON>(P, w.p + off, L, site, y, xc, m.rhs);
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const int64_t q = off + (int64_t)(a * 3 + c) * V + site;
          stc(w.v + q, y[a][c]);
          C<double> rh = ldc(w.rhat + q);
          acc[0] += rh.re * y[a][c].re + rh.im * y[a][c].im;
          acc[1] += rh.re * y[a][c].im - rh.im * y[a][c].re;
        }
    }
    if (run_me) tile_publish<NR, 2>(acc, w.tr, m.tile(o), n_tiles(V), m.rhs);
  }
  (void)nchunks;
  if (last_block(w.ticket)) k1_finish<NR, DIST>(w, V);
}

template <int NR, class W>
__device__ __forceinline__ void k2_logic(const W &w, const double (&out)[NR]) {
  const int r = threadIdx.x;
  if (r < NR && w.st[r].status == ST_RUN) {
    BiState &s = w.st[r];
    s.s2 = out[r];
    s.half = (s.s2 <= s.tol2) ? 1 : 0;
  }
}

// K2: s = r - alpha v ; |s|^2
template <int NR, int DIST = 0, typename R = double>
__global__ void __launch_bounds__(kRedBlock) bi_k2(int64_t V, BiWST<R> w_) {
  const BiWST<R> w = w_.at(blockIdx.y);
  if (!any_status<NR>(w.st, ST_RUN)) return;
  RhsMap<NR> m;
  const bool run_me = w.st[m.rhs].status == ST_RUN;
  const C<R> al = cvt<R>(w.st[m.rhs].alpha);
  if (run_me) {
      MGT_CHUNK_LOOP(m, V) {
      double acc[1] = {0.0};
      if (o < V) {
        const int64_t base = (int64_t)m.rhs * 12 * V + o;
#pragma unroll
        for (int c = 0; c < 12; ++c) {
          const int64_t q = base + (int64_t)c * V;
          C<R> ss = ldc(w.r + q) - al * ldc(w.v + q);
          stc(w.s + q, ss);
          acc[0] += dnorm2(ss);
        }
      }
      tile_publish<NR, 1>(acc, w.tr, m.tile(o), n_tiles(V), m.rhs);
    }
  }
  if (last_block(w.ticket)) {
    double out[NR];
    tiles_final<NR>(w.tr, V, w.ticket, out);
    if (DIST)
      store_red<NR>(w, out);
    else
      k2_logic<NR>(w, out);
  }
}

// K3: t = A s ; (t, s), |t|^2
template <int NR, int RECON, int DIST = 0>
__global__ void __launch_bounds__(kRedBlock, 3) bi_k3(WilsonParams P, LinkField<double, RECON> L, BiWS w_) {
  const BiWS w = w_.at(blockIdx.y);
  if (!any_status<NR>(w.st, ST_RUN)) return;
  RhsMap<NR> m;
  const bool run_me = w.st[m.rhs].status == ST_RUN;
  const int64_t V = P.g.V;
  const int64_t off = (int64_t)m.rhs * 12 * V;
  int64_t nchunks = 0;
  MGT_DYN_LOOP(m, V, w.ctr, nchunks) {
    double acc[3] = {0.0, 0.0, 0.0};
    if (run_me && o < V) {
      const int64_t site = sched_site(P.sched, o);
      C<double> y[4][3], xc[4][3];
      wilson_eval<double, RECON>(P, w.s + off, L, site, y, xc, m.rhs);
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          stc(w.t + off + (int64_t)(a * 3 + c) * V + site, y[a][c]);
          const C<double> tt = y[a][c], ss = xc[a][c];
          acc[0] += tt.re * ss.re + tt.im * ss.im;
          acc[1] += tt.re * ss.im - tt.im * ss.re;
          acc[2] += cabs2(tt);
        }
    }
    if (run_me) tile_publish<NR, 3>(acc, w.tr, m.tile(o), n_tiles(V), m.rhs);
  }
  (void)nchunks;
  if (last_block(w.ticket)) k3_finish<NR, DIST>(w, V);
}

template <int NR, class W>
__device__ __forceinline__ void k4_logic(const W &w, const double (&out)[NR * 3]) {
  const int r = threadIdx.x;
  if (r < NR && w.st[r].status == ST_RUN) {
    BiState &s = w.st[r];
    C<double> rho_new(out[3 * r], out[3 * r + 1]);
    s.r2 = out[3 * r + 2];
    s.iters += 1;
    if (s.r2 <= s.tol2 || s.half) {
      s.status = ST_CONV;
    } else if (czero(rho_new) || czero(s.omega) || !isfinite(s.r2)) {
      s.status = ST_BREAK;
      s.reason = 2;
    } else {
      s.beta = cdiv(rho_new, s.rho) * cdiv(s.alpha, s.omega);
      s.rho = rho_new;
      if (s.iters >= s.maxit) {
        s.status = ST_MAXIT;
        s.reason = 1;
      }
    }
  }
}

// K4: x += alpha p + omega s ; r = s - omega t ; rho' = (rhat, r), |r|^2
template <int NR, int DIST = 0, typename R = double>
__global__ void __launch_bounds__(kRedBlock) bi_k4(int64_t V, BiWST<R> w_) {
  const BiWST<R> w = w_.at(blockIdx.y);
  if (!any_status<NR>(w.st, ST_RUN)) return;
  RhsMap<NR> m;
  const bool run_me = w.st[m.rhs].status == ST_RUN;
  const C<R> al = cvt<R>(w.st[m.rhs].alpha), om = cvt<R>(w.st[m.rhs].omega);
  if (run_me) {
      MGT_CHUNK_LOOP(m, V) {
      double acc[3] = {0.0, 0.0, 0.0};
      if (o < V) {
        const int64_t base = (int64_t)m.rhs * 12 * V + o;
#pragma unroll
        for (int c = 0; c < 12; ++c) {
          const int64_t q = base + (int64_t)c * V;
          C<R> xx = ldc(w.x + q), pp = ldc(w.p + q), ss = ldc(w.s + q), tt = ldc(w.t + q), rh = ldc(w.rhat + q);
          xx = xx + al * pp + om * ss;
          C<R> rr = ss - om * tt;
          stc(w.x + q, xx);
          stc(w.r + q, rr);
          acc[0] += dre(rh, rr);
          acc[1] += dim(rh, rr);
          acc[2] += dnorm2(rr);
        }
      }
      tile_publish<NR, 3>(acc, w.tr, m.tile(o), n_tiles(V), m.rhs);
    }
  }
  if (last_block(w.ticket)) {
    double out[NR * 3];
    tiles_final<NR * 3>(w.tr, V, w.ticket, out);
    if (DIST)
      store_red<NR * 3>(w, out);
    else
      k4_logic<NR>(w, out);
  }
}

// K5: p = r + beta (p - omega v)
template <int NR, typename R = double>
__global__ void __launch_bounds__(kRedBlock) bi_k5(int64_t V, BiWST<R> w_) {
  const BiWST<R> w = w_.at(blockIdx.y);
  if (!any_status<NR>(w.st, ST_RUN)) return;
  RhsMap<NR> m;
  if (w.st[m.rhs].status != ST_RUN) return;
  const C<R> be = cvt<R>(w.st[m.rhs].beta), om = cvt<R>(w.st[m.rhs].omega);
  MGT_SITE_LOOP(m, V) {
    const int64_t base = (int64_t)m.rhs * 12 * V + o;
#pragma unroll
    for (int c = 0; c < 12; ++c) {
      const int64_t q = base + (int64_t)c * V;
      stc(w.p + q, ldc(w.r + q) + be * (ldc(w.p + q) - om * ldc(w.v + q)));
    }
  }
}

// fp32 streaming kernels of the mixed solver's inner BiCGStab (K2, K4, K5
// above for R = float): two adjacent sites per thread so every access is one
// 16-byte load/store of two complex<float> (half the memory instructions
// of the one-site form).  A chunk covers 2 SPB ordered sites; a warp's 64
// sites are tiles 2k (lanes 0-15) and 2k+1 (lanes 16-31), reduced with
// tile_publish_pairs.  Needs an even site count (every extent even).
__device__ __forceinline__ void ld2c(const float2 *p, C<float> &a, C<float> &b) {
  const float4 v = __ldg(reinterpret_cast<const float4 *>(p));
  a = C<float>(v.x, v.y);
  b = C<float>(v.z, v.w);
}
__device__ __forceinline__ void st2c(float2 *p, C<float> a, C<float> b) {
  *reinterpret_cast<float4 *>(p) = make_float4(a.re, a.im, b.re, b.im);
}
#define MGT_PAIR_LOOP(M, V)                                                                                      \
  _Pragma("unroll 1") for (int64_t chunk = blockIdx.x, nch_ = ((V) + 2 * (M).SPB - 1) / (2 * (M).SPB),           \
                                   o = chunk * 2 * (M).SPB + 2 * (M).local;                                     \
                           chunk < nch_; chunk += gridDim.x, o = chunk * 2 * (M).SPB + 2 * (M).local)

template <int NR>
__global__ void __launch_bounds__(kRedBlock) bi_k2v(int64_t V, BiWST<float> w_) {
  const BiWST<float> w = w_.at(blockIdx.y);
  if (!any_status<NR>(w.st, ST_RUN)) return;
  RhsMap<NR> m;
  if (w.st[m.rhs].status == ST_RUN) {
    const C<float> al = cvt<float>(w.st[m.rhs].alpha);
    MGT_PAIR_LOOP(m, V) {
      double acc[1] = {0.0};
      if (o < V) {
        const int64_t base = (int64_t)m.rhs * 12 * V + o;
#pragma unroll
        for (int c = 0; c < 12; ++c) {
          const int64_t q = base + (int64_t)c * V;
          C<float> r0, r1, v0, v1;
          ld2c(w.r + q, r0, r1);
          ld2c(w.v + q, v0, v1);
          const C<float> s0 = r0 - al * v0, s1 = r1 - al * v1;
          st2c(w.s + q, s0, s1);
          acc[0] += dnorm2(s0);
          acc[0] += dnorm2(s1);
        }
      }
      tile_publish_pairs<NR, 1>(acc, w.tr, o >> 5, n_tiles(V), m.rhs);
    }
  }
  if (last_block(w.ticket)) {
    double out[NR];
    tiles_final<NR>(w.tr, V, w.ticket, out);
    k2_logic<NR>(w, out);
  }
}

template <int NR>
__global__ void __launch_bounds__(kRedBlock) bi_k4v(int64_t V, BiWST<float> w_) {
  const BiWST<float> w = w_.at(blockIdx.y);
  if (!any_status<NR>(w.st, ST_RUN)) return;
  RhsMap<NR> m;
  if (w.st[m.rhs].status == ST_RUN) {
    const C<float> al = cvt<float>(w.st[m.rhs].alpha), om = cvt<float>(w.st[m.rhs].omega);
    MGT_PAIR_LOOP(m, V) {
      double acc[3] = {0.0, 0.0, 0.0};
      if (o < V) {
        const int64_t base = (int64_t)m.rhs * 12 * V + o;
#pragma unroll
        for (int c = 0; c < 12; ++c) {
          const int64_t q = base + (int64_t)c * V;
          C<float> x0, x1, p0, p1, s0, s1, t0, t1, h0, h1;
          ld2c(w.x + q, x0, x1);
          ld2c(w.p + q, p0, p1);
          ld2c(w.s + q, s0, s1);
          ld2c(w.t + q, t0, t1);
          ld2c(w.rhat + q, h0, h1);
          const C<float> r0 = s0 - om * t0, r1 = s1 - om * t1;
          st2c(w.x + q, x0 + al * p0 + om * s0, x1 + al * p1 + om * s1);
          st2c(w.r + q, r0, r1);
          acc[0] += dre(h0, r0);
          acc[1] += dim(h0, r0);
          acc[2] += dnorm2(r0);
          acc[0] += dre(h1, r1);
          acc[1] += dim(h1, r1);
          acc[2] += dnorm2(r1);
        }
      }
      tile_publish_pairs<NR, 3>(acc, w.tr, o >> 5, n_tiles(V), m.rhs);
    }
  }
  if (last_block(w.ticket)) {
    double out[NR * 3];
    tiles_final<NR * 3>(w.tr, V, w.ticket, out);
    k4_logic<NR>(w, out);
  }
}

template <int NR>
__global__ void __launch_bounds__(kRedBlock) bi_k5v(int64_t V, BiWST<float> w_) {
  const BiWST<float> w = w_.at(blockIdx.y);
  if (!any_status<NR>(w.st, ST_RUN)) return;
  RhsMap<NR> m;
  if (w.st[m.rhs].status != ST_RUN) return;
  const C<float> be = cvt<float>(w.st[m.rhs].beta), om = cvt<float>(w.st[m.rhs].omega);
  MGT_PAIR_LOOP(m, V) {
    if (o < V) {
      const int64_t base = (int64_t)m.rhs * 12 * V + o;
#pragma unroll
      for (int c = 0; c < 12; ++c) {
        const int64_t q = base + (int64_t)c * V;
        C<float> r0, r1, p0, p1, v0, v1;
        ld2c(w.r + q, r0, r1);
        ld2c(w.p + q, p0, p1);
        ld2c(w.v + q, v0, v1);
        st2c(w.p + q, r0 + be * (p0 - om * v0), r1 + be * (p1 - om * v1));
      }
    }
  }
}

// True residual r = b - A x for every rhs that stopped (CONV/MAXIT/BREAK)
template <int NR, int RECON, int DIST = 0>
__global__ void __launch_bounds__(kRedBlock, 3) bi_resid(WilsonParams P, LinkField<double, RECON> L, BiWS w_) {
  const BiWS w = w_.at(blockIdx.y);
  bool any = false;
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    const int st = w.st[r].status;
    any |= (st == ST_CONV || st == ST_MAXIT || st == ST_BREAK);
  }
  if (!any) return;
  RhsMap<NR> m;
  const int st_me = w.st[m.rhs].status;
  const bool act_me = (st_me == ST_CONV || st_me == ST_MAXIT || st_me == ST_BREAK);
  const int64_t V = P.g.V;
  const int64_t off = (int64_t)m.rhs * 12 * V;
  int64_t nchunks = 0;
  MGT_DYN_LOOP(m, V, w.ctr, nchunks) {
    double acc[1] = {0.0};
    if (act_me && o < V) {
      const int64_t site = sched_site(P.sched, o);
      C<double> y[4][3], xc[4][3];
      wilson_eval<double, RECON>(P, w.x + off, L, site, y, xc, m.rhs);
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const int64_t q = off + (int64_t)(a * 3 + c) * V + site;
          C<double> rr = ldc(w.b + q) - y[a][c];
          stc(w.r + q, rr);
          acc[0] += cabs2(rr);
        }
    }
    if (act_me) tile_publish<NR, 1>(acc, w.tr, m.tile(o), n_tiles(V), m.rhs);
  }
  (void)nchunks;
  if (last_block(w.ticket)) resid_finish<NR, DIST>(w, V);
}

template <int NR, class W>
__device__ __forceinline__ void restart_logic(const W &w, const double (&out)[NR]) {
  const int r = threadIdx.x;
  if (r < NR && w.st[r].status == ST_RESTART) {
    BiState &s = w.st[r];
    s.r2 = out[r];
    s.rho = C<double>(s.r2, 0.0);
    s.alpha = C<double>(1.0, 0.0);
    s.omega = C<double>(1.0, 0.0);
    s.half = 0;
    s.status = ST_RUN;
  }
}

// Restart for rhs flagged ST_RESTART: rhat = p = r (r holds the true residual)
template <int NR, int DIST = 0>
__global__ void __launch_bounds__(kRedBlock) bi_restart(int64_t V, BiWS w_) {
  const BiWS w = w_.at(blockIdx.y);
  if (!any_status<NR>(w.st, ST_RESTART)) return;
  RhsMap<NR> m;
  const bool act_me = w.st[m.rhs].status == ST_RESTART;
  if (act_me) {
    MGT_CHUNK_LOOP(m, V) {
      double acc[1] = {0.0};
      if (o < V) {
        const int64_t base = (int64_t)m.rhs * 12 * V + o;
#pragma unroll
        for (int c = 0; c < 12; ++c) {
          const int64_t q = base + (int64_t)c * V;
          double2 rr = w.r[q];
          w.rhat[q] = rr;
          w.p[q] = rr;
          acc[0] += rr.x * rr.x + rr.y * rr.y;
        }
      }
      tile_publish<NR, 1>(acc, w.tr, m.tile(o), n_tiles(V), m.rhs);
    }
  }
  if (last_block(w.ticket)) {
    double out[NR];
    tiles_final<NR>(w.tr, V, w.ticket, out);
    if (DIST)
      store_red<NR>(w, out);
    else
      restart_logic<NR>(w, out);
  }
}

// copy x out and q = vdot(b, x) per rhs (Hutchinson quadratic form, trace.py:104)
template <int NR, int DIST = 0>
__global__ void __launch_bounds__(kRedBlock) bi_final(int64_t V, double2 *__restrict__ xout, BiWS w_) {
  const BiWS w = w_.at(blockIdx.y);
  xout += (int64_t)blockIdx.y * NR * 12 * V;
  RhsMap<NR> m;
  MGT_CHUNK_LOOP(m, V) {
    double acc[2] = {0.0, 0.0};
    if (o < V) {
      const int64_t base = (int64_t)m.rhs * 12 * V + o;
#pragma unroll
      for (int c = 0; c < 12; ++c) {
        const int64_t q = base + (int64_t)c * V;
        C<double> bb = ldc(w.b + q), xx = ldc(w.x + q);
        stc(xout + q, xx);
        acc[0] += bb.re * xx.re + bb.im * xx.im;
        acc[1] += bb.re * xx.im - bb.im * xx.re;
      }
    }
    tile_publish<NR, 2>(acc, w.tr, m.tile(o), n_tiles(V), m.rhs);
  }
  if (last_block(w.ticket)) {
    double out[NR * 2];
    tiles_final<NR * 2>(w.tr, V, w.ticket, out);
    if (DIST)
      store_red<NR * 2>(w, out);
    else if (threadIdx.x < NR)
      w.st[threadIdx.x].dotq = C<double>(out[2 * threadIdx.x], out[2 * threadIdx.x + 1]);
  }
}

// ---------------------------------------------------------------------------
// Even-odd (Schur) solve, eo_core.cuh.  Fields in the workspace are parity
// fields of Vh sites; the BLAS-1 kernels above run unchanged with V = Vh.
struct BiEo {
  EoGeom E;
  Sched sh;  // slab schedule over cb indices
  EoRoles R;
};

// b (full) -> b_e, b_o, tmp = u_o = Dg^-1 G_out b_o ; |b|^2 of the full rhs
template <int NR>
__global__ void __launch_bounds__(kRedBlock) bi_eo_split(BiEo X, const double2 *__restrict__ b, BiWS w_, double g5out) {
  const BiWS w = w_.at(blockIdx.y);
  b += (int64_t)blockIdx.y * NR * 12 * X.E.g.V;
  RhsMap<NR> m;
  const int64_t Vh = X.E.Vh, V = X.E.g.V;
  const C<double> iu(X.R.iu_re, X.R.iu_im), id(X.R.id_re, X.R.id_im);
  MGT_CHUNK_LOOP(m, Vh) {
    double acc[1] = {0.0};
    if (o < Vh) {
      int x[4];
      const int64_t fe = eo_coords(X.E, 0, o, x);
      const int64_t fo = eo_coords(X.E, 1, o, x);
      const double2 *B = b + (int64_t)m.rhs * 12 * V;
      const int64_t hb = (int64_t)m.rhs * 12 * Vh + o;
#pragma unroll
      for (int k = 0; k < 12; ++k) {
        const C<double> e = ldc(B + (int64_t)k * V + fe), od = ldc(B + (int64_t)k * V + fo);
        stc(w.be + hb + (int64_t)k * Vh, e);
        stc(w.bo + hb + (int64_t)k * Vh, od);
        const C<double> u = k < 6 ? iu * od : id * (g5out * od);
        stc(w.tmp + hb + (int64_t)k * Vh, u);
        acc[0] += cabs2(e) + cabs2(od);
      }
    }
    tile_publish<NR, 1>(acc, w.tr, m.tile(o), n_tiles(Vh), m.rhs);
  }
  if (last_block(w.ticket)) {
    double out[NR];
    tiles_final<NR>(w.tr, Vh, w.ticket, out);
    if (threadIdx.x < NR) w.st[threadIdx.x].bfull2 = out[threadIdx.x];
  }
}

// bh_e = G_out [ G_out b_e + 1/2 H_eo u_o ]  -> w.b
template <int NR, int RECON>
__global__ void __launch_bounds__(kRedBlock, 3) bi_eo_rhs(BiEo X, LinkField<double, RECON> le,
                                                          LinkField<double, RECON> lo, BiWS w_) {
  const BiWS w = w_.at(blockIdx.y);
  RhsMap<NR> m;
  const int64_t Vh = X.E.Vh;
  const int64_t off = (int64_t)m.rhs * 12 * Vh;
  MGT_SITE_LOOP(m, Vh) {
    const int64_t c = sched_site(X.sh, o);
    C<double> y[4][3], cc[4][3];
    eo_eval<double, RECON>(X.E, 0, X.R.rhs, w.tmp + off, w.be + off, le, lo, c, y, cc);
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int k = 0; k < 3; ++k) stc(w.b + off + (int64_t)(a * 3 + k) * Vh + c, y[a][k]);
  }
}

// first half of S: tmp = Dg^-1 H_oe (G_in f), f = p / s / x (mode 0: rhs
// still iterating, mode 1: rhs whose true residual is due)
template <int NR, int RECON, typename R = double, int MINB = eo_minb<R>()>
__global__ void __launch_bounds__(kRedBlock, MINB) bi_eo_first(BiEo X, LinkField<R, RECON> le,
                                                            LinkField<R, RECON> lo, const cplx<R> *f, BiWST<R> w_,
                                                            int mode) {
  const BiWST<R> w = w_.at(blockIdx.y);
  f += (int64_t)blockIdx.y * w_.gfield;
  bool any = false;
#pragma unroll
  for (int r = 0; r < NR; ++r) any |= mode ? resid_active<NR>(w.st[r].status) : w.st[r].status == ST_RUN;
  if (!any) return;
  RhsMap<NR> m;
  const int stm = w.st[m.rhs].status;
  const bool act = mode ? resid_active<NR>(stm) : stm == ST_RUN;
  const int64_t Vh = X.E.Vh;
  const int64_t off = (int64_t)m.rhs * 12 * Vh;
  int64_t nchunks = 0;
  MGT_DYN_LOOP(m, Vh, w.ctr2, nchunks) {
    if (act && o < Vh) {
      const int64_t c = sched_site(X.sh, o);
      C<R> y[4][3], cc[4][3];
      constexpr bool BLK = eo_blk<R>();
      eo_eval<R, RECON, BLK>(X.E, 1, X.R.first, f + off, nullptr, lo, le, c, y, cc);
      const int64_t cs = eo_cstride<BLK>(X.E), bc = off + eo_base<BLK>(X.E, c);
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int k = 0; k < 3; ++k) stc(w.tmp + bc + (int64_t)(a * 3 + k) * cs, y[a][k]);
    }
  }
}

// K1 (eo): v = S p = G_out [ Dg G_in p - 1/4 H_eo tmp ] ; sigma = (rhat, v)
template <int NR, int RECON, typename R = double, int MINB = eo_minb<R>()>
__global__ void __launch_bounds__(kRedBlock, MINB) bi_k1_eo(BiEo X, LinkField<R, RECON> le,
                                                         LinkField<R, RECON> lo, BiWST<R> w_) {
  const BiWST<R> w = w_.at(blockIdx.y);
  if (!any_status<NR>(w.st, ST_RUN)) return;
  RhsMap<NR> m;
  const bool run_me = w.st[m.rhs].status == ST_RUN;
  const int64_t Vh = X.E.Vh;
  const int64_t off = (int64_t)m.rhs * 12 * Vh;
  int64_t nchunks = 0;
  MGT_DYN_LOOP(m, Vh, w.ctr, nchunks) {
    double acc[2] = {0.0, 0.0};
    if (run_me && o < Vh) {
      const int64_t c = sched_site(X.sh, o);
      C<R> y[4][3], cc[4][3];
      constexpr bool BLK = eo_blk<R>(), PRE = eo_pre<R>();
      const int64_t cs = eo_cstride<BLK>(X.E), bc = off + eo_base<BLK>(X.E, c);
      C<R> rhp[4][3];
      if constexpr (PRE) {
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int k = 0; k < 3; ++k) rhp[a][k] = ldc(w.rhat + bc + (int64_t)(a * 3 + k) * cs);
      }
      eo_eval<R, RECON, BLK, PRE>(X.E, 0, X.R.second, w.tmp + off, w.p + off, le, lo, c, y, cc);
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const int64_t q = bc + (int64_t)(a * 3 + k) * cs;
          stc(w.v + q, y[a][k]);
          C<R> rh;
          if constexpr (PRE)
            rh = rhp[a][k];
          else
            rh = ldc(w.rhat + q);
          acc[0] += dre(rh, y[a][k]);
          acc[1] += dim(rh, y[a][k]);
        }
    }
    if (run_me) tile_publish<NR, 2>(acc, w.tr, m.tile(o), n_tiles(Vh), m.rhs);
  }
  (void)nchunks;
  if (last_block(w.ticket)) k1_finish<NR>(w, Vh);
}

// K3 (eo): t = S s ; (t, s), |t|^2
template <int NR, int RECON, typename R = double, int MINB = eo_minb<R>()>
__global__ void __launch_bounds__(kRedBlock, MINB) bi_k3_eo(BiEo X, LinkField<R, RECON> le,
                                                         LinkField<R, RECON> lo, BiWST<R> w_) {
  const BiWST<R> w = w_.at(blockIdx.y);
  if (!any_status<NR>(w.st, ST_RUN)) return;
  RhsMap<NR> m;
  const bool run_me = w.st[m.rhs].status == ST_RUN;
  const int64_t Vh = X.E.Vh;
  const int64_t off = (int64_t)m.rhs * 12 * Vh;
  int64_t nchunks = 0;
  MGT_DYN_LOOP(m, Vh, w.ctr, nchunks) {
    double acc[3] = {0.0, 0.0, 0.0};
    if (run_me && o < Vh) {
      const int64_t c = sched_site(X.sh, o);
      C<R> y[4][3], cc[4][3];
      constexpr bool BLK = eo_blk<R>();
      eo_eval<R, RECON, BLK, eo_pre<R>()>(X.E, 0, X.R.second, w.tmp + off, w.s + off, le, lo, c, y, cc);
      const int64_t cs = eo_cstride<BLK>(X.E), bc = off + eo_base<BLK>(X.E, c);
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          stc(w.t + bc + (int64_t)(a * 3 + k) * cs, y[a][k]);
          const C<R> tt = y[a][k], ss = cc[a][k];
          acc[0] += dre(tt, ss);
          acc[1] += dim(tt, ss);
          acc[2] += dnorm2(tt);
        }
    }
    if (run_me) tile_publish<NR, 3>(acc, w.tr, m.tile(o), n_tiles(Vh), m.rhs);
  }
  (void)nchunks;
  if (last_block(w.ticket)) k3_finish<NR>(w, Vh);
}

#if MGT_F32_STENCIL_PAIRS
// ---------------------------------------------------------------------------
// fp32 stencil kernels with two adjacent cb sites per thread (eo_pair.cuh):
// the same three roles as bi_eo_first / bi_k1_eo / bi_k3_eo for lattices with
// L2 % 4 == 0.  A block iteration covers 2 * SPB ordered sites; lanes 0-15 of
// a warp hold one 32-site tile, lanes 16-31 the next (tile_publish_pairs), so
// the reductions stay a function of the site index only (batch-invariant).
#define MGT_DYN_PAIR_LOOP(M, V, CTR, NCH)                                                     \
  NCH = ((V) + 2 * (M).SPB - 1) / (2 * (M).SPB);                                              \
  for (int64_t chunk = next_chunk(CTR), o = chunk * 2 * (M).SPB + 2 * (M).local; chunk < NCH; \
       chunk = next_chunk(CTR), o = chunk * 2 * (M).SPB + 2 * (M).local)

template <int NR, int RECON, int MINB>
__global__ void __launch_bounds__(kRedBlock, MINB) bi_eo_first_v(BiEo X, LinkField<float, RECON> le,
                                                                 LinkField<float, RECON> lo, const float2 *f,
                                                                 BiWST<float> w_) {
  const BiWST<float> w = w_.at(blockIdx.y);
  f += (int64_t)blockIdx.y * w_.gfield;
  if (!any_status<NR>(w.st, ST_RUN)) return;
  RhsMap<NR> m;
  const bool act = w.st[m.rhs].status == ST_RUN;
  const int64_t Vh = X.E.Vh;
  const int64_t off = (int64_t)m.rhs * 12 * Vh;
  int64_t nchunks = 0;
  MGT_DYN_PAIR_LOOP(m, Vh, w.ctr2, nchunks) {
    if (act && o < Vh) {
      const int64_t c = sched_site(X.sh, o);
      C<float> y[2][4][3], cc[2][4][3];
      eo_eval_pair<RECON>(X.E, 1, X.R.first, f + off, nullptr, lo, le, c, y, cc);
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int k = 0; k < 3; ++k) st2(w.tmp + off + (int64_t)(a * 3 + k) * Vh + c, y[0][a][k], y[1][a][k]);
    }
  }
}

template <int NR, int RECON, int MINB>
__global__ void __launch_bounds__(kRedBlock, MINB) bi_k1_eo_v(BiEo X, LinkField<float, RECON> le,
                                                              LinkField<float, RECON> lo, BiWST<float> w_) {
  const BiWST<float> w = w_.at(blockIdx.y);
  if (!any_status<NR>(w.st, ST_RUN)) return;
  RhsMap<NR> m;
  const bool run_me = w.st[m.rhs].status == ST_RUN;
  const int64_t Vh = X.E.Vh;
  const int64_t off = (int64_t)m.rhs * 12 * Vh;
  int64_t nchunks = 0;
  MGT_DYN_PAIR_LOOP(m, Vh, w.ctr, nchunks) {
    double acc[2] = {0.0, 0.0};
    if (run_me && o < Vh) {
      const int64_t c = sched_site(X.sh, o);
      C<float> y[2][4][3], cc[2][4][3];
      eo_eval_pair<RECON>(X.E, 0, X.R.second, w.tmp + off, w.p + off, le, lo, c, y, cc);
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const int64_t q = off + (int64_t)(a * 3 + k) * Vh + c;
          st2(w.v + q, y[0][a][k], y[1][a][k]);
          C<float> rh0, rh1;
          ld2(w.rhat + q, rh0, rh1);
          acc[0] += dre(rh0, y[0][a][k]);
          acc[1] += dim(rh0, y[0][a][k]);
          acc[0] += dre(rh1, y[1][a][k]);
          acc[1] += dim(rh1, y[1][a][k]);
        }
    }
    if (run_me) tile_publish_pairs<NR, 2>(acc, w.tr, o >> 5, n_tiles(Vh), m.rhs);
  }
  (void)nchunks;
  if (last_block(w.ticket)) k1_finish<NR>(w, Vh);
}

template <int NR, int RECON, int MINB>
__global__ void __launch_bounds__(kRedBlock, MINB) bi_k3_eo_v(BiEo X, LinkField<float, RECON> le,
                                                              LinkField<float, RECON> lo, BiWST<float> w_) {
  const BiWST<float> w = w_.at(blockIdx.y);
  if (!any_status<NR>(w.st, ST_RUN)) return;
  RhsMap<NR> m;
  const bool run_me = w.st[m.rhs].status == ST_RUN;
  const int64_t Vh = X.E.Vh;
  const int64_t off = (int64_t)m.rhs * 12 * Vh;
  int64_t nchunks = 0;
  MGT_DYN_PAIR_LOOP(m, Vh, w.ctr, nchunks) {
    double acc[3] = {0.0, 0.0, 0.0};
    if (run_me && o < Vh) {
      const int64_t c = sched_site(X.sh, o);
      C<float> y[2][4][3], cc[2][4][3];
      eo_eval_pair<RECON>(X.E, 0, X.R.second, w.tmp + off, w.s + off, le, lo, c, y, cc);
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          st2(w.t + off + (int64_t)(a * 3 + k) * Vh + c, y[0][a][k], y[1][a][k]);
#pragma unroll
          for (int s = 0; s < 2; ++s) {
            const C<float> tt = y[s][a][k], ss = cc[s][a][k];
            acc[0] += dre(tt, ss);
            acc[1] += dim(tt, ss);
            acc[2] += dnorm2(tt);
          }
        }
    }
    if (run_me) tile_publish_pairs<NR, 3>(acc, w.tr, o >> 5, n_tiles(Vh), m.rhs);
  }
  (void)nchunks;
  if (last_block(w.ticket)) k3_finish<NR>(w, Vh);
}

#endif  // MGT_F32_STENCIL_PAIRS

// true Schur residual r = bh - S x (= the full residual, odd rows exact)
template <int NR, int RECON>
__global__ void __launch_bounds__(kRedBlock, 3) bi_resid_eo(BiEo X, LinkField<double, RECON> le,
                                                            LinkField<double, RECON> lo, BiWS w_) {
  const BiWS w = w_.at(blockIdx.y);
  bool any = false;
#pragma unroll
  for (int r = 0; r < NR; ++r) any |= resid_active<NR>(w.st[r].status);
  if (!any) return;
  RhsMap<NR> m;
  const bool act_me = resid_active<NR>(w.st[m.rhs].status);
  const int64_t Vh = X.E.Vh;
  const int64_t off = (int64_t)m.rhs * 12 * Vh;
  int64_t nchunks = 0;
  MGT_DYN_LOOP(m, Vh, w.ctr, nchunks) {
    double acc[1] = {0.0};
    if (act_me && o < Vh) {
      const int64_t c = sched_site(X.sh, o);
      C<double> y[4][3], cc[4][3];
      eo_eval<double, RECON>(X.E, 0, X.R.second, w.tmp + off, w.x + off, le, lo, c, y, cc);
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const int64_t q = off + (int64_t)(a * 3 + k) * Vh + c;
          C<double> rr = ldc(w.b + q) - y[a][k];
          stc(w.r + q, rr);
          acc[0] += cabs2(rr);
        }
    }
    if (act_me) tile_publish<NR, 1>(acc, w.tr, m.tile(o), n_tiles(Vh), m.rhs);
  }
  (void)nchunks;
  if (last_block(w.ticket)) resid_finish<NR>(w, Vh);
}

// x_full: even sites <- x_e, odd sites <- x_o = G_in Dg^-1 [G_out b_o + 1/2 H_oe G_in x_e];
// q = vdot(b, x) over the full lattice (trace.py:104)
template <int NR, int RECON>
__global__ void __launch_bounds__(kRedBlock, 3) bi_eo_final(BiEo X, LinkField<double, RECON> le,
                                                            LinkField<double, RECON> lo, double2 *__restrict__ xout,
                                                            BiWS w_) {
  const BiWS w = w_.at(blockIdx.y);
  xout += (int64_t)blockIdx.y * NR * 12 * X.E.g.V;
  RhsMap<NR> m;
  const int64_t Vh = X.E.Vh, V = X.E.g.V;
  const int64_t off = (int64_t)m.rhs * 12 * Vh;
  double2 *XO = xout + (int64_t)m.rhs * 12 * V;
  MGT_CHUNK_LOOP(m, Vh) {
    double acc[2] = {0.0, 0.0};
    if (o < Vh) {
      int x[4];
      const int64_t fe = eo_coords(X.E, 0, o, x);
      const int64_t fo = eo_coords(X.E, 1, o, x);
      C<double> y[4][3], cc[4][3];
      eo_eval<double, RECON>(X.E, 1, X.R.recon, w.x + off, w.bo + off, lo, le, o, y, cc);
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const int ck = a * 3 + k;
          const C<double> xe = ldc(w.x + off + (int64_t)ck * Vh + o), bev = ldc(w.be + off + (int64_t)ck * Vh + o);
          stc(XO + (int64_t)ck * V + fe, xe);
          stc(XO + (int64_t)ck * V + fo, y[a][k]);
          const C<double> bov = cc[a][k], xo = y[a][k];
          acc[0] += bev.re * xe.re + bev.im * xe.im + bov.re * xo.re + bov.im * xo.im;
          acc[1] += bev.re * xe.im - bev.im * xe.re + bov.re * xo.im - bov.im * xo.re;
        }
    }
    tile_publish<NR, 2>(acc, w.tr, m.tile(o), n_tiles(Vh), m.rhs);
  }
  if (last_block(w.ticket)) {
    double out[NR * 2];
    tiles_final<NR * 2>(w.tr, Vh, w.ticket, out);
    const int r = threadIdx.x;
    if (r < NR) {
      w.st[r].dotq = C<double>(out[2 * r], out[2 * r + 1]);
      w.st[r].matvecs += 1;  // the odd-site reconstruction (half of A)
    }
  }
}

// ---------------------------------------------------------------------------
static size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

constexpr int kMaxGroup = 4;
constexpr int kChunk = 8;  // iterations per graph replay
constexpr int kMaxGroups = 64;

// Per-rhs relative tolerances (mgt_bicgstab_solve_tols): after bi_init,
// tol2 = tol_r^2 |b_r|^2 for every rhs r of every group.
struct TolPack {
  double t[kMaxGroups * kMaxGroup];
};
template <int NR>
__global__ void bi_set_tols(BiWS w_, TolPack tp) {
  const BiWS w = w_.at(blockIdx.y);
  const int r = threadIdx.x;
  if (r < NR) {
    BiState &s = w.st[r];
    const double t = tp.t[blockIdx.y * NR + r];
    s.tol2 = t * t * s.b2;
  }
}
template <int NR>
static int set_tols(const BiWS &w, const double *tols, int G, cudaStream_t st) {
  if (!tols) return MGT_OK;
  TolPack tp;
  for (int i = 0; i < G * NR; ++i) tp.t[i] = tols[i];
  bi_set_tols<NR><<<dim3(1, G), 32, 0, st>>>(w, tp);
  MGT_LAUNCH_CHECK("bi_set_tols");
  return MGT_OK;
}

struct WSLayout {
  size_t field, partials, total;
  int64_t V;
  int groups;
  size_t gpart;  // tile-partial doubles per group
};

// groups: batched solves of groups * kMaxGroup rhs share one workspace (and
// one launch per kernel, blockIdx.y = group)
static WSLayout ws_layout(int64_t V, int groups = 1) {
  WSLayout L;
  L.V = V;
  L.groups = groups;
  L.field = align_up((size_t)groups * kMaxGroup * 12 * V * sizeof(double2), 512);
  // tile-ordered reductions (reduce.cuh): up to kMaxGroup * 3 doubles per
  // tile of the full lattice (the largest loop)
  L.gpart = align_up((size_t)n_tiles(V) * kMaxGroup * 3, 32);
  L.partials = align_up((size_t)groups * L.gpart * sizeof(double), 256);
  L.total = 8 * L.field + L.partials + 256 * (size_t)groups /*tickets*/ +
            align_up((size_t)groups * kMaxGroup * sizeof(BiState), 256);
  return L;
}

// fp32 inner workspace of the mixed-precision solve (even-odd fields r,
// rhat, p, v, s, t, x, tmp; own partials, tickets and states), placed after
// the fp64 workspace
static size_t ws32_bytes(const WSLayout &L) {
  const size_t f32 = align_up((size_t)L.groups * kMaxGroup * 12 * (L.V / 2) * sizeof(float2), 512);
  return 8 * f32 + L.partials + 256 * (size_t)L.groups + align_up((size_t)L.groups * kMaxGroup * sizeof(BiState), 256);
}

template <typename R>
static void carve_red(BiWST<R> &w, char *q, const WSLayout &Lw) {
  w.tr.tiles = (double *)q;
  w.gpart = (int64_t)Lw.gpart;
}

static BiWST<float> carve32(char *q, const WSLayout &Lw) {
  BiWST<float> w;
  const size_t f32 = align_up((size_t)Lw.groups * kMaxGroup * 12 * (Lw.V / 2) * sizeof(float2), 512);
  float2 **f[8] = {&w.r, &w.rhat, &w.p, &w.v, &w.s, &w.t, &w.x, &w.tmp};
  for (int i = 0; i < 8; ++i) *f[i] = (float2 *)(q + i * f32);
  w.b = w.be = w.bo = nullptr;
  q += 8 * f32;
  carve_red(w, q, Lw);
  q += Lw.partials;
  w.ticket = (unsigned *)q;
  w.ctr = (unsigned long long *)(q + 8);
  w.ctr2 = (unsigned long long *)(q + 16);
  w.red = (double *)(q + 32);
  q += 256 * (size_t)Lw.groups;
  w.st = (BiState *)q;
  w.gfield = (int64_t)kMaxGroup * 12 * (Lw.V / 2);
  return w;
}

// total bytes for G groups (mixed: plus the fp32 inner workspace)
static size_t ws_total(int64_t V, int groups, bool mixed) {
  const WSLayout L = ws_layout(V, groups);
  return L.total + (mixed ? ws32_bytes(L) : 0);
}

static BiWS carve(char *q, const WSLayout &Lw, bool eo = false) {
  BiWS w;
  double2 **f[11] = {&w.r, &w.rhat, &w.p, &w.v, &w.s, &w.t, &w.x, &w.b, &w.be, &w.bo, &w.tmp};
  // full solve: 8 fields of the slot size; even-odd: 11 parity fields of half a slot
  const size_t step = eo ? Lw.field / 2 : Lw.field;
  char *f0 = q;
  for (int i = 0; i < (eo ? 11 : 8); ++i) *f[i] = (double2 *)(f0 + i * step);
  if (!eo) w.be = w.bo = w.tmp = nullptr;
  q += 8 * Lw.field;
  carve_red(w, q, Lw);
  q += Lw.partials;
  w.ticket = (unsigned *)q;
  w.ctr = (unsigned long long *)(q + 8);
  w.ctr2 = (unsigned long long *)(q + 16);
  w.red = (double *)(q + 32);  // up to 28 doubles
  q += 256 * (size_t)Lw.groups;
  w.st = (BiState *)q;
  w.gfield = (int64_t)kMaxGroup * 12 * (eo ? Lw.V / 2 : Lw.V);
  return w;
}

// Graph cache: one instantiated graph of kChunk iterations per
// (workspace, NR, RECON, operator variant).
struct GraphKey {
  const void *h, *ws;
  int nr, recon, flags, eo, groups;
  double tau;
  bool operator<(const GraphKey &o) const {
    return std::tie(h, ws, nr, recon, flags, eo, groups, tau) <
           std::tie(o.h, o.ws, o.nr, o.recon, o.flags, o.eo, o.groups, o.tau);
  }
};
static std::mutex g_graph_mu;
static std::map<GraphKey, cudaGraphExec_t> g_graphs;

void drop_graphs(const void *h) {
  std::lock_guard<std::mutex> lk(g_graph_mu);
  for (auto it = g_graphs.begin(); it != g_graphs.end();) {
    if (it->first.h == h) {
      cudaGraphExecDestroy(it->second);
      it = g_graphs.erase(it);
    } else {
      ++it;
    }
  }
}

template <int NR, int RECON>
static int launch_chunk(const WilsonParams &P, const LinkField<double, RECON> &lf, const BiWS &w, dim3 gd, dim3 grid,
                        cudaStream_t st) {
  const int64_t V = P.g.V;
  for (int it = 0; it < kChunk; ++it) {
    bi_k1<NR, RECON><<<gd, kRedBlock, 0, st>>>(P, lf, w);
    bi_k2<NR><<<grid, kRedBlock, 0, st>>>(V, w);
    bi_k3<NR, RECON><<<gd, kRedBlock, 0, st>>>(P, lf, w);
    bi_k4<NR><<<grid, kRedBlock, 0, st>>>(V, w);
    bi_k5<NR><<<grid, kRedBlock, 0, st>>>(V, w);
  }
  return MGT_OK;
}

template <int NR, int RECON, typename R = double, int MINB = eo_minb<R>(), bool PAIR = false>
static int launch_chunk_eo(const BiEo &X, const LinkField<R, RECON> &le, const LinkField<R, RECON> &lo,
                           const BiWST<R> &w, dim3 gd, dim3 g1, dim3 grid, cudaStream_t st, int iters = kChunk) {
  const int64_t Vh = X.E.Vh;
  for (int it = 0; it < iters; ++it) {
#if MGT_F32_STENCIL_PAIRS
    if constexpr (PAIR) {
      bi_eo_first_v<NR, RECON, MINB><<<g1, kRedBlock, 0, st>>>(X, le, lo, w.p, w);
      bi_k1_eo_v<NR, RECON, MINB><<<gd, kRedBlock, 0, st>>>(X, le, lo, w);
    } else
#endif
    {
      bi_eo_first<NR, RECON, R, MINB><<<g1, kRedBlock, 0, st>>>(X, le, lo, w.p, w, 0);
      bi_k1_eo<NR, RECON, R, MINB><<<gd, kRedBlock, 0, st>>>(X, le, lo, w);
    }
    if constexpr (std::is_same<R, float>::value && MGT_F32_PAIRS)
      bi_k2v<NR><<<grid, kRedBlock, 0, st>>>(Vh, w);
    else
      bi_k2<NR, 0, R><<<grid, kRedBlock, 0, st>>>(Vh, w);
#if MGT_F32_STENCIL_PAIRS
    if constexpr (PAIR) {
      bi_eo_first_v<NR, RECON, MINB><<<g1, kRedBlock, 0, st>>>(X, le, lo, w.s, w);
      bi_k3_eo_v<NR, RECON, MINB><<<gd, kRedBlock, 0, st>>>(X, le, lo, w);
    } else
#endif
    {
      bi_eo_first<NR, RECON, R, MINB><<<g1, kRedBlock, 0, st>>>(X, le, lo, w.s, w, 0);
      bi_k3_eo<NR, RECON, R, MINB><<<gd, kRedBlock, 0, st>>>(X, le, lo, w);
    }
    if constexpr (std::is_same<R, float>::value && MGT_F32_PAIRS) {
      bi_k4v<NR><<<grid, kRedBlock, 0, st>>>(Vh, w);
      bi_k5v<NR><<<grid, kRedBlock, 0, st>>>(Vh, w);
    } else {
      bi_k4<NR, 0, R><<<grid, kRedBlock, 0, st>>>(Vh, w);
      bi_k5<NR, R><<<grid, kRedBlock, 0, st>>>(Vh, w);
    }
  }
  return MGT_OK;
}

// pinned per-thread mailbox for the solver states (concurrent solves on
// several streams may share a handle)
static BiState *state_mailbox(int n) {
  static thread_local BiState *hs = nullptr;
  static thread_local int cap = 0;
  if (n > cap) {
    if (hs) cudaFreeHost(hs);
    cap = std::max(n, 64);
    if (cudaMallocHost((void **)&hs, cap * sizeof(BiState)) != cudaSuccess) {
      hs = nullptr;
      cap = 0;
    }
  }
  return hs;
}

// Solve G groups of NR rhs (G > 1 only with NR = kMaxGroup): one launch per
// kernel for all groups (blockIdx.y = group).
template <int NR, int RECON>
static int solve_group(mgt_wilson_s *h, const WilsonParams &P, int flags, double tau, const double2 *b, double2 *x,
                       char *ws, const WSLayout &Lw, double tol, const double *tols, int max_iter, int64_t *report,
                       double *relres, double *dot_out, bool eo, int G, cudaStream_t st) {
  const int64_t V = h->g.V;
  const int64_t Vs = eo ? V / 2 : V;  // sites of the solved system
  BiWS w = carve(ws, Lw, eo);
  LinkField<double, RECON> lf{reinterpret_cast<const double2 *>(h->links), V};
  // even-odd pieces
  BiEo X;
  LinkField<double, RECON> le{nullptr, V / 2}, lo{nullptr, V / 2};
  if (eo) {
    X.E = make_eo_geom(h->g, h->antiperiodic);
    Geom gh = h->g;
    gh.L[2] /= 2;
    gh.V /= 2;
    gh.stride[1] /= 2;
    gh.stride[0] /= 2;
    gh.stride[3] /= 2;
    X.sh = make_sched(gh, 1024, h->slab_bytes);
    X.R = make_eo_roles(P);
    le.p = reinterpret_cast<const double2 *>(h->links_cb);
    lo.p = reinterpret_cast<const double2 *>((const char *)h->links_cb + h->link_bytes / 2);
  }
  static int g_dsl = 0, g_str = 0, g_e1 = 0, g_e2 = 0;  // resident grids, per template instance
  if (!g_dsl) g_dsl = resident_grid(bi_k1<NR, RECON>, kRedBlock, (int64_t)1 << 40);
  if (!g_str) g_str = resident_grid(bi_k4<NR>, kRedBlock, (int64_t)1 << 40);
  if (eo && !g_e1) g_e1 = resident_grid(bi_eo_first<NR, RECON>, kRedBlock, (int64_t)1 << 40);
  if (eo && !g_e2) g_e2 = resident_grid(bi_k1_eo<NR, RECON>, kRedBlock, (int64_t)1 << 40);
  const int64_t need = (Vs + RhsMap<NR>::SPB - 1) / RhsMap<NR>::SPB;
  auto per_group = [&](int resident) {
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(need, std::max(1, resident / G)));
  };
  const dim3 grid(per_group(g_str), G);
  const dim3 gd(per_group(eo ? g_e2 : g_dsl), G);
  const dim3 g1(eo ? per_group(g_e1) : 1, G);
  MGT_CUDA(cudaMemsetAsync(w.ticket, 0, 256 * (size_t)G, st));  // tickets and chunk counters
  if (eo) {
    bi_eo_split<NR><<<grid, kRedBlock, 0, st>>>(X, b, w, P.g5out);
    bi_eo_rhs<NR, RECON><<<grid, kRedBlock, 0, st>>>(X, le, lo, w);
    bi_init<NR><<<grid, kRedBlock, 0, st>>>(Vs, w.b, w, tol, max_iter, 1);
    note_launch(3);
  } else {
    bi_init<NR><<<grid, kRedBlock, 0, st>>>(V, b, w, tol, max_iter, 0);
    note_launch(1);
  }
  MGT_LAUNCH_CHECK("bi_init");
  if (int rc = set_tols<NR>(w, tols, G, st)) return rc;

  cudaGraphExec_t exec = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_graph_mu);
    GraphKey key{h, ws, NR, RECON, flags, eo ? 1 : 0, G, tau};
    auto it = g_graphs.find(key);
    if (it != g_graphs.end()) {
      exec = it->second;
    } else {
      cudaStream_t cap;
      MGT_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
      cudaGraph_t graph;
      MGT_CUDA(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
      if (eo)
        launch_chunk_eo<NR, RECON>(X, le, lo, w, gd, g1, grid, cap);
      else
        launch_chunk<NR, RECON>(P, lf, w, gd, grid, cap);
      cudaError_t e = cudaStreamEndCapture(cap, &graph);
      cudaStreamDestroy(cap);
      if (e != cudaSuccess) return cuda_fail(e, "bicgstab graph capture");
      e = cudaGraphInstantiate(&exec, graph, 0);
      cudaGraphDestroy(graph);
      if (e != cudaSuccess) return cuda_fail(e, "bicgstab graph instantiate");
      g_graphs[key] = exec;
    }
  }
  const int per_iter = eo ? 7 : 5;
  const int nst = G * NR;  // states of group g at w.st + g * kMaxGroup
  BiState *hs = state_mailbox(G * kMaxGroup);
  if (!hs) return fail(MGT_ERR_CUDA, "pinned state mailbox");
  auto fetch = [&]() -> int {
    MGT_CUDA(cudaMemcpyAsync(hs, w.st, (size_t)G * kMaxGroup * sizeof(BiState), cudaMemcpyDeviceToHost, st));
    MGT_CUDA(cudaStreamSynchronize(st));
    return MGT_OK;
  };
  auto any_state = [&](int want) {
    for (int g = 0; g < G; ++g)
      for (int r = 0; r < NR; ++r)
        if (hs[g * kMaxGroup + r].status == want) return true;
    return false;
  };
  for (int round = 0; round < 1000000; ++round) {
    MGT_CUDA(cudaGraphLaunch(exec, st));
    note_launch(per_iter * kChunk);
    int rc = fetch();
    if (rc) return rc;
    if (any_state(ST_RUN)) continue;
    if (eo) {
      bi_eo_first<NR, RECON><<<g1, kRedBlock, 0, st>>>(X, le, lo, w.x, w, 1);
      bi_resid_eo<NR, RECON><<<gd, kRedBlock, 0, st>>>(X, le, lo, w);
      note_launch(1);
    } else {
      bi_resid<NR, RECON><<<gd, kRedBlock, 0, st>>>(P, lf, w);
    }
    bi_restart<NR><<<grid, kRedBlock, 0, st>>>(Vs, w);
    note_launch(2);
    MGT_LAUNCH_CHECK("bicgstab residual");
    rc = fetch();
    if (rc) return rc;
    if (!any_state(ST_RUN)) break;
  }
  if (eo)
    bi_eo_final<NR, RECON><<<grid, kRedBlock, 0, st>>>(X, le, lo, x, w);
  else
    bi_final<NR><<<grid, kRedBlock, 0, st>>>(V, x, w);
  note_launch(1);
  MGT_LAUNCH_CHECK("bi_final");
  int rc = fetch();
  if (rc) return rc;
  (void)nst;
  for (int g = 0; g < G; ++g)
    for (int r = 0; r < NR; ++r) {
      const BiState &s = hs[g * kMaxGroup + r];
      const int i = g * NR + r;
      const bool zero_rhs = s.b2 == 0.0;
      const double rel = zero_rhs ? 0.0 : sqrt(s.true_r2 / s.b2);
      const bool conv = zero_rhs || s.true_r2 <= s.tol2;
      report[4 * i + 0] = s.iters;
      report[4 * i + 1] = s.matvecs;
      report[4 * i + 2] = conv ? 1 : 0;
      report[4 * i + 3] = conv ? 0 : (s.reason ? s.reason : 1);
      relres[i] = rel;
      if (dot_out) {
        dot_out[2 * i] = s.dotq.re;
        dot_out[2 * i + 1] = s.dotq.im;
      }
    }
  return MGT_OK;
}

// ---------------------------------------------------------------------------
// Mixed-precision even-odd solve (defect correction).  The fp64 workspace
// holds the Schur system (bh_e, x_e and its true residual r); every outer
// cycle solves S e = r with fp32 fields and links (fp64 reductions and
// scalar recurrences) to a relative tolerance delta, accumulates x_e += e in
// fp64 and recomputes r = bh_e - S x_e in fp64: the stopping test is the
// reference's explicit full residual ||b - A x|| <= tol ||b||
// (krylov.py:78-85), unchanged.  An fp32 iteration streams half the bytes
// of an fp64 one.

// inner start: r = rhat = p = (float) r64 for the rhs still running (zero
// otherwise), x = 0; inner tol2 = max(delta^2 |r|^2, 0.81 tol2_64)
template <int NR>
__global__ void __launch_bounds__(kRedBlock) mx_begin(int64_t V, EoGeom E, BiWS w64_, BiWST<float> w_, double delta) {
  const BiWS w64 = w64_.at(blockIdx.y);
  const BiWST<float> w = w_.at(blockIdx.y);
  RhsMap<NR> m;
  const bool act = w64.st[m.rhs].status == ST_RUN;
  MGT_CHUNK_LOOP(m, V) {
    double acc[1] = {0.0};
    if (o < V) {
      constexpr bool BLK = eo_blk<float>();
      const int64_t base = (int64_t)m.rhs * 12 * V + o;
      const int64_t b32 = (int64_t)m.rhs * 12 * V + eo_base<BLK>(E, o), cs = eo_cstride<BLK>(E);
#pragma unroll
      for (int c = 0; c < 12; ++c) {
        const int64_t q = base + (int64_t)c * V, q32 = b32 + (int64_t)c * cs;
        const C<float> bb = act ? cvt<float>(ldc(w64.r + q)) : C<float>(0.f, 0.f);
        stc(w.r + q32, bb);
        stc(w.rhat + q32, bb);
        stc(w.p + q32, bb);
        stc(w.x + q32, C<float>(0.f, 0.f));
        acc[0] += dnorm2(bb);
      }
    }
    tile_publish<NR, 1>(acc, w.tr, m.tile(o), n_tiles(V), m.rhs);
  }
  if (last_block(w.ticket)) {
    double out[NR];
    tiles_final<NR>(w.tr, V, w.ticket, out);
    const int r = threadIdx.x;
    if (r < NR) {
      BiState &s = w.st[r];
      const BiState &s64 = w64.st[r];
      const double b2 = out[r];
      s.b2 = s.r2 = s.s2 = s.true_r2 = b2;
      s.tol2 = fmax(delta * delta * b2, 0.81 * s64.tol2);
      s.rho = C<double>(b2, 0.0);
      s.alpha = s.omega = C<double>(1.0, 0.0);
      s.beta = s.dotq = C<double>(0.0, 0.0);
      s.half = 0;
      s.iters = 0;
      s.maxit = max(1, s64.maxit - s64.iters);
      s.matvecs = 0;
      s.reason = 0;
      s.status = (s64.status == ST_RUN && b2 > 0.0) ? ST_RUN : ST_DONE;
    }
  }
}

// x_e += (double) e for the rhs whose inner cycle ran; they are marked CONV so
// the fp64 residual kernels recompute their true residual
template <int NR>
__global__ void __launch_bounds__(kRedBlock) mx_accum(int64_t V, EoGeom E, BiWS w64_, BiWST<float> w_) {
  const BiWS w64 = w64_.at(blockIdx.y);
  const BiWST<float> w = w_.at(blockIdx.y);
  RhsMap<NR> m;
  if (w64.st[m.rhs].status == ST_RUN) {
    MGT_SITE_LOOP(m, V) {
      constexpr bool BLK = eo_blk<float>();
      const int64_t base = (int64_t)m.rhs * 12 * V + o;
      const int64_t b32 = (int64_t)m.rhs * 12 * V + eo_base<BLK>(E, o), cs = eo_cstride<BLK>(E);
#pragma unroll
      for (int c = 0; c < 12; ++c) {
        const int64_t q = base + (int64_t)c * V;
        const C<float> e = ldc(w.x + b32 + (int64_t)c * cs);
        const C<double> xx = ldc(w64.x + q);
        stc(w64.x + q, C<double>(xx.re + (double)e.re, xx.im + (double)e.im));
      }
    }
  }
  if (last_block(w64.ticket)) {
    const int r = threadIdx.x;
    if (r == 0) *w64.ticket = 0u;
    if (r < NR) {
      BiState &s = w64.st[r];
      const BiState &t = w.st[r];
      if (s.status == ST_RUN) {
        s.iters += t.iters;
        s.matvecs += t.matvecs;
        s.status = ST_CONV;
      }
    }
  }
}

// rhs whose true residual is still above tol start another cycle unless
// the last one failed to halve it (stagnation -> reported as breakdown)
template <int NR>
__global__ void mx_next(BiWS w_, int cycle, int max_cycles) {
  const BiWS w = w_.at(blockIdx.y);
  const int r = threadIdx.x;
  if (r < NR && w.st[r].status == ST_RESTART) {
    BiState &s = w.st[r];
    if (cycle + 1 >= max_cycles || s.true_r2 > 0.25 * s.s2) {
      s.status = ST_DONE;
      s.reason = 2;
    } else {
      s.s2 = s.true_r2;  // the residual this cycle must improve on
      s.status = ST_RUN;
    }
  }
}

// Device-side loop control of the inner iterations (CUDA conditional graph
// node, WHILE): the body -- kWhileBody iterations and this kernel -- repeats
// while any rhs of the launch is still running, so a cycle of the mixed
// solve is ONE graph launch with no host round trip between iteration
// chunks and at most kWhileBody - 1 early-exit iterations past convergence
// (the chunked replay costs a status copy + synchronise + graph launch,
// ~60 us, per 8 iterations: 16 % of an 8^4 solve, 3 % at 16^4).
#ifndef MGT_WHILE_BODY
#define MGT_WHILE_BODY 2
#endif
constexpr int kWhileBody = MGT_WHILE_BODY;
__global__ void bi_while_cond(cudaGraphConditionalHandle handle, const BiState *st, int G, int NR) {
  bool any = false;
  for (int i = threadIdx.x; i < G * kMaxGroup; i += 32)
    if ((i % kMaxGroup) < NR && st[i].status == ST_RUN) any = true;
  any = __any_sync(0xffffffffu, any);
  if (threadIdx.x == 0) cudaGraphSetConditional(handle, any ? 1u : 0u);
}

// Build the WHILE graph around `body(stream)`; nullptr when the runtime
// refuses (the caller falls back to the chunked replay).
template <class Body>
static cudaGraphExec_t build_while_graph(const BiState *st_dev, int G, int NR, Body body) {
  cudaGraph_t g = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaStream_t cap = nullptr;
  bool ok = cudaGraphCreate(&g, 0) == cudaSuccess;
  cudaGraphConditionalHandle handle{};
  ok = ok && cudaGraphConditionalHandleCreate(&handle, g, 1, cudaGraphCondAssignDefault) == cudaSuccess;
  cudaGraphNodeParams cp = {cudaGraphNodeTypeConditional};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = handle;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  ok = ok && cudaGraphAddNode(&node, g, nullptr, 0, &cp) == cudaSuccess;
  if (ok) {
    cudaGraph_t bodyg = cp.conditional.phGraph_out[0];
    ok = cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking) == cudaSuccess;
    ok = ok && cudaStreamBeginCaptureToGraph(cap, bodyg, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal) ==
                   cudaSuccess;
    if (ok) {
      body(cap);
      bi_while_cond<<<1, 32, 0, cap>>>(handle, st_dev, G, NR);
      cudaGraph_t out = nullptr;
      ok = cudaStreamEndCapture(cap, &out) == cudaSuccess;
    }
  }
  ok = ok && cudaGraphInstantiate(&exec, g, 0) == cudaSuccess;
  if (cap) cudaStreamDestroy(cap);
  if (g) cudaGraphDestroy(g);
  if (!ok) {
    cudaGetLastError();
    if (exec) cudaGraphExecDestroy(exec);
    return nullptr;
  }
  return exec;
}

// MINB32: resident blocks per SM of the fp32 stencil kernels (their launch
// bounds).  Small lattices run at 4 (128 registers, 16 warps/SM: at 8^4 the
// 2,048 rhs-warps of a 32-rhs stencil pass fit one wave instead of 1.15;
// config-1 probes/s +10 %); large ones at 3 (168 registers, no spills, the
// better choice once the pass is many waves long).
template <int NR, int RECON, int MINB32 = eo_minb<float>(), bool PAIR = false>
static int solve_group_mixed(mgt_wilson_s *h, const WilsonParams &P, int flags, double tau, const double2 *b,
                             double2 *x, char *ws, const WSLayout &Lw, double tol, const double *tols, int max_iter,
                             int64_t *report, double *relres, double *dot_out, int G, cudaStream_t st) {
  const int64_t V = h->g.V, Vs = V / 2;
  BiWS w = carve(ws, Lw, true);
  BiWST<float> w32 = carve32(ws + Lw.total, Lw);
  BiEo X;
  X.E = make_eo_geom(h->g, h->antiperiodic);
  Geom gh = h->g;
  gh.L[2] /= 2;
  gh.V /= 2;
  gh.stride[1] /= 2;
  gh.stride[0] /= 2;
  gh.stride[3] /= 2;
  X.sh = make_sched(gh, 1024, h->slab_bytes);
  X.R = make_eo_roles(P);
  LinkField<double, RECON> le{reinterpret_cast<const double2 *>(h->links_cb), Vs};
  LinkField<double, RECON> lo{reinterpret_cast<const double2 *>((const char *)h->links_cb + h->link_bytes / 2), Vs};
  // fp32 links: the handle's storage narrowed, or (MGT_MIXED_L18) full 3x3
  constexpr int R32 = MGT_MIXED_L18 ? 18 : RECON;
  LinkField<float, R32> le32{reinterpret_cast<const float2 *>(h->links_cb32), Vs};
  LinkField<float, R32> lo32{reinterpret_cast<const float2 *>(h->links_cb32) + (R32 / 2) * 4 * Vs, Vs};
  static int g_str = 0, g_e1 = 0, g_e2 = 0, g_f1 = 0, g_f2 = 0;  // resident grids, per template instance
  if (!g_str) g_str = resident_grid(bi_k4<NR>, kRedBlock, (int64_t)1 << 40);
  if (!g_e1) g_e1 = resident_grid(bi_eo_first<NR, RECON>, kRedBlock, (int64_t)1 << 40);
  if (!g_e2) g_e2 = resident_grid(bi_k1_eo<NR, RECON>, kRedBlock, (int64_t)1 << 40);
#if MGT_F32_STENCIL_PAIRS
  if constexpr (PAIR) {
    if (!g_f1) g_f1 = resident_grid(bi_eo_first_v<NR, R32, MINB32>, kRedBlock, (int64_t)1 << 40);
    if (!g_f2) g_f2 = resident_grid(bi_k1_eo_v<NR, R32, MINB32>, kRedBlock, (int64_t)1 << 40);
  } else
#endif
  {
    if (!g_f1) g_f1 = resident_grid(bi_eo_first<NR, R32, float, MINB32>, kRedBlock, (int64_t)1 << 40);
    if (!g_f2) g_f2 = resident_grid(bi_k1_eo<NR, R32, float, MINB32>, kRedBlock, (int64_t)1 << 40);
  }
  const int64_t need = (Vs + RhsMap<NR>::SPB - 1) / RhsMap<NR>::SPB;
  auto per_group_n = [&](int resident, int64_t n) {
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(n, std::max(1, resident / G)));
  };
  auto per_group = [&](int resident) { return per_group_n(resident, need); };
  // the pair stencils take 2 * SPB sites per block iteration
  const int64_t need32 = PAIR ? (need + 1) / 2 : need;
  const dim3 grid(per_group(g_str), G), gd(per_group(g_e2), G), g1(per_group(g_e1), G);
  const dim3 fd(per_group_n(g_f2, need32), G), f1(per_group_n(g_f1, need32), G);
  MGT_CUDA(cudaMemsetAsync(w.ticket, 0, 256 * (size_t)G, st));
  MGT_CUDA(cudaMemsetAsync(w32.ticket, 0, 256 * (size_t)G, st));
  bi_eo_split<NR><<<grid, kRedBlock, 0, st>>>(X, b, w, P.g5out);
  bi_eo_rhs<NR, RECON><<<grid, kRedBlock, 0, st>>>(X, le, lo, w);
  bi_init<NR><<<grid, kRedBlock, 0, st>>>(Vs, w.b, w, tol, max_iter, 1);
  note_launch(3);
  MGT_LAUNCH_CHECK("bi_init (mixed)");
  if (int rc = set_tols<NR>(w, tols, G, st)) return rc;

  cudaGraphExec_t exec = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_graph_mu);
    GraphKey key{h, ws, NR, RECON, flags, PAIR ? 3 : 2, G, tau};
    auto it = g_graphs.find(key);
    if (it != g_graphs.end()) {
      exec = it->second;
    } else {
      cudaStream_t cap;
      MGT_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
      cudaGraph_t graph;
      MGT_CUDA(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
      launch_chunk_eo<NR, R32, float, MINB32, PAIR>(X, le32, lo32, w32, fd, f1, grid, cap);
      cudaError_t e = cudaStreamEndCapture(cap, &graph);
      cudaStreamDestroy(cap);
      if (e != cudaSuccess) return cuda_fail(e, "mixed bicgstab graph capture");
      e = cudaGraphInstantiate(&exec, graph, 0);
      cudaGraphDestroy(graph);
      if (e != cudaSuccess) return cuda_fail(e, "mixed bicgstab graph instantiate");
      g_graphs[key] = exec;
    }
  }
  // the device-controlled loop: opt-in (MGT_SOLVE_WHILE=1).  Measured equal
  // to the chunked replay within 1 % at 8^4 .. 32^4 (a loop trip of the
  // conditional node costs about what the host round trip it removes does;
  // profiles/r02s6_while_graph_ab.txt), so the default stays the simpler path.
  static bool while_unsupported = false;
  const char *wv = getenv("MGT_SOLVE_WHILE");
  const bool use_while = wv && atoi(wv) != 0 && !while_unsupported;
  cudaGraphExec_t exec_w = nullptr;
  if (use_while) {
    std::lock_guard<std::mutex> lk(g_graph_mu);
    GraphKey key{h, ws, NR, RECON, flags, PAIR ? 13 : 12, G, tau};
    auto it = g_graphs.find(key);
    if (it != g_graphs.end()) {
      exec_w = it->second;
    } else {
      exec_w = build_while_graph(w32.st, G, NR, [&](cudaStream_t cap) {
        launch_chunk_eo<NR, R32, float, MINB32, PAIR>(X, le32, lo32, w32, fd, f1, grid, cap, kWhileBody);
      });
      if (exec_w)
        g_graphs[key] = exec_w;
      else
        while_unsupported = true;  // not supported here: keep the chunked replay
    }
  }
  BiState *hs = state_mailbox(G * kMaxGroup);
  if (!hs) return fail(MGT_ERR_CUDA, "pinned state mailbox");
  auto fetch = [&](const BiState *dst) -> int {
    MGT_CUDA(cudaMemcpyAsync(hs, dst, (size_t)G * kMaxGroup * sizeof(BiState), cudaMemcpyDeviceToHost, st));
    MGT_CUDA(cudaStreamSynchronize(st));
    return MGT_OK;
  };
  auto any_run = [&]() {
    for (int g = 0; g < G; ++g)
      for (int r = 0; r < NR; ++r)
        if (hs[g * kMaxGroup + r].status == ST_RUN) return true;
    return false;
  };
  static double delta = 0.0;
  if (delta == 0.0) {
    const char *v = getenv("MGT_MIXED_DELTA");
    delta = v ? atof(v) : 1e-4;
  }
  constexpr int kMaxCycles = 64;
  int rc = fetch(w.st);
  if (rc) return rc;
  for (int cycle = 0; cycle < kMaxCycles && any_run(); ++cycle) {
    mx_begin<NR><<<grid, kRedBlock, 0, st>>>(Vs, X.E, w, w32, delta);
    MGT_LAUNCH_CHECK("mx_begin");
    if (exec_w) {
      MGT_CUDA(cudaGraphLaunch(exec_w, st));  // iterates on the device until no rhs is running
    } else {
      for (int round = 0; round < 1000000; ++round) {
        MGT_CUDA(cudaGraphLaunch(exec, st));
        note_launch(7 * kChunk);
        rc = fetch(w32.st);
        if (rc) return rc;
        if (!any_run()) break;
      }
    }
    int its_before = 0;
    if (exec_w)
      for (int g = 0; g < G; ++g)
        for (int r = 0; r < NR; ++r) its_before = std::max(its_before, hs[g * kMaxGroup + r].iters);
    mx_accum<NR><<<grid, kRedBlock, 0, st>>>(Vs, X.E, w, w32);
    bi_eo_first<NR, RECON><<<g1, kRedBlock, 0, st>>>(X, le, lo, w.x, w, 1);
    bi_resid_eo<NR, RECON><<<gd, kRedBlock, 0, st>>>(X, le, lo, w);
    mx_next<NR><<<dim3(1, G), 32, 0, st>>>(w, cycle, kMaxCycles);
    note_launch(3);
    MGT_LAUNCH_CHECK("mixed residual");
    rc = fetch(w.st);
    if (rc) return rc;
    if (exec_w) {  // launches of the device-controlled loop, from the iterations it added
      int its_after = 0;
      for (int g = 0; g < G; ++g)
        for (int r = 0; r < NR; ++r) its_after = std::max(its_after, hs[g * kMaxGroup + r].iters);
      const int trips = std::max(1, (its_after - its_before + kWhileBody - 1) / kWhileBody);
      note_launch((uint64_t)trips * (7 * kWhileBody + 1));
    }
  }
  bi_eo_final<NR, RECON><<<grid, kRedBlock, 0, st>>>(X, le, lo, x, w);
  MGT_LAUNCH_CHECK("bi_eo_final (mixed)");
  rc = fetch(w.st);
  if (rc) return rc;
  for (int g = 0; g < G; ++g)
    for (int r = 0; r < NR; ++r) {
      const BiState &s = hs[g * kMaxGroup + r];
      const int i = g * NR + r;
      const bool zero_rhs = s.b2 == 0.0;
      const double rel = zero_rhs ? 0.0 : sqrt(s.true_r2 / s.b2);
      const bool conv = zero_rhs || s.true_r2 <= s.tol2;
      report[4 * i + 0] = s.iters;
      report[4 * i + 1] = s.matvecs;
      report[4 * i + 2] = conv ? 1 : 0;
      report[4 * i + 3] = conv ? 0 : (s.reason ? s.reason : 1);
      relres[i] = rel;
      if (dot_out) {
        dot_out[2 * i] = s.dotq.re;
        dot_out[2 * i + 1] = s.dotq.im;
      }
    }
  return MGT_OK;
}

// small lattices (at most 2^13 sites per parity: 8^4, 8^3 x 16) take the
// 4-blocks-per-SM fp32 stencils
constexpr int64_t kSmallMixedVh = 8192;
static int64_t small_mixed_vh() {  // MGT_SMALL_VH overrides (A/B)
  static int64_t v = -1;
  if (v < 0) {
    const char *e = getenv("MGT_SMALL_VH");
    v = e ? atoll(e) : kSmallMixedVh;
  }
  return v;
}
#if MGT_F32_STENCIL_PAIRS
// MGT_F32_STENCIL_PAIRS=0 keeps the one-site fp32 stencils (A/B);
// MGT_PAIR_MIN_VH: smallest half volume that takes the pair stencils
static bool f32_pair_stencils() {
  static int v = -1;
  if (v < 0) {
    const char *e = getenv("MGT_F32_STENCIL_PAIRS");
    v = e ? atoi(e) : 1;
  }
  return v != 0;
}
static int64_t pair_min_vh() {
  static int64_t v = -1;
  if (v < 0) {
    const char *e = getenv("MGT_PAIR_MIN_VH");
    v = e ? atoll(e) : 0;
  }
  return v;
}
#endif
template <int NR, int RECON>
static int solve_group_mixed_any(mgt_wilson_s *h, const WilsonParams &P, int flags, double tau, const double2 *b,
                                 double2 *x, char *ws, const WSLayout &Lw, double tol, const double *tols,
                                 int max_iter, int64_t *report, double *relres, double *dot_out, int G,
                                 cudaStream_t st) {
#if MGT_F32_STENCIL_PAIRS
  // two-sites-per-thread fp32 stencils (eo_pair.cuh) need L2/2 even
  if (f32_pair_stencils() && h->g.L[2] % 4 == 0 && h->g.V / 2 > pair_min_vh())
    return solve_group_mixed<NR, RECON, eo_minb<float>(), true>(h, P, flags, tau, b, x, ws, Lw, tol, tols, max_iter,
                                                                report, relres, dot_out, G, st);
#endif
  if (h->g.V / 2 <= small_mixed_vh())
    return solve_group_mixed<NR, RECON, 4>(h, P, flags, tau, b, x, ws, Lw, tol, tols, max_iter, report, relres,
                                           dot_out, G, st);
  return solve_group_mixed<NR, RECON>(h, P, flags, tau, b, x, ws, Lw, tol, tols, max_iter, report, relres, dot_out,
                                      G, st);
}

// ---------------------------------------------------------------------------
// Distributed t-slab solve: the same kernels with DIST = 1
// leave their rank-local sums in w.red; one all-reduce per reduction point
// (2 / 1 / 3 / 3 doubles per rhs) and a one-block finisher (bi_fin) apply the
// scalar recurrences identically on every rank, so every rank takes the same
// control path.  Each stencil pass is preceded by the spin-projected face
// exchange (halo pack + grouped NCCL send/recv).
enum : int { FIN_INIT, FIN_K1, FIN_K2, FIN_K3, FIN_K4, FIN_RESID, FIN_RESTART, FIN_FINAL };

template <int NR, int KIND>
__global__ void __launch_bounds__(kRedBlock) bi_fin(BiWS w_, double tol, int maxit) {
  const BiWS w = w_.at(blockIdx.y);
  constexpr int M = (KIND == FIN_K1 || KIND == FIN_FINAL) ? 2 * NR : ((KIND == FIN_K3 || KIND == FIN_K4) ? 3 * NR : NR);
  double out[M];
#pragma unroll
  for (int j = 0; j < M; ++j) out[j] = w.red[j];
  if constexpr (KIND == FIN_INIT) init_logic<NR>(w, out, tol, maxit, 0);
  if constexpr (KIND == FIN_K1) k1_logic<NR>(w, out);
  if constexpr (KIND == FIN_K2) k2_logic<NR>(w, out);
  if constexpr (KIND == FIN_K3) k3_logic<NR>(w, out);
  if constexpr (KIND == FIN_K4) k4_logic<NR>(w, out);
  if constexpr (KIND == FIN_RESID) resid_logic<NR>(w, out);
  if constexpr (KIND == FIN_RESTART) restart_logic<NR>(w, out);
  if constexpr (KIND == FIN_FINAL)
    if (threadIdx.x < NR) w.st[threadIdx.x].dotq = C<double>(out[2 * threadIdx.x], out[2 * threadIdx.x + 1]);
}

static size_t slab_face_bytes(const mgt_wilson_s *h) {
  return align_up((size_t)kMaxGroup * 6 * h->g.stride[3] * sizeof(double2), 256);
}

template <int NR, int RECON>
static int solve_group_slab(mgt_wilson_s *h, mgt_comm_s *comm, const WilsonParams &P0, const double2 *b, double2 *x,
                            char *ws, const WSLayout &Lw, double tol, int max_iter, int64_t *report, double *relres,
                            double *dot_out, cudaStream_t st) {
  const int64_t V = h->g.V;
  BiWS w = carve(ws, Lw);
  const size_t fb = slab_face_bytes(h);
  char *hb = ws + Lw.total;
  void *to_prev = hb, *to_next = hb + fb, *from_next = hb + 2 * fb, *from_prev = hb + 3 * fb;
  const size_t face = (size_t)NR * 6 * h->g.stride[3] * sizeof(double2);
  WilsonParams P = P0;
  P.slab = 1;
  P.halo_next = from_next;
  P.halo_prev = from_prev;
  LinkField<double, RECON> lf{reinterpret_cast<const double2 *>(h->links), V};
  static int g_dsl = 0, g_str = 0;
  if (!g_dsl) g_dsl = resident_grid(bi_k1<NR, RECON, 1>, kRedBlock, (int64_t)1 << 40);
  if (!g_str) g_str = resident_grid(bi_k4<NR, 1>, kRedBlock, (int64_t)1 << 40);
  const int64_t need = (V + RhsMap<NR>::SPB - 1) / RhsMap<NR>::SPB;
  const int gd = (int)std::min<int64_t>(g_dsl, need), grid = (int)std::min<int64_t>(g_str, need);
  MGT_CUDA(cudaMemsetAsync(w.ticket, 0, 24, st));
  auto fin = [&](auto kind_tag, int m) -> int {
    constexpr int KIND = decltype(kind_tag)::value;
    int rc = comm_allreduce_sum(comm, w.red, (size_t)m, st);
    if (rc) return rc;
    bi_fin<NR, KIND><<<1, kRedBlock, 0, st>>>(w, tol, max_iter);
    note_launch(1);
    return MGT_OK;
  };
  auto exchange = [&](const double2 *f) -> int {
    int rc = halo_pack_native(h, P0, f, to_prev, to_next, NR, st);
    if (rc) return rc;
    note_launch(1);
    return comm_halo(comm, to_prev, to_next, from_next, from_prev, face, st);
  };
#define MGT_FIN(K, M)                                             \
  do {                                                            \
    int rc_ = fin(std::integral_constant<int, K>{}, M);           \
    if (rc_) return rc_;                                          \
  } while (0)
#define MGT_XCH(F)              \
  do {                          \
    int rc_ = exchange(F);      \
    if (rc_) return rc_;        \
  } while (0)
  bi_init<NR, 1><<<grid, kRedBlock, 0, st>>>(V, b, w, tol, max_iter, 0);
  note_launch(1);
  MGT_FIN(FIN_INIT, NR);
  static thread_local int *hf = nullptr;
  if (!hf) MGT_CUDA(cudaMallocHost((void **)&hf, 64 * sizeof(int)));
  for (int round = 0; round < 1000000; ++round) {
    for (int it = 0; it < kChunk; ++it) {
      MGT_XCH(w.p);
      bi_k1<NR, RECON, 1><<<gd, kRedBlock, 0, st>>>(P, lf, w);
      MGT_FIN(FIN_K1, 2 * NR);
      bi_k2<NR, 1><<<grid, kRedBlock, 0, st>>>(V, w);
      MGT_FIN(FIN_K2, NR);
      MGT_XCH(w.s);
      bi_k3<NR, RECON, 1><<<gd, kRedBlock, 0, st>>>(P, lf, w);
      MGT_FIN(FIN_K3, 3 * NR);
      bi_k4<NR, 1><<<grid, kRedBlock, 0, st>>>(V, w);
      MGT_FIN(FIN_K4, 3 * NR);
      bi_k5<NR><<<grid, kRedBlock, 0, st>>>(V, w);
      note_launch(5);
    }
    MGT_LAUNCH_CHECK("distributed bicgstab chunk");
    for (int r = 0; r < NR; ++r)
      MGT_CUDA(cudaMemcpyAsync(hf + r, &w.st[r].status, sizeof(int), cudaMemcpyDeviceToHost, st));
    MGT_CUDA(cudaStreamSynchronize(st));
    bool running = false;
    for (int r = 0; r < NR; ++r) running |= (hf[r] == ST_RUN);
    if (running) continue;
    MGT_XCH(w.x);
    bi_resid<NR, RECON, 1><<<gd, kRedBlock, 0, st>>>(P, lf, w);
    MGT_FIN(FIN_RESID, NR);
    bi_restart<NR, 1><<<grid, kRedBlock, 0, st>>>(V, w);
    MGT_FIN(FIN_RESTART, NR);
    note_launch(2);
    MGT_LAUNCH_CHECK("distributed bicgstab residual");
    for (int r = 0; r < NR; ++r)
      MGT_CUDA(cudaMemcpyAsync(hf + r, &w.st[r].status, sizeof(int), cudaMemcpyDeviceToHost, st));
    MGT_CUDA(cudaStreamSynchronize(st));
    bool again = false;
    for (int r = 0; r < NR; ++r) again |= (hf[r] == ST_RUN);
    if (!again) break;
  }
  bi_final<NR, 1><<<grid, kRedBlock, 0, st>>>(V, x, w);
  note_launch(1);
  MGT_FIN(FIN_FINAL, 2 * NR);
#undef MGT_FIN
#undef MGT_XCH
  MGT_LAUNCH_CHECK("bi_final (distributed)");
  std::vector<BiState> hs(NR);
  MGT_CUDA(cudaMemcpyAsync(hs.data(), w.st, NR * sizeof(BiState), cudaMemcpyDeviceToHost, st));
  MGT_CUDA(cudaStreamSynchronize(st));
  for (int r = 0; r < NR; ++r) {
    const BiState &s = hs[r];
    const bool zero_rhs = s.b2 == 0.0;
    const double rel = zero_rhs ? 0.0 : sqrt(s.true_r2 / s.b2);
    const bool conv = zero_rhs || s.true_r2 <= s.tol2;
    report[4 * r + 0] = s.iters;
    report[4 * r + 1] = s.matvecs;
    report[4 * r + 2] = conv ? 1 : 0;
    report[4 * r + 3] = conv ? 0 : (s.reason ? s.reason : 1);
    relres[r] = rel;
    if (dot_out) {
      dot_out[2 * r] = s.dotq.re;
      dot_out[2 * r + 1] = s.dotq.im;
    }
  }
  return MGT_OK;
}

}  // namespace mgt

using namespace mgt;

extern "C" {

size_t mgt_bicgstab_workspace_bytes(mgt_wilson_t h, int n_rhs) {
  if (!h) return 0;
  // room for the fp32 inner fields of a mixed-precision solve as well
  return ws_total(h->g.V, std::max(1, n_rhs / kMaxGroup), eo_available(h));
}

static int bicgstab_solve_impl(mgt_wilson_t h, const void *b_dev, void *x_dev, int n_rhs, int flags, double tau,
                               double tol, const double *tols, int max_iter, void *workspace_dev,
                               size_t workspace_bytes, int64_t *report_out, double *relres_out, double *dot_out_host,
                               void *stream) {
  if (!h || !b_dev || !x_dev || !workspace_dev || !report_out || !relres_out)
    return fail(MGT_ERR_INVALID, "mgt_bicgstab_solve: null argument");
  if (h->prec != 64) return fail(MGT_ERR_INVALID, "mgt_bicgstab_solve: needs a complex128 operator");
  if (tols) {
    for (int i = 0; i < n_rhs; ++i)
      if (!(tols[i] > 0.0 && tols[i] < 1.0)) return fail(MGT_ERR_INVALID, "every tol must be in (0,1)");
    tol = tols[0];
  }
  if (!(tol > 0.0 && tol < 1.0)) return fail(MGT_ERR_INVALID, "tol must be in (0,1)");
  if (max_iter < 1) return fail(MGT_ERR_INVALID, "max_iter must be >= 1");
  if (n_rhs < 1) return fail(MGT_ERR_INVALID, "n_rhs must be >= 1");
  cudaStream_t st = as_stream(stream);
  // even-odd Schur solve unless disabled (handle / MGT_SOLVE_FULL) or an extent is odd
  const bool eo = h->solve_eo && !(flags & MGT_SOLVE_FULL) && eo_available(h);
  const bool mixed = eo && (flags & MGT_SOLVE_MIXED);
  flags &= ~(MGT_SOLVE_FULL | MGT_SOLVE_MIXED);
  if (eo) {
    int rc = mixed ? eo_prepare_mixed(h, st) : eo_prepare(h, st);
    if (rc) return rc;
  }
  WilsonParams P = make_params(h, flags, tau);
  const int64_t V = h->g.V;
  // groups of kMaxGroup rhs batched into one launch per kernel, as many as
  // the workspace holds
  int gmax = 1;
  while (gmax < kMaxGroups && ws_total(V, gmax + 1, mixed) <= workspace_bytes) ++gmax;
  if (ws_total(V, 1, mixed) > workspace_bytes) return fail(MGT_ERR_INVALID, "mgt_bicgstab_solve: workspace too small");
  const size_t field = (size_t)12 * V;
  int r0 = 0;
  while (r0 < n_rhs) {
    const int left = n_rhs - r0;
    const int G = std::min(gmax, left / kMaxGroup);
    const int nr = G >= 1 ? 4 : (left >= 2 ? 2 : 1);
    const int Gc = std::max(G, 1);
    const WSLayout Lw = ws_layout(V, Gc);
    const double2 *b = (const double2 *)b_dev + r0 * field;
    double2 *x = (double2 *)x_dev + r0 * field;
    double *dot = dot_out_host ? dot_out_host + 2 * r0 : nullptr;
    const double *tl = tols ? tols + r0 : nullptr;
    char *ws = (char *)workspace_dev;
    int rc;
#define MGT_SOLVE(NR, GG)                                                                                          \
  (mixed ? (h->recon == 18 ? solve_group_mixed_any<NR, 18>(h, P, flags, tau, b, x, ws, Lw, tol, tl, max_iter,     \
                                                           report_out + 4 * r0, relres_out + r0, dot, GG, st)     \
                           : solve_group_mixed_any<NR, 12>(h, P, flags, tau, b, x, ws, Lw, tol, tl, max_iter,     \
                                                           report_out + 4 * r0, relres_out + r0, dot, GG, st))    \
   : (h->recon == 18 ? solve_group<NR, 18>(h, P, flags, tau, b, x, ws, Lw, tol, tl, max_iter, report_out + 4 * r0, \
                                            relres_out + r0, dot, eo, GG, st)                                       \
                     : solve_group<NR, 12>(h, P, flags, tau, b, x, ws, Lw, tol, tl, max_iter, report_out + 4 * r0, \
                                            relres_out + r0, dot, eo, GG, st)))
    if (nr == 4)
      rc = MGT_SOLVE(4, Gc);
    else if (nr == 2)
      rc = MGT_SOLVE(2, 1);
    else
      rc = MGT_SOLVE(1, 1);
#undef MGT_SOLVE
    if (rc) return rc;
    r0 += nr * Gc;
  }
  return MGT_OK;
}

int mgt_bicgstab_solve(mgt_wilson_t h, const void *b_dev, void *x_dev, int n_rhs, int flags, double tau, double tol,
                       int max_iter, void *workspace_dev, int64_t *report_out, double *relres_out,
                       double *dot_out_host, void *stream) {
  if (!h) return fail(MGT_ERR_INVALID, "mgt_bicgstab_solve: null argument");
  return bicgstab_solve_impl(h, b_dev, x_dev, n_rhs, flags, tau, tol, nullptr, max_iter, workspace_dev,
                             ws_total(h->g.V, 1, eo_available(h)), report_out, relres_out, dot_out_host, stream);
}

int mgt_bicgstab_solve_ws(mgt_wilson_t h, const void *b_dev, void *x_dev, int n_rhs, int flags, double tau,
                          double tol, int max_iter, void *workspace_dev, size_t workspace_bytes, int64_t *report_out,
                          double *relres_out, double *dot_out_host, void *stream) {
  return bicgstab_solve_impl(h, b_dev, x_dev, n_rhs, flags, tau, tol, nullptr, max_iter, workspace_dev,
                             workspace_bytes, report_out, relres_out, dot_out_host, stream);
}

int mgt_bicgstab_solve_tols(mgt_wilson_t h, const void *b_dev, void *x_dev, int n_rhs, int flags, double tau,
                            const double *tols, int max_iter, void *workspace_dev, size_t workspace_bytes,
                            int64_t *report_out, double *relres_out, double *dot_out_host, void *stream) {
  if (!tols) return fail(MGT_ERR_INVALID, "mgt_bicgstab_solve_tols: null tolerance array");
  return bicgstab_solve_impl(h, b_dev, x_dev, n_rhs, flags, tau, 0.0, tols, max_iter, workspace_dev,
                             workspace_bytes, report_out, relres_out, dot_out_host, stream);
}

size_t mgt_bicgstab_slab_workspace_bytes(mgt_wilson_t h, int n_rhs) {
  if (!h) return 0;
  return ws_layout(h->g.V).total + 4 * slab_face_bytes(h);
}

int mgt_bicgstab_solve_slab(mgt_wilson_t h, mgt_comm_t comm, const void *b_dev, void *x_dev, int n_rhs, int flags,
                            double tau, double tol, int max_iter, void *workspace_dev, int64_t *report_out,
                            double *relres_out, double *dot_out_host, void *stream) {
  if (!h || !comm || !b_dev || !x_dev || !workspace_dev || !report_out || !relres_out)
    return fail(MGT_ERR_INVALID, "mgt_bicgstab_solve_slab: null argument");
  if (!h->slab) return fail(MGT_ERR_INVALID, "mgt_bicgstab_solve_slab: needs a slab handle");
  if (h->prec != 64) return fail(MGT_ERR_INVALID, "mgt_bicgstab_solve_slab: needs a complex128 operator");
  if (!(tol > 0.0 && tol < 1.0)) return fail(MGT_ERR_INVALID, "tol must be in (0,1)");
  if (max_iter < 1) return fail(MGT_ERR_INVALID, "max_iter must be >= 1");
  if (n_rhs < 1) return fail(MGT_ERR_INVALID, "n_rhs must be >= 1");
  if (comm->nranks * h->g.L[3] != h->T_global)
    return fail(MGT_ERR_INVALID, "mgt_bicgstab_solve_slab: communicator size does not match the slab decomposition");
  cudaStream_t st = as_stream(stream);
  WilsonParams P = make_params(h, flags & ~MGT_SOLVE_FULL, tau);
  const int64_t V = h->g.V;
  WSLayout Lw = ws_layout(V);
  const size_t field = (size_t)12 * V;
  int r0 = 0;
  while (r0 < n_rhs) {
    const int left = n_rhs - r0;
    const int nr = left >= 4 ? 4 : (left >= 2 ? 2 : 1);
    const double2 *b = (const double2 *)b_dev + r0 * field;
    double2 *x = (double2 *)x_dev + r0 * field;
    double *dot = dot_out_host ? dot_out_host + 2 * r0 : nullptr;
    char *ws = (char *)workspace_dev;
    int rc;
#define MGT_SOLVE(NR)                                                                                          \
  (h->recon == 18 ? solve_group_slab<NR, 18>(h, comm, P, b, x, ws, Lw, tol, max_iter, report_out + 4 * r0,     \
                                              relres_out + r0, dot, st)                                        \
                  : solve_group_slab<NR, 12>(h, comm, P, b, x, ws, Lw, tol, max_iter, report_out + 4 * r0,     \
                                              relres_out + r0, dot, st))
    rc = nr == 4 ? MGT_SOLVE(4) : (nr == 2 ? MGT_SOLVE(2) : MGT_SOLVE(1));
#undef MGT_SOLVE
    if (rc) return rc;
    r0 += nr;
  }
  return MGT_OK;
}

}  // extern "C"
