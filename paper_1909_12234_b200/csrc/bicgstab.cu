// GPU-resident BiCGStab for the Wilson operator -- the TruncatedInverse solver
// plugin (reference: krylov.py:200-229; the reference's own solver is GCR,
// krylov.py:52-118, BASELINE.json names BiCGStab).
//
// Per iteration (complex BiCGStab, x0 = 0):
//   K1  v = A p                       sigma = (rhat, v)      alpha = rho/sigma
//   K2  s = r - alpha v               |s|^2  (early exit when s is converged)
//   K3  t = A s                       (t, s), |t|^2          omega = (t,s)/|t|^2
//   K4  x += alpha p + omega s; r = s - omega t;  rho' = (rhat, r), |r|^2, beta
//   K5  p = r + beta (p - omega v)
// Every reduction is fused into the producing kernel (reduce.cuh) and the
// scalar recurrences run in that kernel's last block, so the host only
// launches; it reads the per-rhs status word once per chunk of iterations.
// Convergence is confirmed on the explicitly recomputed residual b - A x
// (krylov.py:78-85, :113-118); a recursion/true-residual mismatch restarts
// with rhat = r.
#include <algorithm>
#include <vector>

#include "handle.cuh"
#include "reduce.cuh"

namespace mgt {

enum : int { ST_RUN = 0, ST_CONV = 1, ST_BREAK = 2, ST_MAXIT = 3, ST_RESTART = 4, ST_DONE = 5 };

struct BiState {
  C<double> rho, alpha, omega, beta, dotq;
  double b2, r2, s2, true_r2, tol2;
  int status, half, iters, maxit, matvecs, reason, pad0, pad1;
};

struct BiWS {
  double2 *r, *rhat, *p, *v, *s, *t;
  double *partials;
  unsigned *ticket;
  BiState *st;
};

template <int NR>
__device__ __forceinline__ bool any_running(const BiState *st, int want = ST_RUN) {
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

#define FOR_SITES(NR)                                                                          \
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n;                  \
       idx += (int64_t)gridDim.x * blockDim.x)

// ---------------------------------------------------------------------------
template <int NR>
__global__ void __launch_bounds__(kRedBlock) bi_init(int64_t V, const double2 *__restrict__ b, double2 *__restrict__ x,
                                                     BiWS w, double tol, int maxit) {
  const int64_t n = V * NR;
  double acc[1] = {0.0};
  FOR_SITES(NR) {
    const int64_t site = idx / NR;
    const int rhs = (int)(idx % NR);
    const int64_t base = (int64_t)rhs * 12 * V + site;
#pragma unroll
    for (int c = 0; c < 12; ++c) {
      const int64_t o = base + (int64_t)c * V;
      double2 bb = b[o];
      w.r[o] = bb;
      w.rhat[o] = bb;
      w.p[o] = bb;
      x[o] = make_double2(0.0, 0.0);
      acc[0] += bb.x * bb.x + bb.y * bb.y;
    }
  }
  if (reduce_publish<NR, 1>(acc, w.partials, w.ticket)) {
    double out[NR];
    reduce_finish<NR>(w.partials, w.ticket, out);
    if (threadIdx.x < NR) {
      BiState &s = w.st[threadIdx.x];
      const double b2 = out[threadIdx.x];
      s.b2 = b2;
      s.r2 = b2;
      s.s2 = b2;
      s.true_r2 = b2;
      s.tol2 = tol * tol * b2;
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
}

// K1: v = A p ; sigma = (rhat, v)
template <int NR, int RECON>
__global__ void __launch_bounds__(kRedBlock, 3) bi_k1(WilsonParams P, LinkField<double, RECON> L, BiWS w) {
  if (!any_running<NR>(w.st)) return;
  const int my = threadIdx.x % NR;  // blockDim and the grid stride are multiples of NR
  const bool run_me = (w.st[my].status == ST_RUN);
  const int64_t V = P.g.V, n = V * NR;
  double acc[2] = {0.0, 0.0};
  FOR_SITES(NR) {
    const int64_t site = sched_site(P.sched, idx / NR);
    const int rhs = (int)(idx % NR);
    if (!run_me) continue;
    const int64_t off = (int64_t)rhs * 12 * V;
    C<double> y[4][3], xc[4][3];
    wilson_eval<double, RECON>(P, w.p + off, L, site, y, xc);
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const int64_t o = off + (int64_t)(a * 3 + c) * V + site;
        stc(w.v + o, y[a][c]);
        C<double> rh = ldc(w.rhat + o);
        acc[0] += rh.re * y[a][c].re + rh.im * y[a][c].im;
        acc[1] += rh.re * y[a][c].im - rh.im * y[a][c].re;
      }
  }
  if (reduce_publish<NR, 2>(acc, w.partials, w.ticket)) {
    double out[NR * 2];
    reduce_finish<NR * 2>(w.partials, w.ticket, out);
    if (threadIdx.x < NR && run_me) {
      BiState &s = w.st[threadIdx.x];
      C<double> sigma(out[2 * threadIdx.x], out[2 * threadIdx.x + 1]);
      s.matvecs += 1;
      if (czero(sigma) || !isfinite(sigma.re) || !isfinite(sigma.im)) {
        s.status = ST_BREAK;
        s.reason = 2;
      } else {
        s.alpha = cdiv(s.rho, sigma);
      }
    }
  }
}

// K2: s = r - alpha v ; |s|^2
template <int NR>
__global__ void __launch_bounds__(kRedBlock) bi_k2(int64_t V, BiWS w) {
  if (!any_running<NR>(w.st)) return;
  const int my = threadIdx.x % NR;
  const bool run_me = (w.st[my].status == ST_RUN);
  const C<double> al = w.st[my].alpha;
  const int64_t n = V * NR;
  double acc[1] = {0.0};
  FOR_SITES(NR) {
    const int64_t site = idx / NR;
    const int rhs = (int)(idx % NR);
    if (!run_me) continue;
    const int64_t base = (int64_t)rhs * 12 * V + site;
#pragma unroll
    for (int c = 0; c < 12; ++c) {
      const int64_t o = base + (int64_t)c * V;
      C<double> rr = ldc(w.r + o), vv = ldc(w.v + o);
      C<double> ss = rr - al * vv;
      stc(w.s + o, ss);
      acc[0] += cabs2(ss);
    }
  }
  if (reduce_publish<NR, 1>(acc, w.partials, w.ticket)) {
    double out[NR];
    reduce_finish<NR>(w.partials, w.ticket, out);
    if (threadIdx.x < NR && run_me) {
      BiState &s = w.st[threadIdx.x];
      s.s2 = out[threadIdx.x];
      s.half = (s.s2 <= s.tol2) ? 1 : 0;
    }
  }
}

// K3: t = A s ; (t, s), |t|^2
template <int NR, int RECON>
__global__ void __launch_bounds__(kRedBlock, 3) bi_k3(WilsonParams P, LinkField<double, RECON> L, BiWS w) {
  if (!any_running<NR>(w.st)) return;
  const int my = threadIdx.x % NR;  // blockDim and the grid stride are multiples of NR
  const bool run_me = (w.st[my].status == ST_RUN);
  const int64_t V = P.g.V, n = V * NR;
  double acc[3] = {0.0, 0.0, 0.0};
  FOR_SITES(NR) {
    const int64_t site = sched_site(P.sched, idx / NR);
    const int rhs = (int)(idx % NR);
    if (!run_me) continue;
    const int64_t off = (int64_t)rhs * 12 * V;
    C<double> y[4][3], xc[4][3];
    wilson_eval<double, RECON>(P, w.s + off, L, site, y, xc);
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const int64_t o = off + (int64_t)(a * 3 + c) * V + site;
        stc(w.t + o, y[a][c]);
        const C<double> tt = y[a][c], ss = xc[a][c];
        acc[0] += tt.re * ss.re + tt.im * ss.im;
        acc[1] += tt.re * ss.im - tt.im * ss.re;
        acc[2] += cabs2(tt);
      }
  }
  if (reduce_publish<NR, 3>(acc, w.partials, w.ticket)) {
    double out[NR * 3];
    reduce_finish<NR * 3>(w.partials, w.ticket, out);
    if (threadIdx.x < NR && run_me) {
      BiState &s = w.st[threadIdx.x];
      C<double> ts(out[3 * threadIdx.x], out[3 * threadIdx.x + 1]);
      const double tt = out[3 * threadIdx.x + 2];
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
}

// K4: x += alpha p + omega s ; r = s - omega t ; rho' = (rhat, r), |r|^2
template <int NR>
__global__ void __launch_bounds__(kRedBlock) bi_k4(int64_t V, double2 *__restrict__ x, BiWS w) {
  if (!any_running<NR>(w.st)) return;
  const int my = threadIdx.x % NR;
  const bool run_me = (w.st[my].status == ST_RUN);
  const C<double> al = w.st[my].alpha, om = w.st[my].omega;
  const int64_t n = V * NR;
  double acc[3] = {0.0, 0.0, 0.0};
  FOR_SITES(NR) {
    const int64_t site = idx / NR;
    const int rhs = (int)(idx % NR);
    if (!run_me) continue;
    const int64_t base = (int64_t)rhs * 12 * V + site;
#pragma unroll
    for (int c = 0; c < 12; ++c) {
      const int64_t o = base + (int64_t)c * V;
      C<double> xx = ldc(x + o), pp = ldc(w.p + o), ss = ldc(w.s + o), tt = ldc(w.t + o), rh = ldc(w.rhat + o);
      xx = xx + al * pp + om * ss;
      C<double> rr = ss - om * tt;
      stc(x + o, xx);
      stc(w.r + o, rr);
      acc[0] += rh.re * rr.re + rh.im * rr.im;
      acc[1] += rh.re * rr.im - rh.im * rr.re;
      acc[2] += cabs2(rr);
    }
  }
  if (reduce_publish<NR, 3>(acc, w.partials, w.ticket)) {
    double out[NR * 3];
    reduce_finish<NR * 3>(w.partials, w.ticket, out);
    if (threadIdx.x < NR && run_me) {
      BiState &s = w.st[threadIdx.x];
      C<double> rho_new(out[3 * threadIdx.x], out[3 * threadIdx.x + 1]);
      s.r2 = out[3 * threadIdx.x + 2];
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
}

// K5: p = r + beta (p - omega v)
template <int NR>
__global__ void __launch_bounds__(kRedBlock) bi_k5(int64_t V, BiWS w) {
  if (!any_running<NR>(w.st)) return;
  const int my = threadIdx.x % NR;
  const bool run_me = (w.st[my].status == ST_RUN);
  const C<double> be = w.st[my].beta, om = w.st[my].omega;
  const int64_t n = V * NR;
  FOR_SITES(NR) {
    const int64_t site = idx / NR;
    const int rhs = (int)(idx % NR);
    if (!run_me) continue;
    const int64_t base = (int64_t)rhs * 12 * V + site;
#pragma unroll
    for (int c = 0; c < 12; ++c) {
      const int64_t o = base + (int64_t)c * V;
      C<double> rr = ldc(w.r + o), pp = ldc(w.p + o), vv = ldc(w.v + o);
      stc(w.p + o, rr + be * (pp - om * vv));
    }
  }
}

// True residual r = b - A x for every rhs that stopped (status CONV/MAXIT/
// BREAK); records |r|^2 in true_r2.
template <int NR, int RECON>
__global__ void __launch_bounds__(kRedBlock, 3) bi_resid(WilsonParams P, LinkField<double, RECON> L, const double2 *__restrict__ b,
                                                      const double2 *__restrict__ x, BiWS w) {
  bool any = false;
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    const int st = w.st[r].status;
    any |= (st == ST_CONV || st == ST_MAXIT || st == ST_BREAK);
  }
  if (!any) return;
  const int my = threadIdx.x % NR;
  const int st_me = w.st[my].status;
  const bool act_me = (st_me == ST_CONV || st_me == ST_MAXIT || st_me == ST_BREAK);
  const int64_t V = P.g.V, n = V * NR;
  double acc[1] = {0.0};
  FOR_SITES(NR) {
    const int64_t site = sched_site(P.sched, idx / NR);
    const int rhs = (int)(idx % NR);
    if (!act_me) continue;
    const int64_t off = (int64_t)rhs * 12 * V;
    C<double> y[4][3], xc[4][3];
    wilson_eval<double, RECON>(P, x + off, L, site, y, xc);
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const int64_t o = off + (int64_t)(a * 3 + c) * V + site;
        C<double> rr = ldc(b + o) - y[a][c];
        stc(w.r + o, rr);
        acc[0] += cabs2(rr);
      }
  }
  if (reduce_publish<NR, 1>(acc, w.partials, w.ticket)) {
    double out[NR];
    reduce_finish<NR>(w.partials, w.ticket, out);
    if (threadIdx.x < NR && act_me) {
      BiState &s = w.st[threadIdx.x];
      s.true_r2 = out[threadIdx.x];
      s.matvecs += 1;
      const bool ok = s.true_r2 <= s.tol2;
      if (ok) {
        s.status = ST_DONE;
        s.reason = 0;
      } else if (s.status == ST_CONV && s.iters < s.maxit) {
        s.status = ST_RESTART;  // recursion drifted from the true residual
      } else {
        s.status = ST_DONE;
        if (s.reason == 0) s.reason = 1;
      }
    }
  }
}

// Restart for rhs flagged ST_RESTART: rhat = p = r (r holds the true residual)
template <int NR>
__global__ void __launch_bounds__(kRedBlock) bi_restart(int64_t V, BiWS w) {
  if (!any_running<NR>(w.st, ST_RESTART)) return;
  const int my = threadIdx.x % NR;
  const bool act_me = (w.st[my].status == ST_RESTART);
  const int64_t n = V * NR;
  double acc[1] = {0.0};
  FOR_SITES(NR) {
    const int64_t site = idx / NR;
    const int rhs = (int)(idx % NR);
    if (!act_me) continue;
    const int64_t base = (int64_t)rhs * 12 * V + site;
#pragma unroll
    for (int c = 0; c < 12; ++c) {
      const int64_t o = base + (int64_t)c * V;
      double2 rr = w.r[o];
      w.rhat[o] = rr;
      w.p[o] = rr;
      acc[0] += rr.x * rr.x + rr.y * rr.y;
    }
  }
  if (reduce_publish<NR, 1>(acc, w.partials, w.ticket)) {
    double out[NR];
    reduce_finish<NR>(w.partials, w.ticket, out);
    if (threadIdx.x < NR && act_me) {
      BiState &s = w.st[threadIdx.x];
      s.r2 = out[threadIdx.x];
      s.rho = C<double>(s.r2, 0.0);
      s.alpha = C<double>(1.0, 0.0);
      s.omega = C<double>(1.0, 0.0);
      s.half = 0;
      s.status = ST_RUN;
    }
  }
}

// q = vdot(b, x) per rhs (Hutchinson quadratic form, trace.py:104)
template <int NR>
__global__ void __launch_bounds__(kRedBlock) bi_dot(int64_t V, const double2 *__restrict__ b, const double2 *__restrict__ x,
                                                    BiWS w) {
  const int64_t n = V * NR;
  double acc[2] = {0.0, 0.0};
  FOR_SITES(NR) {
    const int64_t site = idx / NR;
    const int rhs = (int)(idx % NR);
    const int64_t base = (int64_t)rhs * 12 * V + site;
#pragma unroll
    for (int c = 0; c < 12; ++c) {
      const int64_t o = base + (int64_t)c * V;
      C<double> bb = ldc(b + o), xx = ldc(x + o);
      acc[0] += bb.re * xx.re + bb.im * xx.im;
      acc[1] += bb.re * xx.im - bb.im * xx.re;
    }
  }
  if (reduce_publish<NR, 2>(acc, w.partials, w.ticket)) {
    double out[NR * 2];
    reduce_finish<NR * 2>(w.partials, w.ticket, out);
    if (threadIdx.x < NR) w.st[threadIdx.x].dotq = C<double>(out[2 * threadIdx.x], out[2 * threadIdx.x + 1]);
  }
}

// ---------------------------------------------------------------------------
static size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

struct WSLayout {
  size_t field, partials, total;
  int grid;
};

static WSLayout ws_layout(int64_t V, int NRmax) {
  WSLayout L;
  L.field = align_up((size_t)NRmax * 12 * V * sizeof(double2), 256);
  L.grid = kNumSMs * 16;  // upper bound of any resident grid at 128 threads
  L.partials = align_up((size_t)L.grid * NRmax * 4 * sizeof(double), 256);
  L.total = 6 * L.field + L.partials + 256 /*ticket*/ + align_up(NRmax * sizeof(BiState), 256);
  return L;
}

template <int NR, int RECON>
static int solve_group(mgt_wilson_s *h, const WilsonParams &P, const double2 *b, double2 *x, int64_t V, char *ws,
                       const WSLayout &Lw, double tol, int max_iter, int64_t *report, double *relres,
                       double *dot_out, cudaStream_t st) {
  BiWS w;
  char *q = ws;
  w.r = (double2 *)q; q += Lw.field;
  w.rhat = (double2 *)q; q += Lw.field;
  w.p = (double2 *)q; q += Lw.field;
  w.v = (double2 *)q; q += Lw.field;
  w.s = (double2 *)q; q += Lw.field;
  w.t = (double2 *)q; q += Lw.field;
  w.partials = (double *)q; q += Lw.partials;
  w.ticket = (unsigned *)q; q += 256;
  w.st = (BiState *)q;
  LinkField<double, RECON> lf{reinterpret_cast<const double2 *>(h->links), V};
  // resident grids (occupancy-derived), cached per template instance
  static int g_dsl = 0, g_str = 0;
  if (!g_dsl) g_dsl = resident_grid(bi_k1<NR, RECON>, kRedBlock, (int64_t)1 << 40);
  if (!g_str) g_str = resident_grid(bi_k4<NR>, kRedBlock, (int64_t)1 << 40);
  const int64_t need = (V * NR + kRedBlock - 1) / kRedBlock;
  const int gd = (int)std::min<int64_t>(g_dsl, need), grid = (int)std::min<int64_t>(g_str, need);
  MGT_CUDA(cudaMemsetAsync(w.ticket, 0, sizeof(unsigned), st));
  bi_init<NR><<<grid, kRedBlock, 0, st>>>(V, b, x, w, tol, max_iter);
  MGT_LAUNCH_CHECK("bi_init");
  int *flags = h->host_flags;
  int chunk = 4;
  for (int round = 0; round < 1000000; ++round) {
    for (int it = 0; it < chunk; ++it) {
      bi_k1<NR, RECON><<<gd, kRedBlock, 0, st>>>(P, lf, w);
      bi_k2<NR><<<grid, kRedBlock, 0, st>>>(V, w);
      bi_k3<NR, RECON><<<gd, kRedBlock, 0, st>>>(P, lf, w);
      bi_k4<NR><<<grid, kRedBlock, 0, st>>>(V, x, w);
      bi_k5<NR><<<grid, kRedBlock, 0, st>>>(V, w);
      note_launch(5);
    }
    MGT_LAUNCH_CHECK("bicgstab iteration");
    for (int r = 0; r < NR; ++r)
      MGT_CUDA(cudaMemcpyAsync(flags + r, &w.st[r].status, sizeof(int), cudaMemcpyDeviceToHost, st));
    MGT_CUDA(cudaStreamSynchronize(st));
    bool running = false;
    for (int r = 0; r < NR; ++r) running |= (flags[r] == ST_RUN);
    if (running) {
      chunk = std::min(chunk * 2, 16);
      continue;
    }
    bi_resid<NR, RECON><<<gd, kRedBlock, 0, st>>>(P, lf, b, x, w);
    bi_restart<NR><<<grid, kRedBlock, 0, st>>>(V, w);
    note_launch(2);
    MGT_LAUNCH_CHECK("bicgstab residual");
    for (int r = 0; r < NR; ++r)
      MGT_CUDA(cudaMemcpyAsync(flags + r, &w.st[r].status, sizeof(int), cudaMemcpyDeviceToHost, st));
    MGT_CUDA(cudaStreamSynchronize(st));
    bool again = false;
    for (int r = 0; r < NR; ++r) again |= (flags[r] == ST_RUN);
    if (!again) break;
    chunk = 4;
  }
  if (dot_out) {
    bi_dot<NR><<<grid, kRedBlock, 0, st>>>(V, b, x, w);
    MGT_LAUNCH_CHECK("bi_dot");
  }
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
  return ws_layout(h->g.V, 4).total;
}

int mgt_bicgstab_solve(mgt_wilson_t h, const void *b_dev, void *x_dev, int n_rhs, int flags, double tau, double tol,
                       int max_iter, void *workspace_dev, int64_t *report_out, double *relres_out,
                       double *dot_out_host, void *stream) {
  if (!h || !b_dev || !x_dev || !workspace_dev || !report_out || !relres_out)
    return fail(MGT_ERR_INVALID, "mgt_bicgstab_solve: null argument");
  if (h->prec != 64) return fail(MGT_ERR_INVALID, "mgt_bicgstab_solve: needs a complex128 operator");
  if (!(tol > 0.0 && tol < 1.0)) return fail(MGT_ERR_INVALID, "tol must be in (0,1)");
  if (max_iter < 1) return fail(MGT_ERR_INVALID, "max_iter must be >= 1");
  if (n_rhs < 1) return fail(MGT_ERR_INVALID, "n_rhs must be >= 1");
  cudaStream_t st = as_stream(stream);
  WilsonParams P = make_params(h, flags, tau);
  const int64_t V = h->g.V;
  WSLayout Lw = ws_layout(V, 4);
  const size_t field = (size_t)12 * V;
  int r0 = 0;
  while (r0 < n_rhs) {
    const int left = n_rhs - r0;
    const int nr = left >= 4 ? 4 : (left >= 2 ? 2 : 1);
    const double2 *b = (const double2 *)b_dev + r0 * field;
    double2 *x = (double2 *)x_dev + r0 * field;
    double *dot = dot_out_host ? dot_out_host + 2 * r0 : nullptr;
    int rc;
    char *ws = (char *)workspace_dev;
#define MGT_SOLVE(NR)                                                                                        \
  (h->recon == 18 ? solve_group<NR, 18>(h, P, b, x, V, ws, Lw, tol, max_iter, report_out + 4 * r0,           \
                                         relres_out + r0, dot, st)                                            \
                  : solve_group<NR, 12>(h, P, b, x, V, ws, Lw, tol, max_iter, report_out + 4 * r0,           \
                                         relres_out + r0, dot, st))
    if (nr == 4)
      rc = MGT_SOLVE(4);
    else if (nr == 2)
      rc = MGT_SOLVE(2);
    else
      rc = MGT_SOLVE(1);
#undef MGT_SOLVE
    if (rc) return rc;
    r0 += nr;
  }
  return MGT_OK;
}

}  // extern "C"
