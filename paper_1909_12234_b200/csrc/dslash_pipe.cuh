// Wilson-Dirac plain apply with the neighbour spinors staged through shared
// memory by asynchronous copies (cp.async / LDGSTS), sm_100a.  Opt-in
// (MGT_DSLASH_VARIANT=2): measured SLOWER than the register-staged kernel.
//
// The thread-per-site kernel (dslash_core.cuh) keeps one hop's loads in
// flight per thread in registers and then waits for them (ncu: 4.9 TB/s of
// DRAM traffic, long-scoreboard stalls at 12 warps per SM).  Here every
// thread copies the 12 neighbour components of the hops DEPTH items ahead
// straight into its own shared-memory slots -- loads in flight hold no
// registers -- and the links of the next LD hops are staged in registers.
// The pipeline runs across chunk boundaries (the next chunk's index is
// fetched one chunk ahead, one block barrier per chunk), so a thread always
// has DEPTH spinor items and LD links in flight.
//
// Result (profiles/r02s5_smem_staged_dslash_ab_rejected.txt): 0.62-0.68x
// the default at 32^4 / 48^3 x 96 in fp64 (263 vs 178 us, 2.73 vs 1.79 ms),
// 0.65-0.72x in fp32.  Every staged byte crosses the L1 data banks twice
// (LDGSTS write + LDS read: l1tex throughput 61 % at 3.1 TB/s of DRAM
// traffic, against 33 % for the register-staged kernel at 4.9 TB/s), so the
// shared-memory path saturates before HBM does; deeper pipelines (DEPTH 3)
// and a two-hop link lookahead (spills) do not change that.  Kept as the
// measured answer to "stage the neighbour sites through shared memory".
//
// Same per-site arithmetic, in the same order, as wilson_eval (equal to the
// default kernel up to FMA contraction, tests/test_operator_gpu.py).
// (Operator definition: reference lattice.py:274-318 restated in 4D, see
// dslash_core.cuh.)
#pragma once
#include <type_traits>

#include "dslash_core.cuh"

namespace mgt {

#ifndef MGT_PIPE_DEPTH
#define MGT_PIPE_DEPTH 2
#endif
#ifndef MGT_PIPE_LD
#define MGT_PIPE_LD 1
#endif

template <int BYTES>
__device__ __forceinline__ void cp_async_ca(uint32_t dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(dst), "l"(src), "n"(BYTES) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// the raw (stored) elements of one link, before the third-row reconstruction
template <typename R, int RECON>
struct RawLink {
  cplx<R> e[RECON / 2];
};

template <typename R, int RECON>
__device__ __forceinline__ void raw_link_load(const LinkField<R, RECON> &lf, int mu, int64_t site,
                                              RawLink<R, RECON> &r) {
  if constexpr (RECON == 12 && MGT_LINK_PAIRS) {
    const cpair<R> *q = reinterpret_cast<const cpair<R> *>(lf.p) + (int64_t)mu * 3 * lf.V + site;
#pragma unroll
    for (int pp = 0; pp < 3; ++pp) {
      const cpair<R> v = q[pp * lf.V];
      r.e[2 * pp] = v.a;
      r.e[2 * pp + 1] = v.b;
    }
  } else {
    const cplx<R> *q = lf.p + (int64_t)mu * (RECON / 2) * lf.V + site;
#pragma unroll
    for (int e = 0; e < RECON / 2; ++e) r.e[e] = __ldg(q + e * lf.V);
  }
}

template <typename R, int RECON>
__device__ __forceinline__ void raw_link_expand(const RawLink<R, RECON> &r, C<R> (&u)[3][3]) {
#pragma unroll
  for (int e = 0; e < RECON / 2; ++e) u[e / 3][e % 3] = C<R>(r.e[e].x, r.e[e].y);
  if constexpr (RECON == 12) {
    u[2][0] = conj(u[0][1] * u[1][2] - u[0][2] * u[1][1]);
    u[2][1] = conj(u[0][2] * u[1][0] - u[0][0] * u[1][2]);
    u[2][2] = conj(u[0][0] * u[1][1] - u[0][1] * u[1][0]);
  }
}

struct PipeSite {
  int64_t site;
  int x[4];
  int valid;
};

// item K of a site: hops t+, t-, x0+, x0-, x1+, x1-, x2+, x2- (the order of
// wilson_eval), then the centre (K = 8)
template <int K>
struct PipeItem {
  static constexpr int MU = (K / 2 + 3) & 3;
  static constexpr bool FWD = (K & 1) == 0;
};

template <int K>
__device__ __forceinline__ int64_t pipe_neighbour(const Geom &g, const PipeSite &s) {
  if constexpr (K == 8) {
    return s.site;
  } else {
    constexpr int MU = PipeItem<K>::MU;
    const int L = g.L[MU];
    const int64_t st = g.stride[MU];
    if constexpr (PipeItem<K>::FWD)
      return (s.x[MU] == L - 1) ? s.site - (int64_t)(L - 1) * st : s.site + st;
    else
      return (s.x[MU] == 0) ? s.site + (int64_t)(L - 1) * st : s.site - st;
  }
}

// copy the 12 components of item K's spinor into this thread's slots of a
// stage; always commits a group (empty for an idle thread) so that group
// counting is uniform
template <int K, typename R>
__device__ __forceinline__ void pipe_issue(const Geom &g, const cplx<R> *__restrict__ in, const PipeSite &s,
                                           uint32_t slot) {
  if (s.valid) {
    const cplx<R> *src = in + pipe_neighbour<K>(g, s);
#pragma unroll
    for (int j = 0; j < 12; ++j)
      cp_async_ca<sizeof(cplx<R>)>(slot + j * 128 * (uint32_t)sizeof(cplx<R>), src + (int64_t)j * g.V);
  }
  cp_async_commit();
}

template <int K, typename R, int RECON>
__device__ __forceinline__ void pipe_link(const Geom &g, const LinkField<R, RECON> &lf, const PipeSite &s,
                                          RawLink<R, RECON> &r) {
  if constexpr (K < 8) {
    if (s.valid) raw_link_load(lf, PipeItem<K>::MU, PipeItem<K>::FWD ? s.site : pipe_neighbour<K>(g, s), r);
  }
}

// spin projection of item K's staged neighbour (12 components at sb[j * 128])
template <int K, typename R>
__device__ __forceinline__ void pipe_project(const cplx<R> *sb, R g5in, C<R> (&h)[2][3]) {
  constexpr int MU = PipeItem<K>::MU;
  constexpr bool FWD = PipeItem<K>::FWD;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const cplx<R> v0 = sb[(0 * 3 + c) * 128], v1 = sb[(1 * 3 + c) * 128];
    const cplx<R> v2 = sb[(2 * 3 + c) * 128], v3 = sb[(3 * 3 + c) * 128];
    C<R> p0(v0.x, v0.y), p1(v1.x, v1.y);
    C<R> p2 = g5in * C<R>(v2.x, v2.y);
    C<R> p3 = g5in * C<R>(v3.x, v3.y);
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
}

// colour multiply and reconstruction of hop K (the arithmetic of wilson_hop)
template <int K, typename R, int RECON>
__device__ __forceinline__ void pipe_multiply(const C<R> (&h)[2][3], const RawLink<R, RECON> &raw,
                                              const PipeSite &s, const Geom &g, bool antiperiodic,
                                              C<R> (&acc)[4][3]) {
  constexpr int MU = PipeItem<K>::MU;
  constexpr bool FWD = PipeItem<K>::FWD;
  R ph = R(1);
  if constexpr (MU == 3) {
    if (antiperiodic && s.x[3] == (FWD ? g.L[3] - 1 : 0)) ph = R(-1);
  }
  C<R> u[3][3];
  raw_link_expand(raw, u);
  C<R> w[2][3];
#pragma unroll
  for (int a = 0; a < 2; ++a) {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      C<R> t(R(0), R(0));
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        if constexpr (FWD)
          t = cfma(u[i][j], h[a][j], t);
        else
          t = cfma_conj(u[j][i], h[a][j], t);
      }
      w[a][i] = ph * t;
    }
  }
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

template <typename R>
struct PipeTraits {
  // resident blocks per SM (registers): as the register-staged kernel
  static constexpr int MINB = sizeof(R) == 8 ? 3 : 5;
};

template <typename R, int RECON, int DEPTH, int LD>
__global__ void __launch_bounds__(128, PipeTraits<R>::MINB)
    wilson_apply_pipe_kernel(WilsonParams P, const cplx<R> *__restrict__ in, cplx<R> *__restrict__ out,
                             LinkField<R, RECON> links, unsigned long long *ctr) {
  extern __shared__ __align__(16) unsigned char pipe_smem[];
  __shared__ long long cnext[2];
  static_assert(DEPTH >= 1 && DEPTH <= 4 && LD >= 1 && LD <= 4, "pipeline depths");
  constexpr int AHEAD = DEPTH > LD ? DEPTH : LD;
  constexpr int KSYNC = 9 - AHEAD;  // first step that touches the next chunk's site
  constexpr uint32_t STAGE = 12 * 128 * (uint32_t)sizeof(cplx<R>);
  cplx<R> *buf = reinterpret_cast<cplx<R> *>(pipe_smem);
  const int tid = threadIdx.x;
  const uint32_t slot0 = (uint32_t)__cvta_generic_to_shared(buf + tid);
  const int64_t V = P.g.V;
  const int64_t nch = (V + 127) / 128;
  const R g5in = (R)P.g5in;
  const bool ap = P.antiperiodic != 0;

  auto make_site = [&](int64_t chunk) {
    PipeSite s;
    const int64_t o = chunk * 128 + tid;
    s.valid = (chunk < nch && o < V) ? 1 : 0;
    s.site = sched_site(P.sched, s.valid ? o : 0);
    native_coords(P.g, s.site, s.x);
    return s;
  };

  if (tid == 0) cnext[0] = (long long)atomicAdd(ctr, 1ull);
  __syncthreads();
  int64_t chunk = cnext[0];
  int par = 1;
  PipeSite cur = make_site(chunk), nxt = cur;
  int stage = 0;  // stage of the item being consumed
  RawLink<R, RECON> raw[LD + 1];

  // prologue: items 0 .. DEPTH-1 and links 0 .. LD-1 of the first chunk
  {
    int st = 0;
    auto pro = [&](auto kc) {
      constexpr int K = decltype(kc)::value;
      if constexpr (K < DEPTH) {
        pipe_issue<K, R>(P.g, in, cur, slot0 + st * STAGE);
        st = (st + 1 == DEPTH) ? 0 : st + 1;
      }
      if constexpr (K < LD) pipe_link<K, R, RECON>(P.g, links, cur, raw[K]);
    };
    pro(std::integral_constant<int, 0>{});
    pro(std::integral_constant<int, 1>{});
    pro(std::integral_constant<int, 2>{});
    pro(std::integral_constant<int, 3>{});
  }

  while (chunk < nch) {
    if (tid == 0) cnext[par] = (long long)atomicAdd(ctr, 1ull);
    int64_t nchunk = nch;
    C<R> acc[4][3];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int c = 0; c < 3; ++c) acc[a][c] = C<R>(R(0), R(0));
    C<R> xc[4][3];

    auto step = [&](auto kc) {
      constexpr int K = decltype(kc)::value;
      if constexpr (K == KSYNC) {
        __syncthreads();
        nchunk = cnext[par];
        nxt = make_site(nchunk);
      }
      cp_async_wait<DEPTH - 1>();
      const cplx<R> *sb = buf + (size_t)stage * (12 * 128) + tid;
      // link of item K + LD: a hop of this chunk, the centre (none) or a hop of the next chunk
      if constexpr (K + LD < 8)
        pipe_link<K + LD, R, RECON>(P.g, links, cur, raw[LD]);
      else if constexpr (K + LD > 8)
        pipe_link<K + LD - 9, R, RECON>(P.g, links, nxt, raw[LD]);
      C<R> h[2][3];
      if constexpr (K < 8) {
        pipe_project<K, R>(sb, g5in, h);
      } else {
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const cplx<R> v = sb[(a * 3 + c) * 128];
            xc[a][c] = C<R>(v.x, v.y);
          }
      }
      // the stage just read is free: item K + DEPTH goes into it
      if constexpr (K + DEPTH <= 8)
        pipe_issue<K + DEPTH, R>(P.g, in, cur, slot0 + stage * STAGE);
      else
        pipe_issue<K + DEPTH - 9, R>(P.g, in, nxt, slot0 + stage * STAGE);
      if constexpr (K < 8) pipe_multiply<K, R, RECON>(h, raw[0], cur, P.g, ap, acc);
#pragma unroll
      for (int i = 0; i < LD; ++i) raw[i] = raw[i + 1];
      stage = (stage + 1 == DEPTH) ? 0 : stage + 1;
    };
    step(std::integral_constant<int, 0>{});
    step(std::integral_constant<int, 1>{});
    step(std::integral_constant<int, 2>{});
    step(std::integral_constant<int, 3>{});
    step(std::integral_constant<int, 4>{});
    step(std::integral_constant<int, 5>{});
    step(std::integral_constant<int, 6>{});
    step(std::integral_constant<int, 7>{});
    step(std::integral_constant<int, 8>{});

    if (cur.valid) {
      const C<R> dup((R)P.diag_up_re, (R)P.diag_up_im);
      const C<R> ddn((R)P.diag_dn_re, (R)P.diag_dn_im);
      const R half = R(0.5);
      const R g5out = (R)P.g5out;
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          C<R> v = xc[a][c], y;
          if (a >= 2) {
            v = g5in * v;
            C<R> r = ddn * v - half * acc[a][c];
            y = g5out * r;
          } else {
            y = dup * v - half * acc[a][c];
          }
          stc_cs(out + (a * 3 + c) * V + cur.site, y);
        }
    }
    cur = nxt;
    chunk = nchunk;
    par ^= 1;
  }
  cp_async_wait<0>();
}

}  // namespace mgt
