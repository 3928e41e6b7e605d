// Wilson-Dirac operator handle and the plain apply kernel (C ABI).
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>

#include "dslash_pipe.cuh"
#include "handle.cuh"
#include "reduce.cuh"

namespace mgt {

static thread_local std::string g_last_error;
static std::atomic<uint64_t> g_launches{0};

void set_error(const std::string &msg) { g_last_error = msg; }
int fail(int code, const std::string &msg) {
  g_last_error = msg;
  return code;
}
int cuda_fail(cudaError_t e, const char *what) {
  g_last_error = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
  return MGT_ERR_CUDA;
}
void note_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

cudaError_t scratch_alloc(void **p, size_t bytes, cudaStream_t st) {
  static thread_local int pool_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (pool_dev != dev) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    pool_dev = dev;
  }
  return cudaMallocAsync(p, bytes, st);
}

int num_sms() {
  static std::atomic<int> cache[64];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  int v = cache[dev].load(std::memory_order_relaxed);
  if (v > 0) return v;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v < 1) {
    cudaGetLastError();
    return 148;  // B200; only reached without a usable device (no launch can follow)
  }
  cache[dev].store(v, std::memory_order_relaxed);
  return v;
}

int blocks_per_sm(const void *kernel, int block, size_t smem) {
  static std::mutex mu;
  static std::map<std::tuple<int, const void *, int, size_t>, int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_tuple(dev, kernel, block, smem);
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  int per_sm = 0;
  const cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, smem);
  if (e != cudaSuccess) {
    cuda_fail(e, "cudaOccupancyMaxActiveBlocksPerMultiprocessor");
    return -1;
  }
  std::lock_guard<std::mutex> lk(mu);
  cache[key] = per_sm;
  return per_sm;
}

// ---------------------------------------------------------------------------
// links: reference layout (V_ref, 4, 3, 3) complex128 -> native SoA
template <typename R, int RECON>
__global__ void links_from_ref_kernel(Geom g, const double2 *__restrict__ ref, cplx<R> *__restrict__ out) {
  constexpr int NL = RECON / 2;
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < g.V; s += (int64_t)gridDim.x * blockDim.x) {
    int x[4];
    native_coords(g, s, x);
    const int64_t r = ref_site(g, x);
#pragma unroll
    for (int mu = 0; mu < 4; ++mu) {
#pragma unroll
      for (int e = 0; e < NL; ++e) {
        double2 v = ref[(r * 4 + mu) * 9 + e];
        cplx<R> o;
        o.x = (R)v.x;
        o.y = (R)v.y;
        out[link_index<RECON>(mu, e, s, g.V)] = o;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// plain apply: one thread per (site, rhs-in-group of NR), links shared by the
// NR threads of a site through L1 broadcast.
// resident blocks per SM of the plain apply (tools/f32_apply_ab.sh): fp32
// at 5 (102 registers) -- 8.5 % faster than 4 at 32^4 and 48^3 x 96 (3, 6:
// slower); fp64 at 3 (168 registers, no spills)
#ifndef MGT_F32_APPLY_MINB
#define MGT_F32_APPLY_MINB 5
#endif
#ifndef MGT_F64_APPLY_MINB
#define MGT_F64_APPLY_MINB 3
#endif
// 1: the plain apply loads the centre with the first hop (wilson_eval EARLY,
// 8 instead of 9 dependent memory phases per site).  Measured 5-6 % SLOWER at
// every lattice (48^3 x 96 fp64 1.77 -> 1.88 ms): off.
#ifndef MGT_APPLY_EARLY_CENTRE
#define MGT_APPLY_EARLY_CENTRE 0
#endif
template <typename R, int RECON, int NR>
__global__ void __launch_bounds__(128, (sizeof(R) == 8 ? MGT_F64_APPLY_MINB : MGT_F32_APPLY_MINB))
    wilson_apply_kernel(WilsonParams P, const cplx<R> *__restrict__ in, cplx<R> *__restrict__ out,
                        LinkField<R, RECON> links, unsigned long long *ctr) {
  // warp w of the block serves rhs w % NR on 32 consecutive sites: every load
  // instruction streams one field (like NR = 1) and the NR warps of a site
  // group share its links through L1.
  constexpr int SPB = 128 / NR;  // sites per block iteration
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int rhs = w % NR;
  const int local = (w / NR) * 32 + lane;
  for (int64_t step = 0;; ++step) {
    const int64_t chunk = ctr ? next_chunk(ctr) : blockIdx.x + step * (int64_t)gridDim.x;
    if (chunk * SPB >= P.g.V) break;
    const int64_t o = chunk * SPB + local;
    if (o >= P.g.V) continue;
    const int64_t site = sched_site(P.sched, o);
    const cplx<R> *inr = in + (int64_t)rhs * 12 * P.g.V;
    cplx<R> *outr = out + (int64_t)rhs * 12 * P.g.V;
    C<R> y[4][3], xc[4][3];
    wilson_eval<R, RECON, 1, MGT_APPLY_EARLY_CENTRE != 0>(P, inr, links, site, y, xc);
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int c = 0; c < 3; ++c) stc_cs(outr + (a * 3 + c) * P.g.V + site, y[a][c]);
  }
}

// split variant: two threads per site (single rhs)
template <typename R, int RECON>
__global__ void __launch_bounds__(128, 3) wilson_apply_split2_kernel(WilsonParams P, const cplx<R> *__restrict__ in,
                                                                    cplx<R> *__restrict__ out,
                                                                    LinkField<R, RECON> links) {
  const int64_t n = P.g.V * 2;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t site = sched_site(P.sched, idx >> 1);
    const int h = (int)(idx & 1);
    C<R> y[2][3], xc[2][3];
    wilson_eval_split2<R, RECON>(P, in, links, site, h, y, xc);
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int c = 0; c < 3; ++c) stc_cs(out + ((2 * h + a) * 3 + c) * P.g.V + site, y[a][c]);
  }
}

template <typename R, int RECON>
static int launch_split2(const mgt_wilson_s *h, const WilsonParams &P, const void *x, void *y, cudaStream_t st) {
  LinkField<R, RECON> lf{reinterpret_cast<const cplx<R> *>(h->links), h->g.V};
  const int block = 128;
  static int grid_cache = 0;
  if (!grid_cache) grid_cache = resident_grid(wilson_apply_split2_kernel<R, RECON>, block, (int64_t)1 << 40);
  int64_t need = (h->g.V * 2 + block - 1) / block;
  const int grid = (int)std::min<int64_t>(grid_cache, need);
  wilson_apply_split2_kernel<R, RECON><<<grid, block, 0, st>>>(P, reinterpret_cast<const cplx<R> *>(x),
                                                               reinterpret_cast<cplx<R> *>(y), lf);
  MGT_LAUNCH_CHECK("wilson_apply_split2_kernel");
  return MGT_OK;
}

template <typename R, int RECON, int NR>
static int launch_apply(const mgt_wilson_s *h, const WilsonParams &P, const void *x, void *y, cudaStream_t st) {
  LinkField<R, RECON> lf{reinterpret_cast<const cplx<R> *>(h->links), h->g.V};
  const int block = 128;
  static int grid_cache = 0;  // per template instance; V-independent part
  if (!grid_cache) grid_cache = resident_grid(wilson_apply_kernel<R, RECON, NR>, block, (int64_t)1 << 40);
  int64_t need = (h->g.V * NR + block - 1) / block;
  const int grid = (int)std::min<int64_t>(grid_cache, need);
  unsigned long long *ctr = take_counter(h, st);
  wilson_apply_kernel<R, RECON, NR><<<grid, block, 0, st>>>(P, reinterpret_cast<const cplx<R> *>(x),
                                                             reinterpret_cast<cplx<R> *>(y), lf, ctr);
  MGT_LAUNCH_CHECK("wilson_apply_kernel");
  return MGT_OK;
}

// cp.async-staged apply (dslash_pipe.cuh): single rhs, dynamic chunks
template <typename R, int RECON>
static int launch_pipe(const mgt_wilson_s *h, const WilsonParams &P, const void *x, void *y, cudaStream_t st) {
  constexpr int DEPTH = MGT_PIPE_DEPTH, LD = MGT_PIPE_LD;
  auto kern = wilson_apply_pipe_kernel<R, RECON, DEPTH, LD>;
  constexpr size_t smem = (size_t)DEPTH * 12 * 128 * sizeof(cplx<R>);
  LinkField<R, RECON> lf{reinterpret_cast<const cplx<R> *>(h->links), h->g.V};
  static int per_sm = 0;  // per template instance
  if (!per_sm) {
    MGT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int carve = 100;
    if (const char *v = getenv("MGT_PIPE_CARVEOUT")) carve = atoi(v);
    MGT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, carve));
    const int b = blocks_per_sm(reinterpret_cast<const void *>(kern), 128, smem);
    if (b < 1) return b < 0 ? MGT_ERR_CUDA : fail(MGT_ERR_CUDA, "wilson_apply_pipe_kernel does not fit an SM");
    per_sm = b;
  }
  const int64_t need = (h->g.V + 127) / 128;
  const int grid = (int)std::min<int64_t>((int64_t)num_sms() * per_sm, need);
  unsigned long long *ctr = take_counter(h, st);
  kern<<<grid, 128, smem, st>>>(P, reinterpret_cast<const cplx<R> *>(x), reinterpret_cast<cplx<R> *>(y), lf, ctr);
  MGT_LAUNCH_CHECK("wilson_apply_pipe_kernel");
  return MGT_OK;
}

// rhs-interleaved apply: fields at ((comp*V + site)*NR + rhs).  Thread
// (site, rhs) = (tid / NR, tid % NR): the NR lanes of a site load the same
// link address in one request (one sector set per NR rhs) and a warp's
// spinor loads are 512 contiguous bytes, as for NR = 1.
template <typename R, int RECON, int NR>
__global__ void __launch_bounds__(128, (sizeof(R) == 8 ? 3 : 4))
    wilson_apply_il_kernel(WilsonParams P, const cplx<R> *__restrict__ in, cplx<R> *__restrict__ out,
                           LinkField<R, RECON> links, unsigned long long *ctr) {
  constexpr int BLOCK = (128 / NR) * NR;
  constexpr int SPB = BLOCK / NR;
  if (threadIdx.x >= BLOCK) return;  // never: launched with BLOCK threads
  const int rhs = threadIdx.x % NR;
  const int local = threadIdx.x / NR;
  for (int64_t step = 0;; ++step) {
    const int64_t chunk = ctr ? next_chunk(ctr) : blockIdx.x + step * (int64_t)gridDim.x;
    if (chunk * SPB >= P.g.V) break;
    const int64_t o = chunk * SPB + local;
    if (o >= P.g.V) continue;
    const int64_t site = sched_site(P.sched, o);
    C<R> y[4][3], xc[4][3];
    wilson_eval<R, RECON, NR>(P, in + rhs, links, site, y, xc);
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int c = 0; c < 3; ++c) stc_cs(out + ((a * 3 + c) * P.g.V + site) * NR + rhs, y[a][c]);
  }
}

template <typename R, int RECON, int NR>
static int launch_apply_il(const mgt_wilson_s *h, const WilsonParams &P, const void *x, void *y, cudaStream_t st) {
  LinkField<R, RECON> lf{reinterpret_cast<const cplx<R> *>(h->links), h->g.V};
  constexpr int block = (128 / NR) * NR;
  static int grid_cache = 0;
  if (!grid_cache) grid_cache = resident_grid(wilson_apply_il_kernel<R, RECON, NR>, block, (int64_t)1 << 40);
  const int64_t need = (h->g.V + block / NR - 1) / (block / NR);
  const int grid = (int)std::min<int64_t>(grid_cache, need);
  unsigned long long *ctr = take_counter(h, st);
  wilson_apply_il_kernel<R, RECON, NR><<<grid, block, 0, st>>>(P, reinterpret_cast<const cplx<R> *>(x),
                                                                reinterpret_cast<cplx<R> *>(y), lf, ctr);
  MGT_LAUNCH_CHECK("wilson_apply_il_kernel");
  return MGT_OK;
}

template <typename R, int RECON>
static int apply_il(const mgt_wilson_s *h, const WilsonParams &P, const void *x, void *y, int n_rhs,
                    cudaStream_t st) {
  switch (n_rhs) {
    case 1: return launch_apply_il<R, RECON, 1>(h, P, x, y, st);
    case 2: return launch_apply_il<R, RECON, 2>(h, P, x, y, st);
    case 4: return launch_apply_il<R, RECON, 4>(h, P, x, y, st);
    case 8: return launch_apply_il<R, RECON, 8>(h, P, x, y, st);
    case 12: return launch_apply_il<R, RECON, 12>(h, P, x, y, st);
    default: return fail(MGT_ERR_INVALID, "interleaved apply: n_rhs must be 1, 2, 4, 8 or 12");
  }
}

int wilson_apply_il_native(const mgt_wilson_s *h, const void *x, void *y, int n_rhs, int flags, double tau,
                           cudaStream_t st) {
  WilsonParams P = make_params(h, flags, tau);
  if (h->prec == 64) {
    if (h->recon == 18) return apply_il<double, 18>(h, P, x, y, n_rhs, st);
    return apply_il<double, 12>(h, P, x, y, n_rhs, st);
  }
  if (h->recon == 18) return apply_il<float, 18>(h, P, x, y, n_rhs, st);
  return apply_il<float, 12>(h, P, x, y, n_rhs, st);
}

template <typename R, int RECON>
static int apply_groups(const mgt_wilson_s *h, const WilsonParams &P, const void *x, void *y, int n_rhs,
                        cudaStream_t st) {
  const size_t field = (size_t)12 * h->g.V * sizeof(cplx<R>);
  const char *xb = reinterpret_cast<const char *>(x);
  char *yb = reinterpret_cast<char *>(y);
  // Multi-rhs launches share a site group's links through L1, which pays up
  // to ~2^21 sites; on larger lattices the rhs-warps' 4x footprint breaks
  // the L2 blocking and single-rhs launches are faster (48^3 x 96, 4 rhs:
  // 7.9 vs 7.3 ms fp64, 4.6 vs 4.0 ms fp32).
  const bool group = h->g.V < ((int64_t)1 << 22);
  int r = 0;
  while (r < n_rhs) {
    int left = group ? n_rhs - r : 1, rc;
    if (left >= 4) {
      rc = launch_apply<R, RECON, 4>(h, P, xb + r * field, yb + r * field, st);
      r += 4;
    } else if (left >= 2) {
      rc = launch_apply<R, RECON, 2>(h, P, xb + r * field, yb + r * field, st);
      r += 2;
    } else {
      if (h->variant == 1)
        rc = launch_split2<R, RECON>(h, P, xb + r * field, yb + r * field, st);
      else if (h->variant == 2 && h->dyn_sched)
        rc = launch_pipe<R, RECON>(h, P, xb + r * field, yb + r * field, st);
      else
        rc = launch_apply<R, RECON, 1>(h, P, xb + r * field, yb + r * field, st);
      r += 1;
    }
    if (rc) return rc;
  }
  return MGT_OK;
}

int wilson_apply_native(const mgt_wilson_s *h, const void *x, void *y, int n_rhs, int flags, double tau,
                        cudaStream_t st) {
  WilsonParams P = make_params(h, flags, tau);
  if (h->prec == 64) {
    if (h->recon == 18) return apply_groups<double, 18>(h, P, x, y, n_rhs, st);
    return apply_groups<double, 12>(h, P, x, y, n_rhs, st);
  }
  if (h->recon == 18) return apply_groups<float, 18>(h, P, x, y, n_rhs, st);
  return apply_groups<float, 12>(h, P, x, y, n_rhs, st);
}

// ---------------------------------------------------------------------------
// Fused y = A' x and d = (u, y) (numpy vdot) for an external Krylov loop
// (SURVEY 8(b) "fused wd_apply_axpy_dot": the sigma = (rhat, A p) step of
// BiCGStab or the first Arnoldi dot): the dot rides on the stencil's
// epilogue instead of re-reading y.  fp64; dynamically scheduled chunks
// publish per-chunk partials, summed in chunk order by the last block
// (deterministic).
template <int RECON>
__global__ void __launch_bounds__(128, 3)
    wilson_apply_dot_kernel(WilsonParams P, const double2 *__restrict__ in, double2 *__restrict__ out,
                            const double2 *__restrict__ u, LinkField<double, RECON> links, unsigned long long *ctr,
                            unsigned *ticket, double *partials, double *dot_out) {
  const int64_t V = P.g.V;
  const int64_t nch = (V + 127) / 128;
  for (int64_t chunk = next_chunk(ctr); chunk < nch; chunk = next_chunk(ctr)) {
    const int64_t o = chunk * 128 + threadIdx.x;
    double acc[2] = {0.0, 0.0};
    if (o < V) {
      const int64_t site = sched_site(P.sched, o);
      C<double> y[4][3], xc[4][3];
      wilson_eval<double, RECON>(P, in, links, site, y, xc);
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const int64_t q = (int64_t)(a * 3 + c) * V + site;
          stc(out + q, y[a][c]);
          const C<double> uu = ldc(u + q);
          acc[0] += uu.re * y[a][c].re + uu.im * y[a][c].im;
          acc[1] += uu.re * y[a][c].im - uu.im * y[a][c].re;
        }
    }
    chunk_publish<1, 2>(acc, partials + chunk * 2);
  }
  if (last_block(ticket)) {
    double r[2];
    reduce_finish_n<2>(partials, nch, ticket, r);
    if (threadIdx.x == 0) {
      dot_out[0] = r[0];
      dot_out[1] = r[1];
    }
  }
}

template <int RECON>
static int apply_dot(const mgt_wilson_s *h, const WilsonParams &P, const double2 *x, double2 *y, const double2 *u,
                     int n_rhs, double *dot_dev, cudaStream_t st) {
  LinkField<double, RECON> lf{reinterpret_cast<const double2 *>(h->links), h->g.V};
  const int64_t V = h->g.V, nch = (V + 127) / 128;
  static int grid_cache = 0;
  if (!grid_cache) grid_cache = resident_grid(wilson_apply_dot_kernel<RECON>, 128, (int64_t)1 << 40);
  const int grid = (int)std::min<int64_t>(grid_cache, nch);
  char *scr = nullptr;
  MGT_CUDA(scratch_alloc((void **)&scr, 256 + (size_t)nch * 2 * sizeof(double), st));
  for (int r = 0; r < n_rhs; ++r) {
    MGT_CUDA(cudaMemsetAsync(scr, 0, 256, st));
    wilson_apply_dot_kernel<RECON><<<grid, 128, 0, st>>>(
        P, x + (int64_t)r * 12 * V, y + (int64_t)r * 12 * V, u + (int64_t)r * 12 * V, lf,
        reinterpret_cast<unsigned long long *>(scr + 8), reinterpret_cast<unsigned *>(scr),
        reinterpret_cast<double *>(scr + 256), dot_dev + 2 * r);
    MGT_LAUNCH_CHECK("wilson_apply_dot_kernel");
  }
  MGT_CUDA(cudaFreeAsync(scr, st));
  return MGT_OK;
}

}  // namespace mgt

using namespace mgt;

extern "C" {

const char *mgt_last_error(void) { return g_last_error.c_str(); }
int mgt_version(void) { return 1; }
uint64_t mgt_launch_count(void) { return g_launches.load(); }

int mgt_wilson_create(mgt_wilson_t *out, const int dims[4], int antiperiodic, double mass, int prec, int recon,
                      const void *links_ref_dev, void *stream) {
  if (!out || !dims || !links_ref_dev) return fail(MGT_ERR_INVALID, "mgt_wilson_create: null argument");
  for (int i = 0; i < 4; ++i)
    if (dims[i] < 2) return fail(MGT_ERR_INVALID, "extent < 2 is not a valid lattice");
  if (prec != 64 && prec != 32) return fail(MGT_ERR_INVALID, "prec must be 64 or 32");
  if (recon != 18 && recon != 12) return fail(MGT_ERR_INVALID, "recon must be 18 or 12");
  Geom g = make_geom(dims);
  if (g.V * 12 * 8 >= ((int64_t)1 << 31) * 8) return fail(MGT_ERR_INVALID, "lattice too large for one GPU handle");
  auto *h = new mgt_wilson_s();
  h->g = g;
  h->antiperiodic = antiperiodic;
  h->mass = mass;
  h->prec = prec;
  h->recon = recon;
  h->slab = 0;
  h->t_begin = 0;
  h->T_global = dims[3];
  h->variant = 0;
  if (const char *v = getenv("MGT_DSLASH_VARIANT")) h->variant = atoi(v);
  h->slab_bytes = (int64_t)32 << 20;
  if (const char *v = getenv("MGT_SLAB_MB")) h->slab_bytes = (int64_t)atoi(v) << 20;
  const size_t csz = prec == 64 ? sizeof(double2) : sizeof(float2);
  h->link_bytes = (size_t)4 * (recon / 2) * g.V * csz;
  cudaError_t e = cudaMalloc(&h->links, h->link_bytes);
  if (e != cudaSuccess) {
    delete h;
    return cuda_fail(e, "cudaMalloc(links)");
  }
  e = cudaMallocHost(&h->host_flags, 64 * sizeof(int));
  if (e != cudaSuccess) {
    cudaFree(h->links);
    delete h;
    return cuda_fail(e, "cudaMallocHost(flags)");
  }
  h->dyn_sched = 1;
  if (const char *v = getenv("MGT_DYN_SCHED")) h->dyn_sched = atoi(v);
  h->links_cb = nullptr;
  h->links_cb32 = nullptr;
  h->solve_eo = 1;
  if (const char *v = getenv("MGT_SOLVE_EO")) h->solve_eo = atoi(v);
  h->ctr_next = 0;
  e = cudaMalloc(&h->ctr_ring, kCtrRing * sizeof(unsigned long long));
  if (e != cudaSuccess) {
    cudaFree(h->links);
    cudaFreeHost(h->host_flags);
    delete h;
    return cuda_fail(e, "cudaMalloc(counters)");
  }
  cudaStream_t st = as_stream(stream);
  const int block = 256, grid = grid_for(g.V, block, 8);
  const double2 *ref = reinterpret_cast<const double2 *>(links_ref_dev);
  if (prec == 64 && recon == 18)
    links_from_ref_kernel<double, 18><<<grid, block, 0, st>>>(g, ref, (double2 *)h->links);
  else if (prec == 64)
    links_from_ref_kernel<double, 12><<<grid, block, 0, st>>>(g, ref, (double2 *)h->links);
  else if (recon == 18)
    links_from_ref_kernel<float, 18><<<grid, block, 0, st>>>(g, ref, (float2 *)h->links);
  else
    links_from_ref_kernel<float, 12><<<grid, block, 0, st>>>(g, ref, (float2 *)h->links);
  note_launch();
  e = cudaGetLastError();
  if (e != cudaSuccess) {
    cudaFree(h->links);
    cudaFreeHost(h->host_flags);
    delete h;
    return cuda_fail(e, "links_from_ref_kernel");
  }
  *out = h;
  return MGT_OK;
}

int mgt_wilson_destroy(mgt_wilson_t h) {
  if (!h) return MGT_OK;
  drop_graphs(h);
  cudaFree(h->links);
  if (h->links_cb) cudaFree(h->links_cb);
  if (h->links_cb32) cudaFree(h->links_cb32);
  cudaFree(h->ctr_ring);
  cudaFreeHost(h->host_flags);
  delete h;
  return MGT_OK;
}

int mgt_wilson_info(mgt_wilson_t h, int dims[4], int *prec, int *recon, int64_t *volume) {
  if (!h) return fail(MGT_ERR_INVALID, "null handle");
  if (dims)
    for (int i = 0; i < 4; ++i) dims[i] = h->g.L[i];
  if (prec) *prec = h->prec;
  if (recon) *recon = h->recon;
  if (volume) *volume = h->g.V;
  return MGT_OK;
}

int mgt_wilson_apply(mgt_wilson_t h, const void *x_dev, void *y_dev, int n_rhs, int flags, double tau,
                     void *stream) {
  if (!h || !x_dev || !y_dev) return fail(MGT_ERR_INVALID, "mgt_wilson_apply: null argument");
  if (n_rhs < 1) return fail(MGT_ERR_INVALID, "n_rhs must be >= 1");
  if (x_dev == y_dev) return fail(MGT_ERR_INVALID, "mgt_wilson_apply: in-place apply is not supported");
  if (h->slab) return fail(MGT_ERR_INVALID, "mgt_wilson_apply: slab handles apply through mgt_wilson_apply_slab");
  return wilson_apply_native(h, x_dev, y_dev, n_rhs, flags, tau, as_stream(stream));
}

int mgt_wilson_apply_il(mgt_wilson_t h, const void *x_dev, void *y_dev, int n_rhs, int flags, double tau,
                        void *stream) {
  if (!h || !x_dev || !y_dev) return fail(MGT_ERR_INVALID, "mgt_wilson_apply_il: null argument");
  if (x_dev == y_dev) return fail(MGT_ERR_INVALID, "mgt_wilson_apply_il: in-place apply is not supported");
  if (h->slab) return fail(MGT_ERR_INVALID, "mgt_wilson_apply_il: slab handles are not supported");
  return wilson_apply_il_native(h, x_dev, y_dev, n_rhs, flags, tau, as_stream(stream));
}

int mgt_wilson_apply_dot(mgt_wilson_t h, const void *x_dev, void *y_dev, const void *u_dev, int n_rhs, int flags,
                         double tau, double *dot_out_dev, void *stream) {
  if (!h || !x_dev || !y_dev || !u_dev || !dot_out_dev || n_rhs < 1)
    return fail(MGT_ERR_INVALID, "mgt_wilson_apply_dot: bad argument");
  if (h->prec != 64) return fail(MGT_ERR_INVALID, "mgt_wilson_apply_dot: needs a complex128 operator");
  if (h->slab) return fail(MGT_ERR_INVALID, "mgt_wilson_apply_dot: slab handles use mgt_wilson_apply_slab");
  if (x_dev == y_dev) return fail(MGT_ERR_INVALID, "mgt_wilson_apply_dot: in-place apply is not supported");
  const WilsonParams P = make_params(h, flags, tau);
  cudaStream_t st = as_stream(stream);
  const double2 *x = (const double2 *)x_dev, *u = (const double2 *)u_dev;
  double2 *y = (double2 *)y_dev;
  note_launch(n_rhs);
  return h->recon == 18 ? apply_dot<18>(h, P, x, y, u, n_rhs, dot_out_dev, st)
                        : apply_dot<12>(h, P, x, y, u, n_rhs, dot_out_dev, st);
}

}  // extern "C"
