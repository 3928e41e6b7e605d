// t-slab domain decomposition of the Wilson operator (multi-GPU, SURVEY.md
// 8(e).2).  Rank r owns global t in [t_begin, t_begin + T_local) of T_global;
// the native layout has t slowest, so a slab is one contiguous block of every
// field.  Each apply needs one face from each t neighbour, sent already spin
// projected (6 complex per spatial site instead of 12):
//   to_prev (-> rank-1):  (1 - g_4) z  of this rank's FIRST slice,
//   to_next (-> rank+1):  U_4^dag (1 + g_4) z  of this rank's LAST slice
// (z = G_in x), so the receiver finishes the forward hop with its own link
// and the backward hop needs no link at all.  The antiperiodic sign is
// applied by the receiver from its global t.  Interior sites (t in
// 1 .. T_local-2) need no halo, so their kernel can overlap the exchange.
#include <cstring>
#include <string>

#include "handle.cuh"

namespace mgt {

template <typename R, int RECON>
__global__ void halo_pack_kernel(WilsonParams P, const cplx<R> *__restrict__ in, LinkField<R, RECON> links,
                                 cplx<R> *__restrict__ to_prev, cplx<R> *__restrict__ to_next, int peer) {
  const int64_t S3 = P.g.stride[3], V = P.g.V;
  const int rhs = blockIdx.y;
  const cplx<R> *x = in + (int64_t)rhs * 12 * V;
  const R g5in = (R)P.g5in;
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < S3; s += (int64_t)gridDim.x * blockDim.x) {
    // first slice: (1 - g_4) projection, h_a = z_a - z_{a+2}
    cplx<R> *tp = to_prev + (int64_t)rhs * 6 * S3 + s;
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        C<R> up = ldc(x + (a * 3 + c) * V + s), dn = g5in * ldc(x + ((a + 2) * 3 + c) * V + s);
        C<R> h = up - dn;
        stc(tp + (a * 3 + c) * S3, h);
      }
    // last slice: U_4^dag (1 + g_4) projection, h_a = z_a + z_{a+2}
    const int64_t site = (int64_t)(P.g.L[3] - 1) * S3 + s;
    C<R> h[2][3];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int c = 0; c < 3; ++c)
        h[a][c] = ldc(x + (a * 3 + c) * V + site) + g5in * ldc(x + ((a + 2) * 3 + c) * V + site);
    C<R> u[3][3];
    links.load(3, site, u);
    cplx<R> *tn = to_next + (int64_t)rhs * 6 * S3 + s;
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        C<R> t(R(0), R(0));
#pragma unroll
        for (int j = 0; j < 3; ++j) t = cfma_conj(u[j][i], h[a][j], t);
        stc(tn + (a * 3 + i) * S3, t);
      }
  }
  // peer-mapped faces: the stores above went over NVLink straight into the
  // neighbours' receive windows; make them visible system-wide before the
  // stream-ordered barrier that releases the neighbours' boundary kernels
  if (peer) __threadfence_system();
}

// part 0: every site; 1: interior slices 1 .. L3-2; 2: boundary slices
template <typename R, int RECON>
__global__ void __launch_bounds__(128, (sizeof(R) == 8 ? 3 : 4))
    wilson_slab_kernel(WilsonParams P, const cplx<R> *__restrict__ in, cplx<R> *__restrict__ out,
                       LinkField<R, RECON> links, int part) {
  const int64_t S3 = P.g.stride[3], V = P.g.V;
  const int L3 = P.g.L[3];
  int64_t n;
  if (part == 0)
    n = V;
  else if (part == 1)
    n = L3 > 2 ? (int64_t)(L3 - 2) * S3 : 0;
  else
    n = (L3 == 1 ? 1 : 2) * S3;
  const int rhs = blockIdx.y;
  const cplx<R> *inr = in + (int64_t)rhs * 12 * V;
  cplx<R> *outr = out + (int64_t)rhs * 12 * V;
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < n; o += (int64_t)gridDim.x * blockDim.x) {
    int64_t site;
    if (part == 0)
      site = o;
    else if (part == 1)
      site = S3 + o;
    else
      site = o < S3 ? o : (int64_t)(L3 - 1) * S3 + (o - S3);
    C<R> y[4][3], xc[4][3];
    wilson_eval<R, RECON>(P, inr, links, site, y, xc, rhs);
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int c = 0; c < 3; ++c) stc_cs(outr + (a * 3 + c) * V + site, y[a][c]);
  }
}

template <typename R, int RECON>
static int pack_t(const mgt_wilson_s *h, const WilsonParams &P, const void *x, void *to_prev, void *to_next,
                  int n_rhs, int peer, cudaStream_t st) {
  LinkField<R, RECON> lf{reinterpret_cast<const cplx<R> *>(h->links), h->g.V};
  dim3 grid(grid_for(h->g.stride[3], 128, 4), n_rhs);
  halo_pack_kernel<R, RECON><<<grid, 128, 0, st>>>(P, (const cplx<R> *)x, lf, (cplx<R> *)to_prev, (cplx<R> *)to_next,
                                                    peer);
  MGT_LAUNCH_CHECK("halo_pack_kernel");
  return MGT_OK;
}

template <typename R, int RECON>
static int slab_t(const mgt_wilson_s *h, const WilsonParams &P, const void *x, void *y, int n_rhs, int part,
                  cudaStream_t st) {
  LinkField<R, RECON> lf{reinterpret_cast<const cplx<R> *>(h->links), h->g.V};
  static int per = 0;
  if (!per) per = resident_grid(wilson_slab_kernel<R, RECON>, 128, (int64_t)1 << 40);
  const int64_t n = part == 0 ? h->g.V : (part == 1 ? h->g.V : 2 * h->g.stride[3]);
  dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 127) / 128, std::max(1, per / n_rhs))), n_rhs);
  wilson_slab_kernel<R, RECON><<<grid, 128, 0, st>>>(P, (const cplx<R> *)x, (cplx<R> *)y, lf, part);
  MGT_LAUNCH_CHECK("wilson_slab_kernel");
  return MGT_OK;
}

int halo_pack_native(const mgt_wilson_s *h, const WilsonParams &P, const void *x, void *to_prev, void *to_next,
                     int n_rhs, cudaStream_t st) {
  if (h->prec == 64)
    return h->recon == 18 ? pack_t<double, 18>(h, P, x, to_prev, to_next, n_rhs, 0, st)
                          : pack_t<double, 12>(h, P, x, to_prev, to_next, n_rhs, 0, st);
  return h->recon == 18 ? pack_t<float, 18>(h, P, x, to_prev, to_next, n_rhs, 0, st)
                        : pack_t<float, 12>(h, P, x, to_prev, to_next, n_rhs, 0, st);
}

}  // namespace mgt

using namespace mgt;

extern "C" {

int mgt_wilson_create_slab(mgt_wilson_t *out, const int dims_local[4], int t_begin, int T_global, int antiperiodic,
                           double mass, int prec, int recon, const void *links_ref_local_dev, void *stream) {
  if (!dims_local || T_global < 1 || t_begin < 0 || t_begin + dims_local[3] > T_global)
    return fail(MGT_ERR_INVALID, "mgt_wilson_create_slab: slab outside the global t range");
  // the local t extent may be 1 (T_global / world); create() validates the other extents
  int d[4] = {dims_local[0], dims_local[1], dims_local[2], dims_local[3] < 2 ? 2 : dims_local[3]};
  if (dims_local[3] < 1) return fail(MGT_ERR_INVALID, "mgt_wilson_create_slab: empty slab");
  if (dims_local[3] == 1) return fail(MGT_ERR_INVALID, "mgt_wilson_create_slab: slabs need >= 2 t slices");
  int rc = mgt_wilson_create(out, d, antiperiodic, mass, prec, recon, links_ref_local_dev, stream);
  if (rc) return rc;
  (*out)->slab = 1;
  (*out)->t_begin = t_begin;
  (*out)->T_global = T_global;
  return MGT_OK;
}

int mgt_halo_pack(mgt_wilson_t h, const void *x_dev, void *to_prev_dev, void *to_next_dev, int n_rhs, int flags,
                  double tau, void *stream) {
  if (!h || !x_dev || !to_prev_dev || !to_next_dev || n_rhs < 1) return fail(MGT_ERR_INVALID, "mgt_halo_pack: bad argument");
  const int peer = (flags & MGT_HALO_PEER) ? 1 : 0;
  WilsonParams P = make_params(h, flags & ~MGT_HALO_PEER, tau);
  cudaStream_t st = as_stream(stream);
  if (h->prec == 64)
    return h->recon == 18 ? pack_t<double, 18>(h, P, x_dev, to_prev_dev, to_next_dev, n_rhs, peer, st)
                          : pack_t<double, 12>(h, P, x_dev, to_prev_dev, to_next_dev, n_rhs, peer, st);
  return h->recon == 18 ? pack_t<float, 18>(h, P, x_dev, to_prev_dev, to_next_dev, n_rhs, peer, st)
                        : pack_t<float, 12>(h, P, x_dev, to_prev_dev, to_next_dev, n_rhs, peer, st);
}

int mgt_wilson_apply_slab(mgt_wilson_t h, const void *x_dev, void *y_dev, const void *halo_next_dev,
                          const void *halo_prev_dev, int n_rhs, int flags, double tau, int part, void *stream) {
  if (!h || !x_dev || !y_dev || n_rhs < 1 || part < 0 || part > 2)
    return fail(MGT_ERR_INVALID, "mgt_wilson_apply_slab: bad argument");
  if (!h->slab) return fail(MGT_ERR_INVALID, "mgt_wilson_apply_slab: not a slab handle");
  if (part != 1 && (!halo_next_dev || !halo_prev_dev))
    return fail(MGT_ERR_INVALID, "mgt_wilson_apply_slab: boundary sites need both halos");
  WilsonParams P = make_params(h, flags, tau);
  P.slab = 1;
  P.halo_next = halo_next_dev;
  P.halo_prev = halo_prev_dev;
  cudaStream_t st = as_stream(stream);
  if (h->prec == 64)
    return h->recon == 18 ? slab_t<double, 18>(h, P, x_dev, y_dev, n_rhs, part, st)
                          : slab_t<double, 12>(h, P, x_dev, y_dev, n_rhs, part, st);
  return h->recon == 18 ? slab_t<float, 18>(h, P, x_dev, y_dev, n_rhs, part, st)
                        : slab_t<float, 12>(h, P, x_dev, y_dev, n_rhs, part, st);
}

// ---- CUDA IPC windows (the peer-memory transport of the slab halos) -------
int mgt_ipc_alloc(size_t bytes, void **dev_ptr, void *handle_out) {
  if (!dev_ptr || !handle_out || bytes == 0) return fail(MGT_ERR_INVALID, "mgt_ipc_alloc: bad argument");
  void *p = nullptr;
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e != cudaSuccess) return fail(MGT_ERR_CUDA, std::string("mgt_ipc_alloc: ") + cudaGetErrorString(e));
  cudaMemset(p, 0, bytes);
  cudaIpcMemHandle_t hd;
  e = cudaIpcGetMemHandle(&hd, p);
  if (e != cudaSuccess) {
    cudaFree(p);
    return fail(MGT_ERR_CUDA, std::string("cudaIpcGetMemHandle: ") + cudaGetErrorString(e));
  }
  static_assert(sizeof(cudaIpcMemHandle_t) == MGT_IPC_HANDLE_BYTES, "IPC handle size");
  memcpy(handle_out, &hd, sizeof(hd));
  *dev_ptr = p;
  return MGT_OK;
}

int mgt_ipc_free(void *dev_ptr) {
  if (!dev_ptr) return MGT_OK;
  cudaError_t e = cudaFree(dev_ptr);
  return e == cudaSuccess ? MGT_OK : fail(MGT_ERR_CUDA, std::string("mgt_ipc_free: ") + cudaGetErrorString(e));
}

int mgt_ipc_open(const void *handle, void **dev_ptr) {
  if (!handle || !dev_ptr) return fail(MGT_ERR_INVALID, "mgt_ipc_open: bad argument");
  cudaIpcMemHandle_t hd;
  memcpy(&hd, handle, sizeof(hd));
  cudaError_t e = cudaIpcOpenMemHandle(dev_ptr, hd, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(MGT_ERR_CUDA, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
  }
  return MGT_OK;
}

int mgt_ipc_close(void *dev_ptr) {
  if (!dev_ptr) return MGT_OK;
  cudaError_t e = cudaIpcCloseMemHandle(dev_ptr);
  return e == cudaSuccess ? MGT_OK : fail(MGT_ERR_CUDA, std::string("mgt_ipc_close: ") + cudaGetErrorString(e));
}

}  // extern "C"
