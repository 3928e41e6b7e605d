// The opaque Wilson operator handle shared by the operator / solver units.
#pragma once
#include <atomic>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include "common.cuh"
#include "dslash_core.cuh"

struct mgt_wilson_s {
  mgt::Geom g;
  int antiperiodic;
  double mass;
  int prec;   // 64 or 32
  int recon;  // 18 or 12
  int variant;         // dslash kernel variant (0: thread/site, 1: 2 threads/site)
  int64_t slab_bytes;  // L2 budget of one slab t-plane (schedule)
  void *links;  // native link storage (owned)
  size_t link_bytes;
  // pinned host mailbox for solver convergence flags
  int *host_flags;
  // t-slab decomposition: this handle owns global t in [t_begin, t_begin+L3)
  int slab, t_begin, T_global;
  // ring of chunk counters for the dynamic in-order scheduler (one slot per
  // launch, so concurrent launches on different streams never share one)
  unsigned long long *ctr_ring;
  mutable std::atomic<unsigned> ctr_next;
  int dyn_sched;
  // even-odd form: per-parity link copy, built on first use (eo.cu)
  void *links_cb;
  void *links_cb32;  // fp32 copy of links_cb (mixed-precision solves), built on first use
  std::mutex eo_mu;
  int solve_eo;  // BiCGStab solves the even-odd Schur system (default 1)
};

namespace mgt {
constexpr unsigned kCtrRing = 4096;
// a zeroed counter for the next launch on stream st
inline unsigned long long *take_counter(const mgt_wilson_s *h, cudaStream_t st) {
  if (!h->dyn_sched) return nullptr;
  unsigned long long *c = h->ctr_ring + (h->ctr_next.fetch_add(1) % kCtrRing);
  cudaMemsetAsync(c, 0, sizeof(unsigned long long), st);
  return c;
}
}  // namespace mgt

namespace mgt {

inline WilsonParams make_params(const mgt_wilson_s *h, int flags, double tau) {
  WilsonParams P;
  P.g = h->g;
  P.sched = make_sched(h->g, h->prec == 64 ? 1024 : 512, h->slab_bytes);
  P.antiperiodic = h->antiperiodic;
  double g5in = 1.0, g5out = 1.0, t = tau;
  if (flags & MGT_G5_IN) g5in = -g5in;
  if (flags & MGT_G5_OUT) g5out = -g5out;
  if (flags & MGT_DAGGER) {
    // (A + i tau g5)^dag = g5 (A - i tau g5) g5
    g5in = -g5in;
    g5out = -g5out;
    t = -t;
  }
  P.diag_up_re = 4.0 + h->mass;
  P.diag_up_im = t;
  P.diag_dn_re = 4.0 + h->mass;
  P.diag_dn_im = -t;
  P.g5in = g5in;
  P.g5out = g5out;
  P.slab = 0;  // a slab handle turns this on per apply, with its halo buffers
  P.t_begin = h->t_begin;
  P.T_global = h->T_global;
  P.halo_next = nullptr;
  P.halo_prev = nullptr;
  return P;
}

// build the per-parity links if needed; false if the lattice has an odd extent (eo.cu)
bool eo_available(const mgt_wilson_s *h);
int eo_prepare(mgt_wilson_s *h, cudaStream_t st);
// fp32 copy of the per-parity links of an fp64 handle (eo.cu)
int eo_prepare_mixed(mgt_wilson_s *h, cudaStream_t st);

// the two spin-projected t-faces of x (slab.cu; no peer fence)
int halo_pack_native(const mgt_wilson_s *h, const WilsonParams &P, const void *x, void *to_prev, void *to_next,
                     int n_rhs, cudaStream_t st);

// forget cached solver graphs of a handle (bicgstab.cu)
void drop_graphs(const void *h);

// launch y = op(x) for n_rhs native fields (defined in wilson.cu)

int wilson_apply_native(const mgt_wilson_s *h, const void *x, void *y, int n_rhs, int flags,
                        double tau, cudaStream_t st);

}  // namespace mgt
