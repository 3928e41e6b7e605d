/*
 * mgtrace-b200 C ABI -- the drop-in boundary for the deflated-Hutchinson hot
 * path of arXiv:1909.12234 (reference: /root/reference/pkg/src/mgtrace).
 *
 * The reference has no C ABI: its boundary is a duck-typed Python protocol
 * (SURVEY.md section 8(b)).  Every entry point below replaces one reference
 * interface, cited as file:line; the Python host package
 * `paper_1909_12234_b200` binds these through ctypes and re-exports the
 * reference's Python signatures on top of them.
 *
 * Conventions
 *  - Plain pointers and sizes only.  Every `*_dev` pointer is CUDA device
 *    memory owned by the caller; every call is stream-ordered on `stream`
 *    (a cudaStream_t passed as void*, NULL = legacy default stream).
 *  - Return value: MGT_OK (0) or an error code; mgt_last_error() returns the
 *    message of the last failing call on the calling thread.  No C++
 *    exception crosses the ABI.
 *  - Reference layout ("ref"): complex128 index `site*12 + spin*3 + colour`,
 *    site lexicographic over dims[0..3] with dims[3] (= t) FASTEST
 *    (lattice.py:10, :70-74).  Links ref layout: (V, 4, 3, 3) complex.
 *  - Native layout ("native", what the kernels stream): structure of arrays,
 *    element (rhs, comp, site) at ((rhs*12 + comp)*V + site), one complex
 *    (double2 / float2) per element, site order with t SLOWEST:
 *        site = ((x3*L0 + x0)*L1 + x1)*L2 + x2.
 *  - prec: 64 = complex128 (double2), 32 = complex64 (float2).
 */
#ifndef MGTRACE_B200_H
#define MGTRACE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MGT_OK 0
#define MGT_ERR_INVALID 1  /* bad argument -> ValueError in the shim       */
#define MGT_ERR_CUDA 2     /* CUDA runtime failure -> RuntimeError          */
#define MGT_ERR_SIZE 3     /* dimension mismatch (lattice.py:215-216)       */
#define MGT_ERR_BLOCKING 4 /* BlockingError (multigrid.py:24, :39-44)       */

/* apply flags (lattice.py:219-247) */
#define MGT_G5_IN 1  /* y = A (g5 x)          : a_gamma5()        lattice.py:244-247 */
#define MGT_G5_OUT 2 /* y = g5 (A x)          : hermitian_form()  lattice.py:240-242 */
#define MGT_DAGGER 4 /* y = A^dag x = g5 A g5 : apply_dagger()    lattice.py:219-222 */
/* mgt_halo_pack only: the face pointers are peer-mapped receive windows of
 * the neighbouring ranks (CUDA IPC over NVLink); the pack kernel stores the
 * projected faces straight into them and fences system-wide. */
#define MGT_HALO_PEER 8
/* mgt_bicgstab_solve only: solve the full system instead of the even-odd
 * Schur complement (the default whenever every extent is even). */
#define MGT_SOLVE_FULL 16
/* mgt_bicgstab_solve only: mixed-precision even-odd solve -- defect
 * correction with fp32 inner BiCGStab cycles (fp64 reductions and scalars)
 * and the fp64 explicit residual b - A x as the stopping test (the same
 * contract ||b - A x|| <= tol ||b||).  Ignored when the full system is
 * solved. */
#define MGT_SOLVE_MIXED 32

typedef struct mgt_wilson_s *mgt_wilson_t;

/* ---- diagnostics --------------------------------------------------------- */
const char *mgt_last_error(void);
int mgt_version(void);
/* number of kernel launches issued by this library since load (evidence). */
uint64_t mgt_launch_count(void);

/* ---- layout (reference <-> native) -------------------------------------- */
/* Replaces the implicit reference ordering of lattice.py:70-74; n_rhs fields
 * stored back to back in both layouts. */
int mgt_spinor_from_ref(const int dims[4], int prec, const void *ref_dev,
                        void *native_dev, int n_rhs, void *stream);
int mgt_spinor_to_ref(const int dims[4], int prec, const void *native_dev,
                      void *ref_dev, int n_rhs, void *stream);

/* native (n_rhs, 12, V) <-> rhs-interleaved (12, V, n_rhs) (inverse = 1 goes
 * interleaved -> native).  The interleaved layout is the multi-rhs form of
 * the dilution / hierarchical-probing slot batches (probing.py:110-165,
 * SURVEY 8(f) f2): the rhs of one site share every link load. */
int mgt_rhs_interleave(int64_t volume, int prec, int n_rhs, int inverse,
                       const void *in_dev, void *out_dev, void *stream);

/* ---- gauge links --------------------------------------------------------- */
/* SU(3) U = expm(i eps H) for `nsites` reference-order sites starting at
 * `site_begin`; normals_dev holds (nsites, 4, 8) float64 draws (the draw
 * order is defined in paper_1909_12234_b200/gauge.py).  Output: ref layout
 * (V,4,3,3) complex128.  Replaces generate_gauge (lattice.py:126-144), which
 * only knows U(1). */
int mgt_su3_expm(double eps, const double *normals_dev, int64_t site_begin,
                 int64_t nsites, void *links_ref_dev, void *stream);

/* ---- Wilson-Dirac operator ----------------------------------------------- */
/* Replaces build_wilson (lattice.py:274-318) + LatticeOperator
 * (lattice.py:194-256).  Copies the ref-layout links into the handle's own
 * native link layout (precision `prec`; recon = 18 full links or 12 =
 * two rows + unitarity reconstruction).  antiperiodic != 0: -1 phase on
 * links wrapping in dims[3] (lattice.py:91-102). */
int mgt_wilson_create(mgt_wilson_t *out, const int dims[4], int antiperiodic,
                      double mass, int prec, int recon,
                      const void *links_ref_dev, void *stream);
int mgt_wilson_destroy(mgt_wilson_t h);
int mgt_wilson_info(mgt_wilson_t h, int dims[4], int *prec, int *recon,
                    int64_t *volume);

/* y = flags-variant of (A + i tau g5) applied to x; native layout, n_rhs
 * fields.  Replaces LatticeOperator.apply / apply_dagger / apply_shifted /
 * hermitian_form / a_gamma5 (lattice.py:214-247) and _ShiftedOperator.apply
 * (eigen.py:140-151). */
int mgt_wilson_apply(mgt_wilson_t h, const void *x_dev, void *y_dev, int n_rhs,
                     int flags, double tau, void *stream);

/* Fused y = A' x and dot_out[2r..2r+1] = vdot(u_r, y_r) (re, im; device
 * doubles) for n_rhs native fields: the (rhat, A p) / Arnoldi dot of an
 * external Krylov loop on the stencil's epilogue (SURVEY 8(b) fused
 * apply+dot; LatticeOperator.apply + numpy vdot, lattice.py:214-217).
 * complex128 handles; flags / tau as mgt_wilson_apply. */
int mgt_wilson_apply_dot(mgt_wilson_t h, const void *x_dev, void *y_dev,
                         const void *u_dev, int n_rhs, int flags, double tau,
                         double *dot_out_dev, void *stream);

/* The same operator on n_rhs rhs-interleaved fields ((comp*V + site)*n_rhs +
 * rhs), n_rhs in {1, 2, 4, 8, 12}: one pass over the links for all rhs
 * (LatticeOperator.apply on an (N, k) block, lattice.py:214-217). */
int mgt_wilson_apply_il(mgt_wilson_t h, const void *x_dev, void *y_dev, int n_rhs,
                        int flags, double tau, void *stream);

/* Even-odd (checkerboard) form, every extent even.  Parity fields are
 * (n_rhs, 12, V/2) with cb index = native site >> 1.  split/merge convert a
 * native field to/from its even and odd halves; mgt_wilson_schur_apply
 * applies the even-site Schur complement
 *   S = G_out [ Dg - 1/4 H_eo Dg^-1 H_oe ] G_in   (Dg = 4 + m0 +- i tau)
 * of the flags/tau variant.  mgt_bicgstab_solve runs on S (full residual
 * ||b - A x|| <= tol ||b|| exactly as krylov.py:78-85 tests it). */
int mgt_wilson_eo_split(mgt_wilson_t h, const void *x_full_dev, void *x_even_dev,
                        void *x_odd_dev, int n_rhs, void *stream);
int mgt_wilson_eo_merge(mgt_wilson_t h, const void *x_even_dev, const void *x_odd_dev,
                        void *x_full_dev, int n_rhs, void *stream);
int mgt_wilson_schur_apply(mgt_wilson_t h, const void *x_even_dev, void *y_even_dev,
                           int n_rhs, int flags, double tau, void *stream);

/* Host-buffer apply: y_host = variant(A) x_host for n_rhs REFERENCE-layout
 * complex128 vectors in host memory (LatticeOperator.apply with numpy
 * arrays, lattice.py:214-217).  The host->device copies, the layout
 * permutation, the stencil and the device->host copies are pipelined over
 * `nchunks` x0-slabs on internal streams (pinned host buffers overlap fully).
 * Returns after y_host is written. */
int mgt_wilson_apply_host(mgt_wilson_t h, const void *x_host, void *y_host,
                          int n_rhs, int flags, double tau, int nchunks,
                          void *stream);

/* ---- t-slab decomposition (multi-GPU) ------------------ */
/* The reference is single-process.  A slab handle owns
 * global t in [t_begin, t_begin + dims_local[3]) of T_global (>= 2 slices);
 * links: the slab's own links in the reference layout of the LOCAL dims.
 * mgt_halo_pack writes the two faces this rank sends (n_rhs x 6 x S3
 * complex, S3 = L0*L1*L2): to_prev = (1 - g4) z of the first slice,
 * to_next = U_4^dag (1 + g4) z of the last slice (z = G_in x).
 * mgt_wilson_apply_slab applies the operator with the faces received from
 * rank+1 (halo_next) and rank-1 (halo_prev); part 0 = all sites, 1 = interior
 * slices only (no halo needed; overlaps the exchange), 2 = the two boundary
 * slices.  The plain mgt_wilson_apply rejects slab handles. */
int mgt_wilson_create_slab(mgt_wilson_t *out, const int dims_local[4],
                           int t_begin, int T_global, int antiperiodic,
                           double mass, int prec, int recon,
                           const void *links_ref_local_dev, void *stream);
int mgt_halo_pack(mgt_wilson_t h, const void *x_dev, void *to_prev_dev,
                  void *to_next_dev, int n_rhs, int flags, double tau,
                  void *stream);
int mgt_wilson_apply_slab(mgt_wilson_t h, const void *x_dev, void *y_dev,
                          const void *halo_next_dev, const void *halo_prev_dev,
                          int n_rhs, int flags, double tau, int part,
                          void *stream);

/* Peer-memory transport for the slab halos (replaces the NCCL send/recv of
 * the faces): every rank allocates one receive window with mgt_ipc_alloc,
 * the 64-byte handles are all-gathered by the caller (torch.distributed),
 * each rank maps its t neighbours' windows with mgt_ipc_open, and
 * mgt_halo_pack(..., flags | MGT_HALO_PEER) writes the faces directly into
 * them.  A stream-ordered barrier (one tiny NCCL all-reduce) then releases
 * the boundary kernels; windows are double-buffered by apply parity so the
 * next pack never overwrites a face a neighbour may still be reading. */
#define MGT_IPC_HANDLE_BYTES 64
int mgt_ipc_alloc(size_t bytes, void **dev_ptr, void *handle_out);
int mgt_ipc_free(void *dev_ptr);
int mgt_ipc_open(const void *handle, void **dev_ptr);
int mgt_ipc_close(void *dev_ptr);

/* ---- distributed (t-slab) solve ------------------------------------------- */
/* One communicator per rank (NCCL, loaded at run time): rank 0 makes the
 * 128-byte unique id, the host broadcasts it (torch.distributed), every rank
 * calls mgt_comm_create with its rank after selecting its device.
 * mgt_bicgstab_solve_slab is mgt_bicgstab_solve for a slab handle: the same
 * kernels leave rank-local sums for one all-reduce per reduction point, and
 * every stencil pass exchanges the spin-projected t-faces (SURVEY 8(e).2,
 * "Krylov dots: local partials + ncclAllReduce").  It solves the full
 * system; reports, relres and the quadratic forms are global. */
typedef struct mgt_comm_s *mgt_comm_t;
int mgt_comm_unique_id(void *id_out /* 128 bytes */);
int mgt_comm_create(mgt_comm_t *out, const void *id, int nranks, int rank);
int mgt_comm_destroy(mgt_comm_t comm);
int mgt_comm_allreduce(mgt_comm_t comm, double *buf_dev, int64_t n, void *stream);
size_t mgt_bicgstab_slab_workspace_bytes(mgt_wilson_t h, int n_rhs);
int mgt_bicgstab_solve_slab(mgt_wilson_t h, mgt_comm_t comm, const void *b_dev, void *x_dev,
                            int n_rhs, int flags, double tau, double tol, int max_iter,
                            void *workspace_dev, int64_t *report_out, double *relres_out,
                            double *dot_out_host, void *stream);

/* ---- BLAS-1 on native fields (fp64) -------------------------------------- */
/* out[r] = sum_i conj(a_i) b_i for each of n_rhs fields of `len` complex
 * entries (deterministic fixed-order reduction; numpy vdot semantics). */
int mgt_cdot(const void *a_dev, const void *b_dev, int64_t len, int n_rhs,
             double *out_dev /* 2*n_rhs doubles */, void *stream);

/* ---- Krylov solver -------------------------------------------------------- */
/* Replaces gcr_solve (krylov.py:52-118) as the TruncatedInverse solver
 * plugin (krylov.py:200-229): GPU-resident BiCGStab for (A + i tau g5) x = b
 * (flags as in mgt_wilson_apply), zero initial guess, convergence confirmed
 * on the explicitly recomputed residual ||b - A x|| <= tol ||b||
 * (krylov.py:78-85, :113-118).  b_dev/x_dev: native layout, n_rhs
 * independent systems solved together (shared link loads).
 * report_out: per rhs, 4 int64 {iterations, matvecs, converged, reason}
 * reason: 0 none, 1 max_iter, 2 breakdown; relres_out: per rhs final
 * explicit relative residual.  If dot_out_host != NULL it receives per rhs
 * the complex vdot(b, x) (2 doubles; the Hutchinson quadratic form,
 * trace.py:104).  Host report arrays are written before the call returns. */
size_t mgt_bicgstab_workspace_bytes(mgt_wilson_t h, int n_rhs);
int mgt_bicgstab_solve(mgt_wilson_t h, const void *b_dev, void *x_dev,
                       int n_rhs, int flags, double tau, double tol,
                       int max_iter, void *workspace_dev,
                       int64_t *report_out, double *relres_out,
                       double *dot_out_host, void *stream);
/* Same, with the workspace size: groups of 4 rhs are batched into one launch
 * per solver kernel (blockIdx.y = group), as many groups as a workspace of
 * mgt_bicgstab_workspace_bytes(h, 4 * G) holds -- the small-lattice form
 * (BASELINE configs 1/3/4) that replaces several concurrent 4-rhs solves.
 * mgt_bicgstab_solve assumes the 4-rhs workspace. */
int mgt_bicgstab_solve_ws(mgt_wilson_t h, const void *b_dev, void *x_dev,
                          int n_rhs, int flags, double tau, double tol,
                          int max_iter, void *workspace_dev, size_t workspace_bytes,
                          int64_t *report_out, double *relres_out,
                          double *dot_out_host, void *stream);
/* mgt_bicgstab_solve_ws with one relative tolerance per rhs (tols: host
 * array of n_rhs values in (0,1)): rhs r stops at ||b_r - A x_r|| <=
 * tols[r] ||b_r||.  Used by the deflated-start estimator (the reference's
 * tol ||z|| bound on A e = z - A x0 is tol ||z|| / ||r0|| relative to r0,
 * trace.py:161-188 with krylov.py:78-85). */
int mgt_bicgstab_solve_tols(mgt_wilson_t h, const void *b_dev, void *x_dev,
                            int n_rhs, int flags, double tau, const double *tols,
                            int max_iter, void *workspace_dev, size_t workspace_bytes,
                            int64_t *report_out, double *relres_out,
                            double *dot_out_host, void *stream);

/* Fixed-iteration restarted GCR(m) with zero start (krylov.py:52-118 with
 * max_iter = restart = m, as called by generate_null_vectors,
 * multigrid.py:87-94): x <- GCR_m(A, b).  Returns the report like above. */
size_t mgt_gcr_workspace_bytes(mgt_wilson_t h, int m);
int mgt_gcr_solve(mgt_wilson_t h, const void *b_dev, void *x_dev, int m,
                  int max_iter, double tol, void *workspace_dev,
                  int64_t *report_out, double *relres_out, void *stream);
/* Restarted GMRES(m) from x0 = 0 on the operator variant (flags, tau) of
 * mgt_wilson_apply: Arnoldi (modified Gram-Schmidt) on the device, Givens /
 * least squares on the host, explicit residual b - A x between cycles and
 * as the stopping test (the reference's contract, krylov.py:78-85, 113-118;
 * the north star's GPU-resident "BiCGStab/GMRES", SURVEY 8(b) solve_gmres).
 * max_iter counts Arnoldi steps over all cycles; report as above
 * (reason 2 = Arnoldi breakdown before convergence). */
size_t mgt_gmres_workspace_bytes(mgt_wilson_t h, int m);
int mgt_gmres_solve(mgt_wilson_t h, const void *b_dev, void *x_dev, int m,
                    int max_iter, double tol, int flags, double tau,
                    void *workspace_dev, int64_t *report_out,
                    double *relres_out, void *stream);

/* ---- probes -------------------------------------------------------------- */
/* Bit-exact numpy PCG64 noise (probing.py:94-107): field j of n_fields is
 * make_noise(N, kind, seed0 + j) with N = 12 V, given the seeded 128-bit
 * states/incs of those seeds (host SeedSequence, 4 uint64 per field:
 * state_hi, state_lo, inc_hi, inc_lo).  kind: 0 rademacher, 1 z4.
 * Written in NATIVE layout (layout != 0) or ref layout (layout == 0). */
int mgt_noise(const int dims[4], int kind, const uint64_t *seeds_host,
              int n_fields, int native_layout, void *out_dev, void *stream);
/* The same probes restricted to a t-slab [t_begin, t_begin + t_local) of
 * the global lattice, in the slab's native layout: bit-identical to the
 * corresponding sites of the global mgt_noise field (probe sharding of a
 * t-sharded solve). */
int mgt_noise_slab(const int dims_global[4], int t_begin, int t_local, int kind,
                   const uint64_t *seeds_host, int n_fields, void *out_native_dev,
                   void *stream);

/* ---- prolongator ------------------------------------------------------------ */
/* Block-orthonormal chirality-split prolongator (multigrid.py:116-225).
 * P storage (native): for aggregate b (native coarse order, t slowest),
 * chirality c, vector k < nv: bs = 6*S entries (S sites per aggregate)
 * P[((b*2 + c)*nv + k)*bs + j], j = q*S + s, q < 6 the spin-colour index
 * within the chirality, s the site within the aggregate (native order).
 * Coarse vectors: (coarse_site_native, 2*nv) complex128, column order
 * c*nv + k (multigrid.py:189-216).
 * mgt_prolong_build replaces build_prolongator (multigrid.py:163-225):
 * gathers the nv native null-vector fields and runs the per-(block,
 * chirality) modified Gram-Schmidt twice with the < 1e-8 drop rule;
 * keep_host (nb*2*nv ints, may be NULL) receives 1 per surviving column.
 * Errors: MGT_ERR_BLOCKING if a block extent does not divide the lattice
 * (BlockingScheme.validate, multigrid.py:39-44). */
int mgt_prolong_build(const int dims[4], const int block[4], int nv,
                      const void *null_native_dev /* nv native fields */,
                      void *P_dev, int *keep_host, void *stream);
/* x = P xc (Prolongator.prolong, multigrid.py:156-157) */
int mgt_prolong(const int dims[4], const int block[4], int nv,
                const void *P_dev, const void *xc_dev, void *x_native_dev,
                int n_rhs, void *stream);
/* xc = P^H x, or P^H (g5 x) = g5_c P^H x if gamma5_in (Prolongator.restrict,
 * multigrid.py:153-154; trace.py:266) */
int mgt_restrict(const int dims[4], const int block[4], int nv,
                 const void *P_dev, const void *x_native_dev, void *xc_dev,
                 int n_rhs, int gamma5_in, void *stream);
/* coarse vectors native <-> reference order (coarse site lexicographic,
 * last coarse dim fastest; multigrid.py:52-57, :144-147) */
int mgt_coarse_perm(const int dims[4], const int block[4], int nc, int n_rhs,
                    const void *in_dev, void *out_dev, int to_ref,
                    void *stream);

/* ---- coarse operator (multigrid.py:228-259) ------------------------------ */
/* C = P^H A P as 9 dense (2nv x 2nv) blocks per aggregate, column-major:
 * C[((b*9 + dir)*nc + col)*nc + row], dir 0 = self, 1 + 2 mu + s the
 * neighbour in direction mu (s = 0 forward, 1 backward).  Replaces the
 * SpGEMM of build_coarse_operator (multigrid.py:248). */
int mgt_coarse_build(mgt_wilson_t h, const int block[4], int nv,
                     const void *P_dev, void *C_dev, void *stream);
/* y = C x on native coarse vectors (CoarseOperator.apply) */
int mgt_coarse_apply(const int dims[4], const int block[4], int nv,
                     const void *C_dev, const void *xc_dev, void *yc_dev,
                     int n_rhs, void *stream);
/* The same stencil with the fp32 copy of C (half the bytes; fp64 vectors and
 * accumulation): used for the loose (tol >= 1e-5) inner solves of the coarse
 * Davidson, whose explicit-residual confirmation stays on the fp64 C. */
int mgt_coarse_apply_c32(const int dims[4], const int block[4], int nv,
                         const void *C32_dev, const void *xc_dev, void *yc_dev,
                         int n_rhs, void *stream);
/* One BiCGStab iteration on (C + i tau g5_c) for n_rhs independent native
 * coarse systems (the inner solves of coarse Davidson / Algorithm 2,
 * multigrid.coarse_bicgstab; the reference runs GCR on C through
 * LatticeOperator.apply, krylov.py:52-118 / multigrid.py:228-243).  C is the
 * fp64 operator, or its fp32 copy when c_fp32 != 0.  Vectors (n_rhs, Nc)
 * complex128 on the device: x, r, p, v, s, t updated in place, rhat read.
 * state: n_rhs rows of 16 doubles [rho re, im, alpha re, im, omega re, im,
 * beta re, im, |r|^2, active, tol^2, converged, iterations, freeze, -, -],
 * read and written on the device (the caller seeds rho, active, tol^2,
 * freeze and reads |r|^2 / converged / iterations; with freeze != 0 a
 * converged rhs clears its own active flag). */
int mgt_coarse_bicgstab_iter(const int dims[4], const int block[4], int nv,
                             const void *C_dev, int c_fp32, double tau,
                             int n_rhs, void *x, void *r, const void *rhat,
                             void *p, void *v, void *s, void *t,
                             double *state, void *stream);

/* Coarse even-odd (checkerboard) form, every coarse extent even.  Parity
 * fields are compact: aggregate b (native coarse order) has cb index b >> 1;
 * vectors (n_rhs, nb / 2, 2nv) complex128.  Blocks of one parity's
 * aggregates, column-major: M[((c * nd + d) * nc + col) * nc + row].
 * mgt_coarse_half_apply: y[c] = sum_d M[c][d] src_d for output parity par;
 * nd = 8: the 8 hops (d -> direction d + 1) from x_other; nd = 9: d = 0 the
 * self block on x_self (dropped when skip_self) and the hops from x_other.
 * M in fp64, or fp32 when m_fp32 != 0 (fp64 vectors). */
int mgt_coarse_half_apply(const int dims[4], const int block[4], int nv,
                          const void *M_dev, int nd, int par, int m_fp32,
                          int skip_self, const void *x_self, const void *x_other,
                          void *y, int n_rhs, void *stream);
/* Schur complement S = C_ee - C_eo C_oo^-1 C_oe of (C + i tau g5_c) on the
 * even aggregates from D (odd, nd = 8: C_oo^-1 C_o,dir) and E (even, nd = 9:
 * C_ee and -C_e,dir): y_e = S x_e, t_o: odd scratch (n_rhs fields). */
int mgt_coarse_schur_apply(const int dims[4], const int block[4], int nv,
                           const void *D_dev, const void *E_dev, int m_fp32,
                           const void *x_e, void *y_e, void *t_o, int n_rhs,
                           void *stream);
/* n_iters BiCGStab iterations on S for n_rhs even-parity systems, every
 * scalar on the device (state rows as mgt_coarse_bicgstab_iter; set freeze
 * so converged rhs stop themselves); t_o: odd scratch.  The caller confirms
 * convergence on the explicit residual between calls
 * (multigrid.coarse_bicgstab). */
int mgt_coarse_schur_bicgstab(const int dims[4], const int block[4], int nv,
                              const void *D_dev, const void *E_dev, int m_fp32,
                              int n_rhs, int n_iters, void *x, void *r,
                              const void *rhat, void *p, void *v, void *s,
                              void *t, void *t_o, double *state, void *stream);

/* ---- deflation projection (trace.py:161-188, :266-267; eigen.py:79-86) --- */
/* H (k x s, column major, complex128) = V^H X;  V: (k, len) row-major
 * vectors, X: (s, len). */
int mgt_proj_vhx(const void *V_dev, const void *X_dev, int64_t len, int k,
                 int s, void *H_dev, void *stream);
/* X[j] <- X[j] - sum_i V[i] H[i, j]   (X - V (V^H X) when H = V^H X) */
int mgt_proj_sub(const void *V_dev, const void *H_dev, void *X_dev,
                 int64_t len, int k, int s, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* MGTRACE_B200_H */
