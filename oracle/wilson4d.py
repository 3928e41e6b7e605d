"""4D SU(3) Wilson-Dirac operator, CPU restatement (TEST INFRASTRUCTURE ONLY).

The reference assembles the 2D U(1) Wilson operator in
`/root/reference/pkg/src/mgtrace/lattice.py:274-318`:

    A = (mass + D) I - 1/2 sum_mu [ (I - g_mu) U_mu(x) d_{x+mu}
                                   + (I + g_mu) U_mu(x-mu)^dag d_{x-mu} ]

(diag block `:289`, hop blocks `:297-298`, forward link times boundary phase
`:299`, backward conj link times phase `:300`, block scatter `:310-318`).
This module generalises exactly that assembly to D = 4, DeGrand-Rossi 4x4
gammas and 3x3 SU(3) links (the block is kron(spin, colour) so that the
component index is `spin*3 + colour`), with the reference conventions:

* site order lexicographic, first coordinate slowest (`lattice.py:10`,
  `:70-74`), so t = the last dimension is the FASTEST-varying site index;
* antiperiodic phase -1 on links that wrap in the last dimension
  (`lattice.py:91-102`);
* gamma5 = +1 on the first dof/2 components of every site
  (`lattice.py:266-271`) -- for DeGrand-Rossi gamma5 = diag(1,1,-1,-1), so
  with `comp = spin*3 + colour` this is +1 on comps 0-5, -1 on comps 6-11.

The SU(3) link generator `U = expm(i eps H)` is not in the reference (it only
has U(1) phases, `lattice.py:126-144`).  Its draw order is defined here and in
the product (`paper_1909_12234_b200/gauge.py`) identically:
`rng = numpy.random.default_rng(seed)`, then `rng.normal(size=(V, 4, 8))` with
V in reference site order, and the 8 normals n0..n7 of one link give the
traceless Hermitian

    H01 = (n0 + i n1)/sqrt2, H02 = (n2 + i n3)/sqrt2, H12 = (n4 + i n5)/sqrt2,
    diag = (n6/sqrt2 + n7/sqrt6, -n6/sqrt2 + n7/sqrt6, -2 n7/sqrt6).
"""

import numpy as np
import scipy.sparse as sp

NSPIN = 4
NCOLOR = 3
DOF = NSPIN * NCOLOR

_I = 1j
GAMMAS = (
    np.array([[0, 0, 0, _I], [0, 0, _I, 0], [0, -_I, 0, 0], [-_I, 0, 0, 0]], dtype=np.complex128),
    np.array([[0, 0, 0, -1], [0, 0, 1, 0], [0, 1, 0, 0], [-1, 0, 0, 0]], dtype=np.complex128),
    np.array([[0, 0, _I, 0], [0, 0, 0, -_I], [-_I, 0, 0, 0], [0, _I, 0, 0]], dtype=np.complex128),
    np.array([[0, 0, 1, 0], [0, 0, 0, 1], [1, 0, 0, 0], [0, 1, 0, 0]], dtype=np.complex128),
)
GAMMA5 = GAMMAS[0] @ GAMMAS[1] @ GAMMAS[2] @ GAMMAS[3]


def gamma5_diag(site_count):
    """+1 on the first 6 comps of each site, -1 on the last 6
    (`lattice.py:266-271` with dof = 12)."""
    per_site = np.concatenate([np.ones(DOF // 2), -np.ones(DOF // 2)])
    return np.tile(per_site, site_count)


def neighbor_tables(dims, antiperiodic=True):
    """Forward/backward site tables and boundary phases, shape (ndim, V), in
    the reference site order (restates `lattice.py:82-103`)."""
    dims = tuple(int(L) for L in dims)
    V = int(np.prod(dims))
    coords = np.stack(np.unravel_index(np.arange(V), dims))
    nd = len(dims)
    fwd = np.empty((nd, V), dtype=np.int64)
    bwd = np.empty((nd, V), dtype=np.int64)
    fph = np.ones((nd, V))
    bph = np.ones((nd, V))
    for mu in range(nd):
        up = coords.copy()
        up[mu] = (up[mu] + 1) % dims[mu]
        dn = coords.copy()
        dn[mu] = (dn[mu] - 1) % dims[mu]
        fwd[mu] = np.ravel_multi_index(up, dims)
        bwd[mu] = np.ravel_multi_index(dn, dims)
        if antiperiodic and mu == nd - 1:
            fph[mu, coords[mu] == dims[mu] - 1] = -1.0
            bph[mu, coords[mu] == 0] = -1.0
    return fwd, bwd, fph, bph


# ---------------------------------------------------------------------------
# SU(3) links


def gauge_normals(dims, seed, chunk_sites=None):
    """The (V, 4, 8) Gaussian draws behind the links, reference site order."""
    V = int(np.prod(dims))
    rng = np.random.default_rng(seed)
    if chunk_sites is None:
        return rng.normal(size=(V, 4, 8))
    parts = []
    for s0 in range(0, V, chunk_sites):
        parts.append(rng.normal(size=(min(chunk_sites, V - s0), 4, 8)))
    return np.concatenate(parts)


def hermitian_from_normals(n):
    """Traceless Hermitian 3x3 matrices from (..., 8) normals."""
    r2, r6 = np.sqrt(2.0), np.sqrt(6.0)
    H = np.zeros(n.shape[:-1] + (3, 3), dtype=np.complex128)
    H[..., 0, 1] = (n[..., 0] + 1j * n[..., 1]) / r2
    H[..., 0, 2] = (n[..., 2] + 1j * n[..., 3]) / r2
    H[..., 1, 2] = (n[..., 4] + 1j * n[..., 5]) / r2
    H[..., 1, 0] = np.conj(H[..., 0, 1])
    H[..., 2, 0] = np.conj(H[..., 0, 2])
    H[..., 2, 1] = np.conj(H[..., 1, 2])
    H[..., 0, 0] = n[..., 6] / r2 + n[..., 7] / r6
    H[..., 1, 1] = -n[..., 6] / r2 + n[..., 7] / r6
    H[..., 2, 2] = -2.0 * n[..., 7] / r6
    return H


def su3_links(dims, eps, seed):
    """U_mu(x) = expm(i eps H), (V, 4, 3, 3) complex128, reference site order.
    expm through the Hermitian eigendecomposition H = Q diag(l) Q^dag."""
    H = hermitian_from_normals(gauge_normals(dims, seed))
    lam, Q = np.linalg.eigh(H)
    ph = np.exp(1j * eps * lam)
    return np.einsum("...ij,...j,...kj->...ik", Q, ph, Q.conj())


def unit_links(dims):
    V = int(np.prod(dims))
    U = np.zeros((V, 4, 3, 3), dtype=np.complex128)
    U[..., 0, 0] = U[..., 1, 1] = U[..., 2, 2] = 1.0
    return U


# ---------------------------------------------------------------------------
# operator


def build_wilson4d_csr(links, dims, mass, antiperiodic=True):
    """Sparse (N x N) 4D Wilson operator, N = 12 V, reference index order
    `site*12 + spin*3 + colour` (restatement of `lattice.py:274-318`)."""
    dims = tuple(int(L) for L in dims)
    V = int(np.prod(dims))
    nd = 4
    fwd, bwd, fph, bph = neighbor_tables(dims, antiperiodic)
    eye4 = np.eye(NSPIN, dtype=np.complex128)
    nblk = V * (2 * nd + 1)
    blocks = np.empty((nblk, DOF, DOF), dtype=np.complex128)
    rsite = np.empty(nblk, dtype=np.int64)
    csite = np.empty(nblk, dtype=np.int64)
    sites = np.arange(V)
    blocks[:V] = (mass + nd) * np.eye(DOF)
    rsite[:V] = sites
    csite[:V] = sites
    k = V
    for mu in range(nd):
        pf = -0.5 * (eye4 - GAMMAS[mu])
        pb = -0.5 * (eye4 + GAMMAS[mu])
        uf = links[:, mu] * fph[mu][:, None, None]
        ub = np.conj(np.swapaxes(links[bwd[mu], mu], -1, -2)) * bph[mu][:, None, None]
        blocks[k:k + V] = np.einsum("ab,sij->saibj", pf, uf).reshape(V, DOF, DOF)
        rsite[k:k + V] = sites
        csite[k:k + V] = fwd[mu]
        k += V
        blocks[k:k + V] = np.einsum("ab,sij->saibj", pb, ub).reshape(V, DOF, DOF)
        rsite[k:k + V] = sites
        csite[k:k + V] = bwd[mu]
        k += V
    comp = np.arange(DOF)
    rows = (rsite[:, None, None] * DOF + comp[None, :, None])
    cols = (csite[:, None, None] * DOF + comp[None, None, :])
    rows = np.broadcast_to(rows, blocks.shape).ravel()
    cols = np.broadcast_to(cols, blocks.shape).ravel()
    data = blocks.ravel()
    keep = data != 0
    mat = sp.coo_matrix((data[keep], (rows[keep], cols[keep])), shape=(V * DOF, V * DOF)).tocsr()
    mat.eliminate_zeros()
    return mat


def apply_stencil(links, dims, mass, x, antiperiodic=True):
    """Matrix-free A x with the same conventions as `build_wilson4d_csr`
    (used where the CSR does not fit host memory). x: (N,) or (N, k)."""
    dims = tuple(int(L) for L in dims)
    V = int(np.prod(dims))
    squeeze = x.ndim == 1
    X = x.reshape(V, NSPIN, NCOLOR, -1)
    U = links.reshape(dims + (4, 3, 3))
    Xg = X.reshape(dims + (NSPIN, NCOLOR, X.shape[-1]))
    eye4 = np.eye(NSPIN, dtype=np.complex128)
    acc = np.zeros_like(Xg)
    for mu in range(4):
        L = dims[mu]
        # forward: U_mu(x) psi(x + mu), phase -1 where x_mu = L-1 (t only)
        xf = np.roll(Xg, -1, axis=mu)
        uf = U[..., mu, :, :]
        if antiperiodic and mu == 3:
            sl = [slice(None)] * 4
            sl[mu] = L - 1
            xf = xf.copy()
            xf[tuple(sl)] *= -1.0
        hf = np.einsum("...ij,...sjk->...sik", uf, xf)
        acc += np.einsum("ab,...bik->...aik", eye4 - GAMMAS[mu], hf)
        # backward: U_mu(x - mu)^dag psi(x - mu), phase -1 where x_mu = 0
        xb = np.roll(Xg, 1, axis=mu)
        ub = np.roll(U[..., mu, :, :], 1, axis=mu)
        if antiperiodic and mu == 3:
            sl = [slice(None)] * 4
            sl[mu] = 0
            xb = xb.copy()
            xb[tuple(sl)] *= -1.0
        hb = np.einsum("...ji,...sjk->...sik", ub.conj(), xb)
        acc += np.einsum("ab,...bik->...aik", eye4 + GAMMAS[mu], hb)
    y = (mass + 4.0) * Xg - 0.5 * acc
    y = y.reshape(V * DOF, -1)
    return y[:, 0] if squeeze else y


def apply_at_sites(links, dims, mass, x, sites, antiperiodic=True):
    """(A x) at the given reference-order sites only, (len(sites), 12): the
    same stencil as build_wilson4d_csr evaluated site by site, for spot checks
    on lattices whose full CSR or stencil does not fit host memory.
    links: (V, 4, 3, 3); x: (N,)."""
    dims = tuple(int(L) for L in dims)
    X = x.reshape(-1, NSPIN, NCOLOR)
    U = links
    eye4 = np.eye(NSPIN, dtype=np.complex128)
    out = np.empty((len(sites), DOF), dtype=np.complex128)
    for n, s in enumerate(sites):
        c = list(np.unravel_index(int(s), dims))
        acc = np.zeros((NSPIN, NCOLOR), dtype=np.complex128)
        for mu in range(4):
            up, dn = list(c), list(c)
            up[mu] = (c[mu] + 1) % dims[mu]
            dn[mu] = (c[mu] - 1) % dims[mu]
            sf = np.ravel_multi_index(up, dims)
            sb = np.ravel_multi_index(dn, dims)
            pf = -1.0 if (antiperiodic and mu == 3 and c[3] == dims[3] - 1) else 1.0
            pb = -1.0 if (antiperiodic and mu == 3 and c[3] == 0) else 1.0
            acc += pf * (eye4 - GAMMAS[mu]) @ (X[sf] @ U[s, mu].T)
            acc += pb * (eye4 + GAMMAS[mu]) @ (X[sb] @ U[sb, mu].conj())
        out[n] = ((mass + 4.0) * X[s] - 0.5 * acc).reshape(-1)
    return out


def plane_wave_symbol(dims, mass, mom_index, antiperiodic=True):
    """Unit-gauge plane-wave KAT: A e^{ipx} chi = M(p) e^{ipx} chi with
    M(p) = (m + sum(1 - cos p)) I + i sum gamma_mu sin p_mu (the 4D version of
    `lattice.py:321-338`).  Returns (p, M(p) 4x4)."""
    p = []
    for mu, (L, k) in enumerate(zip(dims, mom_index)):
        if antiperiodic and mu == 3:
            p.append(2 * np.pi * (k + 0.5) / L)
        else:
            p.append(2 * np.pi * k / L)
    p = np.array(p)
    M = (mass + np.sum(1 - np.cos(p))) * np.eye(4, dtype=np.complex128)
    for mu in range(4):
        M = M + 1j * np.sin(p[mu]) * GAMMAS[mu]
    return p, M


def plane_wave(dims, p, chi):
    """e^{ipx} (chi (x) colour vector) in reference order; chi: (4, 3)."""
    coords = np.stack(np.unravel_index(np.arange(int(np.prod(dims))), dims))
    ph = np.exp(1j * (p[:, None] * coords).sum(axis=0))
    return (ph[:, None, None] * chi[None]).reshape(-1)
