"""Anderson Hamiltonian oracle (TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py).

PAPER.md sect. 3, Eq. (eigenequation), l.182-186:

    x_{i-1;j;k} + x_{i+1;j;k} + x_{i;j-1;k} + x_{i;j+1;k} + x_{i;j;k-1} + x_{i;j;k+1}
        + eps_{i;j;k} x_{i;j;k} = lambda x_{i;j;k}

with eps drawn from the box distribution [-w/2, w/2] (l.191-193) and periodic
boundary conditions (Fig. 1 caption, l.220).  The hopping amplitude is the
parameter `hop` (the paper writes +1; BASELINE.json's configs use -1 -- for
even L the two spectra coincide, reading R1).

Site index (reading R2): s = i + L*(j + L*k), i (x) fastest, 0-based.

Disorder generator (reading R3, shared *definition* with the CUDA path, no
shared code): SplitMix64 counter stream.  Output i of stream key `s` is
    h_i = mix64(s + (i+1) * 0x9E3779B97F4A7C15)   (mod 2^64)
(identical to the classic SplitMix64 sequence seeded with `s`), then
    u_i   = (h_i >> 11) * 2^-53          in [0, 1)
    eps_i = (u_i - 0.5) * W              in [-W/2, W/2)
The disorder stream key is the config seed itself.
"""
import numpy as np
import scipy.sparse as sp

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)


def mix64(z):
    """SplitMix64 finaliser on uint64 numpy arrays (wrapping arithmetic)."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * M1
        z = (z ^ (z >> np.uint64(27))) * M2
        z = z ^ (z >> np.uint64(31))
    return z


def splitmix_stream(key, n, offset=0):
    """h_i = mix64(key + (i+1)*GOLDEN) for i in [offset, offset+n)."""
    i = np.arange(offset, offset + n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(key) + (i + np.uint64(1)) * GOLDEN
    return mix64(z)


def uniform01(key, n, offset=0):
    """u_i = (h_i >> 11) * 2^-53, exactly representable doubles in [0,1)."""
    h = splitmix_stream(key, n, offset)
    return (h >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def disorder(L, W, seed):
    """eps_s for s in [0, L^3): box distribution [-W/2, W/2)."""
    u = uniform01(seed, L ** 3)
    return (u - 0.5) * W


def site_index(i, j, k, L):
    """0-based Cartesian coordinates -> linear index (reading R2)."""
    return i + L * (j + L * k)


def site_coords(s, L):
    s = np.asarray(s)
    return s % L, (s // L) % L, s // (L * L)


def neighbours(L):
    """(n, 6) array: periodic neighbours of every site in the order
    -x, +x, -y, +y, -z, +z (PAPER.md Eq. (eigenequation) terms 1..6)."""
    s = np.arange(L ** 3)
    i, j, k = site_coords(s, L)
    out = np.empty((L ** 3, 6), dtype=np.int64)
    out[:, 0] = site_index((i - 1) % L, j, k, L)
    out[:, 1] = site_index((i + 1) % L, j, k, L)
    out[:, 2] = site_index(i, (j - 1) % L, k, L)
    out[:, 3] = site_index(i, (j + 1) % L, k, L)
    out[:, 4] = site_index(i, j, (k - 1) % L, L)
    out[:, 5] = site_index(i, j, (k + 1) % L, L)
    return out


def matrix(L, eps, hop=1.0, sigma=0.0):
    """A - sigma*I as a scipy CSR matrix (all 7 entries per row explicit).

    Requires L >= 3 so that the 6 periodic neighbours are distinct
    (for L <= 2 neighbours coincide; the paper's lattices have M >= 30)."""
    if L < 3:
        raise ValueError("periodic lattice needs L >= 3")
    n = L ** 3
    nb = neighbours(L)
    rows = np.repeat(np.arange(n), 7)
    cols = np.concatenate([np.arange(n)[:, None], nb], axis=1).ravel()
    vals = np.concatenate([(np.asarray(eps) - sigma)[:, None],
                           np.full((n, 6), float(hop))], axis=1).ravel()
    return sp.csr_matrix((vals, (rows, cols)), shape=(n, n))


def stencil_apply(L, eps, x, hop=1.0, sigma=0.0):
    """Matrix-free y = (A - sigma I) x written directly from Eq. (eigenequation)
    with np.roll on the (k, j, i)-shaped field (periodic wrap)."""
    X = np.asarray(x, dtype=np.float64).reshape(L, L, L)  # axes (k, j, i)
    nbsum = (np.roll(X, 1, axis=2) + np.roll(X, -1, axis=2) +
             np.roll(X, 1, axis=1) + np.roll(X, -1, axis=1) +
             np.roll(X, 1, axis=0) + np.roll(X, -1, axis=0))
    E = np.asarray(eps, dtype=np.float64).reshape(L, L, L)
    return (hop * nbsum + (E - sigma) * X).ravel()


def red_sites(L):
    """Reading R6: the bipartite red set used as level-0 independent set:
    (i+j+k) even, and for odd L additionally i, j, k < L-1 (so that no two
    red sites are periodic neighbours)."""
    s = np.arange(L ** 3)
    i, j, k = site_coords(s, L)
    red = (i + j + k) % 2 == 0
    if L % 2 == 1:
        red &= (i < L - 1) & (j < L - 1) & (k < L - 1)
    return red


def slab_rows(L, z0, nz):
    """Sites of planes [z0, z0 + nz) (a z-slab shard, DESIGN.md sect. 6), ascending."""
    return np.arange(z0 * L * L, (z0 + nz) * L * L)


def slab_block(L, z0, nz, eps, hop=1.0, sigma=0.0):
    """The diagonal block of A - sigma I on the planes of a slab: the block-Jacobi piece
    of the sharded preconditioner (couplings to other slabs dropped; for nz = L the
    whole periodic matrix).  eps: the full lattice."""
    r = slab_rows(L, z0, nz)
    return sp.csr_matrix(matrix(L, eps, hop=hop, sigma=sigma)[r][:, r])
