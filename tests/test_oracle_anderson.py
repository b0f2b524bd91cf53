"""Pins for oracle/anderson.py against closed forms and invariants.

PAPER.md sect. 3, Eq. (eigenequation) l.182-186; box distribution l.191-194.
"""
import numpy as np
import pytest

from oracle import anderson as an
from oracle import eigs


# Published SplitMix64 reference outputs (Steele, Lea & Flood, OOPSLA 2014;
# the reference C implementation splitmix64.c by S. Vigna): seed 1234567 and
# seed 0.  Reading R3 defines our stream as exactly this sequence.
SPLITMIX_1234567 = [6457827717110365317, 3203168211198807973, 9817491932198370423,
                    4593380528125082431, 16408922859458223821]
SPLITMIX_0 = [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


def test_splitmix_known_answers():
    assert [int(v) for v in an.splitmix_stream(1234567, 5)] == SPLITMIX_1234567
    assert [int(v) for v in an.splitmix_stream(0, 3)] == SPLITMIX_0


def test_stream_offset_consistency():
    full = an.splitmix_stream(99, 20)
    part = an.splitmix_stream(99, 7, offset=13)
    assert np.array_equal(full[13:], part)


def test_disorder_box_distribution():
    # eps in [-W/2, W/2), mean 0, variance W^2/12 (box distribution, l.191-193)
    W = 16.5
    e = an.disorder(100, W, 3)
    assert e.min() >= -W / 2 and e.max() < W / 2
    n = e.size
    assert abs(e.mean()) < 5 * W / np.sqrt(12 * n)
    assert abs(e.var() - W * W / 12) < 5 * (W * W / 12) * np.sqrt(0.8 / n)
    # deterministic
    assert np.array_equal(e, an.disorder(100, W, 3))
    assert not np.array_equal(e, an.disorder(100, W, 4))


def test_site_index_bijection():
    L = 5
    s = np.arange(L ** 3)
    i, j, k = an.site_coords(s, L)
    assert np.array_equal(an.site_index(i, j, k, L), s)
    assert an.site_index(0, 0, 0, L) == 0 and an.site_index(L - 1, L - 1, L - 1, L) == L ** 3 - 1
    assert an.site_index(1, 0, 0, L) == 1          # x fastest (reading R2)


@pytest.mark.parametrize("L", [3, 4, 5, 6])
@pytest.mark.parametrize("hop", [1.0, -1.0])
def test_clean_spectrum_closed_form(L, hop):
    # W = 0 periodic lattice: eigenvalues 2*hop*(cos kx + cos ky + cos kz), k = 2 pi m / L
    A = an.matrix(L, np.zeros(L ** 3), hop=hop)
    lam = np.linalg.eigh(A.toarray())[0]
    c = np.cos(2 * np.pi * np.arange(L) / L)
    ref = np.sort((2 * hop * (c[:, None, None] + c[None, :, None] + c[None, None, :])).ravel())
    assert np.allclose(lam, ref, atol=1e-12)


@pytest.mark.parametrize("L", [3, 4, 7])
def test_stencil_plane_wave(L):
    # Any plane wave x = cos(k.r + phi) satisfies (A x)_s = (2 hop sum cos k_a + eps_s - sigma) x_s
    # (the disorder acts pointwise) -- pins neighbours, wrap and signs.
    hop, sigma = -1.0, 0.3
    eps = an.disorder(L, 16.5, 11)
    s = np.arange(L ** 3)
    i, j, k = an.site_coords(s, L)
    m = (1, L - 2, 2 % L)
    kv = [2 * np.pi * mm / L for mm in m]
    x = np.cos(kv[0] * i + kv[1] * j + kv[2] * k + 0.37)
    lam0 = 2 * hop * sum(np.cos(q) for q in kv)
    y = an.stencil_apply(L, eps, x, hop=hop, sigma=sigma)
    assert np.allclose(y, (lam0 + eps - sigma) * x, atol=1e-12)
    assert np.allclose(an.matrix(L, eps, hop=hop, sigma=sigma) @ x, y, atol=1e-12)


def test_all_ones_row_sum():
    # SPEC example: W = 0 periodic, x = ones -> 6 * hop everywhere
    L = 3
    y = an.stencil_apply(L, np.zeros(27), np.ones(27), hop=1.0)
    assert np.allclose(y, 6.0)


def test_matrix_structure_and_trace():
    L, W = 6, 16.5
    eps = an.disorder(L, W, 5)
    A = an.matrix(L, eps, hop=-1.0)
    n = L ** 3
    assert A.nnz == 7 * n
    assert (abs(A - A.T)).max() == 0.0
    assert np.isclose(A.diagonal().sum(), eps.sum())
    lam = np.linalg.eigvalsh(A.toarray())
    assert np.isclose(lam.sum(), eps.sum())
    # Gershgorin / PAPER.md l.193-194: spectrum within [-6 - w/2, 6 + w/2]
    assert lam.min() >= -6 - W / 2 and lam.max() <= 6 + W / 2


def test_gauge_equivalence_even_L():
    # bipartite lattice (even L): hop -> -hop is the similarity x_s -> (-1)^(i+j+k) x_s
    L = 6
    eps = an.disorder(L, 16.5, 7)
    l1 = np.linalg.eigvalsh(an.matrix(L, eps, hop=1.0).toarray())
    l2 = np.linalg.eigvalsh(an.matrix(L, eps, hop=-1.0).toarray())
    assert np.allclose(l1, l2, atol=1e-11)


@pytest.mark.parametrize("L", [4, 5])
def test_red_sites_independent(L):
    red = an.red_sites(L)
    nb = an.neighbours(L)
    r = np.where(red)[0]
    assert not red[nb[r]].any()
    if L % 2 == 0:
        assert red.sum() == L ** 3 // 2


def test_symmetric_stencil():
    L = 5
    eps = an.disorder(L, 12.0, 2)
    rng = np.random.default_rng(0)
    x, y = rng.standard_normal((2, L ** 3))
    ax = an.stencil_apply(L, eps, x, hop=-1.0, sigma=0.5)
    ay = an.stencil_apply(L, eps, y, hop=-1.0, sigma=0.5)
    assert np.isclose(y @ ax, x @ ay, rtol=1e-13)


def test_nearest_eigs_order_on_diagonal():
    # SPEC example: diag(1..10), target 5.4 -> {5, 6, 4, 7, 3}
    lam, _ = eigs.dense_nearest(np.diag(np.arange(1.0, 11.0)), 5, sigma=5.4)
    assert list(lam) == [5.0, 6.0, 4.0, 7.0, 3.0]
