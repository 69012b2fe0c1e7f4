"""Pins for oracle/sort.py (Alg. 2) — CPU only."""
import numpy as np
import pytest

from oracle import sort as osort


@pytest.mark.parametrize("dim,p,p0", [(2, 16, 8), (2, 20, 20), (3, 8, 4)])
def test_dft_constant_field(dim, p, p0):
    # constant field c -> DC = c * p^d, every other kept mode 0
    c = 3.25
    S = osort.trunc_dft(np.full(p ** dim, c), dim, p, p0).reshape((p0,) * dim)
    dc = (p0 // 2,) * dim                                  # k = 0 sits at index p0/2 (centred crop)
    assert abs(S[dc] - c * p ** dim) < 1e-10 * p ** dim
    S[dc] = 0
    assert np.abs(S).max() < 1e-10 * p ** dim


def test_dft_single_cosine_mode():
    # cos(2 pi k0 x / p) -> two coefficients p^2/2 at kx = +-k0, ky = 0
    p, p0, k0 = 24, 12, 3
    x = np.arange(p)
    P = np.tile(np.cos(2 * np.pi * k0 * x / p), (p, 1))   # P[y, x]
    S = osort.trunc_dft(P.reshape(-1), 2, p, p0).reshape(p0, p0)
    z = p0 // 2
    for kx in (z + k0, z - k0):
        assert abs(S[z, kx] - p * p / 2) < 1e-9
    S[z, z + k0] = S[z, z - k0] = 0
    assert np.abs(S).max() < 1e-9


@pytest.mark.parametrize("dim,p,p0", [(2, 10, 6), (2, 9, 4), (3, 6, 4)])
def test_dft_matches_library_fft_centred_crop(dim, p, p0):
    # special case reducing to a library routine: numpy FFT, fftshift-centred crop (reading R1)
    rng = np.random.default_rng(1)
    P = rng.standard_normal((p,) * dim)
    F = np.fft.fftshift(np.fft.fftn(P))
    c = p // 2
    sl = tuple(slice(c - p0 // 2, c + p0 - p0 // 2) for _ in range(dim))
    S = osort.trunc_dft(P.reshape(-1), dim, p, p0).reshape((p0,) * dim)
    assert np.abs(S - F[sl]).max() < 1e-12 * np.abs(F).max()


@pytest.mark.parametrize("dim,p", [(2, 12), (3, 6)])
def test_parseval_full_crop(dim, p):
    # with p0 = p the kept modes are all residues mod p: sum |S|^2 = p^d sum P^2
    rng = np.random.default_rng(2)
    P = rng.standard_normal(p ** dim)
    S = osort.trunc_dft(P, dim, p, p)
    assert abs(np.sum(np.abs(S) ** 2) - p ** dim * np.sum(P ** 2)) < 1e-10 * p ** dim * np.sum(P ** 2)


def test_truncation_energy_monotone():
    rng = np.random.default_rng(3)
    P = rng.standard_normal(16 * 16)
    e = [np.sum(np.abs(osort.trunc_dft(P, 2, 16, p0)) ** 2) for p0 in (2, 4, 8, 16)]
    assert all(a <= b + 1e-9 for a, b in zip(e, e[1:]))


def test_greedy_hand_instance():
    # constant fields {0, 10, 1} -> order [0, 2, 1]
    p = 8
    params = np.stack([np.full((1, p * p), v) for v in (0.0, 10.0, 1.0)])
    order, best, gap, near = osort.sort_problems(params, 2, p, 4)
    assert order.tolist() == [0, 2, 1]
    assert np.allclose(best, [p ** 4 * 1.0, p ** 4 * 81.0])


def test_greedy_identical_fields_identity_order():
    # SPEC S:275 + strict `<`: exact ties resolve to the lowest index
    params = np.ones((5, 1, 36))
    order, best, gap, near = osort.sort_problems(params, 2, 6, 4)
    assert order.tolist() == [0, 1, 2, 3, 4]
    assert np.all(best == 0) and near.tolist() == [0, 1, 2]   # last step has one candidate


def test_greedy_single_problem():
    order, best, gap, near = osort.sort_problems(np.zeros((1, 1, 16)), 2, 4, 2)
    assert order.tolist() == [0] and len(best) == 0


def test_greedy_tie_lowest_index():
    D2 = np.array([[0, 5, 2, 2], [5, 0, 1, 1], [2, 1, 0, 3], [2, 1, 3, 0]], dtype=float)
    order, best, second = osort.greedy_order(D2, 0)
    assert order.tolist() == [0, 2, 1, 3]                  # 2 beats 3 on the tie at step 1


def test_greedy_start_argument():
    D2 = np.array([[0, 1, 4], [1, 0, 2], [4, 2, 0]], dtype=float)
    assert osort.greedy_order(D2, 2)[0].tolist() == [2, 1, 0]


@pytest.mark.parametrize("dim,p,N,F", [(2, 8, 12, 1), (2, 6, 9, 2), (3, 4, 7, 1)])
def test_full_crop_equals_raw_field_greedy(dim, p, N, F):
    # SPEC S:276 / SURVEY O2: with p0 = p, D2_sig = p^d ||P_i - P_j||_F^2 (Parseval), so the
    # truncated-FFT sort equals the brute-force greedy on the raw fields (FFT-free pin)
    rng = np.random.default_rng(4)
    params = rng.standard_normal((N, F, p ** dim))
    order, best, gap, near = osort.sort_problems(params, dim, p, p)
    flat = params.reshape(N, -1)
    D2raw = np.array([[np.sum((flat[i] - flat[j]) ** 2) for j in range(N)] for i in range(N)])
    o2, b2, s2 = osort.greedy_order(D2raw * p ** dim, 0)
    assert order.tolist() == o2.tolist()
    assert np.allclose(best, b2, rtol=1e-12)


def test_pair_d2_properties():
    rng = np.random.default_rng(5)
    sig = rng.standard_normal((6, 10)) + 1j * rng.standard_normal((6, 10))
    D2 = osort.pair_d2(sig)
    assert np.all(np.diag(D2) == 0)
    assert np.allclose(D2, D2.T, rtol=0, atol=1e-12)
    # triangle inequality on the (non-squared) distance
    D = np.sqrt(D2)
    for i in range(6):
        for j in range(6):
            assert np.all(D[i, j] <= D[i, :] + D[:, j] + 1e-12)


def test_invalid_p0():
    with pytest.raises(ValueError):
        osort.trunc_dft(np.zeros(16), 2, 4, 3)
    with pytest.raises(ValueError):
        osort.trunc_dft(np.zeros(16), 2, 4, 6)
