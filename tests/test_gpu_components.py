"""Parity of the component entry points (Alg. 3 building blocks) — GPU.

Dense contractions are checked against float64 numpy (a library routine);
the Cholesky inverse against numpy's Cholesky; the small eigensolver against
LAPACK eigh (eigenvalues) and by its own residual / orthogonality.
Tolerances: contractions 1e-13 relative to sum |x||y| bounds.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2510_23215_b200 import scsf
    scsf.load_library()
    return scsf


def _blk(a, ld=None):
    """numpy n x k -> torch [k, ld] column-major block on the GPU (padding = NaN to catch leaks)."""
    import torch
    n, k = a.shape
    ld = ld or (n + 31) // 32 * 32
    t = torch.full((k, ld), float("nan"), dtype=torch.float64, device="cuda")
    t[:, :n] = torch.from_numpy(a.T.copy())
    return t


@pytest.mark.parametrize("n,b1,b2", [(10000, 120, 120), (1000, 20, 20), (777, 33, 65), (4000, 240, 240),
                                     (64, 5, 130), (50, 1, 1), (100000, 64, 64)])
def test_gemm_tn(lib, n, b1, b2):
    rng = np.random.default_rng(n + b1)
    X = rng.standard_normal((n, b1))
    Y = rng.standard_normal((n, b2))
    C = lib.gemm_tn(_blk(X), _blk(Y), n, alpha=0.5).cpu().numpy().T
    ref = 0.5 * X.T @ Y
    bound = 0.5 * np.abs(X).T @ np.abs(Y)
    assert np.all(np.abs(C - ref) <= 1e-13 * bound + 1e-300)


@pytest.mark.parametrize("n,b1,b2,ld", [(1000, 65, 64, 1001), (4103, 200, 130, 4160), (40000, 240, 240, 40000),
                                        (63, 3, 70, 64), (250000, 100, 37, 250016)])
def test_gemm_tn_leading_dimensions(lib, n, b1, b2, ld):
    """Odd ld (the cp.async kernel) and even ld (the TMA-fed kernel: 16-row boxes, rows past n and
    columns past b zero-filled by the tensor map), ragged n and b, both against numpy."""
    rng = np.random.default_rng(ld)
    X = rng.standard_normal((n, b1))
    Y = rng.standard_normal((n, b2))
    C = lib.gemm_tn(_blk(X, ld), _blk(Y, ld), n).cpu().numpy().T
    bound = np.abs(X).T @ np.abs(Y)
    assert np.all(np.abs(C - X.T @ Y) <= 1e-13 * bound + 1e-300)


@pytest.mark.parametrize("n,b", [(10000, 120), (3000, 70), (500, 240)])
def test_gemm_tn_upper(lib, n, b):
    rng = np.random.default_rng(b)
    X = rng.standard_normal((n, b))
    C = lib.gemm_tn(_blk(X), _blk(X), n, upper=True).cpu().numpy().T
    ref = X.T @ X
    iu = np.triu_indices(b)
    assert np.allclose(C[iu], ref[iu], rtol=1e-13, atol=1e-13 * np.abs(ref).max())


@pytest.mark.parametrize("n,b1,b2,beta", [(10000, 120, 120, 0.0), (1001, 7, 130, -1.0), (333, 128, 33, 0.5),
                                          (5000, 240, 240, 0.0), (64, 1, 1, 1.0), (3001, 360, 360, 0.0),
                                          (777, 300, 70, 1.0), (100, 257, 129, -0.5), (4099, 130, 250, 1.0),
                                          (70001, 368, 300, -1.0), (2000, 200, 384, 0.0), (65, 144, 129, 0.5),
                                          (3000, 200, 100, 0.0), (5000, 129, 180, 2.0)])
def test_gemm_nn(lib, n, b1, b2, beta):
    """Every NN kernel: b1 > 128, b2 > 64 with even leading dimensions take the TMA-fed whole-row
    kernel (k_gemm_nn_tma<NI>, NI = ceil(b2 / 64) = 2..6; ragged n, b1, b2 zero-filled by the
    tensor maps); odd ldm, b1 <= 128 or b2 <= 64 the cp.async kernels."""
    import torch
    rng = np.random.default_rng(n + b2)
    X = rng.standard_normal((n, b1))
    M = rng.standard_normal((b1, b2))
    O = rng.standard_normal((n, b2))
    ld = (n + 31) // 32 * 32
    out = _blk(O, ld)
    res = lib.gemm_nn(_blk(X, ld), _blk(M, b1), n, alpha=2.0, beta=beta, out=out)
    got = res[:, :n].cpu().numpy().T
    ref = 2.0 * X @ M + beta * O
    bound = 2.0 * np.abs(X) @ np.abs(M) + abs(beta) * np.abs(O)
    assert np.all(np.abs(got - ref) <= 1e-13 * bound + 1e-300)


@pytest.mark.parametrize("n,b", [(10000, 120), (4097, 64), (300, 240), (2501, 360), (999, 300)])
def test_gemm_nn_in_place(lib, n, b):
    rng = np.random.default_rng(b)
    X = rng.standard_normal((n, b))
    M = rng.standard_normal((b, b))
    Xd = _blk(X)
    lib.gemm_nn(Xd, _blk(M, b), n, out=Xd)
    got = Xd[:, :n].cpu().numpy().T
    ref = X @ M
    assert np.allclose(got, ref, rtol=0, atol=1e-13 * (np.abs(X) @ np.abs(M)).max())


@pytest.mark.parametrize("b", [1, 20, 120, 157, 240])
def test_chol_inv(lib, b):
    import torch
    rng = np.random.default_rng(b)
    Y = rng.standard_normal((4 * b + 10, b))
    S = Y.T @ Y
    St = np.triu(S) + np.tril(np.full((b, b), np.nan), -1)     # only the upper triangle may be read
    Sd = torch.from_numpy(St.T.copy()).cuda()
    Rinv = lib.chol_inv(Sd).cpu().numpy().T
    R = np.linalg.cholesky(S).T
    ref = np.linalg.inv(R)
    assert np.allclose(np.tril(Rinv, -1), 0.0)
    assert np.abs(Rinv - ref).max() <= 1e-10 * np.abs(ref).max()
    assert np.abs(Rinv.T @ S @ Rinv - np.eye(b)).max() <= 1e-10


def test_chol_inv_fallback_flag(lib):
    import torch
    b = 16
    Y = np.random.default_rng(0).standard_normal((40, b))
    Y[:, 5] = Y[:, 3]                                          # exactly rank deficient
    S = torch.from_numpy((Y.T @ Y).T.copy()).cuda()
    with pytest.raises(lib.NotConverged):
        lib.chol_inv(S, nrows=40)


@pytest.mark.parametrize("b,kind", [(1, "dense"), (2, "dense"), (19, "dense"), (120, "dense"), (120, "warm"),
                                    (133, "dense"), (160, "dense"), (240, "warm"), (64, "degenerate"),
                                    (129, "warm"), (240, "dense"), (360, "warm"), (300, "degenerate")])
def test_syev_small(lib, b, kind):
    import torch
    rng = np.random.default_rng(b)
    if kind == "dense":
        B = rng.standard_normal((b, b))
        G = B + B.T
    elif kind == "warm":
        d = np.sort(rng.uniform(10, 2000, b))
        E = rng.standard_normal((b, b)) * 1e-6 * d.max()
        G = np.diag(d) + (E + E.T)
    else:
        d = np.repeat(np.arange(1, b // 2 + 1, dtype=float), 2)
        Q, _ = np.linalg.qr(rng.standard_normal((b, b)))
        G = Q @ np.diag(d) @ Q.T
        G = 0.5 * (G + G.T)
    theta, Z = lib.syev_small(torch.from_numpy(G.T.copy()).cuda())
    th = theta.cpu().numpy()
    Zn = Z.cpu().numpy().T
    w = np.linalg.eigvalsh(G)
    scale = np.abs(w).max()
    # b > 128 runs the block Jacobi (k_blockjac.cu): each round rotates the whole matrix with
    # n-long products, so rounding accumulates ~ n eps per round; the bar is the north-star 1e-12
    tol = 1e-13 if b <= 128 else 1e-12
    assert np.all(np.diff(th) >= 0)
    assert np.abs(th - w).max() <= tol * scale
    assert np.abs(Zn.T @ Zn - np.eye(b)).max() <= tol
    assert np.abs(G @ Zn - Zn * th).max() <= tol * scale
