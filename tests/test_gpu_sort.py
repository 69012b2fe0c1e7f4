"""Parity of scsf_signatures / scsf_sort (Alg. 2) against the oracle — GPU."""
import numpy as np
import pytest

import synth
from oracle import sort as osort

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2510_23215_b200 import scsf
    scsf.load_library()
    return scsf


def _params_dev(params):
    import torch
    return torch.from_numpy(np.ascontiguousarray(params)).cuda()


@pytest.mark.parametrize("cfg_name,N", [("C1", 64), ("C3", 6), ("C4", 5), ("C5", 3)])
def test_signatures_match_oracle(lib, cfg_name, N):
    cfg = synth.get_config(cfg_name)
    f = synth.make_batch(cfg, N)
    sig = lib.signatures(_params_dev(f.params), cfg.dim, cfg.nx, cfg.p0).cpu().numpy()
    ref = osort.signatures(f.params, cfg.dim, cfg.nx, cfg.p0)
    scale = np.abs(ref).max()
    assert np.abs(sig - ref).max() <= 1e-13 * scale


@pytest.mark.parametrize("dim,p,p0", [(2, 9, 4), (2, 16, 16), (3, 6, 6), (2, 33, 2)])
def test_signatures_ragged_and_full_crop(lib, dim, p, p0):
    rng = np.random.default_rng(11)
    params = rng.standard_normal((7, 2, p ** dim))
    sig = lib.signatures(_params_dev(params), dim, p, p0).cpu().numpy()
    ref = osort.signatures(params, dim, p, p0)
    assert np.abs(sig - ref).max() <= 1e-13 * np.abs(ref).max()


@pytest.mark.parametrize("cfg_name", ["C1", "C2", "C3", "C4", "C5"])
def test_sort_permutation_full_size(lib, cfg_name):
    """Exact permutation at BASELINE.json's full N, near-ties reported (none expected)."""
    cfg = synth.get_config(cfg_name)
    f = synth.make_batch(cfg)
    perm, best, second = lib.sort(_params_dev(f.params), cfg.dim, cfg.nx, cfg.p0)
    o_perm, o_best, o_gap, o_near = osort.sort_problems(f.params, cfg.dim, cfg.nx, cfg.p0)
    assert perm.tolist() == o_perm.tolist()
    assert np.allclose(best, o_best, rtol=1e-12, atol=0)
    gap = osort.rel_gaps(best, second)
    assert len(o_near) == 0 and np.all(gap[:-1] >= 1e-12)


def test_sort_ties_lowest_index(lib):
    params = np.ones((6, 1, 64))
    params[3] += 1.0
    perm, best, second = lib.sort(_params_dev(params), 2, 8, 4)
    assert perm.tolist() == [0, 1, 2, 4, 5, 3]
    assert np.all(best[:4] == 0.0) and np.all(second[:3] == 0.0)


def test_sort_hand_instance_and_start(lib):
    params = np.stack([np.full((1, 64), v) for v in (0.0, 10.0, 1.0)])
    perm, best, _ = lib.sort(_params_dev(params), 2, 8, 4)
    assert perm.tolist() == [0, 2, 1]
    perm, _, _ = lib.sort(_params_dev(params), 2, 8, 4, start=1)
    assert perm.tolist() == [1, 2, 0]


def test_sort_single_and_pair(lib):
    perm, best, _ = lib.sort(_params_dev(np.zeros((1, 1, 16))), 2, 4, 2)
    assert perm.tolist() == [0] and len(best) == 0
    perm, best, _ = lib.sort(_params_dev(np.arange(32.0).reshape(2, 1, 16)), 2, 4, 4)
    assert perm.tolist() == [0, 1]


def test_sort_full_crop_equals_raw_greedy(lib):
    rng = np.random.default_rng(3)
    N, p = 40, 8
    params = rng.standard_normal((N, 1, p * p))
    perm, _, _ = lib.sort(_params_dev(params), 2, p, p)
    flat = params.reshape(N, -1)
    D2 = ((flat[:, None, :] - flat[None, :, :]) ** 2).sum(-1) * p * p
    o, _, _ = osort.greedy_order(D2, 0)
    assert perm.tolist() == o.tolist()


def test_sort_bad_args(lib):
    with pytest.raises(lib.ScsfError) as ei:
        lib.sort(_params_dev(np.zeros((3, 1, 16))), 2, 4, 3)
    assert ei.value.code == lib.SCSF_ERR_ARG
    with pytest.raises(lib.ScsfError):
        lib.sort(_params_dev(np.zeros((3, 1, 16))), 2, 4, 2, start=3)
