"""Device-side coefficient fields (scsf_grf_fields) against the host recipe — GPU.

synth.make_batch evaluates DESIGN.md §3's GRF series with numpy (separable matrix products,
numpy's sin/exp); scsf_grf_fields evaluates the same draws on the device.  The two differ
only by summation order and libm rounding, so every array must agree to a few ulps of the
exponent's argument: |rel| <= 1e-12.  Constant arrays (lapv faces, diva reaction) are exact.
"""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

CASES = [("C1", 5), ("C2", 4), ("C3", 3), ("C4", 3), ("C5", 2)]


@pytest.fixture(scope="module")
def lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2510_23215_b200 import scsf
    scsf.load_library()
    return scsf


def _rel(a, b):
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))


@pytest.mark.parametrize("name,N", CASES)
def test_grf_fields_match_host_recipe(lib, name, N):
    import torch
    cfg = synth.get_config(name)
    start = 17
    f = synth.make_batch(cfg, N, start=start)
    xi = torch.from_numpy(synth.draw_xi(cfg, N, start=start)).cuda()
    faces, c, params = lib.grf_fields(cfg.dim, cfg.nx, cfg.K, cfg.s, cfg.sigma, cfg.vscale, cfg.family, xi)
    torch.cuda.synchronize()
    assert _rel(params.cpu().numpy(), f.params) <= 1e-12
    for ax in range(cfg.dim):
        got = faces[ax].cpu().numpy()
        assert got.shape == f.faces[ax].shape
        if cfg.family == "lapv":
            assert np.all(got == 1.0)
        else:
            assert _rel(got, f.faces[ax]) <= 1e-12
    cg = c.cpu().numpy()
    if cfg.family == "diva":
        assert np.all(cg == 0.0)
    else:
        assert _rel(cg, f.c) <= 1e-12


def test_grf_fields_feed_assembly(lib):
    """Fields made on the device assemble to the operators the host fields give."""
    import torch
    from tests.helpers import device_problem
    cfg = synth.get_config("C3")
    f = synth.make_batch(cfg, 3)
    ops_h, _ = device_problem(f)
    xi = torch.from_numpy(synth.draw_xi(cfg, 3)).cuda()
    faces, c, params = lib.grf_fields(cfg.dim, cfg.nx, cfg.K, cfg.s, cfg.sigma, cfg.vscale, cfg.family, xi)
    ops_d = lib.assemble(cfg.dim, cfg.nx, cfg.h, faces, c)
    a, b = ops_d.coef.cpu().numpy(), ops_h.coef.cpu().numpy()
    assert float(np.max(np.abs(a - b))) <= 1e-12 * float(np.max(np.abs(b)))


def test_grf_fields_bad_args(lib):
    import torch
    xi = torch.zeros((1, 1, 33 * 33), dtype=torch.float64, device="cuda")
    with pytest.raises(lib.ScsfError):
        lib.grf_fields(2, 16, 33, 1.0, None, 1.0, "diva", xi)         # K > 32
    xi3 = torch.zeros((1, 1, 6 ** 3), dtype=torch.float64, device="cuda")
    with pytest.raises(lib.ScsfError):
        lib.grf_fields(3, 64, 6, 1.0, None, 1.0, "diva", xi3)         # 3-D nx > 63
    with pytest.raises(ValueError):
        lib.grf_fields(2, 16, 4, 1.0, None, 1.0, "divac", torch.zeros((1, 1, 16), dtype=torch.float64,
                                                                        device="cuda"))
