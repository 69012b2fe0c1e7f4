"""Gaussian-random-field coefficient sampling (input synthesis only).

Recipe; the paper only says the coefficient
fields are "derived using GRF":

    g(x) = sum_{k in {1..K}^d} xi_k (1 + |k|^2)^(-s) prod_d sin(k_d pi x_d),
    xi_k ~ N(0, 1) from numpy default_rng(SeedSequence([23215, cfg, i, f])),
    drawn in C order with shape (K,)*d indexed [k_x, k_y(, k_z)].

Where the config gives sigma, g <- sigma * g / s_K with s_K the analytic
domain-RMS standard deviation of the raw series (`grf_std`).  The coefficient
is vscale * exp(g).  Unit square/cube, Dirichlet, h = 1/(nx+1); node i sits at
x = (i+1) h and the face between node i-1 and node i at x = (i+1/2) h,
i = 0..nx (i = 0 and i = nx are the boundary faces).

Outputs per operator: the face coefficients a on every axis, the nodal
reaction c (zero for -div(a grad u)) and the nodal parameter fields P used by
the sort ("parameter matrices P"; P:1106 p = grid side).
No FD assembly happens here: both the CUDA path and the oracle assemble A
from these arrays with their own code.
"""
from __future__ import annotations

from dataclasses import dataclass
import numpy as np

from .configs import Config, CONFIGS, EXTRA_CONFIGS

_CFG_INDEX = {name: i for i, name in enumerate(list(CONFIGS) + list(EXTRA_CONFIGS))}


def grf_std(K: int, s: float, dim: int) -> float:
    """Analytic domain-RMS std of the raw series: sqrt(sum_k w_k^2 (1/2)^d)."""
    k = np.arange(1, K + 1, dtype=np.float64)
    kk = np.zeros((K,) * dim)
    for ax in range(dim):
        shape = [1] * dim
        shape[ax] = K
        kk = kk + (k ** 2).reshape(shape)
    return float(np.sqrt(((1.0 + kk) ** (-2.0 * s)).sum() * 0.5 ** dim))


def _weights(K: int, s: float, dim: int) -> np.ndarray:
    k = np.arange(1, K + 1, dtype=np.float64)
    kk = np.zeros((K,) * dim)
    for ax in range(dim):
        shape = [1] * dim
        shape[ax] = K
        kk = kk + (k ** 2).reshape(shape)
    return (1.0 + kk) ** (-s)


def _sin_basis(coords: np.ndarray, K: int) -> np.ndarray:
    k = np.arange(1, K + 1, dtype=np.float64)
    return np.sin(np.pi * np.outer(coords, k))          # [len(coords), K]


def _eval(coef: np.ndarray, bases: list[np.ndarray]) -> np.ndarray:
    """g on the tensor grid given per-axis sine bases [x, y(, z)]; C order (z,) y, x."""
    if len(bases) == 2:
        bx, by = bases
        return by @ coef.T @ bx.T                        # coef[kx, ky] -> g[y, x]
    bx, by, bz = bases
    return np.einsum("xa,yb,zc,abc->zyx", bx, by, bz, coef, optimize=True)


@dataclass
class OperatorFields:
    """Coefficient arrays for a batch of N operators on one grid (float64, C order).

    faces[ax] holds a at the face midpoints normal to axis ax:
      2-D: faces[0] [N, ny, nx+1], faces[1] [N, ny+1, nx]
      3-D: faces[0] [N, nz, ny, nx+1], faces[1] [N, nz, ny+1, nx], faces[2] [N, nz+1, ny, nx]
    c: nodal reaction [N, n] (x fastest).  params: sort fields [N, F, n] (x fastest).
    Vibration family (family == "vib"): no faces and c == 0; the nodal
    rigidity D and density rho are params[:, 0] and params[:, 1].
    """
    dim: int
    nx: int
    h: float
    faces: list
    c: np.ndarray
    params: np.ndarray
    family: str = "flux"

    @property
    def is_vib(self) -> bool:
        return self.family == "vib"

    @property
    def n_ops(self) -> int:
        return self.params.shape[0]

    @property
    def n(self) -> int:
        return self.nx ** self.dim

    def subset(self, idx) -> "OperatorFields":
        idx = np.asarray(idx)
        return OperatorFields(self.dim, self.nx, self.h,
                              [np.ascontiguousarray(f[idx]) for f in self.faces],
                              np.ascontiguousarray(self.c[idx]),
                              np.ascontiguousarray(self.params[idx]), self.family)


def _xi(cfg_index: int, i: int, f: int, K: int, dim: int) -> np.ndarray:
    rng = np.random.default_rng(np.random.SeedSequence([23215, cfg_index, i, f]))
    return rng.standard_normal((K,) * dim)


def draw_xi(cfg: Config, n_ops: int | None = None, start: int = 0, indices=None) -> np.ndarray:
    """The normal draws of operators start..start+n_ops-1 (or `indices`): [N, F, K^dim], C order
    per field — the input of the device-side field evaluation (scsf_grf_fields); make_batch
    evaluates the same draws on the host."""
    if indices is None:
        N = cfg.n_ops if n_ops is None else n_ops
        indices = range(start, start + N)
    ci = _CFG_INDEX.get(cfg.name, 0)
    out = np.empty((len(indices), cfg.fields, cfg.K ** cfg.dim))
    for j, i in enumerate(indices):
        for f in range(cfg.fields):
            out[j, f] = _xi(ci, int(i), f, cfg.K, cfg.dim).reshape(-1)
    return out


def make_fields(cfg: Config, i: int, f: int, cfg_index: int | None = None):
    """One GRF sample (operator i, field f) -> (nodal g, [face g per axis])."""
    ci = _CFG_INDEX.get(cfg.name, 0) if cfg_index is None else cfg_index
    dim, nx, K = cfg.dim, cfg.nx, cfg.K
    h = cfg.h
    coef = _xi(ci, i, f, K, dim) * _weights(K, cfg.s, dim)
    if cfg.sigma is not None:
        coef = coef * (cfg.sigma / grf_std(K, cfg.s, dim))
    nodes = (np.arange(nx) + 1.0) * h
    faces = (np.arange(nx + 1) + 0.5) * h
    bn = _sin_basis(nodes, K)
    bf = _sin_basis(faces, K)
    g_node = _eval(coef, [bn] * dim)
    g_face = []
    for ax in range(dim):
        bases = [bn] * dim
        bases[ax] = bf
        g_face.append(_eval(coef, bases))
    return g_node, g_face


def make_batch(cfg: Config, n_ops: int | None = None, start: int = 0, indices=None,
               params_only: bool = False) -> OperatorFields:
    """Operators start..start+n_ops-1 (or the given global `indices`) of config `cfg`.

    Operator i is a pure function of (cfg, i): seeded, deterministic.
    params_only: skip the face/reaction arrays (the sort needs only P).
    """
    if indices is None:
        N = cfg.n_ops if n_ops is None else n_ops
        indices = range(start, start + N)
    indices = [int(i) for i in indices]
    N = len(indices)
    dim, nx = cfg.dim, cfg.nx
    n = nx ** dim
    shape_node = (nx,) * dim
    face_shapes = []
    for ax in range(dim):
        s = [nx] * dim
        s[dim - 1 - ax] = nx + 1                        # C order: axis x is last
        face_shapes.append(tuple(s))
    nf = 0 if params_only else N
    if cfg.family == "vib":
        params = np.empty((N, 2, n))
        for j, i in enumerate(indices):
            for f in range(2):
                g_node, _ = make_fields(cfg, i, f)
                params[j, f] = np.exp(g_node).reshape(n)
        return OperatorFields(dim, nx, cfg.h, [], np.zeros((nf, n)), params, "vib")
    faces = [np.empty((nf,) + fs) for fs in face_shapes]
    c = np.zeros((nf, n))
    params = np.empty((N, cfg.fields, n))
    for j, i in enumerate(indices):
        if cfg.family == "lapv":
            g_node, _ = make_fields(cfg, i, 0)
            v = cfg.vscale * np.exp(g_node)
            params[j, 0] = v.reshape(n)
            if not params_only:
                for ax in range(dim):
                    faces[ax][j] = 1.0
                c[j] = v.reshape(n)
        elif cfg.family == "diva":
            g_node, g_face = make_fields(cfg, i, 0)
            params[j, 0] = (cfg.vscale * np.exp(g_node)).reshape(n)
            if not params_only:
                for ax in range(dim):
                    faces[ax][j] = cfg.vscale * np.exp(g_face[ax])
        elif cfg.family == "divac":
            ga_node, ga_face = make_fields(cfg, i, 0)
            gc_node, _ = make_fields(cfg, i, 1)
            params[j, 0] = np.exp(ga_node).reshape(n)
            params[j, 1] = np.exp(gc_node).reshape(n)
            if not params_only:
                for ax in range(dim):
                    faces[ax][j] = np.exp(ga_face[ax])
                c[j] = params[j, 1]
        else:
            raise ValueError(cfg.family)
    assert all(f.shape[1:] == fs for f, fs in zip(faces, face_shapes))
    del shape_node
    return OperatorFields(dim, nx, cfg.h, faces, c, params)


def constant_fields(dim: int, nx: int, n_ops: int = 1, a: float = 1.0, c: float = 0.0) -> OperatorFields:
    """Constant-coefficient batch (closed-form Laplacian spectrum cases)."""
    n = nx ** dim
    faces = []
    for ax in range(dim):
        s = [nx] * dim
        s[dim - 1 - ax] = nx + 1
        faces.append(np.full((n_ops,) + tuple(s), float(a)))
    cc = np.full((n_ops, n), float(c))
    params = np.full((n_ops, 1, n), float(a))
    return OperatorFields(dim, nx, 1.0 / (nx + 1), faces, cc, params)


def make_perturbed(cfg: Config, n_ops: int, size: float, base: int = 0) -> OperatorFields:
    """SURVEY f1, the paper's similarity experiment (tab:perturbation_impact): n_ops
    perturbations of one base operator of a "lapv" config (-Lap u + V u, the paper's Helmholtz
    stand-in).  V_i = V_base * exp(size * g_i / s_K), g_i an independent GRF of the config's recipe
    scaled to unit domain-RMS, so `size` is the RMS relative perturbation (0.5, 0.1, 0.01, 0 in the
    paper's table).  Deterministic: seeds (23215, 90, i, 0) for the perturbations."""
    if cfg.family != "lapv":
        raise ValueError("perturbation batches are defined for the -Lap u + V u family")
    n = cfg.nx ** cfg.dim
    g0, _ = make_fields(cfg, base, 0)
    unit = cfg.with_(sigma=1.0)
    faces = []
    for ax in range(cfg.dim):
        s = [cfg.nx] * cfg.dim
        s[cfg.dim - 1 - ax] = cfg.nx + 1
        faces.append(np.ones((n_ops,) + tuple(s)))
    c = np.empty((n_ops, n))
    for i in range(n_ops):
        gi, _ = make_fields(unit, i, 0, cfg_index=90)
        c[i] = (cfg.vscale * np.exp(g0 + size * gi)).reshape(n)
    return OperatorFields(cfg.dim, cfg.nx, cfg.h, faces, c, c[:, None, :].copy())
